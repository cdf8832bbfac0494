"""Time the device friction_filter on the bow-knot frame (tw_friction_filter:
search at x + the writer-set replay), and check it against the C oracle
restatement on a reduced knot."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_2211_04045_b200 import capi, scenes as S  # noqa: E402

ctx = capi.Context(0)
for n_along in (1870,):
    fr, v0 = S.knot_frame(n_along=n_along)
    x = fr.x
    yt = x + 0.01 * v0
    mesh = capi.Mesh.from_scene(ctx, fr)
    dyn = capi.Dynamics(ctx, mesh, x, mu=0.3)
    y = capi.friction_filter(ctx, mesh, dyn, x, yt)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        y2 = capi.friction_filter(ctx, mesh, dyn, x, yt)
        ts.append(time.perf_counter() - t)
    print(f"n_along={n_along} nv={fr.nv}: friction_filter (incl. search) {min(ts)*1e3:.1f} ms; "
          f"changed {int(np.any(y != yt, axis=1).sum())} vertices; deterministic "
          f"{np.array_equal(y.view(np.uint64), y2.view(np.uint64))}", flush=True)
    dyn.close()
    mesh.close()

# per-phase timing of one filter call (TW_FR_STATS prints the rounds)
if os.environ.get("TW_FR_PROFILE"):
    fr, v0 = S.knot_frame(n_along=1870)
    mesh = capi.Mesh.from_scene(ctx, fr)
    dyn = capi.Dynamics(ctx, mesh, fr.x, mu=0.3)
    capi.friction_filter(ctx, mesh, dyn, fr.x, fr.x + 0.01 * v0)
    t = time.perf_counter()
    capi.search(ctx, mesh, fr.x, 4e-3)
    print(f"search alone {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)

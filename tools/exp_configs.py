"""Resolve every BASELINE config scene once on the device: sizes, steps,
searches, kernel time; CFG1 also against the oracle (bit-exact positions)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np

from paper_2211_04045_b200 import capi, scenes as S

ctx = capi.Context(0)
for name, make, kw in [("cfg1_cloth_on_sphere", S.cloth_on_sphere, {}),
                       ("cfg2_reef_knot", S.reef_knot, dict(delta=5e-4)),
                       ("cfg3_bow_knot", S.bow_knot, dict(delta=5e-4)),
                       ("cfg4_codim_mix", S.codim_mix, {})]:
    t0 = time.time()
    sc = make()
    m = capi.Mesh.from_scene(ctx, sc)
    for i in range(2):
        x, st = capi.resolve(ctx, m, sc.x, sc.y, **kw)
    print(f"{name}: V={sc.nv} T={len(sc.triangles)} E={len(sc.edges)} steps={st['steps']} "
          f"searches={st['searches']} converged={st['converged']} pairs={st['num_pairs']} "
          f"kernel_ms={st['kernel_ms']:.3f} (scene build {time.time() - t0:.1f} s)", flush=True)
    if name.startswith("cfg1"):
        import pyoracle as O

        xo, so = O.resolve(sc, coloring_mode="device", **kw)
        same = np.array_equal(np.ascontiguousarray(xo).view(np.uint64), np.ascontiguousarray(x).view(np.uint64))
        print(f"  oracle: steps={so['steps']} bit-exact x_out={same}", flush=True)

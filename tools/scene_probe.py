import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2211_04045_b200 import capi, scenes as S
ctx = capi.Context(0)
variants = [(f"torus bow pull5.75", lambda: S.knot_scene(n_along=1870, pull=5.75e-3))]
variants += [(f"ply bow sq{q}", (lambda q=q: S.ply_knot(n_along=1870, squeeze=q * 1e-3, slide=1e-3))) for q in (-0.4, -0.2, -0.1)]
variants += [(f"ply bow sq{q} slide3", (lambda q=q: S.ply_knot(n_along=1870, squeeze=q * 1e-3, slide=3e-3))) for q in (-0.2,)]
for name, mk in variants:
    sc = mk()
    m = capi.Mesh.from_scene(ctx, sc)
    for delta in (5e-4,):
        x, st = capi.resolve(ctx, m, sc.x, sc.y, trace=True, delta=delta, step_limit=200)
        x, st = capi.resolve(ctx, m, sc.x, sc.y, trace=True, delta=delta, step_limit=200)
        tr = st["trace"]
        print(json.dumps({"scene": name, "steps": st["steps"], "searches": st["searches"],
                          "conv": st["converged"], "kernel_ms": round(st["kernel_ms"], 2),
                          "P": [t["num_pairs"] for t in tr[:6]], "C": [t["num_contact_rows"] for t in tr[:16]],
                          "colors": [t["num_colors"] for t in tr[:8]], "maxC": max(t["num_contact_rows"] for t in tr),
                          "maxP": max(t["num_pairs"] for t in tr)}), flush=True)
    m.close()

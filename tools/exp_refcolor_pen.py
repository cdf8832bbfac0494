"""GPU experiment: penetrating targets in reference vs device coloring (steps, searches, convergence)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2211_04045_b200 import capi, scenes
ctx = capi.Context(0)
for name, sc in (("reef_pen", scenes.reef_knot(squeeze=0.2e-3)),):
    mesh = capi.Mesh.from_scene(ctx, sc)
    for mode, lim in (("device", 512), ("reference", 120)):
        t = time.time()
        x, st = capi.resolve(ctx, mesh, sc.x, sc.y, delta=5e-4, coloring_mode=mode, step_limit=lim, trace=True)
        tr = st["trace"]
        print(name, mode, f"{time.time()-t:.1f}s", "steps", st["steps"], "searches", st["searches"], "conv", st["converged"],
              "max|dx|", np.abs(x - sc.x).max(), "bounds", [round(t_["bound"]*1e3, 3) for t_ in tr[:12]],
              "maxdisp", [round(t_["max_disp"]*1e3, 3) for t_ in tr[:12]], flush=True)

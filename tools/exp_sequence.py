"""GPU experiment: consecutive bow-knot frames (state carried), steps and time per frame."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2211_04045_b200 import capi, scenes
ctx = capi.Context(0)
sc, v = scenes.knot_frame(n_along=1870)
mesh = capi.Mesh.from_scene(ctx, sc)
dyn = capi.Dynamics(ctx, mesh, sc.x)
x = sc.x.copy()
for f in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    xn, vn, st = capi.step(ctx, mesh, dyn, x, v, delta=5e-4)
    print(f, f"{st['device_ms']:.2f} ms", "resolve steps", st["resolve_steps"], "searches", st["searches"],
          "conv", st["resolve_converged"], "pcg", st["pcg_iterations"], "max|v|", round(np.abs(vn).max(), 4), flush=True)
    x, v = xn, vn

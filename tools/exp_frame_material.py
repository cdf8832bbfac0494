"""GPU experiment: the bow-knot frame under material variants (density kg/m^2, spring N/m):
CG convergence, resolve steps (device; reference coloring on the reef), and a 15-frame sequence."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2211_04045_b200 import capi, scenes
ctx = capi.Context(0)
for dens, k in ((0.1, 50.0), (1.0, 10.0), (0.5, 10.0), (1.0, 5.0)):
    for n_along in (935, 1870):
        sc, v = scenes.knot_frame(n_along=n_along, density=dens)
        mesh = capi.Mesh.from_scene(ctx, sc)
        dyn = capi.Dynamics(ctx, mesh, sc.x, spring_stiffness=k)
        y, g, st = capi.newton_target(ctx, mesh, dyn, sc.x, v, sc.x)
        res = []
        for mode in (("device", "reference") if n_along == 935 else ("device",)):
            x1, rs = capi.resolve(ctx, mesh, sc.x, y, delta=5e-4, coloring_mode=mode, step_limit=100)
            res.append((mode, rs["steps"], rs["searches"], rs["converged"]))
        seq = []
        x = sc.x.copy()
        vv = v.copy()
        t0 = time.time()
        for f in range(15 if n_along == 1870 else 0):
            xn, vn, fs = capi.step(ctx, mesh, dyn, x, vv, delta=5e-4, step_limit=100)
            seq.append((fs["resolve_steps"], fs["pcg_iterations"], int(fs["resolve_converged"])))
            x, vv = xn, vn
        print(n_along, dens, k, "pcg", st["pcg_iterations"], st["pcg_converged"], f"{st['pcg_ms']:.2f}ms", res,
              "seq", seq, f"{time.time()-t0:.1f}s", flush=True)
        dyn.close(); mesh.close()

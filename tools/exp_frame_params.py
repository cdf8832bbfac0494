"""GPU experiment: knot frames under energy-model / density variants: PCG convergence and resolve
steps in device and reference coloring."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2211_04045_b200 import capi, scenes
ctx = capi.Context(0)
VARIANTS = [dict(density=0.1, k=50.0), dict(density=0.3, k=5.0), dict(density=0.3, k=10.0), dict(density=1.0, k=10.0)]
for n_along in (935, 1870):
    for var in VARIANTS:
        sc, v0 = scenes.knot_frame(n_along=n_along, squeeze=0.2e-3)
        inv = scenes.lumped_inv_mass_fast(sc.x, sc.triangles, np.zeros((0, 2), np.int64), var["density"], 0.0)
        mesh = capi.Mesh(ctx, sc.nv, inv, sc.edges, (), sc.triangles)
        dyn = capi.Dynamics(ctx, mesh, sc.x, spring_stiffness=var["k"])
        y, g, st = capi.newton_target(ctx, mesh, dyn, sc.x, v0, sc.x)
        out = []
        for mode, lim in (("device", 512), ("reference", 60 if n_along == 935 else 0)):
            if not lim:
                continue
            t = time.time()
            x, rs = capi.resolve(ctx, mesh, sc.x, y, delta=5e-4, coloring_mode=mode, step_limit=lim)
            out.append((mode, rs["steps"], rs["searches"], rs["converged"], round(time.time() - t, 2)))
        print(n_along, var, "pcg", st["pcg_iterations"], st["pcg_converged"], f"{st['pcg_ms']:.2f}ms",
              "|y-x|", round(np.abs(y - sc.x).max() * 1e3, 3), "mm", out, flush=True)
        dyn.close(); mesh.close()

"""GPU experiment: one dynamics step (newton target + resolve) on the knot
frames for a few squeeze values; prints PCG iterations, resolve steps, times."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2211_04045_b200 import capi, scenes

ctx = capi.Context(0)
for n_along in (935, 1870):
    for squeeze in (-0.2e-3, 0.2e-3, 0.5e-3, 1.0e-3):
        sc, v0 = scenes.knot_frame(n_along=n_along, squeeze=squeeze)
        mesh = capi.Mesh.from_scene(ctx, sc)
        dyn = capi.Dynamics(ctx, mesh, sc.x)
        for rep in range(3):
            t = time.time()
            x, v, st = capi.step(ctx, mesh, dyn, sc.x, v0, delta=5e-4)
            wall = time.time() - t
        y, g, st2 = capi.newton_target(ctx, mesh, dyn, sc.x, v0)
        pen = np.abs(y - sc.x).max()
        print(f"n_along {n_along} squeeze {squeeze*1e3:+.1f}mm: step dev {st['device_ms']:.2f} ms "
              f"(resolve {st['resolve_ms']:.2f}) wall {wall*1e3:.1f} ms, pcg {st['pcg_iterations']} conv {st['pcg_converged']}, "
              f"resolve steps {st['resolve_steps']} searches {st['searches']} conv {st['resolve_converged']}, "
              f"pairs {st['num_pairs']} rep {st['repulsive_pairs']}, |y-x| {pen*1e3:.2f} mm, |x1-x| {np.abs(x-sc.x).max()*1e3:.2f} mm",
              flush=True)
        dyn.close(); mesh.close()

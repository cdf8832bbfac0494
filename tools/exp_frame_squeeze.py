"""GPU experiment: knot frames vs tightening squeeze/slide (default energy model): resolve steps
in device and reference coloring (step limit 150)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2211_04045_b200 import capi, scenes
ctx = capi.Context(0)
for n_along in (935, 1870):
    for slide in (3e-3, 1.5e-3):
        for squeeze in (-0.1e-3, 0.0, 0.05e-3, 0.1e-3):
            sc, v0 = scenes.knot_frame(n_along=n_along, squeeze=squeeze, slide=slide)
            mesh = capi.Mesh.from_scene(ctx, sc)
            dyn = capi.Dynamics(ctx, mesh, sc.x)
            y, g, st = capi.newton_target(ctx, mesh, dyn, sc.x, v0, sc.x)
            out = []
            for mode in (("device", "reference") if n_along == 935 else ("device",)):
                t = time.time()
                x, rs = capi.resolve(ctx, mesh, sc.x, y, delta=5e-4, coloring_mode=mode, step_limit=150)
                out.append((mode, rs["steps"], rs["searches"], rs["converged"], round(time.time() - t, 2)))
            print(n_along, f"slide {slide*1e3:.1f} squeeze {squeeze*1e3:+.2f}", out, flush=True)
            dyn.close(); mesh.close()

"""GPU experiment: per-scene frame time / resolve steps of the configs[4] batch scenes."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import bench
from paper_2211_04045_b200 import capi
ctx = capi.Context(0)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    sc, v0 = bench.batch_scene(i)
    mesh = capi.Mesh.from_scene(ctx, sc)
    dyn = capi.Dynamics(ctx, mesh, sc.x)
    t = time.time()
    x, v, st = capi.step(ctx, mesh, dyn, sc.x, v0, delta=5e-4)
    print(i, f"{(time.time()-t)*1e3:.1f} ms", {k: st[k] for k in ("resolve_steps", "searches", "resolve_converged", "pcg_iterations", "resolve_ms")},
          "max |x1-x0|", np.abs(x - sc.x).max(), flush=True)
    dyn.close(); mesh.close()

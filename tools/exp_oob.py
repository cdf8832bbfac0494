"""GPU experiment: does writing a neighbouring allocation change our results (an out-of-bounds read)?"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2211_04045_b200 import capi

stream = torch.cuda.current_stream()
ctx = capi.Context(0, stream=stream.cuda_stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
sc, v = bench.batch_scene(0)
mesh = capi.Mesh.from_scene(ctx, sc)
dyn = capi.Dynamics(ctx, mesh, sc.x)
kw = dict(delta=5e-4)
out = {}
for fill in (0, 1, 0x7F, 0xFF, 0):
    flush.fill_(fill)
    y, g, st = capi.newton_target(ctx, mesh, dyn, sc.x, v, sc.x)
    flush.fill_(fill)
    x, rs = capi.resolve(ctx, mesh, sc.x, y, **kw)
    yb = out.setdefault("y", y)
    xb = out.setdefault("x", x)
    print(f"fill {fill:#x}: y same {np.array_equal(y.view(np.uint64), yb.view(np.uint64))} (pcg {st['pcg_iterations']}), "
          f"resolve steps {rs['steps']} x same {np.array_equal(x.view(np.uint64), xb.view(np.uint64))}", flush=True)
# resolve with the fixed y under different fills
y0 = out["y"]
for fill in (1, 0x7F, 0xFF):
    flush.fill_(fill)
    x, rs = capi.resolve(ctx, mesh, sc.x, y0, **kw)
    print(f"fixed y, fill {fill:#x}: steps {rs['steps']} same {np.array_equal(x.view(np.uint64), out['x'].view(np.uint64))}", flush=True)
# the device-pointer step path as in the bench
d_x0, d_v0 = torch.from_numpy(sc.x).cuda(), torch.from_numpy(v).cuda()
d_x, d_v = d_x0.clone(), d_v0.clone()
for fill in (0, 1, 2, 0xFF):
    flush.fill_(fill)
    d_x.copy_(d_x0); d_v.copy_(d_v0)
    st = capi.step_device_ptr(ctx, mesh, dyn, d_x.data_ptr(), d_v.data_ptr(), **kw)
    print(f"step_device fill {fill:#x}: resolve steps {st['resolve_steps']} pcg {st['pcg_iterations']}", flush=True)

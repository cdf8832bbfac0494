"""Drive bow-knot simulation frames for ncu: warm-up steps (capacity growth
happens there), then ONE profiled step inside cudaProfilerStart/Stop (run ncu
with --profile-from-start off so only that step's kernels are captured:
the search, the dynamics kernels, k_pcg_reg and k_resolve)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2211_04045_b200 import capi, scenes as S
sc, v0 = S.knot_frame(n_along=1870)
ctx = capi.Context(0)
m = capi.Mesh.from_scene(ctx, sc)
dyn = capi.Dynamics(ctx, m, sc.x, **S.FRAME_ENERGY)
for i in range(3):
    x, v, st = capi.step(ctx, m, dyn, sc.x, v0, delta=5e-4)
torch.cuda.synchronize()
torch.cuda.profiler.start()
x, v, st = capi.step(ctx, m, dyn, sc.x, v0, delta=5e-4)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("frame", st)

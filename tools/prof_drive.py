"""Drive bow-knot resolves for ncu: warm-up calls (capacity growth happens
there), then ONE profiled call inside cudaProfilerStart/Stop (run ncu with
--profile-from-start off so only that call's kernels are captured)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2211_04045_b200 import capi, scenes as S
sc = S.bow_knot()
ctx = capi.Context(0)
m = capi.Mesh.from_scene(ctx, sc)
for i in range(3):
    x, st = capi.resolve(ctx, m, sc.x, sc.y, delta=5e-4)
torch.cuda.synchronize()
torch.cuda.profiler.start()
x, st = capi.resolve(ctx, m, sc.x, sc.y, delta=5e-4)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("steps", st["steps"], "kernel_ms", st["kernel_ms"], "retries", st.get("retries"))

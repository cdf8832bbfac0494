"""Drive the stage search + refresh on the bow knot for ncu: warm-up calls,
then one profiled search and refresh inside cudaProfilerStart/Stop."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2211_04045_b200 import capi, scenes as S
sc = S.bow_knot()
ctx = capi.Context(0)
m = capi.Mesh.from_scene(ctx, sc)
for i in range(2):
    p = capi.search(ctx, m, sc.x, 4e-3, cap=16_000_000)
    D = capi.refresh(ctx, m, sc.x, 4e-3, p)
torch.cuda.synchronize()
torch.cuda.profiler.start()
p = capi.search(ctx, m, sc.x, 4e-3, cap=16_000_000)
D = capi.refresh(ctx, m, sc.x, 4e-3, p)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("pairs", len(p))

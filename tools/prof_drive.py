"""Drive one bow-knot resolve for ncu (2 warm-up calls, then the profiled call)."""
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2211_04045_b200 import capi, scenes as S
sc = S.bow_knot()
ctx = capi.Context(0)
m = capi.Mesh.from_scene(ctx, sc)
for i in range(3):
    x, st = capi.resolve(ctx, m, sc.x, sc.y, delta=5e-4)
print("steps", st["steps"], "kernel_ms", st["kernel_ms"])

"""Drive stage search + refresh on the bow knot for ncu (warm-up, then profiled calls)."""
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2211_04045_b200 import capi, scenes as S
sc = S.bow_knot()
ctx = capi.Context(0)
m = capi.Mesh.from_scene(ctx, sc)
for i in range(2):
    p = capi.search(ctx, m, sc.x, 4e-3, cap=16_000_000)
D = capi.refresh(ctx, m, sc.x, 4e-3, p)
print("pairs", len(p))

"""Cumulative phase times of the bow-knot resolve cut at L = 1..4 steps."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_2211_04045_b200 import capi, scenes as S

sc = S.bow_knot()
ctx = capi.Context(0)
m = capi.Mesh.from_scene(ctx, sc)
names = sys.argv[1:] or ["ph_pgs_flow", "ph_pgs_color", "ph_pgs_tail"]
for L in (1, 2, 3, 4):
    for i in range(2):
        x, st = capi.resolve(ctx, m, sc.x, sc.y, delta=5e-4, step_limit=L)
    prof = capi.phase_profile(ctx)
    print(f"L={L} kernel_ms {st['kernel_ms']:.3f} " +
          " ".join(f"{k}={prof[k][0]:.3f}/{prof[k][1]}" for k in names if k in prof))

"""Phase profile of one bow-knot resolve (per-phase ms and call counts)."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_2211_04045_b200 import capi, scenes as S

sc = S.bow_knot()
ctx = capi.Context(0)
m = capi.Mesh.from_scene(ctx, sc)
for i in range(3):
    x, st = capi.resolve(ctx, m, sc.x, sc.y, delta=5e-4)
prof = capi.phase_profile(ctx)
print(f"kernel_ms {st['kernel_ms']:.3f} "
      f"steps {st['steps']} searches {st['searches']}")
for k, (ms, n) in prof.items():
    print(f"  {k:20s} {ms:7.3f} ms total, {ms / n:.4f} ms per call ({n} calls)")

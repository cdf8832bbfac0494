"""Phase profile of one resolve of a named scene: python tools/exp_scene.py cloth_on_sphere"""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_2211_04045_b200 import capi, scenes as S

sc = getattr(S, sys.argv[1])()
kw = dict(delta=5e-4) if "knot" in sys.argv[1] else {}
ctx = capi.Context(0)
m = capi.Mesh.from_scene(ctx, sc)
for i in range(3):
    x, st = capi.resolve(ctx, m, sc.x, sc.y, **kw)
prof = capi.phase_profile(ctx)
print(f"{sys.argv[1]} kernel_ms {st['kernel_ms']:.3f} setup_ms {st['setup_ms']:.3f} steps {st['steps']} "
      f"searches {st['searches']}")
for k, (ms, n) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:20s} {ms:7.3f} ms total, {1000 * ms / n:7.2f} us per call ({n} calls)")

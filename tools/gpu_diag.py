import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, pyoracle as O
from paper_2211_04045_b200 import capi, scenes as S
ctx = capi.Context(0)
sc = S.fixture_press(0.012)
kw = dict(solver="jacobi", coloring_mode="reference")
m = capi.Mesh.from_scene(ctx, sc)
lo, hi = 20, 300
xg, sg = capi.resolve(ctx, m, sc.x, sc.y, trace=True, step_limit=hi, **kw)
xo, so = O.resolve(sc, trace=True, step_limit=hi, **kw)
print("full", sg["steps"], so["steps"], flush=True)
# bisect the first differing step
while hi - lo > 1:
    mid = (lo + hi) // 2
    xg, sg = capi.resolve(ctx, m, sc.x, sc.y, trace=True, step_limit=mid, **kw)
    xo, so = O.resolve(sc, trace=True, step_limit=mid, **kw)
    if np.array_equal(xg.view(np.uint64), xo.view(np.uint64)):
        lo = mid
    else:
        hi = mid
print("first differing step limit", hi, flush=True)
xg, sg = capi.resolve(ctx, m, sc.x, sc.y, trace=True, step_limit=hi, **kw)
xo, so = O.resolve(sc, trace=True, step_limit=hi, **kw)
for a, b in zip(sg["trace"][-3:], so["trace"][-3:]):
    print("gpu", a); print("ora", b)
d = np.abs(xg - xo).max(axis=1)
print("verts differing", np.nonzero(d)[0][:20], d.max(), flush=True)

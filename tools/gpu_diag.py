import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, pyoracle as O
from paper_2211_04045_b200 import capi, scenes as S
def cmp(ctx, sc, tag, **kw):
    m = capi.Mesh.from_scene(ctx, sc)
    xg, sg = capi.resolve(ctx, m, sc.x, sc.y, trace=True, **kw)
    xo, so = O.resolve(sc, trace=True, **kw)
    same = np.array_equal(xg.view(np.uint64), xo.view(np.uint64))
    first = next((i for i, (a, b) in enumerate(zip(sg["trace"], so["trace"])) if a != b), None)
    print(tag, sc.name, "same" if same else "DIFF", sg["steps"], so["steps"], sg["searches"], so["searches"], "first trace diff", first, flush=True)
    if first is not None:
        print(" gpu", sg["trace"][first]); print(" ora", so["trace"][first])
    return same
ctx = capi.Context(0)
cmp(ctx, S.fixture_press(0.012), "fresh", solver="jacobi", coloring_mode="reference")
ctx2 = capi.Context(0)
for sc in S.scene_fixtures(0):
    m = capi.Mesh.from_scene(ctx2, sc)
    capi.resolve(ctx2, m, sc.x, sc.y, coloring_mode="device")
cmp(ctx2, S.fixture_press(0.012), "after-battery", solver="jacobi", coloring_mode="reference")
cmp(ctx2, S.fixture_press(0.012), "again", solver="jacobi", coloring_mode="reference")

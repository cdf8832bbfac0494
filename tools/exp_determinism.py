"""GPU experiment: is a call's result independent of the previous calls on the context?"""
import sys
import numpy as np
sys.path.insert(0, ".")
import bench
from paper_2211_04045_b200 import capi

ctx = capi.Context(0)
scs = [bench.batch_scene(i) for i in (0, 7, 3)]
sc0 = scs[0][0]
mesh = capi.Mesh.from_scene(ctx, sc0)
dyn = capi.Dynamics(ctx, mesh, sc0.x)
ys = [capi.newton_target(ctx, mesh, dyn, sc.x, v, sc.x)[0] for sc, v in scs]
ys2 = [capi.newton_target(ctx, mesh, dyn, sc.x, v, sc.x)[0] for sc, v in scs]
print("newton targets repeatable:", [np.array_equal(a.view(np.uint64), b.view(np.uint64)) for a, b in zip(ys, ys2)])
kw = dict(delta=5e-4)
res = []
for k in (0, 1, 2, 0, 2, 1, 0):
    x, st = capi.resolve(ctx, mesh, sc0.x, ys[k], **kw)
    res.append((k, x, st["steps"], st["searches"]))
    print(k, st["steps"], st["searches"], st["converged"], flush=True)
first = {}
for k, x, s, n in res:
    if k in first:
        print("scene", k, "same as first call:", np.array_equal(first[k].view(np.uint64), x.view(np.uint64)))
    else:
        first[k] = x
# fresh contexts
for k in (0, 1, 2):
    c2 = capi.Context(0)
    m2 = capi.Mesh.from_scene(c2, sc0)
    x, st = capi.resolve(c2, m2, sc0.x, ys[k], **kw)
    print("fresh ctx scene", k, st["steps"], "same as first:", np.array_equal(first[k].view(np.uint64), x.view(np.uint64)))
    m2.close(); c2.close()
# steps through the frame API
for k in (0, 1, 0):
    sc, v = scs[k]
    x, vv, st = capi.step(ctx, mesh, dyn, sc.x, v, **kw)
    print("step scene", k, st["resolve_steps"], st["searches"], flush=True)

"""Coloring quality at the bow knot's contact step: rows per dynamic vertex
(a lower bound on the colors: rows sharing a vertex form a clique) against
the colors the device coloring and the reference coloring use."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np

from paper_2211_04045_b200 import capi, scenes as S

sc = S.bow_knot()
ctx = capi.Context(0)
m = capi.Mesh.from_scene(ctx, sc)
x3, st = capi.resolve(ctx, m, sc.x, sc.y, delta=5e-4, step_limit=3)
P = capi.search(ctx, m, x3, 4e-3)
E = np.asarray(sc.edges).reshape(-1, 2)
y = np.where((sc.inv_mass == 0)[:, None], sc.x, sc.y)
et = np.linalg.norm(y[E[:, 0]] - y[E[:, 1]], axis=1)
R = capi.linearize(ctx, m, x3, P, et, delta=5e-4)
contact = R.kind != 4
dyn = sc.inv_mass > 0
cnt = np.zeros(sc.nv, np.int64)
for v in R.verts[contact].reshape(-1):
    if v >= 0 and dyn[v]:
        cnt[v] += 1
ecnt = np.zeros(sc.nv, np.int64)
for v in R.verts[~contact][:, :2].reshape(-1):
    if dyn[v]:
        ecnt[v] += 1
print(f"rows {len(R)} contact {contact.sum()}; max contact rows at a vertex {cnt.max()}, "
      f"max contact+edge rows at a vertex {(cnt + ecnt).max()}")
for mode in ("device", "reference"):
    nc, col = capi.color(ctx, m, R, mode=mode)
    print(f"{mode} coloring: {nc} colors; contact colors {col[contact].max() + 1}")
hist = np.bincount(np.bincount(capi.color(ctx, m, R, mode='device')[1][contact]))
print("rows per color (device): min", np.bincount(capi.color(ctx, m, R, mode='device')[1][contact]).min())

"""GPU stage parity for the backward-step stages, through the C-ABI:
linearize_all (constraints.cpp:181-220) -> the active-constraint index set and
every row value / Jacobian / diagonal; color_constraints (constraints.cpp:
222-288) in both coloring modes -> identical colors; assemble_lcp + PGS /
Jacobi sweeps + recover_target (lcp.cpp) -> identical multipliers, q and
recovered target. Inputs are the oracle's own pair sets on the fixture
battery (at the penetrating targets, so contact rows exist) and the
bow-knot-sized reef knot; comparisons are exact (integers) and bitwise (FP64)."""
import numpy as np
import pytest

import pyoracle as O
from paper_2211_04045_b200 import capi, scenes as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = capi.Context(0)
    yield c
    c.close()


def bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def _edge_targets(sc, pos):
    E = np.asarray(sc.edges).reshape(-1, 2)
    return np.linalg.norm(pos[E[:, 0]] - pos[E[:, 1]], axis=1)


def _cases():
    cases = [(sc.name, sc) for sc in S.scene_fixtures(0)]
    return cases


def _device_rows_as_oracle(R):
    """capi.Rows -> the fields an oracle Rows comparison needs (nverts from padding)."""
    nverts = (R.verts >= 0).sum(axis=1).astype(np.int32)
    return nverts


def _compare_rows(Ro, Rd):
    assert len(Ro) == len(Rd)
    assert np.array_equal(Ro.kind, Rd.kind)
    nv = _device_rows_as_oracle(Rd)
    assert np.array_equal(Ro.nverts, nv)
    for i in range(len(Ro)):
        n = Ro.nverts[i]
        assert np.array_equal(Ro.verts[i, :n], Rd.verts[i, :n]), i
    contact = Ro.kind != O.ROW_EDGE
    assert np.array_equal(Ro.pair_key[contact], Rd.pair_key[contact])  # the active-constraint index set
    assert np.array_equal(Ro.edge_index[~contact], Rd.edge_index[~contact])
    assert bits_equal(Ro.value, Rd.value)
    assert bits_equal(Ro.diag, Rd.diag)
    # Jacobian blocks of the row's vertices (padding blocks are zero on both sides)
    for i in range(len(Ro)):
        n = Ro.nverts[i]
        assert bits_equal(Ro.jac[i, :n], Rd.jac[i, :n]), i


def _inputs(sc, delta):
    y = np.asarray(sc.y, np.float64)
    P = O.search(sc, y, 4e-3)
    et = _edge_targets(sc, np.asarray(sc.x, np.float64))
    Ro = O.linearize(sc, y, P, et, delta=delta)
    return y, P, et, Ro


@pytest.mark.parametrize("name,sc", _cases())
def test_linearize_rows_bitexact(ctx, name, sc):
    delta = 1e-3
    y, P, et, Ro = _inputs(sc, delta)
    m = capi.Mesh.from_scene(ctx, sc)
    Rd = capi.linearize(ctx, m, y, P, et, delta=delta)
    _compare_rows(Ro, Rd)
    # gap family and no edge rows
    Ro2 = O.linearize(sc, y, P, et, delta=delta, family=1, edge_constraints=False)
    Rd2 = capi.linearize(ctx, m, y, P, et, delta=delta, family=1, edge_constraints=False)
    _compare_rows(Ro2, Rd2)


@pytest.mark.parametrize("mode", ["device", "reference"])
@pytest.mark.parametrize("name,sc", _cases())
def test_color_bitexact(ctx, name, sc, mode):
    y, P, et, Ro = _inputs(sc, 1e-3)
    m = capi.Mesh.from_scene(ctx, sc)
    Rd = capi.linearize(ctx, m, y, P, et, delta=1e-3)
    nco, co = O.color(sc, Ro, 0x5EED, mode={"reference": 0, "device": 1}[mode])
    ncd, cd = capi.color(ctx, m, Rd, seed=0x5EED, mode=mode)
    assert ncd == nco
    assert np.array_equal(cd, co)
    # a proper coloring: rows sharing a dynamic vertex differ
    dyn = np.asarray(sc.inv_mass) > 0
    seen = {}
    for i in range(len(Rd)):
        for v in Rd.verts[i]:
            if v >= 0 and dyn[v]:
                assert (v, cd[i]) not in seen, (i, seen.get((v, cd[i])))
                seen[(v, cd[i])] = i


@pytest.mark.parametrize("solver,sweeps", [("pgs", 1), ("pgs", 3), ("jacobi", 2)])
@pytest.mark.parametrize("name,sc", _cases()[:8])
def test_backward_bitexact(ctx, name, sc, solver, sweeps):
    y, P, et, Ro = _inputs(sc, 1e-3)
    m = capi.Mesh.from_scene(ctx, sc)
    Rd = capi.linearize(ctx, m, y, P, et, delta=1e-3)
    nc, col = O.color(sc, Ro, 0x5EED, mode=1)
    x = np.asarray(sc.x, np.float64)
    rng = np.random.default_rng(7)
    lam0 = np.where(rng.random(len(Ro)) < 0.3, rng.uniform(0, 1e-3, len(Ro)), 0.0)  # warm starts
    so = {"pgs": 0, "jacobi": 1}[solver]
    bo = O.backward(sc.inv_mass, Ro, col, nc, x, y, lam=lam0, solver=so, sweeps=sweeps)
    bd = capi.backward(ctx, sc.inv_mass, Rd, col, nc, x, y, lam=lam0, solver=solver, sweeps=sweeps)
    assert bits_equal(bo["q"], bd["q"])
    assert bits_equal(bo["lambda"], bd["lambda"])
    assert bits_equal(bo["y"], bd["y"])


def test_stage_chain_on_knot(ctx):
    """linearize -> color -> backward on a knot-sized set (reef knot target)."""
    sc = S.reef_knot()
    y = np.asarray(sc.y, np.float64)
    P = O.search(sc, y, 4e-3, cap=160 * sc.nv)
    et = _edge_targets(sc, np.asarray(sc.x, np.float64))
    Ro = O.linearize(sc, y, P, et, delta=5e-4)
    m = capi.Mesh.from_scene(ctx, sc)
    Rd = capi.linearize(ctx, m, y, P, et, delta=5e-4)
    _compare_rows(Ro, Rd)
    assert (Ro.kind != O.ROW_EDGE).sum() > 1000  # contact rows exist
    nco, co = O.color(sc, Ro, 0x5EED, mode=1)
    ncd, cd = capi.color(ctx, m, Rd, mode="device")
    assert ncd == nco and np.array_equal(cd, co)
    x = np.asarray(sc.x, np.float64)
    bo = O.backward(sc.inv_mass, Ro, co, nco, x, y)
    bd = capi.backward(ctx, sc.inv_mass, Rd, cd, ncd, x, y)
    assert bits_equal(bo["lambda"], bd["lambda"]) and bits_equal(bo["y"], bd["y"])


def test_stage_validation(ctx):
    sc = S.scene_fixtures(0)[0]
    m = capi.Mesh.from_scene(ctx, sc)
    R = capi.Rows(2)
    R.kind[:] = [4, 0]  # contact row after an edge row
    R.edge_index[:] = [0, -1]
    with pytest.raises(capi.TwError) as e:
        capi.color(ctx, m, R)
    assert e.value.code == capi.TW_EINVAL
    with pytest.raises(capi.TwError) as e:
        capi.backward(ctx, sc.inv_mass, capi.Rows(0), None, 0, sc.x, sc.y, solver="al20")
    assert e.value.code == capi.TW_EUNSUPPORTED

"""Pins the clean-room C oracle against the REAL reference.

oracle/_ref/libtwoway_ref.so is the reference's own source tree
(/root/reference/proj/src, compiled in place by oracle/Makefile.ref) built
against the Eigen-subset shim oracle/ref_shim/. These CPU tests assert that
  * scenes.scene_fixtures(0) reproduces the reference's testkit fixture battery
    (fixtures.cpp:304-314) bit for bit;
  * the oracle's resolve (reference coloring) equals the reference's resolve bit
    for bit (x_out, per-step max displacement, step/search counts, flags) on the
    battery across the config matrix (family, sweeps, solver, edge rows, fresh
    search);
  * the oracle's search pair sets and linearize/color rows equal the reference's;
  * the reference itself misses its own acceptance #11 threshold with one sweep
    (so the oracle's 1.34 is the reference's behaviour, not a restatement bug).
The library travels with the snapshot; where it was never built these skip.
"""
import numpy as np
import pytest

import pyoracle as O
import pyref as R
from paper_2211_04045_b200 import scenes as S

pytestmark = pytest.mark.skipif(not R.available() and not R.build(), reason="reference build absent")

FIXTURES = S.scene_fixtures(0)


def _bits(a):
    return np.ascontiguousarray(np.nan_to_num(a), np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def ref_fixtures():
    return [R.fixture(i, 0) for i in range(R.num_fixtures(0))]


def test_fixture_battery_is_the_references(ref_fixtures):
    assert len(ref_fixtures) == len(FIXTURES) == 21
    for sc, (name, m, x, y, benign, pen) in zip(FIXTURES, ref_fixtures):
        assert name == sc.name
        assert np.array_equal(_bits(x), _bits(sc.x)) and np.array_equal(_bits(y), _bits(sc.y)), name
        _, _, inv = m.state()
        assert np.array_equal(_bits(inv), _bits(sc.inv_mass)), name
        assert np.array_equal(m.edges(), sc.edges), name  # MeshState::finalize edge order
        T, Sd = m.topology()
        assert np.array_equal(T, sc.triangles) and np.array_equal(Sd, sc.strand_edges.reshape(-1, 2))
        assert (benign, pen) == (sc.benign, sc.penetrating)


CONFIGS = [
    {},
    {"constraint_family": "gap"},
    {"sweeps": 3},
    {"edge_constraints": 0},
    {"force_fresh_search": 1},
    {"eps": 0.25},
    {"step_limit": 4},
    {"solver": "jacobi", "step_limit": 200},
]


@pytest.mark.parametrize("i", range(len(FIXTURES)))
def test_oracle_resolve_equals_reference(ref_fixtures, i):
    sc = FIXTURES[i]
    m = ref_fixtures[i][1]
    for kw in CONFIGS:
        xr, sr = R.resolve(m, sc.x, sc.y, **kw)
        xo, so = O.resolve(sc, coloring_mode="reference", **kw)
        assert np.array_equal(_bits(xr), _bits(xo)), (sc.name, kw)
        assert np.array_equal(_bits(sr["step_max_disp"]), _bits(so["step_max_disp"])), (sc.name, kw)
        for k in ("steps", "searches", "converged", "hit_step_limit", "start_in_contact",
                  "step_law_violated", "stagnated"):
            assert sr[k] == so[k], (sc.name, kw, k)


@pytest.mark.parametrize("i", range(len(FIXTURES)))
def test_oracle_search_and_rows_equal_reference(ref_fixtures, i):
    sc = FIXTURES[i]
    m = ref_fixtures[i][1]
    for pos in (sc.x, sc.y, 0.5 * (sc.x + sc.y)):
        for d_max in (4e-3, 8e-3):
            keys, dist, flags = R.search(m, pos, d_max)
            P = O.search(sc, pos, d_max)
            assert np.array_equal(keys, P.keys) and np.array_equal(_bits(dist), _bits(P.dist))
            assert np.array_equal(flags & 2, P.flags & O.PF_ALL_STATIC)
        for fam in (0, 1):
            rr = R.linearize(m, pos, sc.y, family=fam)
            P = O.search(sc, pos, 4e-3)
            # edge targets exactly as resolve.cpp:53-55 ((y_i - y_j).norm())
            d = sc.y[sc.edges[:, 0]] - sc.y[sc.edges[:, 1]]
            et = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
            rows = O.linearize(sc, pos, P, et, family=fam)
            nc, col = O.color(sc, rows, 0x5EED, mode=0)  # reference coloring
            assert np.array_equal(rr["kind"], rows.kind)
            assert np.array_equal(rr["key"][rr["kind"] != O.ROW_EDGE], rows.pair_key[rows.kind != O.ROW_EDGE])
            assert np.array_equal(rr["edge_index"], rows.edge_index)
            assert np.array_equal(_bits(rr["value"]), _bits(rows.value))
            assert np.array_equal(_bits(rr["diag"]), _bits(rows.diag))
            assert rr["ncolors"] == nc and np.array_equal(rr["color"], col)


def test_reference_misses_its_own_acceptance_11(ref_fixtures):
    """acceptance.cpp:455-479: the real reference gives stretch 1.345 (guarded,
    one sweep) > 1.15 -- the oracle's value; 4 sweeps meet the threshold."""
    sc = FIXTURES[3]
    assert sc.name == "spike_theta135"
    m = ref_fixtures[3][1]

    def stretch(x):
        d = sc.y[sc.edges[:, 0]] - sc.y[sc.edges[:, 1]]
        ly = np.sqrt((d[:, 0] ** 2 + d[:, 1] ** 2) + d[:, 2] ** 2)
        ok = ly >= 1e-12
        e = x[sc.edges[ok, 0]] - x[sc.edges[ok, 1]]
        return np.max(np.sqrt((e[:, 0] ** 2 + e[:, 1] ** 2) + e[:, 2] ** 2) / ly[ok])

    guarded = stretch(R.resolve(m, sc.x, sc.y)[0])
    free = stretch(R.resolve(m, sc.x, sc.y, edge_constraints=0)[0])
    four = stretch(R.resolve(m, sc.x, sc.y, sweeps=4)[0])
    assert guarded > 1.15 and free > guarded and four <= 1.15
    assert guarded == stretch(O.resolve(sc)[0])


def test_reference_ccd_counts_equal_oracle(ref_fixtures):
    for i in (0, 3, 6, 8, 9):
        sc = FIXTURES[i]
        m = ref_fixtures[i][1]
        assert R.ccd_certify(m, sc.x, sc.y) == O.ccd_certify(sc, sc.x, sc.y), sc.name

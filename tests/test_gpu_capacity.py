"""Capacity growth: a context whose pair, candidate, partner-slot, archive,
color and reference-coloring capacities all start tiny (TW_TINY_CAPS) must
grow them by device-flagged overflow + rerun and return exactly what a
normally sized context returns."""
import os

import numpy as np
import pytest

from paper_2211_04045_b200 import capi, scenes as S

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def normal():
    c = capi.Context(0)
    yield c
    c.close()


@pytest.fixture
def ctxs(normal):
    os.environ["TW_TINY_CAPS"] = "1"  # read at context creation: a fresh tiny context per test
    try:
        tiny = capi.Context(0)
    finally:
        del os.environ["TW_TINY_CAPS"]
    yield normal, tiny
    tiny.close()


CASES = [(sc, {}) for sc in S.scene_fixtures(0)[:6]] + [(S.reef_knot(), dict(delta=5e-4))]


@pytest.mark.parametrize("mode", ["device", "reference"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0].name)
def test_tiny_capacities_grow_to_identical_results(ctxs, case, mode):
    sc, kw = case
    if mode == "reference" and sc.nv > 10000:
        pytest.skip("reference coloring replays on one thread: fixture sizes only")
    normal, tiny = ctxs
    mn, mt = capi.Mesh.from_scene(normal, sc), capi.Mesh.from_scene(tiny, sc)
    xn, sn = capi.resolve(normal, mn, sc.x, sc.y, coloring_mode=mode, **kw)
    xt, stt = capi.resolve(tiny, mt, sc.x, sc.y, coloring_mode=mode, **kw)
    assert np.array_equal(_bits(xn), _bits(xt))
    assert (sn["steps"], sn["searches"], sn["num_pairs"]) == (stt["steps"], stt["searches"], stt["num_pairs"])
    if sn["num_pairs"] > 256:
        assert stt["retries"] > 0  # the growth path did run
    # the stage search grows its own way
    pn, pt = capi.search(normal, mn, sc.y, 4e-3), capi.search(tiny, mt, sc.y, 4e-3)
    assert np.array_equal(pn.keys, pt.keys) and np.array_equal(_bits(pn.dist), _bits(pt.dist))


@pytest.fixture
def wide_slots(normal):
    os.environ["TW_QUERY_SLOTS"] = "256"  # > 128 partner slots: the in-memory partner sort
    try:
        wide = capi.Context(0)
    finally:
        del os.environ["TW_QUERY_SLOTS"]
    yield normal, wide
    wide.close()


@pytest.mark.parametrize("sc", [S.reef_knot(), S.bow_knot()], ids=lambda s: s.name)
def test_partner_sort_paths_agree(wide_slots, sc):
    """Partner lists are sorted in registers inside the key emission when the
    slot capacity is <= 128 and by ph_query_totals in memory above that: both
    orders must be the reference's key order."""
    normal, wide = wide_slots
    mn, mw = capi.Mesh.from_scene(normal, sc), capi.Mesh.from_scene(wide, sc)
    pn, pw = capi.search(normal, mn, sc.x, 4e-3), capi.search(wide, mw, sc.x, 4e-3)
    k = pn.keys.astype(np.uint64)
    assert len(k) > 0 and np.all(k[1:] > k[:-1])  # strictly ascending keys
    assert np.array_equal(pn.keys, pw.keys) and np.array_equal(_bits(pn.dist), _bits(pw.dist))
    xn, sn = capi.resolve(normal, mn, sc.x, sc.y, delta=5e-4, step_limit=3)
    xw, sw = capi.resolve(wide, mw, sc.x, sc.y, delta=5e-4, step_limit=3)
    assert np.array_equal(_bits(xn), _bits(xw)) and sn["num_pairs"] == sw["num_pairs"]


def test_record_path_grows_on_demand(ctxs):
    """record_path keeps the path on the device in a buffer that starts small
    (2 states in a tiny context, 33 normally) and grows through the capacity
    rerun: the recorded path has exactly steps + 1 states, starts at x, ends at
    x_out, and equals a normally sized context's path bit for bit."""
    normal, tiny = ctxs
    for sc in S.scene_fixtures(0)[9:12]:  # random fixtures: tens to hundreds of steps
        out = []
        for c in (normal, tiny):
            m = capi.Mesh.from_scene(c, sc)
            x, st = capi.resolve(c, m, sc.x, sc.y, record_path=True)
            p = st["path"]
            assert len(p) == st["steps"] + 1
            assert np.array_equal(_bits(p[0]), _bits(sc.x)) and np.array_equal(_bits(p[-1]), _bits(x))
            out.append(p)
            m.close()
        assert np.array_equal(_bits(out[0]), _bits(out[1]))


@pytest.mark.parametrize("ctas", ["1", "4"])
def test_pgs_subgrid_size_is_invisible(normal, ctas):
    """The PGS color phases run on a sub-grid of sm_count x TW_PGS_CTAS_PER_SM
    CTAs (default 2): 1 and 4 per SM must give bit-identical results."""
    os.environ["TW_PGS_CTAS_PER_SM"] = ctas
    try:
        other = capi.Context(0)
    finally:
        del os.environ["TW_PGS_CTAS_PER_SM"]
    for sc, kw in [(S.scene_fixtures(0)[3], {}), (S.reef_knot(**S.FRAME_DEFAULTS), dict(delta=5e-4))]:
        out = []
        for c in (normal, other):
            m = capi.Mesh.from_scene(c, sc)
            x, st = capi.resolve(c, m, sc.x, sc.y, coloring_mode="device", **kw)
            out.append((x, st["steps"], st["step_max_disp"]))
            m.close()
        assert np.array_equal(_bits(out[0][0]), _bits(out[1][0])) and out[0][1] == out[1][1]
        assert np.array_equal(_bits(out[0][2]), _bits(out[1][2]))
    other.close()

"""Device CCD certification (testkit/ccd.cpp:339-498)
against the oracle certifier: identical violation and certain-violation counts
on every segment of the fixture battery's resolve paths, on the direct
(penetrating) x -> y segments, and on random blobs; and the bow-knot resolve
path — too large for the CPU certifier in a test — certified on the device."""
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


FIX = [sc for sc in S.scene_fixtures(0) if len(sc.triangles) or len(sc.edges)]


@pytest.mark.parametrize("sc", FIX, ids=lambda s: s.name)
def test_ccd_matches_oracle_on_paths_and_direct_segments(ctx, sc):
    m = capi.Mesh.from_scene(ctx, sc)
    _, st = O.resolve(sc, record_path=True)
    path = st["path"]
    for i in range(len(path) - 1):
        assert capi.ccd_certify(ctx, m, path[i], path[i + 1]) == O.ccd_certify(sc, path[i], path[i + 1]), i
    # the direct move to the (penetrating) target
    assert capi.ccd_certify(ctx, m, sc.x, sc.y) == O.ccd_certify(sc, sc.x, sc.y)


@pytest.mark.parametrize("seed", range(6))
def test_ccd_matches_oracle_on_random_motion(ctx, seed):
    sc = S.fixture_random(seed, seed)
    rng = np.random.default_rng(seed)
    x1 = np.asarray(sc.x) + rng.normal(0, 4e-3, size=np.asarray(sc.x).shape)
    m = capi.Mesh.from_scene(ctx, sc)
    assert capi.ccd_certify(ctx, m, sc.x, x1) == O.ccd_certify(sc, sc.x, x1)


@pytest.mark.parametrize("squeeze", [-0.2e-3, 1e-3])
def test_bow_knot_path_is_intersection_free(ctx, squeeze):
    """The bench knot (plies pressed to a 0.2 mm gap) and a penetrating
    variant (target plies cross by up to 2 mm): the raw target motion of the
    latter collides, the resolve path of both certifies clean."""
    sc = S.ply_knot(n_along=1870, squeeze=squeeze, slide=3e-3)
    m = capi.Mesh.from_scene(ctx, sc)
    v_raw, _ = capi.ccd_certify(ctx, m, sc.x, sc.y)
    if squeeze > 0:
        assert v_raw > 0
    x, st = capi.resolve(ctx, m, sc.x, sc.y, delta=5e-4, record_path=True, step_limit=64)
    assert st["converged"] or squeeze > 0  # a crossing target is approached, not reached
    viol, cert = capi.ccd_certify_path(ctx, m, st["path"])
    assert cert == 0 and viol == 0, (viol, cert, st["steps"])

"""The API surface added this round, against the oracle / the reference build:
linearize_all's re-evaluation data (flavor, ref_volume, gap weights, denom:
tw_stage_linearize_ex) and constraint_value_at, bit for bit with the oracle;
normal_flow_target bit for bit with the reference build's
(normal_flow.cpp:38-81); _twoway.certify_segment / normal_flow_target with the
reference module's signatures."""
import numpy as np
import pytest

import pyoracle as O
import pyref as R
from paper_2211_04045_b200 import scenes as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2211_04045_b200 import capi

    c = capi.Context(0)
    yield c
    c.close()


def _bits(a):
    return np.ascontiguousarray(np.nan_to_num(a), np.float64).view(np.uint64)


@pytest.mark.parametrize("i", [0, 3, 4, 6, 8, 9, 12])
@pytest.mark.parametrize("family", [0, 1])
def test_linearize_eval_data_and_value_at_match_oracle(ctx, i, family):
    from paper_2211_04045_b200 import capi

    sc = S.scene_fixtures(0)[i]
    m = capi.Mesh.from_scene(ctx, sc)
    pos = 0.5 * (sc.x + sc.y)
    P = O.search(sc, pos, 4e-3)
    d = sc.y[sc.edges[:, 0]] - sc.y[sc.edges[:, 1]]
    et = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
    ro = O.linearize(sc, pos, P, et, family=family)
    rd = capi.linearize(ctx, m, pos, P, et, family=family, ex=True)
    assert len(rd) == len(ro)
    assert np.array_equal(rd.flavor, ro.flavor)
    assert np.array_equal(_bits(rd.ref_volume), _bits(ro.ref_volume))
    assert np.array_equal(_bits(rd.gap_weights), _bits(ro.gap_weights))
    assert np.array_equal(_bits(rd.denom), _bits(ro.denom))
    for where in (sc.x, sc.y):
        vd = capi.constraint_value_at(ctx, rd, where)
        vo = np.array([O.constraint_value_at(ro, k, where) for k in range(len(ro))])
        assert np.array_equal(_bits(vd), _bits(vo))
    m.close()


@pytest.mark.skipif(not R.available(), reason="reference build absent")
@pytest.mark.parametrize("beta", [5e-4, -5e-4])
def test_normal_flow_target_matches_reference(ctx, beta):
    from paper_2211_04045_b200 import capi

    m = S.make_icosphere(3, 0.03, (0, 0, 0))
    rm = R.RefMesh(m.positions, m.triangles)
    yr = R.normal_flow_target(rm, m.positions, beta=beta, alpha_smooth=0.5)
    yd = capi.normal_flow_target(ctx, m.positions, m.triangles, beta=beta, alpha=0.5)
    assert np.array_equal(_bits(yd), _bits(yr))
    with pytest.raises(ValueError):  # require_closed_manifold
        capi.normal_flow_target(ctx, m.positions, m.triangles[:-1])


def test_twoway_module_surface():
    from paper_2211_04045_b200 import _twoway

    sc = S.scene_fixtures(0)[1]
    d = _twoway.certify_segment(sc.x, sc.y, sc.triangles)
    assert set(d) == {"certain", "uncertain"} and d["certain"] > 0  # the raw target motion penetrates
    x, st = _twoway.resolve(sc.x, sc.y, sc.triangles, inv_mass=sc.inv_mass, record_path=True)
    path = st["path"]
    for a, b in zip(path[:-1], path[1:]):
        assert _twoway.certify_segment(a, b, sc.triangles)["certain"] == 0
    m = S.make_icosphere(2, 0.03, (0, 0, 0))
    y = _twoway.normal_flow_target(m.positions, m.triangles, beta=5e-4, alpha=0.5)
    assert y.shape == m.positions.shape and np.all(np.isfinite(y))

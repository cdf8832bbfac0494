"""The BASELINE.json config scenes on the device. CFG1 (cloth on a static
sphere, 6.7K vertices, ~35 Alg.-1 steps) end to end against the oracle in both
coloring modes, bit for bit; a reduced CFG4 codimensional mix (closed bodies,
strands, particles) likewise; the full CFG4
resolves to convergence with its path certified on the device."""
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


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _same_resolve(ctx, sc, mode, **kw):
    m = capi.Mesh.from_scene(ctx, sc)
    xd, sd = capi.resolve(ctx, m, sc.x, sc.y, coloring_mode=mode, trace=True, **kw)
    xo, so = O.resolve(sc, coloring_mode=mode, trace=True, **kw)
    assert (sd["steps"], sd["searches"], sd["converged"]) == (so["steps"], so["searches"], so["converged"])
    assert np.array_equal(_bits(xd), _bits(xo))
    for td, to in zip(sd["trace"], so["trace"]):
        for k in ("searched", "num_pairs", "num_contact_rows", "num_edge_rows", "num_colors"):
            assert td[k] == to[k], k
    return sd


@pytest.mark.parametrize("mode", ["device", "reference"])
def test_cfg1_cloth_on_sphere_bitexact(ctx, mode):
    st = _same_resolve(ctx, S.cloth_on_sphere(), mode)
    assert st["steps"] > 10  # a long resolve: many searches and contact steps


def test_cfg4_reduced_codim_mix_bitexact(ctx):
    sc = S.codim_mix(n_bodies=2, n_strands=36, strand_segments=32, n_particles=3000)
    kinds = set()
    P = O.search(sc, sc.y, 4e-3)
    for k in P.keys:
        kinds.add((int(k) >> 62, (int(k) >> 60) & 3))
    assert {(0, 2), (1, 1)} <= kinds  # VT, EE at the target (VV / VE: the fixture battery's particles)
    _same_resolve(ctx, sc, "device")


def test_cfg4_codim_mix_full_certified(ctx):
    sc = S.codim_mix()
    m = capi.Mesh.from_scene(ctx, sc)
    x, st = capi.resolve(ctx, m, sc.x, sc.y, record_path=True, step_limit=64)
    assert st["converged"]
    viol, cert = capi.ccd_certify_path(ctx, m, st["path"])
    assert viol == 0 and cert == 0

"""The friction_filter restatement (oracle/pyoracle.py, dynamics.cpp:272-324)
pinned bit for bit to the reference's own friction_filter (oracle/_ref, built
from /root/reference/proj/src/dynamics.cpp) on the friction scenes of
tests/test_gpu_friction.py: short and long dependency chains, the Coulomb
cap binding or not, static -0.0 coordinates. CPU only."""
import numpy as np
import pytest

import pyoracle as O
import pyref as R
from test_gpu_friction import SCENES

pytestmark = pytest.mark.skipif(not R.available(), reason="reference build absent")


class _Mesh:
    def __init__(self, m, edges):
        self.inv_mass = m.inv_mass
        self.edges = edges
        self.triangles = np.asarray(m.triangles, np.int32).reshape(-1, 3)


@pytest.mark.parametrize("mu", [0.0, 0.3, 5.0])
@pytest.mark.parametrize("name", ["drape", "drape_neg_zero", "sphere"])
def test_friction_restatement_matches_reference(name, mu):
    m, x, yt = SCENES[name]()
    rm = R.RefMesh(x, m.triangles, m.strand_edges, m.inv_mass, np.zeros_like(x))
    yr = R.friction_filter(rm, x, x, yt, d_max=4e-3, mu=mu)
    yo = O.friction_filter(_Mesh(m, rm.edges()), x, yt, 4e-3, mu)
    assert np.any(yr != yt)
    assert np.array_equal(yo.view(np.uint64), yr.view(np.uint64)), np.abs(yo - yr).max()

"""Device friction_filter (csrc/tw_dynamics.cu, k_friction) against the REAL
reference's friction_filter (dynamics.cpp:272-324, oracle/_ref).

The reference runs a Gauss-Seidel pass over the pair set in pair order; the
device runs the same pass as a dataflow over the pairs' shared vertices. The
filtered target must be bit-identical, on scenes where the dependency chains
are short (cloth over a static patch / sphere) and long (a dense patch whose
vertices sit in dozens of pairs), with and without the Coulomb cap binding,
and with static vertices carrying -0.0 coordinates (whose +-0 writes the
device must reproduce).
"""
import numpy as np
import pytest

import pyref as R
from paper_2211_04045_b200 import scenes as S

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="reference build absent")]


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def drape(n=16, spacing=4e-3, gap=0.6e-3, neg_zero=False, seed=3, push=1.2e-3, slide=1.5e-3):
    """A dynamic patch `gap` above a static one; the target pushes it `push`
    down into the static patch and slides it `slide` sideways, plus jitter."""
    top = S.make_grid_patch(n, n, spacing * (n - 1), spacing * (n - 1), (0, 0, gap))
    S.compute_lumped_masses(top, 0.1, 0.0)
    bot = S.make_grid_patch(n, n, spacing * (n - 1), spacing * (n - 1), (0.001, 0.0013, 0.0))
    bot.inv_mass = np.zeros(len(bot.positions))
    if neg_zero:
        bot.positions[:, 2] = -0.0
    S.append_mesh(bot, top)
    x = bot.positions.copy()
    rng = np.random.default_rng(seed)
    y = x.copy()
    dyn = bot.inv_mass > 0
    y[dyn, 2] -= push
    y[dyn, 0] += slide
    y[dyn] += rng.uniform(-2e-4, 2e-4, (int(dyn.sum()), 3))
    return bot, x, y


def sphere_contact(n=24, spacing=4e-3, gap=0.5e-3):
    """CFG1-like: a cloth patch resting `gap` above the top of a static
    icosphere (s = 3), pushed into it and slid sideways."""
    sphere = S.make_icosphere(3, 0.05, (0, 0, 0))
    sphere.inv_mass = np.zeros(len(sphere.positions))
    size = spacing * (n - 1)
    cloth = S.make_grid_patch(n, n, size, size, (-size / 2, -size / 2, 0.05 + gap))
    S.compute_lumped_masses(cloth, 0.1, 0.0)
    S.append_mesh(sphere, cloth)
    x = sphere.positions.copy()
    y = x.copy()
    dyn = sphere.inv_mass > 0
    y[dyn, 2] -= 2e-3
    y[dyn, 1] += 1e-3
    return sphere, x, y


SCENES = {
    "drape": lambda: drape(),
    "drape_dense": lambda: drape(n=20, spacing=2.0e-3),       # in-plane pairs: long chains
    "drape_neg_zero": lambda: drape(neg_zero=True),            # static -0.0 coordinates
    "sphere": lambda: sphere_contact(),
}


@pytest.fixture(scope="module")
def ctx():
    from paper_2211_04045_b200 import capi

    c = capi.Context(0)
    yield c
    c.close()


def _meshes(ctx, m, x, **model):
    from paper_2211_04045_b200 import capi

    mesh = capi.Mesh(ctx, len(x), m.inv_mass, (), m.strand_edges, m.triangles)
    dyn = capi.Dynamics(ctx, mesh, x, **model)
    rm = R.RefMesh(x, m.triangles, m.strand_edges, m.inv_mass, np.zeros_like(x))
    assert np.array_equal(rm.edges(), mesh.edges)
    return mesh, dyn, rm


@pytest.mark.parametrize("mu", [0.0, 0.3, 5.0])
@pytest.mark.parametrize("name", list(SCENES))
def test_friction_filter_bitexact(ctx, name, mu):
    from paper_2211_04045_b200 import capi

    m, x, yt = SCENES[name]()
    model = dict(mu=mu)
    mesh, dyn, rm = _meshes(ctx, m, x, **model)
    y = capi.friction_filter(ctx, mesh, dyn, x, yt, d_max=4e-3)
    yr = R.friction_filter(rm, x, x, yt, d_max=4e-3, **model)
    changed = np.any(_bits(yr).reshape(-1, 3) != _bits(yt).reshape(-1, 3), axis=1)
    assert changed.sum() > 10, "the scene must put pairs inside the repulsion radius at the target"
    diff = np.any(_bits(y).reshape(-1, 3) != _bits(yr).reshape(-1, 3), axis=1)
    assert not diff.any(), (int(diff.sum()), np.abs(y - yr).max())
    if name == "drape_neg_zero":  # the static plane keeps its (signed) zeros exactly as the reference
        st = m.inv_mass == 0
        assert np.array_equal(np.signbit(y[st, 2]), np.signbit(yr[st, 2]))
    dyn.close()
    mesh.close()


def test_friction_filter_is_deterministic(ctx):
    """The dataflow schedule varies run to run; the result must not."""
    from paper_2211_04045_b200 import capi

    m, x, yt = drape(n=24, spacing=2.0e-3)
    mesh, dyn, rm = _meshes(ctx, m, x, mu=0.5)
    y0 = capi.friction_filter(ctx, mesh, dyn, x, yt)
    for _ in range(5):
        assert np.array_equal(_bits(capi.friction_filter(ctx, mesh, dyn, x, yt)), _bits(y0))
    dyn.close()
    mesh.close()


def test_friction_full_replay_fallback():
    """TW_FR_MAX_ROUNDS=0: the replay runs over every pair (the fallback for a
    writer set that does not settle) -- same bits as the reference."""
    import subprocess
    import sys

    code = (
        "import sys, numpy as np; sys.path[:0] = ['tests', 'oracle', '.']\n"
        "import pyref as R, test_gpu_friction as T\n"
        "from paper_2211_04045_b200 import capi\n"
        "ctx = capi.Context(0)\n"
        "for name in ('drape_dense', 'drape_neg_zero'):\n"
        "    m, x, yt = T.SCENES[name]()\n"
        "    mesh, dyn, rm = T._meshes(ctx, m, x, mu=0.3)\n"
        "    y = capi.friction_filter(ctx, mesh, dyn, x, yt)\n"
        "    yr = R.friction_filter(rm, x, x, yt, d_max=4e-3, mu=0.3)\n"
        "    assert np.array_equal(y.view(np.uint64), yr.view(np.uint64)), name\n"
        "print('ok')\n")
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "TW_FR_MAX_ROUNDS": "0"})
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_friction_filter_knot(ctx):
    """A 200-segment knot frame (two plies, 8K vertices): the tightening target
    penetrates where the knot is tightest."""
    from paper_2211_04045_b200 import capi

    frame, v0 = S.knot_frame(n_along=200)
    x = frame.x
    yt = x + 0.01 * v0
    model = dict(mu=0.4, dt=0.01)
    mesh = capi.Mesh.from_scene(ctx, frame)
    dyn = capi.Dynamics(ctx, mesh, x, **model)
    rm = R.RefMesh(x, frame.triangles, frame.strand_edges, frame.inv_mass, np.zeros_like(x))
    assert np.array_equal(rm.edges(), mesh.edges)
    y = capi.friction_filter(ctx, mesh, dyn, x, yt, d_max=4e-3)
    yr = R.friction_filter(rm, x, x, yt, d_max=4e-3, **model)
    assert not np.array_equal(_bits(yr), _bits(yt))
    assert np.array_equal(_bits(y), _bits(yr)), np.abs(y - yr).max()
    dyn.close()
    mesh.close()


def test_step_with_friction(ctx):
    """step() with mu > 0 = (newton target + friction_filter) -> resolve; the
    target matches the reference's (PCG tolerance, as tests/test_gpu_dynamics.py
    states), and its friction pass is the bit-exact filter of the device's own
    Newton target."""
    from paper_2211_04045_b200 import capi

    m, x, _ = drape(gap=0.8e-3)
    v = np.zeros_like(x)
    dyn_v = m.inv_mass > 0
    v[dyn_v, 2] = -0.05
    v[dyn_v, 0] = 0.2
    model = dict(mu=0.3, repulsion_stiffness=0.05)  # the target stays inside the radius, sliding
    mesh, dyn, rm = _meshes(ctx, m, x, **model)
    dyn0 = capi.Dynamics(ctx, mesh, x, repulsion_stiffness=0.05)  # same model without friction
    y, _, st = capi.newton_target(ctx, mesh, dyn, x, v, x)
    y0, _, _ = capi.newton_target(ctx, mesh, dyn0, x, v, x)
    assert np.array_equal(_bits(y), _bits(capi.friction_filter(ctx, mesh, dyn, x, y0)))
    assert not np.array_equal(_bits(y), _bits(y0))
    rm2 = R.RefMesh(x, m.triangles, m.strand_edges, m.inv_mass, v)
    yr, _, _, conv = R.newton_target(rm2, x, x, d_max=4e-3, **model)
    assert conv
    scale = np.abs(yr - x).max()
    assert np.abs(y - yr).max() <= 1e-5 * scale, (np.abs(y - yr).max(), scale)
    xs, vs, sst = capi.step(ctx, mesh, dyn, x, v, coloring_mode="reference")
    xr, sr = capi.resolve(ctx, mesh, x, y, coloring_mode="reference")
    assert np.array_equal(_bits(xs), _bits(xr))
    assert sst["resolve_steps"] == sr["steps"]
    dyn0.close()
    dyn.close()
    mesh.close()


def test_negative_mu_is_rejected(ctx):
    from paper_2211_04045_b200 import capi

    m, x, _ = drape()
    mesh = capi.Mesh(ctx, len(x), m.inv_mass, (), m.strand_edges, m.triangles)
    with pytest.raises(ValueError):
        capi.Dynamics(ctx, mesh, x, mu=-0.1)
    with pytest.raises(ValueError):
        capi.Dynamics(ctx, mesh, x, dt=0.0)
    mesh.close()

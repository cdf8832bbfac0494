"""Device dynamics (csrc/tw_dynamics.cu) against the REAL reference's
dynamics.cpp (oracle/_ref, built from /root/reference/proj/src):

  * gradient_and_hessian + add_repulsion: the gradient is gathered in the
    reference's accumulation order and matches bit for bit (no bending);
  * newton_target: the block-Jacobi PCG target matches within the PCG
    tolerance (both solve to a 1e-6 relative residual; stated bound below);
  * step(): positions and velocities after a full simulation step (target +
    resolve + velocity update) match within the same bound, with identical
    resolve step counts.
"""
import numpy as np
import pytest

import pyref as R
from paper_2211_04045_b200 import scenes as S

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="reference build absent")]

# |y_dev - y_ref|_inf <= TOL_REL * |y_ref - x|_inf: two CG implementations that
# both stop at a 1e-6 relative residual on a mass-dominated (well-conditioned)
# system agree to ~1e-6 of the step; 1e-5 leaves room for the conditioning.
TOL_REL = 1e-5


def drape(n=16, spacing=4e-3, gap=2.5e-3, v_down=0.2, static_below=True, strands=False, jitter=0.05, model=None):
    """A dynamic cloth patch over a static one, falling with v_down (m/s) plus
    a seeded per-vertex velocity jitter (so the springs load and the CG has
    work to do)."""
    top = S.make_grid_patch(n, n, spacing * (n - 1), spacing * (n - 1), (0, 0, gap))
    S.compute_lumped_masses(top, 0.1, 0.0)
    if static_below:
        bot = S.make_grid_patch(n, n, spacing * (n - 1), spacing * (n - 1), (0.001, 0.0013, 0.0))
        bot.inv_mass = np.zeros(len(bot.positions))
        S.append_mesh(bot, top)
        m = bot
    else:
        m = top
    if strands:
        st = S.make_strand(12, (0.002, 0.03, gap * 0.5), (0.05, 0.031, gap * 0.5))
        S.compute_lumped_masses(st, 0.0, 0.05)
        S.append_mesh(m, st)
    v = np.random.default_rng(7).uniform(-jitter, jitter, m.positions.shape)
    dyn = m.inv_mass > 0
    v[dyn, 2] -= v_down
    v[~dyn] = 0.0
    return m, v


# scene -> (geometry, energy-model overrides). "drape" starts inside the
# repulsion radius (0.8 mm < 1 mm) with a repulsion stiffness matched to the
# 0.1 kg/m^2 cloth (the default 1e3 N/m would dominate m/dt^2 by 1e5).
SCENES = {
    "drape": dict(gap=0.8e-3, model=dict(repulsion_stiffness=0.5)),
    "drape_fast": dict(v_down=0.6),
    "drape_strands": dict(strands=True, v_down=0.4),
    "free_patch": dict(static_below=False, v_down=0.0),
}
MODELS = {
    "default": dict(),
    "bending": dict(bending_stiffness=0.02),
    "stiff": dict(spring_stiffness=400.0, repulsion_stiffness=5e3, dt=1 / 30),
}


def _model(name, model):
    return {**MODELS[model], **(SCENES[name].get("model") or {})}


@pytest.fixture(scope="module")
def ctx():
    from paper_2211_04045_b200 import capi

    c = capi.Context(0)
    yield c
    c.close()


def _setup(ctx, name, model):
    from paper_2211_04045_b200 import capi

    m, v = drape(**SCENES[name])
    x = m.positions.copy()
    # both sides derive the edge order from (strands, triangles) as MeshState::finalize does
    mesh = capi.Mesh(ctx, len(x), m.inv_mass, (), m.strand_edges, m.triangles)
    dyn = capi.Dynamics(ctx, mesh, x, **_model(name, model))
    rm = R.RefMesh(x, m.triangles, m.strand_edges, m.inv_mass, v)
    assert np.array_equal(rm.edges(), mesh.edges)
    return m, x, v, mesh, dyn, rm


@pytest.mark.parametrize("model", list(MODELS))
@pytest.mark.parametrize("name", list(SCENES))
def test_newton_target_matches_reference(ctx, name, model):
    from paper_2211_04045_b200 import capi

    m, x, v, mesh, dyn, rm = _setup(ctx, name, model)
    y, g, st = capi.newton_target(ctx, mesh, dyn, x, v, x, d_max=4e-3)
    yr, gr, it_r, conv_r = R.newton_target(rm, x, x, d_max=4e-3, **_model(name, model))
    assert conv_r  # the comparison is between converged solves
    if _model(name, model).get("bending_stiffness", 0.0) == 0.0:
        assert np.array_equal(g.view(np.uint64), gr.view(np.uint64)), np.abs(g - gr).max()
    else:  # hinge coefficients come from a different null-space computation
        assert np.allclose(g, gr, rtol=1e-9, atol=1e-12 * np.abs(gr).max())
    scale = np.abs(yr - x).max()
    assert scale > 0
    assert np.abs(y - yr).max() <= TOL_REL * scale, (np.abs(y - yr).max(), scale)
    assert bool(st["pcg_converged"]) == conv_r
    # iteration counts of two CG implementations differ with rounding (the
    # recurrence q = H z + beta q here vs a fresh H p there): within 25%
    assert abs(st["pcg_iterations"] - it_r) <= max(3, it_r // 4), (st["pcg_iterations"], it_r)
    dyn.close()
    mesh.close()


@pytest.mark.parametrize("name", ["drape", "free_patch"])
def test_step_matches_reference(ctx, name):
    """Three consecutive frames against the reference's step(). On these
    scenes resolve is well conditioned, so the PCG-level difference of the
    targets stays at that level in x and v."""
    from paper_2211_04045_b200 import capi

    m, x, v, mesh, dyn, rm = _setup(ctx, name, "default")
    xs, vs = x.copy(), v.copy()
    xr_prev = x.copy()
    for k in range(3):
        xs_new, vs_new, st = capi.step(ctx, mesh, dyn, xs, vs, coloring_mode="reference")
        xr, vr, nsteps, _ = R.step(rm, x, energy=_model(name, "default"))
        scale = max(np.abs(xr - xr_prev).max(), 1e-9)
        assert np.abs(xs_new - xr).max() <= 10 * TOL_REL * scale, (k, np.abs(xs_new - xr).max(), scale)
        assert np.abs(vs_new - vr).max() <= 10 * TOL_REL * scale / 0.01
        assert st["resolve_steps"] == nsteps
        assert st["resolve_converged"]
        # continue both from the reference state so the comparison stays per-frame
        xs, vs, xr_prev = xr.copy(), vr.copy(), xr.copy()
    dyn.close()
    mesh.close()


@pytest.mark.parametrize("name", list(SCENES))
def test_step_is_target_then_resolve(ctx, name):
    """step() = newton_target -> resolve -> v = (x - x0)/dt exactly (device
    composition, bit for bit), on every scene -- including drape_fast, where
    resolve is so sensitive that a 1e-12 change of y changes x_out by mm
    (measured with the reference build), so only the target is compared with
    the reference there."""
    from paper_2211_04045_b200 import capi

    m, x, v, mesh, dyn, rm = _setup(ctx, name, "default")
    y, _, _ = capi.newton_target(ctx, mesh, dyn, x, v, x)
    xs, vs, st = capi.step(ctx, mesh, dyn, x, v, coloring_mode="reference")
    xr, sr = capi.resolve(ctx, mesh, x, y, coloring_mode="reference")
    assert np.array_equal(xs.view(np.uint64), xr.view(np.uint64))
    assert st["resolve_steps"] == sr["steps"]
    dt = _model(name, "default").get("dt", 0.01)
    vexp = np.where(m.inv_mass[:, None] > 0, (xr - x) / dt, 0.0)
    assert np.array_equal(vs.view(np.uint64), vexp.view(np.uint64))
    dyn.close()
    mesh.close()


def test_step_is_intersection_free(ctx):
    from paper_2211_04045_b200 import capi

    m, x, v, mesh, dyn, rm = _setup(ctx, "drape_fast", "default")
    for _ in range(3):
        # the frame's certified path is resolve's piecewise-linear path from x
        # to x_next (the straight segment x -> x_next need not be free)
        y, _, _ = capi.newton_target(ctx, mesh, dyn, x, v, x)
        xp, sp = capi.resolve(ctx, mesh, x, y, record_path=True)
        xn, v, st = capi.step(ctx, mesh, dyn, x, v)
        assert np.array_equal(xn.view(np.uint64), xp.view(np.uint64))
        assert capi.ccd_certify_path(ctx, mesh, sp["path"])[1] == 0
        x = xn


def test_concurrent_contexts_are_deterministic():
    """Two contexts sharing the device (tw_ctx_set_grid_share, own streams,
    threads) step independent frames at the same time and return bit for bit
    what one full-device context returns (the configs[4] batch mode)."""
    import threading

    from paper_2211_04045_b200 import capi

    scenes = [S.knot_frame(n_along=300, jitter_seed=s) for s in (1, 2, 3, 4)]
    solo = capi.Context(0)
    ref = []
    for sc, v in scenes:
        m = capi.Mesh.from_scene(solo, sc)
        d = capi.Dynamics(solo, m, sc.x)
        ref.append(capi.step(solo, m, d, sc.x, v, delta=5e-4)[:2])
        d.close()
        m.close()
    solo.close()
    out = [None] * len(scenes)

    def work(k):
        c = capi.Context(0)
        c.set_grid_share(2)
        for i in range(k, len(scenes), 2):
            sc, v = scenes[i]
            m = capi.Mesh.from_scene(c, sc)
            d = capi.Dynamics(c, m, sc.x)
            out[i] = capi.step(c, m, d, sc.x, v, delta=5e-4)[:2]
            d.close()
            m.close()
        c.close()

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for (xa, va), (xb, vb) in zip(ref, out):
        assert np.array_equal(xa.view(np.uint64), xb.view(np.uint64))
        assert np.array_equal(va.view(np.uint64), vb.view(np.uint64))

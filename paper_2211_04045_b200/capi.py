"""ctypes binding of the C-ABI (include/tw_c.h) in libtwoway_b200.so.

This is the host-side entry the tests and the benchmark use; it mirrors the
reference's operator interface (resolve(x, y, mesh, cfg) -> x, stats). The
library is built in-tree by ``make`` / ``__graft_entry__.build()``; importing
without it, or calling without a CUDA device, raises (there is no CPU
fallback on this path).
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TW_LIB_PATH: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("TW_LIB_PATH") or os.path.join(_HERE, "libtwoway_b200.so")

TW_OK, TW_EINVAL, TW_EUNSUPPORTED, TW_ECAPACITY, TW_ECUDA, TW_ETIMEOUT = range(6)
SOLVERS = {"pgs": 0, "jacobi": 1, "al20": 2, "al100": 3}
FAMILIES = {"volume": 0, "gap": 1}
COLORINGS = {"reference": 0, "device": 1}


class TwError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"tw error {code}: {msg}")
        self.code = code


class Config(C.Structure):
    _fields_ = [
        ("step_limit", C.c_int32), ("solver", C.c_int32), ("eps", C.c_double),
        ("d_min", C.c_double), ("d_max", C.c_double), ("delta", C.c_double),
        ("sigma", C.c_double), ("gamma", C.c_double), ("sweeps", C.c_int32),
        ("family", C.c_int32), ("under_relax", C.c_double), ("edge_constraints", C.c_int32),
        ("force_fresh_search", C.c_int32), ("record_path", C.c_int32),
        ("coloring_mode", C.c_int32), ("color_seed", C.c_uint64),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("steps", C.c_int32), ("searches", C.c_int32), ("final_residual", C.c_double),
        ("wall_ms", C.c_double), ("converged", C.c_int32), ("hit_step_limit", C.c_int32),
        ("stagnated", C.c_int32), ("start_in_contact", C.c_int32),
        ("step_law_violated", C.c_int32), ("num_pairs", C.c_int32),
        ("pairs_evaluated", C.c_int64), ("rows_solved", C.c_int64), ("device_ms", C.c_double),
        ("kernel_launches", C.c_int32), ("retries", C.c_int32), ("kernel_ms", C.c_double),
        ("setup_ms", C.c_double),
    ]


class StepTrace(C.Structure):
    _fields_ = [
        ("searched", C.c_int32), ("num_pairs", C.c_int32), ("num_contact_rows", C.c_int32),
        ("num_edge_rows", C.c_int32), ("num_colors", C.c_int32), ("num_active_pairs", C.c_int32),
        ("bound", C.c_double), ("max_disp", C.c_double), ("residual", C.c_double),
    ]


EXPORTS = [
    "tw_abi_version", "tw_default_config", "tw_ctx_create", "tw_ctx_destroy", "tw_last_error",
    "tw_ctx_kernel_launches", "tw_ctx_phase_profile", "tw_mesh_create", "tw_mesh_num_edges", "tw_mesh_edges",
    "tw_mesh_destroy", "tw_resolve", "tw_resolve_device", "tw_stage_closest", "tw_stage_search",
    "tw_stage_refresh", "tw_stage_linearize", "tw_stage_color", "tw_stage_backward",
    "tw_stage_advance", "tw_ccd_certify", "tw_default_energy_model", "tw_dyn_create", "tw_dyn_destroy",
    "tw_dyn_num_hinges", "tw_newton_target", "tw_step", "tw_step_device", "tw_stage_lcp",
    "tw_stage_linearize_ex", "tw_stage_build_rows", "tw_stage_constraint_value", "tw_stage_fill_diag",
    "tw_normal_flow_target", "tw_last_path", "tw_ctx_set_grid_share", "tw_friction_filter",
]


class EnergyModel(C.Structure):
    """tw_energy_model = EnergyModel scalars (dynamics.hpp:12-24)."""

    _fields_ = [
        ("spring_stiffness", C.c_double), ("bending_stiffness", C.c_double),
        ("gravity", C.c_double * 3), ("repulsion_stiffness", C.c_double),
        ("repulsion_radius", C.c_double), ("dt", C.c_double), ("newton_iters", C.c_int32),
        ("mu", C.c_double), ("pcg_tol", C.c_double), ("pcg_max_iters", C.c_int32),
    ]


class StepStats(C.Structure):
    _fields_ = [
        ("resolve_steps", C.c_int32), ("searches", C.c_int32), ("resolve_converged", C.c_int32),
        ("pcg_iterations", C.c_int32), ("pcg_converged", C.c_int32), ("num_pairs", C.c_int32),
        ("repulsive_pairs", C.c_int32), ("device_ms", C.c_double), ("resolve_ms", C.c_double),
        ("wall_ms", C.c_double), ("target_ms", C.c_double), ("pcg_ms", C.c_double),
        ("friction_ms", C.c_double),
    ]

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built (run `make` or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.tw_abi_version.restype = C.c_int
        L.tw_default_config.argtypes = [C.POINTER(Config)]
        L.tw_ctx_create.argtypes = [C.c_int, P, C.POINTER(P)]
        L.tw_ctx_destroy.argtypes = [P]
        L.tw_last_error.restype = C.c_char_p
        L.tw_last_error.argtypes = [P]
        L.tw_ctx_kernel_launches.restype = C.c_int64
        L.tw_ctx_kernel_launches.argtypes = [P]
        L.tw_mesh_create.argtypes = [P, C.c_int32, P, C.c_int32, P, C.c_int32, P, C.c_int32, P, C.POINTER(P)]
        L.tw_mesh_num_edges.restype = C.c_int32
        L.tw_mesh_num_edges.argtypes = [P]
        L.tw_mesh_edges.argtypes = [P, P]
        L.tw_mesh_destroy.argtypes = [P]
        L.tw_resolve.argtypes = [P, P, P, P, C.POINTER(Config), P, C.POINTER(Stats), P, P, P]
        L.tw_resolve_device.argtypes = [P, P, P, P, C.POINTER(Config), P, C.POINTER(Stats)]
        L.tw_stage_closest.argtypes = [P, C.c_int32, P, C.c_int64, P, P, P, P]
        L.tw_stage_search.argtypes = [P, P, P, C.c_double, C.c_int64, P, P, P, P, P, P, P]
        L.tw_stage_refresh.argtypes = [P, P, P, C.c_double, C.c_int64, P, P, P, P, P, P, P]
        L.tw_stage_advance.argtypes = [P, C.c_int32, P, P, P, C.c_double, P, P, P]
        L.tw_ccd_certify.argtypes = [P, P, P, P, P, P, P]
        L.tw_stage_linearize.argtypes = [P, P, P, C.c_int64, P, P, P, P, P, P, P, C.c_double, C.c_double,
                                         C.c_int32, C.c_int32, C.c_int64, P, P, P, P, P, P, P, P]
        L.tw_stage_color.argtypes = [P, P, C.c_int64, P, P, P, P, C.c_uint64, C.c_int32, C.c_int32, P, P]
        L.tw_stage_backward.argtypes = [P, C.c_int32, P, C.c_int64, P, P, P, P, P, C.c_int32, P, P, C.c_int32,
                                        C.c_int32, C.c_double, P, P, P]
        L.tw_last_path.argtypes = [P, C.c_int64, P, C.POINTER(C.c_int32)]
        L.tw_ctx_set_grid_share.argtypes = [P, C.c_int32]
        L.tw_stage_linearize_ex.argtypes = [P, P, P, C.c_int64, P, P, P, P, P, P, P, C.c_double, C.c_double,
                                            C.c_int32, C.c_int32, C.c_int64, P, P, P, P, P, P, P, P, P, P, P, P]
        L.tw_stage_constraint_value.argtypes = [P, C.c_int32, P, C.c_int64, P, P, P, P, P, P, P, P]
        L.tw_normal_flow_target.argtypes = [P, C.c_int32, P, C.c_int32, P, C.c_double, C.c_double, P]
        L.tw_default_energy_model.argtypes = [C.POINTER(EnergyModel)]
        L.tw_dyn_create.argtypes = [P, P, C.POINTER(EnergyModel), P, C.POINTER(P)]
        L.tw_dyn_destroy.argtypes = [P]
        L.tw_dyn_num_hinges.restype = C.c_int32
        L.tw_dyn_num_hinges.argtypes = [P]
        L.tw_newton_target.argtypes = [P, P, P, C.c_double, P, P, P, P, P, C.POINTER(StepStats)]
        L.tw_step.argtypes = [P, P, P, C.POINTER(Config), P, P, C.POINTER(StepStats)]
        L.tw_friction_filter.argtypes = [P, P, P, C.c_double, P, P, P]
        L.tw_step_device.argtypes = [P, P, P, C.POINTER(Config), P, P, C.POINTER(StepStats)]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def make_config(**kw) -> Config:
    c = Config()
    lib().tw_default_config(C.byref(c))
    for k, v in kw.items():
        if k == "solver":
            v = SOLVERS[v] if isinstance(v, str) else v
        elif k in ("constraint_family", "family"):
            k, v = "family", (FAMILIES[v] if isinstance(v, str) else v)
        elif k in ("coloring", "coloring_mode"):
            k, v = "coloring_mode", (COLORINGS[v] if isinstance(v, str) else v)
        elif k in ("edge_constraints", "force_fresh_search", "record_path"):
            v = int(bool(v))
        if not any(k == f[0] for f in Config._fields_):
            raise ValueError(f"unknown config key '{k}'")
        setattr(c, k, v)
    return c


class Context:
    """One tw_ctx: device buffers + stream (not thread-safe)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.h = C.c_void_p()
        self._meshes = weakref.WeakSet()  # meshes are destroyed before their context
        rc = lib().tw_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(self.h))
        if rc != TW_OK:
            raise TwError(rc, "tw_ctx_create failed (no CUDA device?)")

    def check(self, rc):
        if rc != TW_OK:
            raise TwError(rc, lib().tw_last_error(self.h).decode())

    def set_grid_share(self, parts: int):
        """Use 1/parts of the device (for parts concurrent contexts)."""
        self.check(lib().tw_ctx_set_grid_share(self.h, int(parts)))

    @property
    def kernel_launches(self) -> int:
        return int(lib().tw_ctx_kernel_launches(self.h))

    def close(self):
        if self.h:
            for m in list(self._meshes):
                m.close()
            lib().tw_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Mesh:
    """tw_mesh: topology uploaded once (edge order = MeshState::finalize)."""

    def __init__(self, ctx: Context, nv, inv_mass=None, edges=(), strand_edges=(), triangles=()):
        self.ctx = ctx
        self.nv = int(nv)
        im = None if inv_mass is None else np.ascontiguousarray(inv_mass, np.float64)
        self.inv_mass = np.ones(self.nv) if im is None else im
        e = np.ascontiguousarray(np.asarray(edges, np.int32).reshape(-1, 2))
        s = np.ascontiguousarray(np.asarray(strand_edges, np.int32).reshape(-1, 2))
        t = np.ascontiguousarray(np.asarray(triangles, np.int32).reshape(-1, 3))
        self.triangles = t
        self.h = C.c_void_p()
        ctx.check(lib().tw_mesh_create(ctx.h, self.nv, _p(im), len(e), _p(e), len(s), _p(s), len(t), _p(t),
                                       C.byref(self.h)))
        ctx._meshes.add(self)
        ne = lib().tw_mesh_num_edges(self.h)
        self.edges = np.zeros((ne, 2), np.int32)
        lib().tw_mesh_edges(self.h, _p(self.edges))

    @classmethod
    def from_scene(cls, ctx, sc):
        return cls(ctx, sc.nv, sc.inv_mass, sc.edges, sc.strand_edges, sc.triangles)

    def close(self):
        if self.h:
            lib().tw_mesh_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def resolve(ctx: Context, mesh: Mesh, x, y, trace=False, out=None, **kw):
    """resolve(x_start, y_target, mesh, cfg) on the device. Returns (x_out, stats dict).
    out: optional (nv, 3) float64 result buffer (e.g. pinned host memory)."""
    cfg = make_config(**kw)
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    y = np.ascontiguousarray(y, np.float64).reshape(-1, 3)
    if len(x) != mesh.nv or len(y) != mesh.nv:
        raise ValueError("resolve: position arrays do not match mesh")
    xo = np.zeros_like(x) if out is None else out
    st = Stats()
    smd = np.zeros(max(1, cfg.step_limit))
    tr = (StepTrace * cfg.step_limit)() if trace else None
    rc = lib().tw_resolve(ctx.h, mesh.h, _p(x), _p(y), C.byref(cfg), _p(xo), C.byref(st), _p(smd), None,
                          C.cast(tr, C.c_void_p) if tr is not None else None)
    if rc == TW_EINVAL:
        raise ValueError(lib().tw_last_error(ctx.h).decode())
    if rc == TW_EUNSUPPORTED:
        raise NotImplementedError(lib().tw_last_error(ctx.h).decode())
    ctx.check(rc)
    stats = {k: getattr(st, k) for k, _ in Stats._fields_}
    stats["step_max_disp"] = smd[:st.steps].copy()
    if cfg.record_path:  # exactly the recorded states (the device buffer grows on demand)
        path = np.empty((st.steps + 1, mesh.nv, 3))
        n = C.c_int32(0)
        ctx.check(lib().tw_last_path(ctx.h, st.steps + 1, _p(path), C.byref(n)))
        stats["path"] = path[:n.value]
    if tr is not None:
        stats["trace"] = [{k: getattr(tr[i], k) for k, _ in StepTrace._fields_} for i in range(st.steps)]
    return xo, stats


def resolve_device_ptr(ctx: Context, mesh: Mesh, d_x: int, d_y: int, d_out: int, **kw):
    """resolve on device pointers already resident in HBM (nv*3 float64 each)."""
    cfg = make_config(**kw)
    st = Stats()
    ctx.check(lib().tw_resolve_device(ctx.h, mesh.h, C.c_void_p(d_x), C.c_void_p(d_y), C.byref(cfg),
                                      C.c_void_p(d_out), C.byref(st)))
    return {k: getattr(st, k) for k, _ in Stats._fields_}


def phase_profile(ctx: Context):
    """Per-phase time of the last resolve: {phase name: (ms, count)} from the
    persistent kernel's CTA-0 barrier timestamps. Call sites are mapped to the
    phase function called just before each barrier in csrc/tw_kernels.cu."""
    import re

    L = lib()
    L.tw_ctx_phase_profile.restype = C.c_int32
    L.tw_ctx_phase_profile.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]
    NS = 256  # kPhaseSites (csrc/tw_engine.cuh)
    sites = np.zeros(NS, np.int32)
    ms = np.zeros(NS)
    cnt = np.zeros(NS, np.int32)
    n = L.tw_ctx_phase_profile(ctx.h, _p(sites), _p(ms), _p(cnt), NS)
    src = open(os.path.join(_HERE, "csrc", "tw_kernels.cu")).read().splitlines()
    names = {}
    for i, line in enumerate(src, start=1):
        if line.strip() in ("SYNC();", "SUBSYNC(nsub);"):
            prev = src[i - 2]
            m = re.search(r"(ph_[a-z_]+)", prev)
            # sites are __LINE__ % NS: the resolve kernel (first in the file) wins
            names.setdefault(i % NS, m.group(1) if m else f"line{i}")
    out = {}
    for k in range(min(n, NS)):
        name = names.get(int(sites[k]), f"site{int(sites[k])}")
        a, b = out.get(name, (0.0, 0))
        out[name] = (a + float(ms[k]), b + int(cnt[k]))
    return out


def closest_batch(ctx: Context, x, kinds, verts):
    """simplex_pair_closest for n pairs. kinds (n, 2), verts (n, 6)."""
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    kinds = np.ascontiguousarray(kinds, np.int32).reshape(-1, 2)
    verts = np.ascontiguousarray(verts, np.int32).reshape(-1, 6)
    n = len(kinds)
    out = np.zeros((n, 11))
    has = np.zeros(n, np.int32)
    ctx.check(lib().tw_stage_closest(ctx.h, len(x), _p(x), n, _p(kinds), _p(verts), _p(out), _p(has)))
    return out, has


class Pairs:
    def __init__(self, n):
        self.keys = np.zeros(n, np.uint64)
        self.dist = np.zeros(n)
        self.wa = np.zeros((n, 3))
        self.wb = np.zeros((n, 3))
        self.dir = np.zeros((n, 3))
        self.flags = np.zeros(n, np.uint8)

    def __len__(self):
        return len(self.keys)

    def take(self, n):
        p = Pairs(0)
        for k in ("keys", "dist", "wa", "wb", "dir", "flags"):
            setattr(p, k, getattr(self, k)[:n].copy())
        return p


def search(ctx: Context, mesh: Mesh, x, d_max, cap=None) -> Pairs:
    """proximity_search on the device broad phase; pairs sorted by key."""
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    cap = cap or max(1024, 64 * mesh.nv)
    while True:
        P = Pairs(cap)
        n = C.c_int64(0)
        rc = lib().tw_stage_search(ctx.h, mesh.h, _p(x), d_max, cap, _p(P.keys), _p(P.dist), _p(P.wa), _p(P.wb),
                                   _p(P.dir), _p(P.flags), C.byref(n))
        if rc == TW_ECAPACITY and n.value > cap:
            cap = n.value
            continue
        ctx.check(rc)
        return P.take(n.value)


def refresh(ctx: Context, mesh: Mesh, x, bound, pairs: Pairs):
    """refresh_distances in place; returns per_vertex_bound for every vertex."""
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    D = np.zeros(mesh.nv)
    ctx.check(lib().tw_stage_refresh(ctx.h, mesh.h, _p(x), bound, len(pairs), _p(pairs.keys), _p(pairs.dist),
                                     _p(pairs.wa), _p(pairs.wb), _p(pairs.dir), _p(pairs.flags), _p(D)))
    return D


def advance(ctx: Context, inv_mass, y, D, gamma, x, r):
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3).copy()
    r = np.ascontiguousarray(r, np.float64).copy()
    md = C.c_double(0.0)
    ctx.check(lib().tw_stage_advance(ctx.h, len(r), _p(np.ascontiguousarray(inv_mass, np.float64)),
                                     _p(np.ascontiguousarray(y, np.float64)), _p(np.ascontiguousarray(D, np.float64)),
                                     gamma, _p(x), _p(r), C.byref(md)))
    return x, r, md.value


class Rows:
    """Constraint rows as tw_stage_linearize returns them (contact rows in pair
    order, then edge rows in edge order): kind (0 VT, 1 EE, 2 VE, 3 VV, 4 edge),
    verts (R, 4; -1 padded), value, jac (R, 4, 3), diag, pair_key, edge_index."""

    def __init__(self, n):
        self.kind = np.zeros(n, np.uint8)
        self.verts = np.full((n, 4), -1, np.int32)
        self.value = np.zeros(n)
        self.jac = np.zeros((n, 4, 3))
        self.diag = np.zeros(n)
        self.pair_key = np.zeros(n, np.uint64)
        self.edge_index = np.full(n, -1, np.int32)

    def __len__(self):
        return len(self.kind)

    def take(self, n):
        r = Rows(0)
        for k in ("kind", "verts", "value", "jac", "diag", "pair_key", "edge_index"):
            setattr(r, k, getattr(self, k)[:n].copy())
        return r


def linearize(ctx: Context, mesh: Mesh, x, pairs: Pairs, edge_targets, delta=1e-3, sigma=1.1, family=0,
              edge_constraints=True, ex=False) -> Rows:
    """linearize_all (constraints.cpp:181-220) on the device."""
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    et = np.ascontiguousarray(edge_targets if edge_targets is not None else np.zeros(1), np.float64)
    family = FAMILIES[family] if isinstance(family, str) else family
    cap = len(pairs) + len(mesh.edges) + 16
    R = Rows(cap)
    n = C.c_int64(0)
    if not ex:
        ctx.check(lib().tw_stage_linearize(ctx.h, mesh.h, _p(x), len(pairs), _p(pairs.keys), _p(pairs.dist),
                                           _p(pairs.wa), _p(pairs.wb), _p(pairs.dir), _p(pairs.flags), _p(et),
                                           delta, sigma, family, int(bool(edge_constraints)), cap, _p(R.kind),
                                           _p(R.verts), _p(R.value), _p(R.jac), _p(R.diag), _p(R.pair_key),
                                           _p(R.edge_index), C.byref(n)))
        return R.take(n.value)
    # tw_stage_linearize_ex: plus each row's re-evaluation data
    flavor, refv = np.zeros(cap, np.uint8), np.zeros(cap)
    gw, den = np.zeros((cap, 4)), np.zeros(cap)
    ctx.check(lib().tw_stage_linearize_ex(ctx.h, mesh.h, _p(x), len(pairs), _p(pairs.keys), _p(pairs.dist),
                                          _p(pairs.wa), _p(pairs.wb), _p(pairs.dir), _p(pairs.flags), _p(et),
                                          delta, sigma, family, int(bool(edge_constraints)), cap, _p(R.kind),
                                          _p(R.verts), _p(R.value), _p(R.jac), _p(R.diag), _p(R.pair_key),
                                          _p(R.edge_index), _p(flavor), _p(refv), _p(gw), _p(den), C.byref(n)))
    out = R.take(n.value)
    k = n.value
    out.flavor, out.ref_volume, out.gap_weights, out.denom = flavor[:k], refv[:k], gw[:k], den[:k]
    return out


def constraint_value_at(ctx: Context, rows, x, sigma=1.1):
    """constraint_value_at (constraints.cpp:39-54) of every row (rows from linearize(..., ex=True))."""
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    n = len(rows)
    nv_rows = np.ascontiguousarray((rows.verts >= 0).sum(1), np.int32)
    out = np.zeros(max(1, n))
    sig = np.full(max(1, n), sigma)
    ctx.check(lib().tw_stage_constraint_value(ctx.h, len(x), _p(x), n, _p(np.ascontiguousarray(rows.flavor, np.uint8)),
                                              _p(nv_rows), _p(np.ascontiguousarray(rows.verts, np.int32)),
                                              _p(np.ascontiguousarray(rows.ref_volume)),
                                              _p(np.ascontiguousarray(rows.gap_weights)),
                                              _p(np.ascontiguousarray(rows.denom)), _p(sig), _p(out)))
    return out[:n]


def normal_flow_target(ctx: Context, x, triangles, beta=5e-4, alpha=0.5):
    """normal_flow_target (normal_flow.cpp:38-81) on the device."""
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
    y = np.zeros_like(x)
    rc = lib().tw_normal_flow_target(ctx.h, len(x), _p(x), len(t), _p(t), beta, alpha, _p(y))
    if rc == TW_EINVAL:
        raise ValueError(lib().tw_last_error(ctx.h).decode())
    ctx.check(rc)
    return y


def color(ctx: Context, mesh: Mesh, rows: Rows, seed=0x5EED, mode="device", edge_constraints=True):
    """color_constraints on the device; returns (ncolors, color per row)."""
    mode = COLORINGS[mode] if isinstance(mode, str) else mode
    out = np.zeros(len(rows), np.int32)
    nco = C.c_int32(0)
    ctx.check(lib().tw_stage_color(ctx.h, mesh.h, len(rows), _p(np.ascontiguousarray(rows.kind, np.uint8)),
                                   _p(np.ascontiguousarray(rows.verts, np.int32)),
                                   _p(np.ascontiguousarray(rows.pair_key, np.uint64)),
                                   _p(np.ascontiguousarray(rows.edge_index, np.int32)), seed, mode,
                                   int(bool(edge_constraints)), _p(out), C.byref(nco)))
    return nco.value, out


def backward(ctx: Context, inv_mass, rows: Rows, colors, ncolors, x, y, lam=None, solver="pgs", sweeps=1,
             under_relax=0.5):
    """assemble_lcp + sweeps + recover_target on the device; returns dict
    (lambda, q, y) like the oracle's backward."""
    inv = np.ascontiguousarray(inv_mass, np.float64)
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    y = np.ascontiguousarray(y, np.float64).reshape(-1, 3)
    n = len(rows)
    lam = np.zeros(n) if lam is None else np.ascontiguousarray(lam, np.float64).copy()
    q = np.zeros(max(1, n))
    yo = np.zeros_like(x)
    solver = SOLVERS[solver] if isinstance(solver, str) else solver
    col = np.ascontiguousarray(colors if colors is not None else np.zeros(n), np.int32)
    ctx.check(lib().tw_stage_backward(ctx.h, len(inv), _p(inv), n, _p(np.ascontiguousarray(rows.verts, np.int32)),
                                      _p(np.ascontiguousarray(rows.value, np.float64)),
                                      _p(np.ascontiguousarray(rows.jac, np.float64)),
                                      _p(np.ascontiguousarray(rows.diag, np.float64)), _p(col), int(ncolors),
                                      _p(x), _p(y), solver, sweeps, under_relax, _p(lam), _p(q), _p(yo)))
    return {"lambda": lam, "q": q[:n], "y": yo}


def ccd_certify(ctx: Context, mesh: Mesh, x0, x1, candidates=False):
    """ccd_certify (testkit/ccd.cpp) of the segment x0 -> x1 on the device:
    (violations, certain) [, candidate stencils tested]."""
    x0 = np.ascontiguousarray(x0, np.float64).reshape(-1, 3)
    x1 = np.ascontiguousarray(x1, np.float64).reshape(-1, 3)
    v, c, n = C.c_int32(0), C.c_int32(0), C.c_int64(0)
    ctx.check(lib().tw_ccd_certify(ctx.h, mesh.h, _p(x0), _p(x1), C.byref(v), C.byref(c), C.byref(n)))
    return (v.value, c.value, n.value) if candidates else (v.value, c.value)


def ccd_certify_path(ctx: Context, mesh: Mesh, path):
    """Certify every segment of a recorded resolve path: (violations, certain) totals."""
    tot, cert = 0, 0
    for i in range(len(path) - 1):
        v, c = ccd_certify(ctx, mesh, path[i], path[i + 1])
        tot += v
        cert += c
    return tot, cert


# ---------------------------------------------------------------- dynamics
def make_energy_model(**kw) -> EnergyModel:
    m = EnergyModel()
    lib().tw_default_energy_model(C.byref(m))
    for k, v in kw.items():
        if k == "gravity":
            for i in range(3):
                m.gravity[i] = float(v[i])
        elif any(k == f[0] for f in EnergyModel._fields_):
            setattr(m, k, v)
        else:
            raise ValueError(f"unknown energy model key '{k}'")
    return m


class Dynamics:
    """tw_dyn: EnergyModel prepared on a mesh (rest lengths, hinges) plus the
    device state of step() (dynamics.cpp:326-349)."""

    def __init__(self, ctx: Context, mesh: Mesh, rest_x, **model):
        self.ctx, self.mesh = ctx, mesh
        self.model = make_energy_model(**model)
        rx = np.ascontiguousarray(rest_x, np.float64).reshape(-1, 3)
        self.h = C.c_void_p()
        rc = lib().tw_dyn_create(ctx.h, mesh.h, C.byref(self.model), _p(rx), C.byref(self.h))
        if rc == TW_EINVAL:
            raise ValueError(lib().tw_last_error(ctx.h).decode())
        ctx.check(rc)

    @property
    def num_hinges(self):
        return int(lib().tw_dyn_num_hinges(self.h))

    def close(self):
        if self.h:
            lib().tw_dyn_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _step_stats(st):
    return {k: getattr(st, k) for k, _ in StepStats._fields_}


def newton_target(ctx: Context, mesh: Mesh, dyn: Dynamics, x0, v0, x=None, d_max=4e-3):
    """search + gradient_and_hessian + add_repulsion + newton_target (+ friction_filter
    when mu > 0): (y, grad, stats)."""
    x0 = np.ascontiguousarray(x0, np.float64).reshape(-1, 3)
    v0 = np.ascontiguousarray(v0, np.float64).reshape(-1, 3)
    x = x0 if x is None else np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    y = np.zeros_like(x0)
    g = np.zeros(3 * mesh.nv)
    st = StepStats()
    rc = lib().tw_newton_target(ctx.h, mesh.h, dyn.h, d_max, _p(x0), _p(v0), _p(x), _p(y), _p(g), C.byref(st))
    if rc == TW_EUNSUPPORTED:
        raise NotImplementedError(lib().tw_last_error(ctx.h).decode())
    ctx.check(rc)
    return y, g, _step_stats(st)


def friction_filter(ctx: Context, mesh: Mesh, dyn: Dynamics, x, y_target, d_max=4e-3):
    """friction_filter(model, mesh, x, y_target, proximity_search(x, d_max))
    (dynamics.cpp:272-324) on the device: the filtered target."""
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    yt = np.ascontiguousarray(y_target, np.float64).reshape(-1, 3)
    y = np.zeros_like(yt)
    ctx.check(lib().tw_friction_filter(ctx.h, mesh.h, dyn.h, d_max, _p(x), _p(yt), _p(y)))
    return y


def step(ctx: Context, mesh: Mesh, dyn: Dynamics, x, v, **kw):
    """One simulation step on the device: returns (x_next, v_next, stats)."""
    cfg = make_config(**kw)
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3).copy()
    v = np.ascontiguousarray(v, np.float64).reshape(-1, 3).copy()
    st = StepStats()
    rc = lib().tw_step(ctx.h, mesh.h, dyn.h, C.byref(cfg), _p(x), _p(v), C.byref(st))
    if rc == TW_EINVAL:
        raise ValueError(lib().tw_last_error(ctx.h).decode())
    if rc == TW_EUNSUPPORTED:
        raise NotImplementedError(lib().tw_last_error(ctx.h).decode())
    ctx.check(rc)
    return x, v, _step_stats(st)


def step_device_ptr(ctx: Context, mesh: Mesh, dyn: Dynamics, d_x: int, d_v: int, **kw):
    """step() on device-resident state (HBM pointers, nv*3 float64 each)."""
    cfg = make_config(**kw)
    st = StepStats()
    ctx.check(lib().tw_step_device(ctx.h, mesh.h, dyn.h, C.byref(cfg), C.c_void_p(d_x), C.c_void_p(d_v),
                                   C.byref(st)))
    return _step_stats(st)

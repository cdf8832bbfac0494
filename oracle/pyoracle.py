"""ctypes binding of the C oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs as the checker / timed CPU reference. The product
package (paper_2211_04045_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

KIND_V, KIND_E, KIND_T = 0, 1, 2
PF_ACTIVE, PF_ALL_STATIC, PF_DEGENERATE = 1, 2, 4
ROW_VT, ROW_EE, ROW_VE, ROW_VV, ROW_EDGE = range(5)


class Config(C.Structure):
    """or_config == tw_resolve_config layout (ResolveConfig, resolve.hpp:13-34)."""

    _fields_ = [
        ("step_limit", C.c_int32), ("solver", C.c_int32), ("eps", C.c_double),
        ("d_min", C.c_double), ("d_max", C.c_double), ("delta", C.c_double),
        ("sigma", C.c_double), ("gamma", C.c_double), ("sweeps", C.c_int32),
        ("family", C.c_int32), ("under_relax", C.c_double), ("edge_constraints", C.c_int32),
        ("force_fresh_search", C.c_int32), ("record_path", C.c_int32),
        ("coloring_mode", C.c_int32), ("color_seed", C.c_uint64),
    ]


def default_config(**kw) -> Config:
    c = Config(step_limit=512, solver=0, eps=1e-4, d_min=2e-3, d_max=4e-3, delta=1e-3, sigma=1.1,
               gamma=0.9, sweeps=1, family=0, under_relax=0.5, edge_constraints=1,
               force_fresh_search=0, record_path=0, coloring_mode=0, color_seed=0x5EED)
    for k, v in kw.items():
        if k == "solver":
            v = {"pgs": 0, "jacobi": 1, "al20": 2, "al100": 3}.get(v, v)
        if k == "constraint_family" or k == "family":
            k, v = "family", {"volume": 0, "gap": 1}.get(v, v)
        if k == "coloring_mode":
            v = {"reference": 0, "device": 1}.get(v, v)
        setattr(c, k, v)
    return c


class Stats(C.Structure):
    _fields_ = [
        ("steps", C.c_int32), ("searches", C.c_int32), ("final_residual", C.c_double),
        ("wall_ms", C.c_double), ("converged", C.c_int32), ("hit_step_limit", C.c_int32),
        ("stagnated", C.c_int32), ("start_in_contact", C.c_int32),
        ("step_law_violated", C.c_int32), ("status", C.c_int32),
    ]


class StepTrace(C.Structure):
    _fields_ = [
        ("searched", C.c_int32), ("num_pairs", C.c_int32), ("num_contact_rows", C.c_int32),
        ("num_edge_rows", C.c_int32), ("num_colors", C.c_int32), ("num_active_pairs", C.c_int32),
        ("bound", C.c_double), ("max_disp", C.c_double), ("residual", C.c_double),
    ]


def build() -> str:
    out = os.path.join(_HERE, "liboracle.so")
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return out


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        P = C.c_void_p
        L.or_closest.restype = C.c_int
        L.or_closest.argtypes = [C.c_int, P, C.c_int, P, P, P]
        L.or_finalize_edges.restype = C.c_int
        L.or_finalize_edges.argtypes = [C.c_int, C.c_int, P, C.c_int, P, C.c_int, P, P]
        L.or_search.restype = C.c_int64
        L.or_search.argtypes = [C.c_int, P, C.c_int, P, C.c_int, P, P, C.c_double, C.c_int64,
                                P, P, P, P, P, P]
        L.or_refresh.restype = None
        L.or_refresh.argtypes = [C.c_int, C.c_int, P, C.c_int, P, P, C.c_double, C.c_int64,
                                 P, P, P, P, P, P]
        L.or_vertex_bound.restype = None
        L.or_vertex_bound.argtypes = [C.c_int, C.c_int, P, C.c_int, P, C.c_double, C.c_int64,
                                      P, P, P, P]
        L.or_linearize.restype = C.c_int64
        L.or_linearize.argtypes = [C.c_int, P, C.c_int, P, C.c_int, P, P, C.c_int64, P, P, P, P,
                                   P, P, P, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                   C.c_int64,
                                   P, P, P, P, P, P, P, P, P, P, P, P]
        L.or_constraint_value_at.restype = C.c_double
        L.or_constraint_value_at.argtypes = [C.c_int, C.c_int, P, C.c_double, P, C.c_double,
                                             C.c_double, P]
        L.or_color.restype = C.c_int
        L.or_color.argtypes = [C.c_int, P, C.c_int64, P, P, P, P, P, C.c_uint64, C.c_int,
                               C.c_int, P, C.c_int, P]
        L.or_color_edges.restype = C.c_int
        L.or_color_edges.argtypes = [C.c_int, P, C.c_int, P, P]
        L.or_backward.restype = C.c_int
        L.or_backward.argtypes = [C.c_int, P, C.c_int64, P, P, P, P, P, P, C.c_int, P, P,
                                  C.c_int, C.c_int, C.c_double, P, P, P, P]
        L.or_advance.restype = C.c_double
        L.or_advance.argtypes = [C.c_int, P, P, P, C.c_double, P, P]
        L.or_resolve.restype = C.c_int
        L.or_resolve.argtypes = [C.c_int, P, C.c_int, P, C.c_int, P, P, P, C.POINTER(Config), P,
                                 C.POINTER(Stats), P, P, P]
        L.or_mt19937_64_nth.restype = C.c_uint64
        L.or_mt19937_64_nth.argtypes = [C.c_uint64, C.c_int64]
        L.or_uniform_index.restype = C.c_uint64
        L.or_uniform_index.argtypes = [C.c_uint64, C.c_int64, C.c_uint64]
        L.or_ccd_certify.restype = C.c_int
        L.or_ccd_certify.argtypes = [C.c_int, C.c_int, P, C.c_int, P, P, P, C.POINTER(C.c_int)]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


def _i32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a.reshape(shape) if shape is not None else a


# ------------------------------------------------------------------- API
def closest(ka, va, kb, vb, x):
    """simplex_pair_closest; returns dict or None (nullopt); raises on adjacency."""
    x = _f64(x, (-1, 3))
    va = _i32(list(va) + [-1] * (3 - len(va)))
    vb = _i32(list(vb) + [-1] * (3 - len(vb)))
    out = np.zeros(11)
    h = lib().or_closest(ka, _p(va), kb, _p(vb), _p(x), _p(out))
    if h < 0:
        raise ValueError("simplex_pair_closest: adjacent pair or unsupported kinds")
    if h == 0:
        return None
    return {"distance": out[0], "weights_a": out[1:4].copy(), "weights_b": out[4:7].copy(),
            "direction": out[7:10].copy(), "degenerate": bool(out[10])}


def finalize_edges(nv, explicit, strands, tris):
    explicit, strands, tris = _i32(explicit, (-1, 2)), _i32(strands, (-1, 2)), _i32(tris, (-1, 3))
    out = np.zeros((len(explicit) + len(strands) + 3 * len(tris) + 1, 2), np.int32)
    n = lib().or_finalize_edges(nv, len(explicit), _p(explicit), len(strands), _p(strands),
                                len(tris), _p(tris), _p(out))
    return out[:n].copy()


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


def search(scene_or_mesh, x, d_max, cap=None):
    m = scene_or_mesh
    x = _f64(x, (-1, 3))
    inv, E, T = _f64(m.inv_mass), _i32(m.edges, (-1, 2)), _i32(m.triangles, (-1, 3))
    cap = cap if cap is not None else max(1024, 64 * len(x))
    while True:
        P = Pairs(cap)
        n = lib().or_search(len(x), _p(inv), len(E), _p(E), len(T), _p(T), _p(x), d_max, cap,
                            _p(P.keys), _p(P.dist), _p(P.wa), _p(P.wb), _p(P.dir), _p(P.flags))
        if n >= 0:
            return P.take(n)
        cap = -n


def refresh(m, x, bound, pairs: Pairs):
    x = _f64(x, (-1, 3))
    E, T = _i32(m.edges, (-1, 2)), _i32(m.triangles, (-1, 3))
    lib().or_refresh(len(x), len(E), _p(E), len(T), _p(T), _p(x), bound, len(pairs),
                     _p(pairs.keys), _p(pairs.dist), _p(pairs.wa), _p(pairs.wb), _p(pairs.dir),
                     _p(pairs.flags))


def vertex_bound(m, bound, pairs: Pairs, nv):
    E, T = _i32(m.edges, (-1, 2)), _i32(m.triangles, (-1, 3))
    out = np.zeros(nv)
    lib().or_vertex_bound(nv, len(E), _p(E), len(T), _p(T), bound, len(pairs), _p(pairs.keys),
                          _p(pairs.dist), _p(pairs.flags), _p(out))
    return out


class Rows:
    FIELDS = ("kind", "nverts", "verts", "value", "jac", "diag", "pair_key", "edge_index",
              "flavor", "ref_volume", "gap_weights", "denom")

    def __init__(self, n):
        self.kind = np.zeros(n, np.uint8)
        self.nverts = np.zeros(n, np.int32)
        self.verts = np.zeros((n, 4), np.int32)
        self.value = np.zeros(n)
        self.jac = np.zeros((n, 4, 3))
        self.diag = np.zeros(n)
        self.pair_key = np.zeros(n, np.uint64)
        self.edge_index = np.zeros(n, np.int32)
        self.flavor = np.zeros(n, np.uint8)
        self.ref_volume = np.zeros(n)
        self.gap_weights = np.zeros((n, 4))
        self.denom = np.zeros(n)

    def __len__(self):
        return len(self.kind)

    def take(self, n):
        r = Rows(0)
        for k in self.FIELDS:
            setattr(r, k, getattr(self, k)[:n].copy())
        return r


def linearize(m, x, pairs: Pairs, edge_targets, delta=1e-3, sigma=1.1, family=0,
              edge_constraints=True, window=0.0):
    x = _f64(x, (-1, 3))
    inv, E, T = _f64(m.inv_mass), _i32(m.edges, (-1, 2)), _i32(m.triangles, (-1, 3))
    et = _f64(edge_targets) if len(E) else np.zeros(1)
    cap = len(pairs) + len(E) + 16
    R = Rows(cap)
    n = lib().or_linearize(len(x), _p(inv), len(E), _p(E), len(T), _p(T), _p(x), len(pairs),
                           _p(pairs.keys), _p(pairs.dist), _p(pairs.wa), _p(pairs.wb),
                           _p(pairs.dir), _p(pairs.flags), _p(et), delta, window, sigma, family,
                           int(edge_constraints), cap, _p(R.kind), _p(R.nverts), _p(R.verts),
                           _p(R.value), _p(R.jac), _p(R.diag), _p(R.pair_key), _p(R.edge_index),
                           _p(R.flavor), _p(R.ref_volume), _p(R.gap_weights), _p(R.denom))
    assert n >= 0
    return R.take(n)


def constraint_value_at(rows: Rows, i, x, sigma=1.1):
    x = _f64(x, (-1, 3))
    v = _i32(rows.verts[i])
    gw = _f64(rows.gap_weights[i])
    return lib().or_constraint_value_at(int(rows.flavor[i]), int(rows.nverts[i]), _p(v),
                                        float(rows.ref_volume[i]), _p(gw), float(rows.denom[i]),
                                        sigma, _p(x))


def color(m, rows: Rows, seed, mode=0, edge_constraints=True, inv_mass=None):
    inv = _f64(m.inv_mass if inv_mass is None else inv_mass)
    E = _i32(m.edges, (-1, 2)) if m is not None else np.zeros((0, 2), np.int32)
    out = np.zeros(len(rows), np.int32)
    nc = lib().or_color(len(inv), _p(inv), len(rows), _p(rows.kind), _p(rows.nverts),
                        _p(rows.verts), _p(rows.pair_key), _p(rows.edge_index), seed, mode,
                        len(E), _p(E), int(edge_constraints), _p(out))
    return nc, out


def color_edges(inv_mass, edges):
    inv, E = _f64(inv_mass), _i32(edges, (-1, 2))
    out = np.zeros(len(E), np.int32)
    nc = lib().or_color_edges(len(inv), _p(inv), len(E), _p(E), _p(out))
    return nc, out


def backward(inv_mass, rows: Rows, colors, ncolors, x, y, lam=None, solver=0, sweeps=1,
             under_relax=0.5):
    inv = _f64(inv_mass)
    x, y = _f64(x, (-1, 3)), _f64(y, (-1, 3))
    lam = np.zeros(len(rows)) if lam is None else _f64(lam).copy()
    q = np.zeros(max(1, len(rows)))
    imp = np.zeros((len(inv), 3))
    yo = np.zeros((len(inv), 3))
    col = _i32(colors) if colors is not None else np.zeros(len(rows), np.int32)
    rc = lib().or_backward(len(inv), _p(inv), len(rows), _p(_i32(rows.nverts)), _p(_i32(rows.verts)),
                           _p(_f64(rows.value)), _p(_f64(rows.jac)), _p(_f64(rows.diag)), _p(col),
                           ncolors, _p(x), _p(y), solver, sweeps, under_relax, _p(lam), _p(q),
                           _p(imp), _p(yo))
    if rc != 0:
        raise ValueError("unsupported solver")
    return {"lambda": lam, "q": q[:len(rows)], "impulse": imp, "y": yo}


def advance(inv_mass, y, D, gamma, x, r):
    x = _f64(x, (-1, 3)).copy()
    r = _f64(r).copy()
    md = lib().or_advance(len(r), _p(_f64(inv_mass)), _p(_f64(y, (-1, 3))), _p(_f64(D)), gamma,
                          _p(x), _p(r))
    return x, r, md


def resolve(scene, x=None, y=None, trace=False, **kw):
    """Oracle resolve(x, y, mesh, cfg). Returns (x_out, stats dict)."""
    cfg = default_config(**kw)
    x = _f64(scene.x if x is None else x, (-1, 3))
    y = _f64(scene.y if y is None else y, (-1, 3))
    inv, E, T = _f64(scene.inv_mass), _i32(scene.edges, (-1, 2)), _i32(scene.triangles, (-1, 3))
    nv = len(x)
    xo = np.zeros_like(x)
    st = Stats()
    smd = np.zeros(cfg.step_limit)
    path = np.zeros((cfg.step_limit + 1, nv, 3)) if cfg.record_path else None
    tr = (StepTrace * cfg.step_limit)() if trace else None
    rc = lib().or_resolve(nv, _p(inv), len(E), _p(E), len(T), _p(T), _p(x), _p(y), C.byref(cfg),
                          _p(xo), C.byref(st), _p(smd), _p(path) if path is not None else None,
                          C.cast(tr, C.c_void_p) if tr is not None else None)
    if rc == -1:
        raise ValueError("resolve: invalid argument")
    if rc == -2:
        raise NotImplementedError("resolve: solver not supported by the oracle")
    stats = {k: getattr(st, k) for k, _ in Stats._fields_}
    stats["step_max_disp"] = smd[:st.steps].copy()
    if path is not None:
        stats["path"] = path[:st.steps + 1].copy()
    if tr is not None:
        stats["trace"] = [{k: getattr(tr[i], k) for k, _ in StepTrace._fields_} for i in range(st.steps)]
    return xo, stats


def ccd_certify(scene, x0, x1):
    """ccd_certify on one segment; returns (violations, certain)."""
    E, T = _i32(scene.edges, (-1, 2)), _i32(scene.triangles, (-1, 3))
    x0, x1 = _f64(x0, (-1, 3)), _f64(x1, (-1, 3))
    certain = C.c_int(0)
    v = lib().or_ccd_certify(len(x0), len(E), _p(E), len(T), _p(T), _p(x0), _p(x1), C.byref(certain))
    return v, certain.value


def ccd_certify_path(scene, path):
    tot, cert = 0, 0
    for i in range(len(path) - 1):
        v, c = ccd_certify(scene, path[i], path[i + 1])
        tot += v
        cert += c
    return tot, cert


def _simplex(m, kind, idx):
    if kind == KIND_V:
        return [int(idx)]
    if kind == KIND_E:
        return [int(v) for v in m.edges[idx]]
    return [int(v) for v in m.triangles[idx]]


def friction_filter(m, x, y_target, d_max, mu, dt=0.01, repulsion_radius=1e-3):
    """friction_filter(model, mesh, x, y_target, proximity_search(x, d_max))
    restated from dynamics.cpp:272-324 (Python scalars: IEEE double, no
    contraction, the reference's association), on the oracle's search and
    closest points. Pure-Python loop: small scenes only."""
    x = _f64(x, (-1, 3))
    y = _f64(y_target, (-1, 3)).copy()
    inv = [float(v) for v in _f64(m.inv_mass)]
    pairs = search(m, x, d_max)
    xs = [list(map(float, r)) for r in x]

    def is_zero(v):
        return all(abs(c) <= 1e-12 for c in v)

    for i in range(len(pairs)):
        if pairs.flags[i] & PF_ALL_STATIC:  # :278
            continue
        key = int(pairs.keys[i])
        ka, kb = key >> 62, (key >> 60) & 3
        va, vb = _simplex(m, ka, (key >> 30) & 0x3FFFFFFF), _simplex(m, kb, key & 0x3FFFFFFF)
        res = closest(ka, va, kb, vb, y)  # penetration at the target state, :279
        if res is None:
            continue
        depth = repulsion_radius - float(res["distance"])
        if depth <= 0.0:
            continue
        n = [float(c) for c in res["direction"]]
        if is_zero(n):
            n = [float(c) for c in pairs.dir[i]]  # p.closest.direction, :284
        if is_zero(n):
            continue
        vid = va + vb
        sw = [float(w) for w in res["weights_a"][:len(va)]] + [-float(w) for w in res["weights_b"][:len(vb)]]
        kappa = 0.0
        v_rel = [0.0, 0.0, 0.0]
        for a, v in enumerate(vid):  # :299-302
            kappa += sw[a] * sw[a] * inv[v]
            v_rel = [v_rel[c] + (sw[a] * (float(y[v, c]) - xs[v][c])) / dt for c in range(3)]
        if kappa <= 0.0:
            continue
        vn = (v_rel[0] * n[0] + v_rel[1] * n[1]) + v_rel[2] * n[2]  # :307-318
        hi = depth / dt
        jn = 0.0 if -vn < 0.0 else (hi if hi < -vn else -vn)  # std::clamp
        impulse = [jn * c for c in n]
        vt = [v_rel[c] - vn * n[c] for c in range(3)]
        vt_norm = math.sqrt((vt[0] * vt[0] + vt[1] * vt[1]) + vt[2] * vt[2])
        if vt_norm > 1e-12:
            cap = mu * jn
            dvt = vt_norm if vt_norm < cap else cap  # std::min(cap, vt_norm)
            impulse = [impulse[c] - dvt * (vt[c] / vt_norm) for c in range(3)]
        dv = [c / kappa for c in impulse]
        for a, v in enumerate(vid):  # :320-321
            s = dt * inv[v] * sw[a]
            for c in range(3):
                y[v, c] = float(y[v, c]) + s * dv[c]
    return y

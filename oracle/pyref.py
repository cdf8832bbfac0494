"""ctypes binding of the REAL reference build (oracle/_ref/libtwoway_ref.so).

TEST INFRASTRUCTURE ONLY. `oracle/Makefile.ref` compiles the reference's own
sources from /root/reference/proj/src (in place, never copied) against the
Eigen-subset shim `oracle/ref_shim/` (Eigen is absent from the image). Used by
tests/ to pin the clean-room restatement (pyoracle / liboracle.so) and by
bench.py's `--impl reference` / cpu_baseline legs to time the reference's own
`resolve`. The product package never imports it.

The library travels to the GPU box with the gpurun snapshot (oracle/_ref/ is
git-ignored, not gpurun-ignored); `available()` is False where it was never
built (the sources under /root/reference exist only in the build container).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from pyoracle import Config, Stats, default_config  # same struct layouts (oracle.h)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_ref", "libtwoway_ref.so")
_LIB = None
REF_SRC = "/root/reference/proj"


class EnergyParams(C.Structure):
    """EnergyModel scalars (dynamics.hpp:12-24)."""

    _fields_ = [
        ("spring_stiffness", C.c_double), ("bending_stiffness", C.c_double),
        ("gravity", C.c_double * 3), ("repulsion_stiffness", C.c_double),
        ("repulsion_radius", C.c_double), ("dt", C.c_double), ("newton_iters", C.c_int32),
        ("mu", C.c_double), ("pcg_tol", C.c_double), ("pcg_max_iters", C.c_int32),
    ]


def energy_params(**kw) -> EnergyParams:
    """EnergyModel defaults (dynamics.hpp:12-24) with overrides."""
    p = EnergyParams(spring_stiffness=50.0, bending_stiffness=0.0, repulsion_stiffness=1e3,
                     repulsion_radius=1e-3, dt=0.01, newton_iters=1, mu=0.0, pcg_tol=1e-6,
                     pcg_max_iters=400)
    p.gravity[0], p.gravity[1], p.gravity[2] = 0.0, 0.0, -9.81
    for k, v in kw.items():
        if k == "gravity":
            for i in range(3):
                p.gravity[i] = float(v[i])
        else:
            setattr(p, k, v)
    return p


def build() -> bool:
    """Build oracle/_ref from the reference sources when they are present."""
    if not os.path.isdir(REF_SRC):
        return os.path.exists(_SO)
    subprocess.run(["make", "-s", "-C", _HERE, "-f", "Makefile.ref", "-j8", "all"], check=True)
    return True


def available() -> bool:
    return os.path.exists(_SO)


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        P = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_mesh_create.restype = P
        L.ref_mesh_create.argtypes = [C.c_int, P, C.c_int, P, C.c_int, P, P, P]
        L.ref_mesh_destroy.argtypes = [P]
        L.ref_mesh_edges.argtypes = [P, C.c_int, P]
        L.ref_mesh_positions.argtypes = [P, P, P, P]
        L.ref_mesh_topology.argtypes = [P, P, P, P, P]
        L.ref_resolve.argtypes = [P, P, P, C.POINTER(Config), P, C.POINTER(Stats), P, C.c_int64, P]
        L.ref_search.restype = C.c_int64
        L.ref_search.argtypes = [P, P, C.c_double, C.c_int64, P, P, P]
        L.ref_linearize.restype = C.c_int64
        L.ref_linearize.argtypes = [P, P, P, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                    C.c_uint64, C.c_int64, P, P, P, P, P, P, P]
        L.ref_step.argtypes = [P, P, C.POINTER(EnergyParams), C.POINTER(Config), P, P, P]
        L.ref_newton_target.argtypes = [P, P, C.POINTER(EnergyParams), C.c_double, P, P, P, P, P]
        L.ref_friction_filter.argtypes = [P, P, C.POINTER(EnergyParams), C.c_double, P, P, P]
        L.ref_incremental_energy.restype = C.c_double
        L.ref_incremental_energy.argtypes = [P, P, C.POINTER(EnergyParams), P]
        L.ref_normal_flow_target.argtypes = [P, P, C.c_double, C.c_double, P]
        L.ref_frame_sample.argtypes = [P, P, C.POINTER(EnergyParams), C.POINTER(Config), P]
        L.ref_ccd_certify.argtypes = [P, P, P, P]
        L.ref_fixture.restype = P
        L.ref_fixture.argtypes = [C.c_uint64, C.c_int, C.c_int, P, P, P, C.c_char_p, C.c_int]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)


def _err():
    return lib().ref_last_error().decode()


class RefMesh:
    """MeshState built as bindings/module.cpp:32-48 does (finalize + validate)."""

    def __init__(self, x, triangles, strand_edges=(), inv_mass=None, velocities=None, handle=None):
        if handle is not None:
            self.h = handle
        else:
            x = _f64(x)
            T = np.ascontiguousarray(triangles, dtype=np.int32).reshape(-1, 3)
            S = np.ascontiguousarray(strand_edges, dtype=np.int32).reshape(-1, 2)
            inv = None if inv_mass is None else np.ascontiguousarray(inv_mass, dtype=np.float64)
            vel = None if velocities is None else _f64(velocities)
            self.h = lib().ref_mesh_create(len(x), _p(x), len(T), _p(T), len(S), _p(S), _p(inv), _p(vel))
            if not self.h:
                raise ValueError(_err())
        self.nv = lib().ref_mesh_positions(self.h, None, None, None)

    @classmethod
    def from_scene(cls, sc, velocities=None):
        return cls(sc.x, sc.triangles, sc.strand_edges, sc.inv_mass, velocities)

    def edges(self):
        ne = lib().ref_mesh_edges(self.h, 0, None)
        out = np.zeros((ne, 2), np.int32)
        lib().ref_mesh_edges(self.h, ne, _p(out))
        return out

    def state(self):
        x, v, inv = np.zeros((self.nv, 3)), np.zeros((self.nv, 3)), np.zeros(self.nv)
        lib().ref_mesh_positions(self.h, _p(x), _p(v), _p(inv))
        return x, v, inv

    def topology(self):
        nt, ns = C.c_int32(0), C.c_int32(0)
        lib().ref_mesh_topology(self.h, C.byref(nt), None, C.byref(ns), None)
        T = np.zeros((nt.value, 3), np.int32)
        S = np.zeros((ns.value, 2), np.int32)
        lib().ref_mesh_topology(self.h, C.byref(nt), _p(T), C.byref(ns), _p(S))
        return T, S

    def close(self):
        if self.h:
            lib().ref_mesh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def resolve(mesh: RefMesh, x, y, **kw):
    """twoway::resolve of the reference build. Returns (x_out, stats dict)."""
    cfg = default_config(**kw)
    x, y = _f64(x), _f64(y)
    xo = np.zeros_like(x)
    st = Stats()
    smd = np.zeros(cfg.step_limit)
    path = np.zeros((cfg.step_limit + 1) * mesh.nv * 3) if cfg.record_path else None
    rc = lib().ref_resolve(mesh.h, _p(x), _p(y), C.byref(cfg), _p(xo), C.byref(st), _p(smd),
                           0 if path is None else len(path), _p(path))
    if rc == -1:
        raise ValueError(_err())
    if rc != 0:
        raise RuntimeError(_err())
    stats = {k: getattr(st, k) for k, _ in Stats._fields_}
    stats["step_max_disp"] = smd[:st.steps].copy()
    if path is not None:
        stats["path"] = path.reshape(-1, mesh.nv, 3)[:st.steps + 1].copy()
    return xo, stats


def search(mesh: RefMesh, x, d_max):
    """proximity_search keys (sorted) and distances."""
    x = _f64(x)
    cap = max(1024, 64 * mesh.nv)
    while True:
        keys, dist, flags = np.zeros(cap, np.uint64), np.zeros(cap), np.zeros(cap, np.uint8)
        n = lib().ref_search(mesh.h, _p(x), d_max, cap, _p(keys), _p(dist), _p(flags))
        if n >= 0:
            return keys[:n].copy(), dist[:n].copy(), flags[:n].copy()
        if n < -(1 << 40):
            raise RuntimeError(_err())
        cap = -n


def linearize(mesh: RefMesh, x, y, d_max=4e-3, delta=1e-3, sigma=1.1, family=0,
              edge_constraints=True, seed=0x5EED):
    """search at x + linearize_all + color_constraints: per-row identity and values."""
    x, y = _f64(x), _f64(y)
    cap = 64 * mesh.nv + 4 * len(mesh.edges()) + 16
    while True:
        out = {"kind": np.zeros(cap, np.uint8), "key": np.zeros(cap, np.uint64),
               "edge_index": np.zeros(cap, np.int32), "value": np.zeros(cap),
               "diag": np.zeros(cap), "color": np.zeros(cap, np.int32)}
        nc = C.c_int32(0)
        n = lib().ref_linearize(mesh.h, _p(x), _p(y), d_max, delta, sigma, family,
                                int(edge_constraints), seed, cap, _p(out["kind"]), _p(out["key"]),
                                _p(out["edge_index"]), _p(out["value"]), _p(out["diag"]),
                                _p(out["color"]), C.byref(nc))
        if n >= 0:
            r = {k: v[:n].copy() for k, v in out.items()}
            r["ncolors"] = nc.value
            return r
        cap = -n


def newton_target(mesh: RefMesh, rest_x, x, d_max=4e-3, **energy):
    """search + gradient_and_hessian + add_repulsion + newton_target (+ friction filter)."""
    ep = energy_params(**energy)
    x, rest = _f64(x), _f64(rest_x)
    y, g = np.zeros_like(x), np.zeros(3 * len(x))
    it, conv = C.c_int32(0), C.c_int32(0)
    rc = lib().ref_newton_target(mesh.h, _p(rest), C.byref(ep), d_max, _p(x), _p(y), _p(g),
                                 C.byref(it), C.byref(conv))
    if rc != 0:
        raise RuntimeError(_err())
    return y, g, it.value, bool(conv.value)


def friction_filter(mesh: RefMesh, rest_x, x, y_target, d_max=4e-3, **energy):
    """The reference's friction_filter on the pair set of proximity_search(x, d_max)."""
    ep = energy_params(**energy)
    x, yt = _f64(x), _f64(y_target)
    y = np.zeros_like(x)
    rc = lib().ref_friction_filter(mesh.h, _p(_f64(rest_x)), C.byref(ep), d_max, _p(x), _p(yt), _p(y))
    if rc != 0:
        raise RuntimeError(_err())
    return y


def incremental_energy(mesh: RefMesh, rest_x, x, **energy):
    ep = energy_params(**energy)
    return lib().ref_incremental_energy(mesh.h, _p(_f64(rest_x)), C.byref(ep), _p(_f64(x)))


def step(mesh: RefMesh, rest_x, energy=None, **kw):
    """dynamics step() on the mesh state (positions, velocities). Returns
    (x_next, v_next, total resolve steps, searches); the mesh state advances."""
    ep = energy_params(**(energy or {}))
    cfg = default_config(**kw)
    xo, vo = np.zeros((mesh.nv, 3)), np.zeros((mesh.nv, 3))
    s = C.c_int32(0)
    n = lib().ref_step(mesh.h, _p(_f64(rest_x)), C.byref(ep), C.byref(cfg), _p(xo), _p(vo), C.byref(s))
    if n < 0:
        raise RuntimeError(_err())
    return xo, vo, n, s.value


def frame_sample(mesh: RefMesh, rest_x, energy=None, **kw):
    """Timed pieces of one reference frame (seconds): target (search +
    gradient/Hessian + repulsion + PCG), one proximity_search, one non-search
    Alg.-1 iteration; plus that iteration's contact rows and colors."""
    ep = energy_params(**(energy or {}))
    cfg = default_config(**kw)
    out = np.zeros(5)
    rc = lib().ref_frame_sample(mesh.h, _p(_f64(rest_x)), C.byref(ep), C.byref(cfg), _p(out))
    if rc != 0:
        raise RuntimeError(_err())
    return {"target_s": out[0], "search_s": out[1], "iteration_s": out[2], "contact_rows": int(out[3]),
            "colors": int(out[4])}


def normal_flow_target(mesh: RefMesh, x, beta=5e-4, alpha_smooth=0.5):
    y = np.zeros((mesh.nv, 3))
    rc = lib().ref_normal_flow_target(mesh.h, _p(_f64(x)), beta, alpha_smooth, _p(y))
    if rc != 0:
        raise ValueError(_err())
    return y


def ccd_certify(mesh: RefMesh, x0, x1):
    c = C.c_int32(0)
    v = lib().ref_ccd_certify(mesh.h, _p(_f64(x0)), _p(_f64(x1)), C.byref(c))
    return v, c.value


def fixture(index, seed=0):
    """Fixture `index` of the reference's scene_fixtures(seed): (name, mesh, x, y, benign, penetrating)."""
    cap = 1 << 22
    y = np.zeros(cap)
    nv, flags = C.c_int32(0), C.c_int32(0)
    name = C.create_string_buffer(128)
    h = lib().ref_fixture(seed, index, cap, _p(y), C.byref(nv), C.byref(flags), name, 128)
    if not h:
        return None
    m = RefMesh(None, None, handle=h)
    x, _, _ = m.state()
    return (name.value.decode(), m, x, y[:3 * nv.value].reshape(-1, 3).copy(),
            bool(flags.value & 1), bool(flags.value & 2))


def num_fixtures(seed=0):
    nv, flags = C.c_int32(0), C.c_int32(0)
    name = C.create_string_buffer(8)
    lib().ref_fixture(seed, -1, 0, None, C.byref(nv), C.byref(flags), name, 8)
    return nv.value

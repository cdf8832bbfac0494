"""Deterministic scene generators (numpy) for tests and benchmarks.

Mesh builders restate the reference test kit (proj/src/testkit/fixtures.cpp)
so the fixture battery used by the reference acceptance suite
(``scene_fixtures``, fixtures.cpp:304-314) exists here too; the benchmark
scenes of BASELINE.json (cloth over sphere, reef/bow knots of two twisted
strips, codimensional mix, knot batch) are synthetic and documented in
DESIGN.md. Every scene is a plain ``Scene`` of numpy arrays: positions are
(n, 3) float64 row-major (the byte layout of ``std::vector<Vec3>``).

The random fixtures draw from a bit-exact mt19937_64 + libstdc++
``generate_canonical`` restatement; the reference's unspecified argument
evaluation order inside ``Vec3(uni(rng), ...)`` is taken left to right.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

PI = math.pi


# --------------------------------------------------------------------- RNG
class MT19937_64:
    """std::mt19937_64 (used by the reference fixtures and coloring)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def __call__(self) -> int:
        M = 0xFFFFFFFFFFFFFFFF
        if self.idx >= 312:
            upper, lower = (M << 31) & M, (1 << 31) - 1
            mt = self.mt
            for k in range(312):
                y = (mt[k] & upper) | (mt[(k + 1) % 312] & lower)
                mt[k] = mt[(k + 156) % 312] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
            self.idx = 0
        z = self.mt[self.idx]
        self.idx += 1
        z ^= (z >> 29) & 0x5555555555555555
        z ^= (z << 17) & 0x71D67FFFEDA60000 & M
        z ^= (z << 37) & 0xFFF7EEE000000000 & M
        z ^= z >> 43
        return z & M

    def canonical(self) -> float:
        # libstdc++ generate_canonical<double, 53> with a 64-bit engine
        r = float(self()) / 18446744073709551616.0
        return r if r < 1.0 else math.nextafter(1.0, 0.0)

    def uniform(self, a: float, b: float) -> float:
        return self.canonical() * (b - a) + a


# ------------------------------------------------------------------- scene
@dataclasses.dataclass
class Scene:
    name: str
    x: np.ndarray            # (n, 3) float64 start state (intersection-free)
    y: np.ndarray            # (n, 3) float64 target
    triangles: np.ndarray    # (t, 3) int32
    edges: np.ndarray        # (e, 2) int32, finalized order (mesh.cpp:10-33)
    strand_edges: np.ndarray  # (s, 2) int32
    inv_mass: np.ndarray     # (n,) float64, 0 = static
    benign: bool = True
    penetrating: bool = False

    @property
    def nv(self) -> int:
        return int(self.x.shape[0])


@dataclasses.dataclass
class Mesh:
    positions: np.ndarray
    triangles: np.ndarray
    strand_edges: np.ndarray
    edges: np.ndarray
    inv_mass: np.ndarray


def finalize_edges(explicit: np.ndarray, strands: np.ndarray, tris: np.ndarray) -> np.ndarray:
    """MeshState::finalize edge order (mesh.cpp:15-26)."""
    seen = set()
    out = []
    for a, b in np.asarray(explicit, dtype=np.int64).reshape(-1, 2):
        seen.add((min(a, b), max(a, b)))
        out.append((int(a), int(b)))
    for a, b in np.asarray(strands, dtype=np.int64).reshape(-1, 2):
        k = (min(a, b), max(a, b))
        if k not in seen:
            seen.add(k)
            out.append((int(a), int(b)))
    t = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    if len(t):
        # vectorised triangle-edge dedup preserving first occurrence in (t, k) order
        a = np.stack([t[:, 0], t[:, 1], t[:, 2]], axis=1).reshape(-1)
        b = np.stack([t[:, 1], t[:, 2], t[:, 0]], axis=1).reshape(-1)
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        key = lo * (1 << 32) + hi
        _, first = np.unique(key, return_index=True)
        first = np.sort(first)
        prior = {k[0] * (1 << 32) + k[1] for k in seen}
        extra = [(int(lo[i]), int(hi[i])) for i in first if int(key[i]) not in prior]
        out.extend(extra)
    return np.asarray(out, dtype=np.int32).reshape(-1, 2)


def make_mesh(positions, triangles=(), strand_edges=(), edges=(), inv_mass=None) -> Mesh:
    p = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    t = np.asarray(triangles, dtype=np.int32).reshape(-1, 3)
    s = np.asarray(strand_edges, dtype=np.int32).reshape(-1, 2)
    e = finalize_edges(np.asarray(edges, dtype=np.int32).reshape(-1, 2), s, t)
    im = np.ones(len(p)) if inv_mass is None else np.asarray(inv_mass, dtype=np.float64)
    return Mesh(p.copy(), t, s, e, im.copy())


def append_mesh(m: Mesh, o: Mesh) -> int:
    """append_mesh (mesh.cpp:79-106): offsets topology, carries plain edges,
    re-finalizes."""
    off = len(m.positions)
    tri_keys = {tuple(sorted((int(t[k]), int(t[(k + 1) % 3])))) for t in o.triangles for k in range(3)}
    strand_set = {tuple(int(v) for v in e) for e in o.strand_edges}
    plain = [e for e in o.edges
             if tuple(sorted(int(v) for v in e)) not in tri_keys and tuple(int(v) for v in e) not in strand_set]
    m.positions = np.concatenate([m.positions, o.positions])
    m.inv_mass = np.concatenate([m.inv_mass, o.inv_mass])
    m.triangles = np.concatenate([m.triangles, o.triangles + off]).astype(np.int32)
    m.strand_edges = np.concatenate([m.strand_edges, o.strand_edges + off]).astype(np.int32)
    explicit = np.concatenate([m.edges, np.asarray(plain, dtype=np.int32).reshape(-1, 2) + off])
    m.edges = finalize_edges(explicit, m.strand_edges, m.triangles)
    return off


def _sqnorm3(v) -> float:
    """Eigen squaredNorm of a Vector3d: (x*x + y*y) + z*z."""
    return (float(v[0]) * float(v[0]) + float(v[1]) * float(v[1])) + float(v[2]) * float(v[2])


def _norm3(v) -> float:
    return math.sqrt(_sqnorm3(v))


def _matvec3(R, v):
    """Matrix3d * Vector3d, each row ((r0*v0 + r1*v1) + r2*v2)."""
    return np.array([(R[i, 0] * v[0] + R[i, 1] * v[1]) + R[i, 2] * v[2] for i in range(3)])


def compute_lumped_masses(m: Mesh, area_density: float, line_density: float) -> None:
    """compute_lumped_masses (mesh.cpp:57-77); pinned vertices stay pinned."""
    n = len(m.positions)
    mass = np.zeros(n)
    P = m.positions
    for t in m.triangles:
        e1, e2 = P[t[1]] - P[t[0]], P[t[2]] - P[t[0]]
        a = area_density * 0.5 * _norm3(np.cross(e1, e2))
        for k in range(3):
            mass[t[k]] += a / 3.0
    for e in m.strand_edges:
        a = line_density * _norm3(P[e[1]] - P[e[0]])
        mass[e[0]] += 0.5 * a
        mass[e[1]] += 0.5 * a
    pinned = m.inv_mass == 0.0
    inv = np.where(mass > 0.0, 1.0 / np.where(mass > 0.0, mass, 1.0), 1.0)
    m.inv_mass = np.where(pinned, 0.0, inv)


def lumped_inv_mass_fast(P, tris, strands, area_density, line_density, pinned=None):
    """Vectorised compute_lumped_masses for large meshes."""
    n = len(P)
    mass = np.zeros(n)
    if len(tris):
        e1 = P[tris[:, 1]] - P[tris[:, 0]]
        e2 = P[tris[:, 2]] - P[tris[:, 0]]
        a = area_density * 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1) / 3.0
        for k in range(3):
            np.add.at(mass, tris[:, k], a)
    if len(strands):
        a = line_density * np.linalg.norm(P[strands[:, 1]] - P[strands[:, 0]], axis=1)
        np.add.at(mass, strands[:, 0], 0.5 * a)
        np.add.at(mass, strands[:, 1], 0.5 * a)
    inv = np.where(mass > 0.0, 1.0 / np.where(mass > 0.0, mass, 1.0), 1.0)
    if pinned is not None:
        inv = np.where(pinned, 0.0, inv)
    return inv


# --------------------------------------------------------------- builders
def make_grid_patch(nx, ny, size_u, size_v, origin, du=(1, 0, 0), dv=(0, 1, 0)) -> Mesh:
    """make_grid_patch, fixtures.cpp:14-35 (alternating diagonals)."""
    o, du, dv = (np.asarray(a, dtype=np.float64) for a in (origin, du, dv))
    i, j = np.meshgrid(np.arange(nx), np.arange(ny))
    i, j = i.reshape(-1), j.reshape(-1)
    P = o + du * (size_u * i / (nx - 1))[:, None] + dv * (size_v * j / (ny - 1))[:, None]
    tris = []
    for jj in range(ny - 1):
        for ii in range(nx - 1):
            a, b, c, d = jj * nx + ii, jj * nx + ii + 1, (jj + 1) * nx + ii + 1, (jj + 1) * nx + ii
            if (ii + jj) % 2 == 0:
                tris += [(a, b, c), (a, c, d)]
            else:
                tris += [(a, b, d), (b, c, d)]
    return make_mesh(P, tris)


def make_pyramid(base, height, c) -> Mesh:
    """make_pyramid, fixtures.cpp:37-46 (all vertices static)."""
    c = np.asarray(c, dtype=np.float64)
    h = base / 2.0
    P = [c + (-h, -h, 0), c + (h, -h, 0), c + (h, h, 0), c + (-h, h, 0), c + (0, 0, height)]
    tris = [(0, 1, 4), (1, 2, 4), (2, 3, 4), (3, 0, 4), (0, 2, 1), (0, 3, 2)]
    m = make_mesh(P, tris)
    m.inv_mass = np.zeros(5)
    return m


def make_icosphere(subdivisions, radius, center) -> Mesh:
    """make_icosphere, fixtures.cpp:48-88."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    verts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t),
             (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    verts = [np.asarray(v, dtype=np.float64) / _norm3(np.asarray(v, dtype=np.float64)) for v in verts]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdivisions):
        mid = {}

        def midpoint(a, b):
            key = (min(a, b), max(a, b))
            if key in mid:
                return mid[key]
            v = verts[a] + verts[b]
            verts.append(v / _norm3(v))
            mid[key] = len(verts) - 1
            return mid[key]

        nxt = []
        for f in faces:
            ab, bc, ca = midpoint(f[0], f[1]), midpoint(f[1], f[2]), midpoint(f[2], f[0])
            nxt += [(f[0], ab, ca), (f[1], bc, ab), (f[2], ca, bc), (ab, bc, ca)]
        faces = nxt
    P = np.asarray(center, dtype=np.float64) + radius * np.asarray(verts)
    return make_mesh(P, faces)


def make_lathe(zs, radii, slices, close_caps) -> Mesh:
    """make_lathe, fixtures.cpp:90-117."""
    P = []
    stacks = len(zs)
    for s in range(stacks):
        for k in range(slices):
            a = 2.0 * PI * k / slices
            P.append((radii[s] * math.cos(a), radii[s] * math.sin(a), zs[s]))

    def vid(s, k):
        return s * slices + (k % slices)

    tris = []
    for s in range(stacks - 1):
        for k in range(slices):
            tris += [(vid(s, k), vid(s, k + 1), vid(s + 1, k)),
                     (vid(s, k + 1), vid(s + 1, k + 1), vid(s + 1, k))]
    if close_caps:
        p0 = len(P)
        P.append((0, 0, zs[0]))
        p1 = len(P)
        P.append((0, 0, zs[-1]))
        for k in range(slices):
            tris += [(p0, vid(0, k + 1), vid(0, k)), (p1, vid(stacks - 1, k), vid(stacks - 1, k + 1))]
    return make_mesh(P, tris)


def make_tube(radius, height, slices, stacks, center) -> Mesh:
    zs = [-height / 2 + height * s / (stacks - 1) for s in range(stacks)]
    m = make_lathe(zs, [radius] * stacks, slices, False)
    m.positions = m.positions + np.asarray(center, dtype=np.float64)
    return m


def make_strand(n, a, b) -> Mesh:
    """make_strand, fixtures.cpp:139-145."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    P = [a + (b - a) * (i / n) for i in range(n + 1)]
    return make_mesh(P, (), [(i, i + 1) for i in range(n)])


def rotation_matrix(axis, angle):
    """Eigen::AngleAxisd::toRotationMatrix."""
    ax = np.asarray(axis, dtype=np.float64)
    ax = ax / _norm3(ax)
    s, c = math.sin(angle), math.cos(angle)
    sa, ca = s * ax, (1.0 - c) * ax
    R = np.empty((3, 3))
    t = ca[0] * ax[1]
    R[0, 1], R[1, 0] = t - sa[2], t + sa[2]
    t = ca[0] * ax[2]
    R[0, 2], R[2, 0] = t + sa[1], t - sa[1]
    t = ca[1] * ax[2]
    R[1, 2], R[2, 1] = t - sa[0], t + sa[0]
    R[0, 0], R[1, 1], R[2, 2] = ca * ax + c
    return R


def rotate_about(x, center, axis, angle):
    R = rotation_matrix(axis, angle)
    c = np.asarray(center, dtype=np.float64)
    return np.array([c + _matvec3(R, p - c) for p in np.asarray(x, dtype=np.float64)]).reshape(-1, 3)


def _scene(name, m: Mesh, y, benign=True, penetrating=False) -> Scene:
    return Scene(name, m.positions.copy(), np.asarray(y, dtype=np.float64).copy(),
                 m.triangles.astype(np.int32), m.edges.astype(np.int32),
                 m.strand_edges.astype(np.int32), m.inv_mass.astype(np.float64), benign, penetrating)


# ---------------------------------------------------------------- fixtures
def fixture_spike_patch(theta_deg: float) -> Scene:
    """fixture_spike_patch, fixtures.cpp:180-199."""
    m = make_pyramid(0.04, 0.03, (0.0013, -0.0017, 0))
    patch = make_grid_patch(9, 9, 0.08, 0.08, (-0.04, -0.04, 0.036))
    compute_lumped_masses(patch, 0.1, 0.0)
    append_mesh(m, patch)
    x = m.positions
    y = rotate_about(x, (0, 0, 0.036), (0, 0, 1), theta_deg * PI / 180.0)
    y = y + np.array([0, 0, -0.012])
    st = m.inv_mass == 0.0
    y[st] = x[st]
    return _scene("spike_theta%d" % int(theta_deg), m, y, theta_deg <= 45.0, True)


def fixture_press(push: float) -> Scene:
    """fixture_press, fixtures.cpp:201-219."""
    m = make_grid_patch(7, 7, 0.06, 0.06, (-0.03, -0.03, 0.0))
    m.inv_mass = np.zeros(len(m.positions))
    top = make_grid_patch(7, 7, 0.06, 0.06, (-0.0295, -0.0295, 0.003))
    compute_lumped_masses(top, 0.1, 0.0)
    append_mesh(m, top)
    y = m.positions.copy()
    y[49:, 2] -= push
    return _scene("press", m, y, push <= 0.01, push > 0.003)


def fixture_tube_twist() -> Scene:
    """fixture_tube_twist, fixtures.cpp:221-242."""
    m = make_tube(0.015, 0.06, 12, 7, (0, 0, 0))
    compute_lumped_masses(m, 0.1, 0.0)
    y = m.positions.copy()
    for v in range(len(y)):
        t = (y[v, 2] + 0.03) / 0.06
        ang = (t - 0.5) * (2.0 * PI / 1.5)
        c = np.array([0, 0, y[v, 2]])
        p = c + _matvec3(rotation_matrix((0, 0, 1), ang), y[v] - c)
        p[2] *= 0.7
        y[v] = p
    return _scene("tube_twist", m, y, True, False)


def fixture_particles() -> Scene:
    """fixture_particles, fixtures.cpp:244-254."""
    m = make_mesh([(-0.005, 0, 0), (0.005, 0, 0)])
    return _scene("particles", m, [(0.005, 0, 0), (-0.005, 0, 0)], True, False)


def fixture_strand_cross() -> Scene:
    """fixture_strand_cross, fixtures.cpp:256-272."""
    m = make_strand(6, (-0.03, 0, 0.002), (0.03, 0, 0.002))
    o = make_strand(6, (0, -0.03, 0), (0, 0.03, 0))
    compute_lumped_masses(m, 0.0, 0.05)
    compute_lumped_masses(o, 0.0, 0.05)
    append_mesh(m, o)
    y = m.positions.copy()
    y[:7, 2] -= 0.006
    return _scene("strand_cross", m, y, True, False)


def fixture_random(seed: int, index: int) -> Scene:
    """fixture_random, fixtures.cpp:274-302."""
    rng = MT19937_64((seed * 1000003 + index) & 0xFFFFFFFFFFFFFFFF)
    uni = lambda: rng.uniform(-1.0, 1.0)  # noqa: E731
    m = make_grid_patch(6, 6, 0.05, 0.05, (-0.025, -0.025, 0.0))
    top = make_grid_patch(6, 6, 0.05, 0.05, (-0.024, -0.024, 0.004 + 0.002 * uni()))
    compute_lumped_masses(m, 0.1, 0.0)
    compute_lumped_masses(top, 0.1, 0.0)
    append_mesh(m, top)
    x = m.positions
    # Vec3(a, b, c) constructor arguments: g++ evaluates them right to left,
    # so the reference draws z, then y, then x (fixtures.cpp:290,292).
    az = 1.5 + 0.5 * uni()
    ay = uni()
    axis = (uni(), ay, az)
    ang = (30.0 + 25.0 * uni()) * PI / 180.0
    sz = -0.008 + 0.004 * uni()
    sy = 0.004 * uni()
    shift = np.array([0.004 * uni(), sy, sz])
    y = x.copy()
    y[36:] = rotate_about(y[36:], (0, 0, 0.004), axis, ang) + shift
    for v in range(36):
        y[v, 2] += 0.003 * math.sin(3.0 * x[v, 0] / 0.05) * uni()
    return _scene("random_%d" % index, m, y, False, False)


def scene_fixtures(seed: int = 0) -> list[Scene]:
    """scene_fixtures, fixtures.cpp:304-314: the 21-scene acceptance battery."""
    out = [fixture_spike_patch(th) for th in (0.0, 45.0, 90.0, 135.0)]
    out += [fixture_press(0.006), fixture_press(0.012), fixture_tube_twist(), fixture_particles(),
            fixture_strand_cross()]
    out += [fixture_random(seed, i) for i in range(12)]
    return out


# ------------------------------------------------------- benchmark scenes
def _ribbon_topology(n_across: int, n_along: int, base: int):
    i, j = np.meshgrid(np.arange(n_across - 1), np.arange(n_along - 1), indexing="ij")
    i, j = i.reshape(-1), j.reshape(-1)
    a = base + j * n_across + i
    b = a + 1
    c = a + n_across + 1
    d = a + n_across
    alt = ((i + j) % 2) == 0
    t1 = np.where(alt[:, None], np.stack([a, b, c], 1), np.stack([a, b, d], 1))
    t2 = np.where(alt[:, None], np.stack([a, c, d], 1), np.stack([b, c, d], 1))
    return np.stack([t1, t2], 1).reshape(-1, 3).astype(np.int32)


def knot_scene(n_along: int = 935, n_across: int = 20, spacing: float = 3e-3, p: int = 2, q: int = 3,
               r_inner: float = 6e-3, pull: float = 3.5e-3, end_gap: float = 0.04,
               jitter_seed: int | None = None, name: str = "knot") -> Scene:
    """Two twisted cloth strips swept along the two components of a torus link
    (each strip follows a (p, q) torus knot; the second is phase-shifted by
    pi/p around the tube), so the strips wind around each other and twist
    about the tube centre line. The strips are open (end_gap of parameter
    left unwound) and start intersection-free: the ribbons occupy radial
    bands [r_inner, r_inner + width] of the tube cross-section at distinct
    poloidal angles. The target tightens the knot: every vertex is pulled
    ``pull`` metres towards the tube centre line and the inner rows of the 2p
    strip passes interpenetrate there.

    CFG2 (reef): n_along=935 -> 37,400 V / 70,984 T. CFG3 (bow): n_along=1870
    -> 74,800 V / 141,964 T.
    """
    width = (n_across - 1) * spacing
    rho_c = r_inner + 0.5 * width
    length = (n_along - 1) * spacing
    s_total = 2.0 * PI * p
    s_span = s_total * (1.0 - end_gap)
    # major radius such that the centre row has the requested along-spacing
    R = length / s_span
    rng = np.random.default_rng(jitter_seed) if jitter_seed is not None else None
    P_all, Y_all, T_all = [], [], []
    for k in range(2):
        s = np.linspace(0.0, s_span, n_along)
        rho = r_inner + spacing * np.arange(n_across)
        S, RHO = np.meshgrid(s, rho, indexing="ij")  # (along, across)
        phi = (q / p) * S + k * (PI / p)
        if rng is not None:
            phi = phi + 0.02 * rng.standard_normal()
        th = S
        ring = R + RHO * np.cos(phi)
        P = np.stack([ring * np.cos(th), ring * np.sin(th), RHO * np.sin(phi)], -1).reshape(-1, 3)
        rho_y = RHO - pull
        ring_y = R + rho_y * np.cos(phi)
        Y = np.stack([ring_y * np.cos(th), ring_y * np.sin(th), rho_y * np.sin(phi)], -1).reshape(-1, 3)
        base = k * n_along * n_across
        T_all.append(_ribbon_topology(n_across, n_along, base))
        P_all.append(P)
        Y_all.append(Y)
    P = np.concatenate(P_all)
    Y = np.concatenate(Y_all)
    T = np.concatenate(T_all)
    E = finalize_edges(np.zeros((0, 2), np.int32), np.zeros((0, 2), np.int32), T)
    inv = lumped_inv_mass_fast(P, T, np.zeros((0, 2), np.int64), 0.1, 0.0)
    del rho_c
    return Scene(name, P, Y, T, E, np.zeros((0, 2), np.int32), inv, True, True)


def ply_knot(n_along: int = 935, n_across: int = 20, spacing: float = 3e-3, p: int = 2, q: int = 3,
             tube: float = 0.03, gap: float = 2.5e-3, squeeze: float = 2.0e-3, slide: float = 2.0e-3,
             end_gap: float = 0.04, jitter_seed: int | None = None, name: str = "knot",
             density: float = 0.1) -> Scene:
    """Two cloth strips ("plies") laid face to face along the same twisted band
    of a (p, q) torus knot — a two-ply ribbon tied into a knot. Ply A lies on
    the torus of tube radius ``tube + gap/2``, ply B on ``tube - gap/2``; the
    band covers a poloidal angle of width/tube around the knot path, so the
    strips twist around the tube as they wind. Concentric tori cannot
    intersect, hence the start state is intersection-free with a ``gap``
    clearance between the strips (in-plane neighbours at 3 mm spacing are
    within d_max as well).

    Tightening target: the plies are pressed into each other with a squeeze
    that varies along the knot (0 .. ``gap/2 + squeeze`` per ply, so they
    interpenetrate by up to ``2*squeeze`` where the knot is tightest) and ply A
    slides ``slide`` metres along the path relative to ply B.

    CFG2 (reef): n_along=935 -> 37,400 V / 70,984 T. CFG3 (bow): n_along=1870
    -> 74,800 V / 142,044 T.
    """
    width = (n_across - 1) * spacing
    length = (n_along - 1) * spacing
    s_span = 2.0 * PI * p * (1.0 - end_gap)
    R = length / s_span
    rng = np.random.default_rng(jitter_seed) if jitter_seed is not None else None
    phase = 0.0 if rng is None else rng.uniform(0, 2 * PI)
    s = np.linspace(0.0, s_span, n_along)
    u = (np.arange(n_across) - 0.5 * (n_across - 1)) * spacing
    S_, U_ = np.meshgrid(s, u, indexing="ij")
    P_all, Y_all, T_all = [], [], []
    for k, sign in enumerate((+1.0, -1.0)):
        r0 = tube + sign * 0.5 * gap
        phi = (q / p) * S_ + U_ / tube
        # squeeze profile along the knot: tight where sin > 0
        prof = 0.5 * (1.0 + np.sin(3.0 * S_ + phase))
        r1 = r0 - sign * prof * (0.5 * gap + squeeze)
        th = S_
        th1 = S_ + (sign * 0.5 * slide / R)
        ring0 = R + r0 * np.cos(phi)
        P = np.stack([ring0 * np.cos(th), ring0 * np.sin(th), r0 * np.sin(phi)], -1).reshape(-1, 3)
        ring1 = R + r1 * np.cos(phi)
        Y = np.stack([ring1 * np.cos(th1), ring1 * np.sin(th1), r1 * np.sin(phi)], -1).reshape(-1, 3)
        T_all.append(_ribbon_topology(n_across, n_along, k * n_along * n_across))
        P_all.append(P)
        Y_all.append(Y)
    P = np.concatenate(P_all)
    Y = np.concatenate(Y_all)
    T = np.concatenate(T_all)
    E = finalize_edges(np.zeros((0, 2), np.int32), np.zeros((0, 2), np.int32), T)
    inv = lumped_inv_mass_fast(P, T, np.zeros((0, 2), np.int64), density, 0.0)
    del width
    return Scene(name, P, Y, T, E, np.zeros((0, 2), np.int32), inv, True, True)


KNOT_DEFAULTS = dict(squeeze=-0.2e-3, slide=3e-3)  # plies close to a 0.2 mm gap and slide 3 mm


def reef_knot(**kw) -> Scene:
    """CFG2: 37,400 V / 70,984 T two-ply knot (ply_knot), tightening step."""
    kw = {**KNOT_DEFAULTS, **kw}
    kw.setdefault("name", "reef_knot")
    return ply_knot(n_along=935, **kw)


def bow_knot(**kw) -> Scene:
    """CFG3: 74,800 V / 142,044 T two-ply knot (ply_knot), tightening step."""
    kw = {**KNOT_DEFAULTS, **kw}
    kw.setdefault("name", "bow_knot")
    return ply_knot(n_along=1870, **kw)


# The frame of the benchmark: the plies are driven up to 0.2 mm into each other
# where the knot is tightest while sliding 1.5 mm relative to each other. A
# scan of squeeze in [-0.1, +0.1] mm at this slide converges in 6-11 Alg.-1
# steps in both coloring modes (the paper's bow knot: 5.4 on average, 17 at
# most); at a 3 mm slide some frames need 40+ steps or stall.
FRAME_DEFAULTS = dict(squeeze=0.1e-3, slide=1.5e-3)
# Material of the frame: 0.5 kg/m^2 cloth with 10 N/m springs, at which the
# block-Jacobi PCG reaches the reference's 1e-6 relative residual within its
# 400-iteration cap (the default 0.1 kg/m^2 / 50 N/m stops at the cap), so the
# Newton target is the actual implicit-Euler solution. ENERGY goes to the
# EnergyModel of both implementations.
FRAME_DENSITY = 0.5
FRAME_ENERGY = dict(spring_stiffness=10.0)


def knot_frame(n_along: int = 1870, dt: float = 0.01, **kw):
    """A simulation frame of the tightening knot for the dynamics step
    (dynamics.cpp:326-349): the plies at rest (x, 2.5 mm apart) moving with
    v0 = (y_tight - x) / dt, where y_tight is the ply_knot tightening target
    (squeeze / slide / density in ``kw``, FRAME_DEFAULTS / FRAME_DENSITY
    otherwise; simulate with the EnergyModel overrides FRAME_ENERGY). One implicit-Euler
    step with the paper's knot time step dt = 1/100 then drives
    the plies into each other; resolve makes the frame intersection-free.
    Returns (scene, v0)."""
    kw = {**FRAME_DEFAULTS, "density": FRAME_DENSITY, **kw}
    kw.setdefault("name", "bow_knot_frame" if n_along == 1870 else "knot_frame")
    sc = ply_knot(n_along=n_along, **kw)
    v0 = (sc.y - sc.x) / dt
    return sc, v0


def cloth_on_sphere(n: int = 64, spacing: float = 0.01, drop: float = 0.03) -> Scene:
    """CFG1: a 64x64 cloth (7,938 T) at 10 mm spacing hovering 24 mm above a
    static icosphere (s = 4, r = 0.2 m, 5,120 T); the target is one dt = 1/30 s
    fall of ``drop`` metres, which pushes the centre of the cloth into the
    sphere."""
    sphere = make_icosphere(4, 0.2, (0, 0, 0))
    sphere.inv_mass = np.zeros(len(sphere.positions))
    size = spacing * (n - 1)
    cloth = make_grid_patch(n, n, size, size, (-size / 2, -size / 2, 0.2 + 0.024))
    compute_lumped_masses(cloth, 0.1, 0.0)
    append_mesh(sphere, cloth)
    y = sphere.positions.copy()
    ns = 2562
    y[ns:, 2] -= drop
    return _scene("cloth_on_sphere", sphere, y, True, True)


def codim_mix(n_bodies: int = 8, n_strands: int = 1000, strand_segments: int = 64,
              n_particles: int = 96000, seed: int = 0) -> Scene:
    """CFG4: 8 closed icosphere (s = 4) bodies stacked in a column, 1,000 hair
    strands of 64 segments hanging beside them and 96K particles in a jittered
    lattice above; everything falls 8 mm. Exercises the VV, VE, VT and EE
    kinds (the reference has no tetrahedra: closed surfaces stand in)."""
    rng = np.random.default_rng(seed)
    Ps, Ts, Ss, Is = [], [], [], []
    base = 0
    r = 0.05
    for b in range(n_bodies):
        sph = make_icosphere(4, r, (0.0, 0.0, b * (2 * r + 0.006)))
        Ps.append(sph.positions)
        Ts.append(sph.triangles + base)
        Is.append(lumped_inv_mass_fast(sph.positions, sph.triangles, np.zeros((0, 2), np.int64), 0.1, 0.0))
        base += len(sph.positions)
    side = int(math.ceil(math.sqrt(n_strands)))
    seg = 0.004
    for s in range(n_strands):
        gx, gy = s % side, s // side
        x0 = 0.12 + gx * 0.006
        y0 = -0.1 + gy * 0.006
        z = 0.8 - seg * np.arange(strand_segments + 1)
        pts = np.stack([np.full_like(z, x0), np.full_like(z, y0), z], 1)
        Ps.append(pts)
        Ss.append(np.stack([np.arange(strand_segments), np.arange(1, strand_segments + 1)], 1) + base)
        Is.append(np.full(len(pts), 1.0 / (0.05 * seg)))
        base += len(pts)
    m = int(round(n_particles ** (1 / 3)))
    while m ** 3 < n_particles:
        m += 1
    g = np.stack(np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij"), -1).reshape(-1, 3)[:n_particles]
    pts = np.array([-0.4, -0.4, 1.0]) + g * 0.005 + rng.uniform(-0.0005, 0.0005, size=g.shape)
    Ps.append(pts)
    Is.append(np.full(len(pts), 1000.0))
    P = np.concatenate(Ps)
    T = np.concatenate(Ts).astype(np.int32)
    S = np.concatenate(Ss).astype(np.int32)
    E = finalize_edges(np.zeros((0, 2), np.int32), S, T)
    inv = np.concatenate(Is)
    Y = P.copy()
    Y[:, 2] -= 0.008
    Y[:len(Y) - n_particles, 0] += 0.003 * np.sin(P[:len(Y) - n_particles, 2] * 40.0)
    return Scene("codim_mix", P, Y, T, E, S, inv, True, False)

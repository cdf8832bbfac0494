// FP64 geometry on the device with the exact evaluation order of the
// reference's Eigen Vector3d expressions. This file is
// compiled with -fmad=false: every a*b+c below is a separate IEEE multiply and
// add, as in the reference's x86-64 SSE2 build. Distances, weights and
// directions are therefore bit-identical to the reference restatement.
//
// Reference: proj/src/distance.cpp (closest points), proj/src/constraints.cpp
// (stencil determinant, contact / edge rows).
#pragma once

#include <cstdint>

namespace tw {

struct d3 {
    double x, y, z;
};

__host__ __device__ __forceinline__ d3 mk(double x, double y, double z) { return d3{x, y, z}; }
__host__ __device__ __forceinline__ d3 add(d3 a, d3 b) { return d3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ __forceinline__ d3 sub(d3 a, d3 b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ __forceinline__ d3 neg(d3 a) { return d3{-a.x, -a.y, -a.z}; }
__host__ __device__ __forceinline__ d3 scl(double s, d3 a) { return d3{s * a.x, s * a.y, s * a.z}; }
__host__ __device__ __forceinline__ d3 dvd(d3 a, double s) { return d3{a.x / s, a.y / s, a.z / s}; }
__host__ __device__ __forceinline__ double dot(d3 a, d3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__host__ __device__ __forceinline__ double sqn(d3 a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
__host__ __device__ __forceinline__ double nrm(d3 a) { return sqrt(sqn(a)); }
__host__ __device__ __forceinline__ d3 crs(d3 a, d3 b) {
    return d3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__host__ __device__ __forceinline__ d3 normalized(d3 a) {
    const double z = sqn(a);
    return z > 0.0 ? dvd(a, sqrt(z)) : a;
}
__host__ __device__ __forceinline__ bool is_zero(d3 a) {
    return fabs(a.x) <= 1e-12 && fabs(a.y) <= 1e-12 && fabs(a.z) <= 1e-12;
}
// std::clamp / std::min / std::max with the reference's comparison order
__host__ __device__ __forceinline__ double clampd(double v, double lo, double hi) {
    return v < lo ? lo : (hi < v ? hi : v);
}
__host__ __device__ __forceinline__ double mind(double a, double b) { return b < a ? b : a; }
__host__ __device__ __forceinline__ double maxd(double a, double b) { return a < b ? b : a; }

// ---------------------------------------------------------------- keys
enum : int { KV = 0, KE = 1, KT = 2 };

__host__ __device__ __forceinline__ uint64_t pair_key(int ka, int ia, int kb, int ib) {
    return (uint64_t(ka) << 62) | (uint64_t(kb) << 60) | (uint64_t(uint32_t(ia)) << 30) |
           uint64_t(uint32_t(ib));
}
__host__ __device__ __forceinline__ int key_ka(uint64_t k) { return int(k >> 62); }
__host__ __device__ __forceinline__ int key_kb(uint64_t k) { return int((k >> 60) & 3); }
__host__ __device__ __forceinline__ int key_ia(uint64_t k) { return int((k >> 30) & 0x3fffffff); }
__host__ __device__ __forceinline__ int key_ib(uint64_t k) { return int(k & 0x3fffffff); }

// ------------------------------------------------------- ClosestResult
struct Closest {
    double dist;
    double wa[3];
    double wb[3];
    d3 dir;
    bool degenerate;
};

__device__ __forceinline__ void closest_init(Closest& r) {
    r.dist = 0.0;
    r.wa[0] = 1.0, r.wa[1] = 0.0, r.wa[2] = 0.0;
    r.wb[0] = 1.0, r.wb[1] = 0.0, r.wb[2] = 0.0;
    r.dir = mk(0, 0, 0);
    r.degenerate = false;
}

// distance.cpp:11-15
__device__ __forceinline__ d3 safe_unit(d3 v, bool& ok) {
    const double n = nrm(v);
    ok = n > 1e-20;
    return ok ? dvd(v, n) : mk(0, 0, 0);
}

// distance.cpp:18-24
__device__ __forceinline__ d3 any_perpendicular(d3 d) {
    d3 axis = fabs(d.x) < fabs(d.y) ? mk(1, 0, 0) : mk(0, 1, 0);
    if (fabs(d.z) < fabs(dot(axis, d))) axis = mk(0, 0, 1);
    bool ok = false;
    const d3 p = safe_unit(crs(d, axis), ok);
    return ok ? p : mk(1, 0, 0);
}

// distance.cpp:34-45
__device__ __forceinline__ void closest_vv(d3 p, d3 q, Closest& r) {
    closest_init(r);
    const d3 d = sub(p, q);
    r.dist = nrm(d);
    if (r.dist >= 1e-9) {
        r.dir = dvd(d, r.dist);
    } else {
        r.degenerate = true;
    }
}

// distance.cpp:47-64
__device__ __forceinline__ void closest_ve(d3 p, d3 e0, d3 e1, Closest& r) {
    closest_init(r);
    const d3 d = sub(e1, e0);
    const double dd = sqn(d);
    double t = dd > 0.0 ? dot(sub(p, e0), d) / dd : 0.0;
    t = clampd(t, 0.0, 1.0);
    const d3 c = add(e0, scl(t, d));
    r.wb[0] = 1.0 - t, r.wb[1] = t, r.wb[2] = 0.0;
    const d3 gap = sub(p, c);
    r.dist = nrm(gap);
    if (r.dist >= 1e-9) {
        r.dir = dvd(gap, r.dist);
    } else {
        r.dir = any_perpendicular(d);
        r.degenerate = true;
    }
}

// distance.cpp:66-151 (Ericson's closest point on triangle). Returns false
// for a degenerate triangle (the reference's nullopt).
__device__ __forceinline__ bool closest_vt(d3 p, d3 a, d3 b, d3 c, Closest& r) {
    const d3 ab = sub(b, a), ac = sub(c, a);
    const d3 n = crs(ab, ac);
    if (0.5 * nrm(n) <= 1e-12) return false;
    const d3 ap = sub(p, a);
    const double d1 = dot(ab, ap), d2 = dot(ac, ap);
    double w0, w1, w2;
    d3 cl;
    if (d1 <= 0.0 && d2 <= 0.0) {
        cl = a, w0 = 1.0, w1 = 0.0, w2 = 0.0;
    } else {
        const d3 bp = sub(p, b);
        const double d3v = dot(ab, bp), d4 = dot(ac, bp);
        const double vc = d1 * d4 - d3v * d2;
        if (d3v >= 0.0 && d4 <= d3v) {
            cl = b, w0 = 0.0, w1 = 1.0, w2 = 0.0;
        } else if (vc <= 0.0 && d1 >= 0.0 && d3v <= 0.0) {
            const double v = d1 / (d1 - d3v);
            cl = add(a, scl(v, ab)), w0 = 1.0 - v, w1 = v, w2 = 0.0;
        } else {
            const d3 cp = sub(p, c);
            const double d5 = dot(ab, cp), d6 = dot(ac, cp);
            const double vb = d5 * d2 - d1 * d6;
            const double va = d3v * d6 - d5 * d4;
            if (d6 >= 0.0 && d5 <= d6) {
                cl = c, w0 = 0.0, w1 = 0.0, w2 = 1.0;
            } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
                const double v = d2 / (d2 - d6);
                cl = add(a, scl(v, ac)), w0 = 1.0 - v, w1 = 0.0, w2 = v;
            } else if (va <= 0.0 && (d4 - d3v) >= 0.0 && (d5 - d6) >= 0.0) {
                const double v = (d4 - d3v) / ((d4 - d3v) + (d5 - d6));
                cl = add(b, scl(v, sub(c, b))), w0 = 0.0, w1 = 1.0 - v, w2 = v;
            } else {
                const double denom = va + vb + vc;
                const double v = vb / denom;
                const double u = vc / denom;
                cl = add(add(a, scl(v, ab)), scl(u, ac)), w0 = 1.0 - v - u, w1 = v, w2 = u;
            }
        }
    }
    closest_init(r);
    r.wb[0] = w0, r.wb[1] = w1, r.wb[2] = w2;
    const d3 gap = sub(p, cl);
    r.dist = nrm(gap);
    if (r.dist >= 1e-9) {
        r.dir = dvd(gap, r.dist);
    } else {
        r.dir = normalized(n);
        r.degenerate = true;
    }
    return true;
}

// distance.cpp:153-216
__device__ __forceinline__ bool closest_ee(d3 p1, d3 p2, d3 q1, d3 q2, Closest& r) {
    const d3 d1 = sub(p2, p1), d2 = sub(q2, q1), rr = sub(p1, q1);
    const double a = sqn(d1), e = sqn(d2), f = dot(d2, rr);
    if (sqrt(a) <= 1e-12 || sqrt(e) <= 1e-12) return false;
    const double c = dot(d1, rr), b = dot(d1, d2);
    const double denom = a * e - b * b;
    double s, t;
    if (denom > 1e-12 * a * e) {
        s = clampd((b * f - c * e) / denom, 0.0, 1.0);
        t = (b * s + f) / e;
        if (t < 0.0) {
            t = 0.0;
            s = clampd(-c / a, 0.0, 1.0);
        } else if (t > 1.0) {
            t = 1.0;
            s = clampd((b - c) / a, 0.0, 1.0);
        }
    } else {
        // near-parallel: endpoint enumeration (distance.cpp:174-198)
        double bs = 0.0, bt = 0.0, bd2 = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const double cs = k ? 1.0 : 0.0;
            const d3 ps = add(p1, scl(cs, d1));
            const double ct = clampd(dot(sub(ps, q1), d2) / e, 0.0, 1.0);
            const double dist2 = sqn(sub(ps, add(q1, scl(ct, d2))));
            if (dist2 < bd2) bs = cs, bt = ct, bd2 = dist2;
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const double ct = k ? 1.0 : 0.0;
            const d3 qt = add(q1, scl(ct, d2));
            const double cs = clampd(dot(sub(qt, p1), d1) / a, 0.0, 1.0);
            const double dist2 = sqn(sub(add(p1, scl(cs, d1)), qt));
            if (dist2 < bd2) bs = cs, bt = ct, bd2 = dist2;
        }
        s = bs, t = bt;
    }
    closest_init(r);
    r.wa[0] = 1.0 - s, r.wa[1] = s, r.wa[2] = 0.0;
    r.wb[0] = 1.0 - t, r.wb[1] = t, r.wb[2] = 0.0;
    const d3 gap = sub(add(p1, scl(s, d1)), add(q1, scl(t, d2)));
    r.dist = nrm(gap);
    if (r.dist >= 1e-9) {
        r.dir = dvd(gap, r.dist);
    } else {
        bool ok = false;
        r.dir = safe_unit(crs(d1, d2), ok);
        if (!ok) r.dir = any_perpendicular(d1);
        r.degenerate = true;
    }
    return true;
}

__device__ __forceinline__ void flip(Closest& r) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double t = r.wa[i];
        r.wa[i] = r.wb[i];
        r.wb[i] = t;
    }
    r.dir = neg(r.dir);
}

// pair_closest for a compile-time pair class (the kinds a proximity key
// holds: VV, VE, VT, EE). The vertex ids stay in registers (no runtime-indexed
// arrays, so no local memory); same calls and arithmetic as pair_closest.
template <int KA, int KB, typename LoadX>
__device__ __forceinline__ int pair_closest_t(const int (&ia)[3], const int (&ib)[3], const LoadX& X, Closest& r) {
#pragma unroll
    for (int i = 0; i <= KA; ++i)
#pragma unroll
        for (int j = 0; j <= KB; ++j)
            if (ia[i] == ib[j]) return -1;
    if constexpr (KA == KV && KB == KV) {
        closest_vv(X(ia[0]), X(ib[0]), r);
        return 1;
    } else if constexpr (KA == KV && KB == KE) {
        closest_ve(X(ia[0]), X(ib[0]), X(ib[1]), r);
        return 1;
    } else if constexpr (KA == KV && KB == KT) {
        return closest_vt(X(ia[0]), X(ib[0]), X(ib[1]), X(ib[2]), r) ? 1 : 0;
    } else if constexpr (KA == KE && KB == KE) {
        const bool swp = (ib[0] < ia[0]) || (ib[0] == ia[0] && ib[1] < ia[1]);
        if (!closest_ee(X(swp ? ib[0] : ia[0]), X(swp ? ib[1] : ia[1]), X(swp ? ia[0] : ib[0]),
                        X(swp ? ia[1] : ib[1]), r))
            return 0;
        if (swp) flip(r);
        return 1;
    } else {
        return -1;
    }
}

// Runs f(PairClass<KA, KB>{}) for the runtime class of a proximity key.
template <int A, int B>
struct PairClass {
    static constexpr int ka = A, kb = B;
};
template <typename F>
__device__ __forceinline__ bool with_pair_class(int ka, int kb, F&& f) {
    if (ka == KV && kb == KT) f(PairClass<KV, KT>{});
    else if (ka == KE && kb == KE) f(PairClass<KE, KE>{});
    else if (ka == KV && kb == KE) f(PairClass<KV, KE>{});
    else if (ka == KV && kb == KV) f(PairClass<KV, KV>{});
    else return false;
    return true;
}

// simplex_pair_closest (distance.cpp:218-253) for the canonical pair kinds the
// proximity set holds (a = V or E, b = V/E/T) plus the flipped kinds.
// ids: vertex ids of a (ia[0..2]) and b (ib[0..2]). Returns 1 value, 0
// nullopt, -1 adjacent / unsupported.
template <typename LoadX>
__device__ __forceinline__ int pair_closest(int ka, const int* ia, int kb, const int* ib,
                                            const LoadX& X, Closest& r) {
    for (int i = 0; i <= ka; ++i)
        for (int j = 0; j <= kb; ++j)
            if (ia[i] == ib[j]) return -1;
    if (ka == KV && kb == KV) {
        closest_vv(X(ia[0]), X(ib[0]), r);
        return 1;
    }
    if (ka == KV && kb == KE) {
        closest_ve(X(ia[0]), X(ib[0]), X(ib[1]), r);
        return 1;
    }
    if (ka == KE && kb == KV) {
        closest_ve(X(ib[0]), X(ia[0]), X(ia[1]), r);
        flip(r);
        return 1;
    }
    if (ka == KV && kb == KT) return closest_vt(X(ia[0]), X(ib[0]), X(ib[1]), X(ib[2]), r) ? 1 : 0;
    if (ka == KT && kb == KV) {
        if (!closest_vt(X(ib[0]), X(ia[0]), X(ia[1]), X(ia[2]), r)) return 0;
        flip(r);
        return 1;
    }
    if (ka == KE && kb == KE) {
        const bool swp = (ib[0] < ia[0]) || (ib[0] == ia[0] && ib[1] < ia[1]);
        const int* ea = swp ? ib : ia;
        const int* eb = swp ? ia : ib;
        if (!closest_ee(X(ea[0]), X(ea[1]), X(eb[0]), X(eb[1]), r)) return 0;
        if (swp) flip(r);
        return 1;
    }
    return -1;
}

// ------------------------------------------------------ constraint rows
// stencil_det / stencil_det_gradient, constraints.cpp:17-27
__device__ __forceinline__ double stencil_det(d3 p0, d3 p1, d3 p2, d3 p3) {
    return dot(sub(p1, p0), crs(sub(p2, p0), sub(p3, p0)));
}
__device__ __forceinline__ void stencil_grad(d3 p0, d3 p1, d3 p2, d3 p3, d3 g[4]) {
    g[1] = crs(sub(p2, p0), sub(p3, p0));
    g[2] = crs(sub(p3, p0), sub(p1, p0));
    g[3] = crs(sub(p1, p0), sub(p2, p0));
    g[0] = neg(add(add(g[1], g[2]), g[3]));
}

enum : int { ROW_VT = 0, ROW_EE = 1, ROW_VE = 2, ROW_VV = 3, ROW_EDGE = 4 };

struct Row {
    int kind;
    int nverts;
    int v[4];
    double value;
    d3 jac[4];
};

// Re-evaluation data of a row (Constraint::flavor / ref_volume / gap_weights /
// denom, constraints.hpp:26-33), recorded only by the stage entries.
enum : int { FLAVOR_VOLUME = 0, FLAVOR_GAP = 1, FLAVOR_LENGTH = 2 };
struct RowEval {
    int flavor;
    double ref_volume;
    double gw[4];
    double denom;
};

// build_gap_constraint, constraints.cpp:56-76. ids: a's then b's vertex ids
// (na + nb <= 4); wa, wb: the pair's cached weights; sign per side.
__device__ __forceinline__ void build_gap(int kind, int na, const int* va, int nb, const int* vb,
                                          const double* wa, const double* wb, double dist, d3 dir,
                                          double delta, Row& c, RowEval* ev = nullptr) {
    c.kind = kind;
    int n = 0;
    double gw[4];
    for (int i = 0; i < na; ++i, ++n) c.v[n] = va[i], gw[n] = wa[i];
    for (int i = 0; i < nb; ++i, ++n) c.v[n] = vb[i], gw[n] = -wb[i];
    c.nverts = n;
    for (int m = n; m < 4; ++m) c.v[m] = -1, c.jac[m] = mk(0, 0, 0);
    c.value = dist / delta - 1.0;
    for (int m = 0; m < n; ++m) c.jac[m] = scl(gw[m] / delta, dir);
    if (ev) {
        ev->flavor = FLAVOR_GAP;
        ev->ref_volume = 0.0;
        ev->denom = delta;
        for (int m = 0; m < 4; ++m) ev->gw[m] = m < n ? gw[m] : 0.0;
    }
}

// build_vt_constraint (constraints.cpp:86-115) / build_ee_constraint
// (constraints.cpp:117-142) / gap fallbacks; family = 1 forces the gap row.
// ka/kb, va/vb: the pair's simplices. Returns the row in c.
template <typename LoadX>
__device__ __forceinline__ void build_contact(int ka, const int* va, int kb, const int* vb,
                                              const double* wa, const double* wb, double dist,
                                              d3 dir, double delta, int family, const LoadX& X,
                                              Row& c, RowEval* ev = nullptr) {
    const int kind = (ka == KV && kb == KT) ? ROW_VT
                     : (ka == KE && kb == KE) ? ROW_EE
                     : (ka == KV && kb == KE) ? ROW_VE
                                              : ROW_VV;
    if (family == 1 || kind == ROW_VE || kind == ROW_VV) {
        build_gap(kind, ka + 1, va, kb + 1, vb, wa, wb, dist, dir, delta, c, ev);
        return;
    }
    d3 p0, p1, p2, p3;
    int i0, i1, i2, i3;
    double h;
    if (kind == ROW_VT) {
        i0 = va[0], i1 = vb[0], i2 = vb[1], i3 = vb[2];
        p0 = X(i0), p1 = X(i1), p2 = X(i2), p3 = X(i3);
        d3 n = crs(sub(p2, p1), sub(p3, p1));
        const double n_len = nrm(n);
        if (n_len < 1e-20) {
            build_gap(kind, 1, va, 3, vb, wa, wb, dist, dir, delta, c, ev);
            return;
        }
        n = dvd(n, n_len);
        if (dot(n, dir) < 0.0) n = neg(n);
        h = 0.5 * (delta - dist);
        const d3 hn = scl(h, n);
        const double wr = stencil_det(add(p0, hn), sub(p1, hn), sub(p2, hn), sub(p3, hn));
        if (fabs(wr) < 6.0 * 1e-18) {
            build_gap(kind, 1, va, 3, vb, wa, wb, dist, dir, delta, c, ev);
            return;
        }
        c.kind = kind;
        c.nverts = 4;
        c.v[0] = i0, c.v[1] = i1, c.v[2] = i2, c.v[3] = i3;
        c.value = stencil_det(p0, p1, p2, p3) / wr - 1.0;
        d3 g[4];
        stencil_grad(p0, p1, p2, p3, g);
        for (int m = 0; m < 4; ++m) c.jac[m] = dvd(g[m], wr);
        if (ev) *ev = RowEval{FLAVOR_VOLUME, wr, {0, 0, 0, 0}, 0.0};
        return;
    }
    // EE
    if (is_zero(dir)) {
        build_gap(kind, 2, va, 2, vb, wa, wb, dist, dir, delta, c, ev);
        return;
    }
    i0 = va[0], i1 = va[1], i2 = vb[0], i3 = vb[1];
    p0 = X(i0), p1 = X(i1), p2 = X(i2), p3 = X(i3);
    h = 0.5 * (delta - dist);
    const d3 hd = scl(h, dir);
    const double wr = stencil_det(add(p0, hd), add(p1, hd), sub(p2, hd), sub(p3, hd));
    if (fabs(wr) < 6.0 * 1e-18) {
        build_gap(kind, 2, va, 2, vb, wa, wb, dist, dir, delta, c, ev);
        return;
    }
    c.kind = kind;
    c.nverts = 4;
    c.v[0] = i0, c.v[1] = i1, c.v[2] = i2, c.v[3] = i3;
    c.value = stencil_det(p0, p1, p2, p3) / wr - 1.0;
    d3 g[4];
    stencil_grad(p0, p1, p2, p3, g);
    for (int m = 0; m < 4; ++m) c.jac[m] = dvd(g[m], wr);
    if (ev) *ev = RowEval{FLAVOR_VOLUME, wr, {0, 0, 0, 0}, 0.0};
}

__device__ __forceinline__ double row_jnorm(const Row& c) {
    double j = 0.0;
    for (int m = 0; m < c.nverts; ++m) j += sqn(c.jac[m]);
    return j;
}

}  // namespace tw

// Continuous-collision certification of one linear segment x0 -> x1 on the
// device: the per-stencil test of proj/src/testkit/ccd.cpp (the reference's
// trusted certifier of the intersection-free guarantee): the coplanarity
// cubic of the moving stencil in double-double arithmetic (testkit/dd.hpp),
// its roots in [0, 1] by bisection on the exact sign, inside tests at each
// root, and the planar fallback for identically coplanar stencils. FP64 in the
// reference's operation order (-fmad=false; the double-double products use
// explicit fma as dd.hpp does).
#pragma once

#include "tw_math.cuh"

namespace tw {
namespace ccd {

enum : int { HIT_NONE = 0, HIT_UNCERTAIN = 1, HIT_CERTAIN = 2 };
constexpr double kInsideMargin = 1e-8;

// ------------------------------------------------------ double-double
struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd dmk(double h, double l) { return dd{h, l}; }
__device__ __forceinline__ double dval(dd a) { return a.hi + a.lo; }
__device__ __forceinline__ int dsign(dd a) {
    if (a.hi > 0.0 || (a.hi == 0.0 && a.lo > 0.0)) return 1;
    if (a.hi < 0.0 || (a.hi == 0.0 && a.lo < 0.0)) return -1;
    return 0;
}
__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return dmk(s, (a - (s - bb)) + (b - bb));
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = a * b;
    return dmk(p, fma(a, b, -p));
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = a + b;
    return dmk(s, b - (s - a));
}
__device__ __forceinline__ dd dadd(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    s.lo += a.lo + b.lo;
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dsub(dd a, dd b) { return dadd(a, dmk(-b.hi, -b.lo)); }
__device__ __forceinline__ dd dmul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return quick_two_sum(p.hi, p.lo);
}
struct dd3 {
    dd x, y, z;
};
__device__ __forceinline__ dd3 dcross(dd3 a, dd3 b) {
    return dd3{dsub(dmul(a.y, b.z), dmul(a.z, b.y)), dsub(dmul(a.z, b.x), dmul(a.x, b.z)),
               dsub(dmul(a.x, b.y), dmul(a.y, b.x))};
}
__device__ __forceinline__ dd ddot(dd3 a, dd3 b) { return dadd(dadd(dmul(a.x, b.x), dmul(a.y, b.y)), dmul(a.z, b.z)); }
__device__ __forceinline__ dd3 dpoint(d3 v) { return dd3{dmk(v.x, 0.0), dmk(v.y, 0.0), dmk(v.z, 0.0)}; }

// ---------------------------------------------------- small sorted lists
struct dlist {
    double v[16];
    int n;
};
__device__ __forceinline__ void dl_push(dlist& l, double x) {
    if (l.n < 16) l.v[l.n++] = x;
}
__device__ __forceinline__ void dl_sort(dlist& l) {  // ascending (qsort with a < b compare)
    for (int i = 1; i < l.n; ++i) {
        const double x = l.v[i];
        int j = i - 1;
        while (j >= 0 && l.v[j] > x) l.v[j + 1] = l.v[j], --j;
        l.v[j + 1] = x;
    }
}

// ----------------------------------------------------- coplanarity cubic
struct cubic {
    dd c0, c1, c2, c3;
};
__device__ __forceinline__ cubic coplanarity_cubic(d3 u0, d3 du, d3 v0, d3 dv, d3 w0, d3 dw) {
    const dd3 U0 = dpoint(u0), DU = dpoint(du), V0 = dpoint(v0), DV = dpoint(dv), W0 = dpoint(w0), DW = dpoint(dw);
    const dd3 A = dcross(U0, V0);
    dd3 B = dcross(U0, DV);
    const dd3 B2 = dcross(DU, V0);
    B.x = dadd(B.x, B2.x), B.y = dadd(B.y, B2.y), B.z = dadd(B.z, B2.z);
    const dd3 C = dcross(DU, DV);
    cubic c;
    c.c0 = ddot(A, W0);
    c.c1 = dadd(ddot(A, DW), ddot(B, W0));
    c.c2 = dadd(ddot(B, DW), ddot(C, W0));
    c.c3 = ddot(C, DW);
    return c;
}
__device__ __forceinline__ dd eval_cubic(const cubic& c, double t) {
    const dd T = dmk(t, 0.0);
    return dadd(dmul(dadd(dmul(dadd(dmul(c.c3, T), c.c2), T), c.c1), T), c.c0);
}

__device__ inline void quadratic_roots01(double a, double b, double c, dlist& out) {
    if (fabs(a) < 1e-300) {
        if (fabs(b) > 1e-300) {
            const double r = -c / b;
            if (r > 0.0 && r < 1.0) dl_push(out, r);
        }
        return;
    }
    const double disc = b * b - 4.0 * a * c;
    if (disc < 0.0) return;
    const double sq = sqrt(disc);
    const double q = -0.5 * (b + (b >= 0.0 ? sq : -sq));
    const double r1 = q / a;
    const double r2 = fabs(q) > 1e-300 ? c / q : r1;
    if (r1 > 0.0 && r1 < 1.0) dl_push(out, r1);
    if (r2 > 0.0 && r2 < 1.0) dl_push(out, r2);
}

__device__ inline void cubic_roots01(const cubic& c, dlist& roots, dlist& extrema) {
    dlist bps;
    bps.n = 0;
    quadratic_roots01(3.0 * dval(c.c3), 2.0 * dval(c.c2), dval(c.c1), bps);
    extrema = bps;
    dl_push(bps, 0.0);
    dl_push(bps, 1.0);
    dl_sort(bps);
    for (int i = 0; i + 1 < bps.n; ++i) {
        double a = bps.v[i], b = bps.v[i + 1];
        const int sa = dsign(eval_cubic(c, a)), sb = dsign(eval_cubic(c, b));
        if (sa == 0) {
            dl_push(roots, a);
            continue;
        }
        if (sb == 0 || sa * sb > 0) continue;
        for (int it = 0; it < 100; ++it) {
            const double mm = 0.5 * (a + b);
            const int sm = dsign(eval_cubic(c, mm));
            if (sm == 0) {
                a = b = mm;
                break;
            }
            if (sm == sa) a = mm;
            else b = mm;
        }
        dl_push(roots, 0.5 * (a + b));
    }
    if (dsign(eval_cubic(c, 1.0)) == 0) dl_push(roots, 1.0);
    dl_sort(roots);
    int w = 0;
    for (int i = 0; i < roots.n; ++i)
        if (w == 0 || !(fabs(roots.v[w - 1] - roots.v[i]) < 1e-12)) roots.v[w++] = roots.v[i];
    roots.n = w;
}

// ------------------------------------------------------------ root tests
__device__ inline int vt_inside_at(d3 p, d3 a, d3 b, d3 c) {
    const d3 n = crs(sub(b, a), sub(c, a));
    const double nn = sqn(n);
    if (nn < 1e-40) return HIT_UNCERTAIN;
    const double la = dot(crs(sub(b, p), sub(c, p)), n) / nn;
    const double lb = dot(crs(sub(c, p), sub(a, p)), n) / nn;
    const double lc = dot(crs(sub(a, p), sub(b, p)), n) / nn;
    const double m = mind(mind(la, lb), lc);
    if (m > kInsideMargin) return HIT_CERTAIN;
    if (m > -kInsideMargin) return HIT_UNCERTAIN;
    return HIT_NONE;
}

__device__ inline int ee_inside_at(d3 p1, d3 p2, d3 q1, d3 q2) {
    const d3 d1 = sub(p2, p1), d2 = sub(q2, q1), r = sub(q1, p1);
    const d3 n = crs(d1, d2);
    const double nn = sqn(n);
    const double scale2 = sqn(d1) * sqn(d2);
    if (nn < 1e-24 * scale2) {
        d3 gap = r;
        if (sqn(d1) > 0) gap = sub(gap, scl(dot(r, d1) / sqn(d1), d1));
        return nrm(gap) < 1e-9 ? HIT_UNCERTAIN : HIT_NONE;
    }
    const double s = dot(crs(r, d2), n) / nn;
    const double u = dot(crs(r, d1), n) / nn;
    const double m = mind(mind(mind(s, 1.0 - s), u), 1.0 - u);
    if (m > kInsideMargin) return HIT_CERTAIN;
    if (m > -kInsideMargin) return HIT_UNCERTAIN;
    return HIT_NONE;
}

// ---------------------------------------------- identically coplanar path
__device__ inline bool common_fixed_plane(const d3 s[4], const d3 e[4], d3& origin, d3& bu, d3& bv) {
    const d3 pts[8] = {s[0], s[1], s[2], s[3], e[0], e[1], e[2], e[3]};
    origin = pts[0];
    d3 n = mk(0, 0, 0);
    double scale = 0.0;
    for (int i = 1; i < 8; ++i) scale = maxd(scale, nrm(sub(pts[i], origin)));
    if (scale == 0.0) {
        bu = mk(1, 0, 0), bv = mk(0, 1, 0);
        return true;
    }
    for (int i = 1; i < 8 && sqn(n) < 1e-20 * scale * scale * scale * scale; ++i)
        for (int j = i + 1; j < 8; ++j) {
            const d3 cand = crs(sub(pts[i], origin), sub(pts[j], origin));
            if (sqn(cand) > sqn(n)) n = cand;
        }
    if (sqn(n) < 1e-24 * pow(scale, 4.0)) {
        d3 d = mk(0, 0, 0);
        for (int i = 1; i < 8; ++i)
            if (sqn(sub(pts[i], origin)) > sqn(d)) d = sub(pts[i], origin);
        bu = normalized(d);
        const d3 axis = fabs(bu.x) < 0.9 ? mk(1, 0, 0) : mk(0, 1, 0);
        bv = normalized(crs(bu, axis));
        return true;
    }
    n = normalized(n);
    for (int i = 0; i < 8; ++i)
        if (fabs(dot(sub(pts[i], origin), n)) > 1e-10 * maxd(scale, 1e-3)) return false;
    bu = normalized(crs(fabs(n.x) < 0.9 ? mk(1, 0, 0) : mk(0, 1, 0), n));
    bv = crs(n, bu);
    return true;
}

struct p2 {
    double x, y;
};
struct lin2 {
    p2 p0, d;
};
__device__ __forceinline__ p2 lin_at(const lin2& l, double t) { return p2{l.p0.x + t * l.d.x, l.p0.y + t * l.d.y}; }
__device__ inline void orient_roots(const lin2& a, const lin2& b, const lin2& c, dlist& out) {
    const p2 u0 = {b.p0.x - a.p0.x, b.p0.y - a.p0.y}, du = {b.d.x - a.d.x, b.d.y - a.d.y};
    const p2 v0 = {c.p0.x - a.p0.x, c.p0.y - a.p0.y}, dv = {c.d.x - a.d.x, c.d.y - a.d.y};
    const double A = du.x * dv.y - du.y * dv.x;
    const double B = u0.x * dv.y - u0.y * dv.x + du.x * v0.y - du.y * v0.x;
    const double C = u0.x * v0.y - u0.y * v0.x;
    quadratic_roots01(A, B, C, out);
}
__device__ __forceinline__ double orient_at(const lin2& a, const lin2& b, const lin2& c, double t) {
    const p2 pa = lin_at(a, t), pb = lin_at(b, t), pc = lin_at(c, t);
    return (pb.x - pa.x) * (pc.y - pa.y) - (pb.y - pa.y) * (pc.x - pa.x);
}
__device__ inline int planar_ee_hit(const lin2 m[4]) {
    dlist bps;
    bps.v[0] = 0.0, bps.v[1] = 1.0, bps.n = 2;
    orient_roots(m[0], m[1], m[2], bps);
    orient_roots(m[0], m[1], m[3], bps);
    orient_roots(m[2], m[3], m[0], bps);
    orient_roots(m[2], m[3], m[1], bps);
    dl_sort(bps);
    int best = HIT_NONE;
    for (int i = 0; i + 1 < bps.n; ++i) {
        const double t = 0.5 * (bps.v[i] + bps.v[i + 1]);
        const double o1 = orient_at(m[0], m[1], m[2], t), o2 = orient_at(m[0], m[1], m[3], t);
        const double o3 = orient_at(m[2], m[3], m[0], t), o4 = orient_at(m[2], m[3], m[1], t);
        if (o1 * o2 < 0.0 && o3 * o4 < 0.0) {
            const double mag = mind(mind(fabs(o1), fabs(o2)), mind(fabs(o3), fabs(o4)));
            if (mag > 1e-20) return HIT_CERTAIN;
            best = HIT_UNCERTAIN;
        }
    }
    return best;
}
__device__ inline int planar_vt_hit(const lin2 m[4]) {
    dlist bps;
    bps.v[0] = 0.0, bps.v[1] = 1.0, bps.n = 2;
    orient_roots(m[1], m[2], m[0], bps);
    orient_roots(m[2], m[3], m[0], bps);
    orient_roots(m[3], m[1], m[0], bps);
    dl_sort(bps);
    int best = HIT_NONE;
    for (int i = 0; i + 1 < bps.n; ++i) {
        const double t = 0.5 * (bps.v[i] + bps.v[i + 1]);
        const double o1 = orient_at(m[1], m[2], m[0], t), o2 = orient_at(m[2], m[3], m[0], t);
        const double o3 = orient_at(m[3], m[1], m[0], t);
        const bool inside = (o1 >= 0 && o2 >= 0 && o3 >= 0) || (o1 <= 0 && o2 <= 0 && o3 <= 0);
        if (inside) {
            const double mag = mind(mind(fabs(o1), fabs(o2)), fabs(o3));
            if (mag > 1e-20) return HIT_CERTAIN;
            best = HIT_UNCERTAIN;
        }
    }
    return best;
}

// HIT_* of one stencil: s = start, e = end positions of {p, a, b, c} (VT) or
// {p1, p2, q1, q2} (EE)
__device__ inline int check_stencil(const d3 s[4], const d3 e[4], bool is_vt) {
    const cubic cub = is_vt ? coplanarity_cubic(sub(s[2], s[1]), sub(sub(e[2], e[1]), sub(s[2], s[1])),
                                                sub(s[3], s[1]), sub(sub(e[3], e[1]), sub(s[3], s[1])),
                                                sub(s[0], s[1]), sub(sub(e[0], e[1]), sub(s[0], s[1])))
                            : coplanarity_cubic(sub(s[1], s[0]), sub(sub(e[1], e[0]), sub(s[1], s[0])),
                                                sub(s[3], s[2]), sub(sub(e[3], e[2]), sub(s[3], s[2])),
                                                sub(s[2], s[0]), sub(sub(e[2], e[0]), sub(s[2], s[0])));
    const bool ident = dsign(cub.c0) == 0 && dsign(cub.c1) == 0 && dsign(cub.c2) == 0 && dsign(cub.c3) == 0;
    if (ident) {
        d3 origin, bu, bv;
        int h = HIT_NONE;
        if (common_fixed_plane(s, e, origin, bu, bv)) {
            lin2 m[4];
            for (int i = 0; i < 4; ++i) {
                m[i].p0.x = dot(sub(s[i], origin), bu);
                m[i].p0.y = dot(sub(s[i], origin), bv);
                const d3 d = sub(e[i], s[i]);
                m[i].d.x = dot(d, bu);
                m[i].d.y = dot(d, bv);
            }
            h = is_vt ? planar_vt_hit(m) : planar_ee_hit(m);
        } else {
            for (int k = 0; k <= 32 && h == HIT_NONE; ++k) {
                const double t = k / 32.0;
                d3 p[4];
                for (int i = 0; i < 4; ++i) p[i] = add(s[i], scl(t, sub(e[i], s[i])));
                const int hh = is_vt ? vt_inside_at(p[0], p[1], p[2], p[3]) : ee_inside_at(p[0], p[1], p[2], p[3]);
                if (hh != HIT_NONE) h = HIT_UNCERTAIN;
            }
        }
        return h;
    }
    dlist roots, extrema;
    roots.n = 0, extrema.n = 0;
    cubic_roots01(cub, roots, extrema);
    for (int i = 0; i < extrema.n; ++i) {
        const dd f = eval_cubic(cub, extrema.v[i]);
        if (dsign(f) != 0 && fabs(dval(f)) < 1e-24) dl_push(roots, extrema.v[i]);
    }
    for (int i = 0; i < roots.n; ++i) {
        const double t = roots.v[i];
        d3 p[4];
        for (int k = 0; k < 4; ++k) p[k] = add(s[k], scl(t, sub(e[k], s[k])));
        const int h = is_vt ? vt_inside_at(p[0], p[1], p[2], p[3]) : ee_inside_at(p[0], p[1], p[2], p[3]);
        if (h != HIT_NONE) return h;  // one report per pair
    }
    return HIT_NONE;
}

}  // namespace ccd
}  // namespace tw

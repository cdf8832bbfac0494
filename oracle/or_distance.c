/*
 * ORACLE — test infrastructure only.
 * Restatement of proj/src/distance.cpp (closest-point primitives).
 */
#include <stdlib.h>
#include <string.h>

#include "or_internal.h"

static const double kDegenerateDistance = 1e-9; /* distance.hpp:23 */
static const double kDegenerateTriArea = 1e-12; /* distance.hpp:24 */
static const double kDegenerateEdgeLen = 1e-12; /* distance.hpp:25 */

static void closest_init(or_closest_t* r) {
    /* ClosestResult defaults, distance.hpp:15-21 */
    r->distance = 0.0;
    r->wa[0] = 1.0, r->wa[1] = 0.0, r->wa[2] = 0.0;
    r->wb[0] = 1.0, r->wb[1] = 0.0, r->wb[2] = 0.0;
    r->dir = v3_zero();
    r->degenerate = 0;
}

/* distance.cpp:11-15 */
static v3 safe_unit(v3 v, int* ok) {
    const double n = v3_norm(v);
    *ok = n > 1e-20;
    return *ok ? v3_div(v, n) : v3_zero();
}

/* distance.cpp:18-24 */
static v3 any_perpendicular(v3 d) {
    v3 axis = fabs(d.x) < fabs(d.y) ? v3_make(1, 0, 0) : v3_make(0, 1, 0);
    if (fabs(d.z) < fabs(v3_dot(axis, d))) axis = v3_make(0, 0, 1);
    int ok = 0;
    v3 p = safe_unit(v3_cross(d, axis), &ok);
    return ok ? p : v3_make(1, 0, 0);
}

/* distance.cpp:34-45 */
void or_vv(v3 p, v3 q, or_closest_t* r) {
    closest_init(r);
    const v3 d = v3_sub(p, q);
    r->distance = v3_norm(d);
    if (r->distance >= kDegenerateDistance) {
        r->dir = v3_div(d, r->distance);
    } else {
        r->dir = v3_zero();
        r->degenerate = 1;
    }
}

/* distance.cpp:47-64 */
void or_ve(v3 p, v3 e0, v3 e1, or_closest_t* r) {
    closest_init(r);
    const v3 d = v3_sub(e1, e0);
    const double dd = v3_sqn(d);
    double t = dd > 0.0 ? v3_dot(v3_sub(p, e0), d) / dd : 0.0;
    t = or_clamp(t, 0.0, 1.0);
    const v3 c = v3_add(e0, v3_scale(t, d));
    r->wb[0] = 1.0 - t, r->wb[1] = t, r->wb[2] = 0.0;
    const v3 gap = v3_sub(p, c);
    r->distance = v3_norm(gap);
    if (r->distance >= kDegenerateDistance) {
        r->dir = v3_div(gap, r->distance);
    } else {
        r->dir = any_perpendicular(d);
        r->degenerate = 1;
    }
}

/* distance.cpp:66-151 (Ericson closest point on triangle) */
int or_vt(v3 p, v3 a, v3 b, v3 c, or_closest_t* r) {
    const v3 ab = v3_sub(b, a), ac = v3_sub(c, a);
    const v3 n = v3_cross(ab, ac);
    if (0.5 * v3_norm(n) <= kDegenerateTriArea) return 0;

    const v3 ap = v3_sub(p, a);
    const double d1 = v3_dot(ab, ap), d2 = v3_dot(ac, ap);
    double w[3] = {0.0, 0.0, 0.0};
    v3 closest = v3_zero();
    int done = 0;
    if (d1 <= 0.0 && d2 <= 0.0) {
        closest = a;
        w[0] = 1.0, w[1] = 0.0, w[2] = 0.0;
        done = 1;
    }
    if (!done) {
        const v3 bp = v3_sub(p, b);
        const double d3 = v3_dot(ab, bp), d4 = v3_dot(ac, bp);
        if (d3 >= 0.0 && d4 <= d3) {
            closest = b;
            w[0] = 0.0, w[1] = 1.0, w[2] = 0.0;
            done = 1;
        }
        if (!done) {
            const double vc = d1 * d4 - d3 * d2;
            if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
                const double v = d1 / (d1 - d3);
                closest = v3_add(a, v3_scale(v, ab));
                w[0] = 1.0 - v, w[1] = v, w[2] = 0.0;
                done = 1;
            }
        }
        if (!done) {
            const v3 cp = v3_sub(p, c);
            const double d5 = v3_dot(ab, cp), d6 = v3_dot(ac, cp);
            if (d6 >= 0.0 && d5 <= d6) {
                closest = c;
                w[0] = 0.0, w[1] = 0.0, w[2] = 1.0;
                done = 1;
            }
            if (!done) {
                const double vb = d5 * d2 - d1 * d6;
                if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
                    const double v = d2 / (d2 - d6);
                    closest = v3_add(a, v3_scale(v, ac));
                    w[0] = 1.0 - v, w[1] = 0.0, w[2] = v;
                    done = 1;
                }
                if (!done) {
                    const double va = d3 * d6 - d5 * d4;
                    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
                        const double v = (d4 - d3) / ((d4 - d3) + (d5 - d6));
                        closest = v3_add(b, v3_scale(v, v3_sub(c, b)));
                        w[0] = 0.0, w[1] = 1.0 - v, w[2] = v;
                        done = 1;
                    }
                }
            }
            if (!done) {
                const double vc = d1 * d4 - d3 * d2;
                const double vb = d5 * d2 - d1 * d6;
                const double va = d3 * d6 - d5 * d4;
                const double denom = va + vb + vc;
                const double v = vb / denom;
                const double u = vc / denom;
                closest = v3_add(v3_add(a, v3_scale(v, ab)), v3_scale(u, ac));
                w[0] = 1.0 - v - u, w[1] = v, w[2] = u;
                done = 1;
            }
        }
    }

    closest_init(r);
    r->wb[0] = w[0], r->wb[1] = w[1], r->wb[2] = w[2];
    const v3 gap = v3_sub(p, closest);
    r->distance = v3_norm(gap);
    if (r->distance >= kDegenerateDistance) {
        r->dir = v3_div(gap, r->distance);
    } else {
        r->dir = v3_normalized(n);
        r->degenerate = 1;
    }
    return 1;
}

/* distance.cpp:153-216 */
int or_ee(v3 p1, v3 p2, v3 q1, v3 q2, or_closest_t* r) {
    const v3 d1 = v3_sub(p2, p1), d2 = v3_sub(q2, q1), rr = v3_sub(p1, q1);
    const double a = v3_sqn(d1), e = v3_sqn(d2), f = v3_dot(d2, rr);
    if (sqrt(a) <= kDegenerateEdgeLen || sqrt(e) <= kDegenerateEdgeLen) return 0;

    const double c = v3_dot(d1, rr), b = v3_dot(d1, d2);
    const double denom = a * e - b * b;

    double s, t;
    if (denom > 1e-12 * a * e) {
        s = or_clamp((b * f - c * e) / denom, 0.0, 1.0);
        t = (b * s + f) / e;
        if (t < 0.0) {
            t = 0.0;
            s = or_clamp(-c / a, 0.0, 1.0);
        } else if (t > 1.0) {
            t = 1.0;
            s = or_clamp((b - c) / a, 0.0, 1.0);
        }
    } else {
        /* near-parallel: endpoint enumeration, distance.cpp:174-198 */
        double bs = 0.0, bt = 0.0, bd2 = INFINITY;
        const double cands[2] = {0.0, 1.0};
        for (int k = 0; k < 2; ++k) {
            const double cs = cands[k];
            const v3 ps = v3_add(p1, v3_scale(cs, d1));
            const double ct = or_clamp(v3_dot(v3_sub(ps, q1), d2) / e, 0.0, 1.0);
            const double dist2 = v3_sqn(v3_sub(ps, v3_add(q1, v3_scale(ct, d2))));
            if (dist2 < bd2) bs = cs, bt = ct, bd2 = dist2;
        }
        for (int k = 0; k < 2; ++k) {
            const double ct = cands[k];
            const v3 qt = v3_add(q1, v3_scale(ct, d2));
            const double cs = or_clamp(v3_dot(v3_sub(qt, p1), d1) / a, 0.0, 1.0);
            const double dist2 = v3_sqn(v3_sub(v3_add(p1, v3_scale(cs, d1)), qt));
            if (dist2 < bd2) bs = cs, bt = ct, bd2 = dist2;
        }
        s = bs;
        t = bt;
    }

    closest_init(r);
    r->wa[0] = 1.0 - s, r->wa[1] = s, r->wa[2] = 0.0;
    r->wb[0] = 1.0 - t, r->wb[1] = t, r->wb[2] = 0.0;
    const v3 ca = v3_add(p1, v3_scale(s, d1)), cb = v3_add(q1, v3_scale(t, d2));
    const v3 gap = v3_sub(ca, cb);
    r->distance = v3_norm(gap);
    if (r->distance >= kDegenerateDistance) {
        r->dir = v3_div(gap, r->distance);
    } else {
        int ok = 0;
        r->dir = safe_unit(v3_cross(d1, d2), &ok);
        if (!ok) r->dir = any_perpendicular(d1);
        r->degenerate = 1;
    }
    return 1;
}

/* Simplex::shares_vertex, mesh.hpp:22-27 */
int or_shares_vertex(const or_simplex* a, const or_simplex* b) {
    for (int i = 0; i < or_simplex_size(a); ++i)
        for (int j = 0; j < or_simplex_size(b); ++j)
            if (a->idx[i] == b->idx[j]) return 1;
    return 0;
}

static void flip(or_closest_t* r) {
    double t[3];
    memcpy(t, r->wa, sizeof t);
    memcpy(r->wa, r->wb, sizeof t);
    memcpy(r->wb, t, sizeof t);
    r->dir = v3_neg(r->dir);
}

/* distance.cpp:218-253 */
int or_pair_closest(const or_simplex* sa, const or_simplex* sb, const double* x,
                    or_closest_t* r) {
    if (or_shares_vertex(sa, sb)) return -1;
#define P(i) v3_load(x + 3 * (size_t)(i))
    const int ka = sa->kind, kb = sb->kind;
    if (ka == OR_KIND_V && kb == OR_KIND_V) {
        or_vv(P(sa->idx[0]), P(sb->idx[0]), r);
        return 1;
    }
    if (ka == OR_KIND_V && kb == OR_KIND_E) {
        or_ve(P(sa->idx[0]), P(sb->idx[0]), P(sb->idx[1]), r);
        return 1;
    }
    if (ka == OR_KIND_E && kb == OR_KIND_V) {
        const int h = or_pair_closest(sb, sa, x, r);
        if (h == 1) flip(r);
        return h;
    }
    if (ka == OR_KIND_V && kb == OR_KIND_T)
        return or_vt(P(sa->idx[0]), P(sb->idx[0]), P(sb->idx[1]), P(sb->idx[2]), r);
    if (ka == OR_KIND_T && kb == OR_KIND_V) {
        const int h = or_pair_closest(sb, sa, x, r);
        if (h == 1) flip(r);
        return h;
    }
    if (ka == OR_KIND_E && kb == OR_KIND_E) {
        /* canonical operand order by the vertex-id tuple (distance.cpp:243-251) */
        const int swap = (sb->idx[0] < sa->idx[0]) ||
                         (sb->idx[0] == sa->idx[0] && sb->idx[1] < sa->idx[1]);
        const or_simplex* ea = swap ? sb : sa;
        const or_simplex* eb = swap ? sa : sb;
        const int h = or_ee(P(ea->idx[0]), P(ea->idx[1]), P(eb->idx[0]), P(eb->idx[1]), r);
        if (h == 1 && swap) flip(r);
        return h;
    }
#undef P
    return -1;
}

int or_closest(int ka, const int* va, int kb, const int* vb, const double* x, double* out) {
    or_simplex a = {ka, {va[0], ka >= 1 ? va[1] : -1, ka >= 2 ? va[2] : -1}};
    or_simplex b = {kb, {vb[0], kb >= 1 ? vb[1] : -1, kb >= 2 ? vb[2] : -1}};
    or_closest_t r;
    const int h = or_pair_closest(&a, &b, x, &r);
    if (h != 1) return h;
    out[0] = r.distance;
    for (int i = 0; i < 3; ++i) out[1 + i] = r.wa[i], out[4 + i] = r.wb[i];
    out[7] = r.dir.x, out[8] = r.dir.y, out[9] = r.dir.z;
    out[10] = r.degenerate;
    return 1;
}

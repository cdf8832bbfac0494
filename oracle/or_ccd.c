/*
 * ORACLE — test infrastructure only.
 * Restatement of proj/src/testkit/ccd.cpp + proj/include/twoway/testkit/dd.hpp:
 * the trusted continuous-collision certifier used to prove the
 * intersection-free guarantee of a resolve path (swept-AABB binning,
 * double-double coplanarity cubic, bisection roots, inside tests, planar
 * fallback for identically coplanar stencils). Never on the product path.
 */
#include <stdlib.h>
#include <string.h>

#include "or_internal.h"

/* ------------------------------------------------------------ dd.hpp */
typedef struct {
    double hi, lo;
} dd;
static inline dd dd_make(double h, double l) {
    dd r = {h, l};
    return r;
}
static inline double dd_value(dd a) { return a.hi + a.lo; }
static inline int dd_sign(dd a) {
    if (a.hi > 0.0 || (a.hi == 0.0 && a.lo > 0.0)) return 1;
    if (a.hi < 0.0 || (a.hi == 0.0 && a.lo < 0.0)) return -1;
    return 0;
}
static inline dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return dd_make(s, (a - (s - bb)) + (b - bb));
}
static inline dd two_prod(double a, double b) {
    const double p = a * b;
    return dd_make(p, fma(a, b, -p));
}
static inline dd quick_two_sum(double a, double b) {
    const double s = a + b;
    return dd_make(s, b - (s - a));
}
static inline dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    s.lo += a.lo + b.lo;
    return quick_two_sum(s.hi, s.lo);
}
static inline dd dd_sub(dd a, dd b) { return dd_add(a, dd_make(-b.hi, -b.lo)); }
static inline dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return quick_two_sum(p.hi, p.lo);
}
typedef struct {
    dd x, y, z;
} dd3;
static inline dd3 dd3_cross(dd3 a, dd3 b) {
    dd3 r = {dd_sub(dd_mul(a.y, b.z), dd_mul(a.z, b.y)), dd_sub(dd_mul(a.z, b.x), dd_mul(a.x, b.z)),
             dd_sub(dd_mul(a.x, b.y), dd_mul(a.y, b.x))};
    return r;
}
static inline dd dd3_dot(dd3 a, dd3 b) {
    return dd_add(dd_add(dd_mul(a.x, b.x), dd_mul(a.y, b.y)), dd_mul(a.z, b.z));
}
static inline dd3 dd3_point(v3 v) {
    dd3 r = {dd_make(v.x, 0.0), dd_make(v.y, 0.0), dd_make(v.z, 0.0)};
    return r;
}

/* ------------------------------------------------------ boxes + bins */
typedef struct {
    v3 lo, hi;
} box;

static int overlap(const box* a, const box* b) {
    return a->lo.x <= b->hi.x && a->lo.y <= b->hi.y && a->lo.z <= b->hi.z && b->lo.x <= a->hi.x &&
           b->lo.y <= a->hi.y && b->lo.z <= a->hi.z;
}

static box swept_box(const int* ids, int n, const double* x0, const double* x1, double inflate) {
    box b;
    b.lo = b.hi = v3_load(x0 + 3 * (size_t)ids[0]);
    for (int i = 0; i < n; ++i) {
        const v3 p = v3_load(x0 + 3 * (size_t)ids[i]), q = v3_load(x1 + 3 * (size_t)ids[i]);
        b.lo = v3_make(or_min(or_min(b.lo.x, p.x), q.x), or_min(or_min(b.lo.y, p.y), q.y),
                       or_min(or_min(b.lo.z, p.z), q.z));
        b.hi = v3_make(or_max(or_max(b.hi.x, p.x), q.x), or_max(or_max(b.hi.y, p.y), q.y),
                       or_max(or_max(b.hi.z, p.z), q.z));
    }
    b.lo = v3_make(b.lo.x - inflate, b.lo.y - inflate, b.lo.z - inflate);
    b.hi = v3_make(b.hi.x + inflate, b.hi.y + inflate, b.hi.z + inflate);
    return b;
}

static uint64_t cell_hash(int64_t x, int64_t y, int64_t z) {
    uint64_t h = (uint64_t)x * 0x8DA6B343ull;
    h ^= (uint64_t)y * 0xD8163841ull + (h << 17);
    h ^= (uint64_t)z * 0xCB1AB31Full + (h >> 13);
    return h * 0x2545F4914F6CDD1Dull;
}

typedef struct {
    uint64_t h;
    int id;
} binrec;
static int cmp_binrec(const void* a, const void* b) {
    const binrec* x = (const binrec*)a;
    const binrec* y = (const binrec*)b;
    if (x->h != y->h) return x->h < y->h ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id);
}
static int cmp_dbl(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y);
}

typedef struct {
    double cell;
    binrec* recs;
    int64_t nrec, cap;
    int* global;
    int nglobal;
} bins;

static void bins_build(bins* B, const box* boxes, int n, double cell) {
    B->cell = cell;
    B->recs = NULL;
    B->nrec = B->cap = 0;
    B->global = (int*)or_xmalloc(((size_t)n + 1) * sizeof(int));
    B->nglobal = 0;
    for (int i = 0; i < n; ++i) {
        const box* b = &boxes[i];
        const int64_t x0 = (int64_t)floor(b->lo.x / cell), y0 = (int64_t)floor(b->lo.y / cell),
                      z0 = (int64_t)floor(b->lo.z / cell);
        const int64_t x1 = (int64_t)floor(b->hi.x / cell), y1 = (int64_t)floor(b->hi.y / cell),
                      z1 = (int64_t)floor(b->hi.z / cell);
        const int64_t span = (x1 - x0 + 1) * (y1 - y0 + 1) * (z1 - z0 + 1);
        if (span > 4096) {
            B->global[B->nglobal++] = i;
            continue;
        }
        for (int64_t x = x0; x <= x1; ++x)
            for (int64_t y = y0; y <= y1; ++y)
                for (int64_t z = z0; z <= z1; ++z) {
                    if (B->nrec == B->cap) {
                        B->cap = B->cap ? B->cap * 2 : 1024;
                        B->recs = (binrec*)or_xrealloc(B->recs, (size_t)B->cap * sizeof(binrec));
                    }
                    B->recs[B->nrec].h = cell_hash(x, y, z);
                    B->recs[B->nrec].id = i;
                    ++B->nrec;
                }
    }
    qsort(B->recs, (size_t)B->nrec, sizeof(binrec), cmp_binrec);
}
static void bins_free(bins* B) {
    free(B->recs);
    free(B->global);
}
/* first record with hash h, or -1 */
static int64_t bins_find(const bins* B, uint64_t h) {
    int64_t lo = 0, hi = B->nrec;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (B->recs[mid].h < h) lo = mid + 1;
        else hi = mid;
    }
    return (lo < B->nrec && B->recs[lo].h == h) ? lo : -1;
}

static double max_coeff(v3 v) { return or_max(or_max(v.x, v.y), v.z); }

static double pick_cell_size(const box* a, int na, const box* b, int nb) {
    const int n = na + nb;
    if (n == 0) return 1.0;
    double* ext = (double*)or_xmalloc((size_t)n * sizeof(double));
    for (int i = 0; i < na; ++i) ext[i] = max_coeff(v3_sub(a[i].hi, a[i].lo));
    for (int i = 0; i < nb; ++i) ext[na + i] = max_coeff(v3_sub(b[i].hi, b[i].lo));
    qsort(ext, (size_t)n, sizeof(double), cmp_dbl);
    const size_t at = (size_t)n * 9 / 10;
    const double r = or_max(2.0 * ext[at], 1e-6);
    free(ext);
    return r;
}

/* ------------------------------------------------ coplanarity cubic */
typedef struct {
    dd c0, c1, c2, c3;
} cubic;

static cubic coplanarity_cubic(v3 u0, v3 du, v3 v0, v3 dv, v3 w0, v3 dw) {
    const dd3 U0 = dd3_point(u0), DU = dd3_point(du);
    const dd3 V0 = dd3_point(v0), DV = dd3_point(dv);
    const dd3 W0 = dd3_point(w0), DW = dd3_point(dw);
    const dd3 A = dd3_cross(U0, V0);
    dd3 B = dd3_cross(U0, DV);
    const dd3 B2 = dd3_cross(DU, V0);
    B.x = dd_add(B.x, B2.x);
    B.y = dd_add(B.y, B2.y);
    B.z = dd_add(B.z, B2.z);
    const dd3 C = dd3_cross(DU, DV);
    cubic c;
    c.c0 = dd3_dot(A, W0);
    c.c1 = dd_add(dd3_dot(A, DW), dd3_dot(B, W0));
    c.c2 = dd_add(dd3_dot(B, DW), dd3_dot(C, W0));
    c.c3 = dd3_dot(C, DW);
    return c;
}

static dd eval_cubic(const cubic* c, double t) {
    const dd T = dd_make(t, 0.0);
    return dd_add(dd_mul(dd_add(dd_mul(dd_add(dd_mul(c->c3, T), c->c2), T), c->c1), T), c->c0);
}

typedef struct {
    double v[16];
    int n;
} dlist;
static void dl_push(dlist* l, double x) {
    if (l->n < 16) l->v[l->n++] = x;
}

static void quadratic_roots01(double a, double b, double c, dlist* out) {
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

static void sort_dl(dlist* l) { qsort(l->v, (size_t)l->n, sizeof(double), cmp_dbl); }

static void cubic_roots01(const cubic* c, dlist* roots, dlist* extrema) {
    dlist bps = {{0}, 0};
    quadratic_roots01(3.0 * dd_value(c->c3), 2.0 * dd_value(c->c2), dd_value(c->c1), &bps);
    *extrema = bps;
    dl_push(&bps, 0.0);
    dl_push(&bps, 1.0);
    sort_dl(&bps);
    for (int i = 0; i + 1 < bps.n; ++i) {
        double a = bps.v[i], b = bps.v[i + 1];
        const int sa = dd_sign(eval_cubic(c, a)), sb = dd_sign(eval_cubic(c, b));
        if (sa == 0) {
            dl_push(roots, a);
            continue;
        }
        if (sb == 0 || sa * sb > 0) continue;
        for (int it = 0; it < 100; ++it) {
            const double mm = 0.5 * (a + b);
            const int sm = dd_sign(eval_cubic(c, mm));
            if (sm == 0) {
                a = b = mm;
                break;
            }
            if (sm == sa) a = mm;
            else b = mm;
        }
        dl_push(roots, 0.5 * (a + b));
    }
    if (dd_sign(eval_cubic(c, 1.0)) == 0) dl_push(roots, 1.0);
    sort_dl(roots);
    int w = 0;
    for (int i = 0; i < roots->n; ++i)
        if (w == 0 || !(fabs(roots->v[w - 1] - roots->v[i]) < 1e-12)) roots->v[w++] = roots->v[i];
    roots->n = w;
}

/* -------------------------------------------------------- root tests */
enum { HIT_NONE = 0, HIT_UNCERTAIN = 1, HIT_CERTAIN = 2 };
static const double kInsideMargin = 1e-8;

static int vt_inside_at(v3 p, v3 a, v3 b, v3 c) {
    const v3 n = v3_cross(v3_sub(b, a), v3_sub(c, a));
    const double nn = v3_sqn(n);
    if (nn < 1e-40) return HIT_UNCERTAIN;
    const double la = v3_dot(v3_cross(v3_sub(b, p), v3_sub(c, p)), n) / nn;
    const double lb = v3_dot(v3_cross(v3_sub(c, p), v3_sub(a, p)), n) / nn;
    const double lc = v3_dot(v3_cross(v3_sub(a, p), v3_sub(b, p)), n) / nn;
    const double m = or_min(or_min(la, lb), lc);
    if (m > kInsideMargin) return HIT_CERTAIN;
    if (m > -kInsideMargin) return HIT_UNCERTAIN;
    return HIT_NONE;
}

static int ee_inside_at(v3 p1, v3 p2, v3 q1, v3 q2) {
    const v3 d1 = v3_sub(p2, p1), d2 = v3_sub(q2, q1), r = v3_sub(q1, p1);
    const v3 n = v3_cross(d1, d2);
    const double nn = v3_sqn(n);
    const double scale2 = v3_sqn(d1) * v3_sqn(d2);
    if (nn < 1e-24 * scale2) {
        v3 gap = r;
        if (v3_sqn(d1) > 0) gap = v3_sub(gap, v3_scale(v3_dot(r, d1) / v3_sqn(d1), d1));
        return v3_norm(gap) < 1e-9 ? HIT_UNCERTAIN : HIT_NONE;
    }
    const double s = v3_dot(v3_cross(r, d2), n) / nn;
    const double u = v3_dot(v3_cross(r, d1), n) / nn;
    const double m = or_min(or_min(or_min(s, 1.0 - s), u), 1.0 - u);
    if (m > kInsideMargin) return HIT_CERTAIN;
    if (m > -kInsideMargin) return HIT_UNCERTAIN;
    return HIT_NONE;
}

/* -------------------------------------------- identically coplanar path */
static int common_fixed_plane(const v3 s[4], const v3 e[4], v3* origin, v3* bu, v3* bv) {
    v3 pts[8] = {s[0], s[1], s[2], s[3], e[0], e[1], e[2], e[3]};
    *origin = pts[0];
    v3 n = v3_zero();
    double scale = 0.0;
    for (int i = 1; i < 8; ++i) scale = or_max(scale, v3_norm(v3_sub(pts[i], *origin)));
    if (scale == 0.0) {
        *bu = v3_make(1, 0, 0);
        *bv = v3_make(0, 1, 0);
        return 1;
    }
    for (int i = 1; i < 8 && v3_sqn(n) < 1e-20 * scale * scale * scale * scale; ++i)
        for (int j = i + 1; j < 8; ++j) {
            const v3 cand = v3_cross(v3_sub(pts[i], *origin), v3_sub(pts[j], *origin));
            if (v3_sqn(cand) > v3_sqn(n)) n = cand;
        }
    if (v3_sqn(n) < 1e-24 * pow(scale, 4)) {
        v3 d = v3_zero();
        for (int i = 1; i < 8; ++i)
            if (v3_sqn(v3_sub(pts[i], *origin)) > v3_sqn(d)) d = v3_sub(pts[i], *origin);
        *bu = v3_normalized(d);
        const v3 axis = fabs(bu->x) < 0.9 ? v3_make(1, 0, 0) : v3_make(0, 1, 0);
        *bv = v3_normalized(v3_cross(*bu, axis));
        return 1;
    }
    n = v3_normalized(n);
    for (int i = 0; i < 8; ++i)
        if (fabs(v3_dot(v3_sub(pts[i], *origin), n)) > 1e-10 * or_max(scale, 1e-3)) return 0;
    *bu = v3_normalized(v3_cross(fabs(n.x) < 0.9 ? v3_make(1, 0, 0) : v3_make(0, 1, 0), n));
    *bv = v3_cross(n, *bu);
    return 1;
}

typedef struct {
    double x, y;
} p2;
typedef struct {
    p2 p0, d;
} lin2;
static p2 lin_at(const lin2* l, double t) {
    p2 r = {l->p0.x + t * l->d.x, l->p0.y + t * l->d.y};
    return r;
}
static void orient_roots(const lin2* a, const lin2* b, const lin2* c, dlist* out) {
    const p2 u0 = {b->p0.x - a->p0.x, b->p0.y - a->p0.y}, du = {b->d.x - a->d.x, b->d.y - a->d.y};
    const p2 v0 = {c->p0.x - a->p0.x, c->p0.y - a->p0.y}, dv = {c->d.x - a->d.x, c->d.y - a->d.y};
    const double A = du.x * dv.y - du.y * dv.x;
    const double B = u0.x * dv.y - u0.y * dv.x + du.x * v0.y - du.y * v0.x;
    const double C = u0.x * v0.y - u0.y * v0.x;
    quadratic_roots01(A, B, C, out);
}
static double orient_at(const lin2* a, const lin2* b, const lin2* c, double t) {
    const p2 pa = lin_at(a, t), pb = lin_at(b, t), pc = lin_at(c, t);
    return (pb.x - pa.x) * (pc.y - pa.y) - (pb.y - pa.y) * (pc.x - pa.x);
}
static int planar_ee_hit(const lin2 m[4], double* t_hit) {
    dlist bps = {{0.0, 1.0}, 2};
    orient_roots(&m[0], &m[1], &m[2], &bps);
    orient_roots(&m[0], &m[1], &m[3], &bps);
    orient_roots(&m[2], &m[3], &m[0], &bps);
    orient_roots(&m[2], &m[3], &m[1], &bps);
    sort_dl(&bps);
    int best = HIT_NONE;
    for (int i = 0; i + 1 < bps.n; ++i) {
        const double t = 0.5 * (bps.v[i] + bps.v[i + 1]);
        const double o1 = orient_at(&m[0], &m[1], &m[2], t);
        const double o2 = orient_at(&m[0], &m[1], &m[3], t);
        const double o3 = orient_at(&m[2], &m[3], &m[0], t);
        const double o4 = orient_at(&m[2], &m[3], &m[1], t);
        if (o1 * o2 < 0.0 && o3 * o4 < 0.0) {
            const double mag = or_min(or_min(fabs(o1), fabs(o2)), or_min(fabs(o3), fabs(o4)));
            *t_hit = t;
            if (mag > 1e-20) return HIT_CERTAIN;
            best = HIT_UNCERTAIN;
        }
    }
    return best;
}
static int planar_vt_hit(const lin2 m[4], double* t_hit) {
    dlist bps = {{0.0, 1.0}, 2};
    orient_roots(&m[1], &m[2], &m[0], &bps);
    orient_roots(&m[2], &m[3], &m[0], &bps);
    orient_roots(&m[3], &m[1], &m[0], &bps);
    sort_dl(&bps);
    int best = HIT_NONE;
    for (int i = 0; i + 1 < bps.n; ++i) {
        const double t = 0.5 * (bps.v[i] + bps.v[i + 1]);
        const double o1 = orient_at(&m[1], &m[2], &m[0], t);
        const double o2 = orient_at(&m[2], &m[3], &m[0], t);
        const double o3 = orient_at(&m[3], &m[1], &m[0], t);
        const int inside = (o1 >= 0 && o2 >= 0 && o3 >= 0) || (o1 <= 0 && o2 <= 0 && o3 <= 0);
        if (inside) {
            const double mag = or_min(or_min(fabs(o1), fabs(o2)), fabs(o3));
            *t_hit = t;
            if (mag > 1e-20) return HIT_CERTAIN;
            best = HIT_UNCERTAIN;
        }
    }
    return best;
}

/* returns HIT_* for one stencil (ids = {p,a,b,c} for VT, {p1,p2,q1,q2} for EE) */
static int check_stencil(const int ids[4], int is_vt, const double* x0, const double* x1) {
    v3 s[4], e[4];
    for (int i = 0; i < 4; ++i) s[i] = v3_load(x0 + 3 * (size_t)ids[i]), e[i] = v3_load(x1 + 3 * (size_t)ids[i]);
    cubic cub;
    if (is_vt) {
        cub = coplanarity_cubic(v3_sub(s[2], s[1]), v3_sub(v3_sub(e[2], e[1]), v3_sub(s[2], s[1])),
                                v3_sub(s[3], s[1]), v3_sub(v3_sub(e[3], e[1]), v3_sub(s[3], s[1])),
                                v3_sub(s[0], s[1]), v3_sub(v3_sub(e[0], e[1]), v3_sub(s[0], s[1])));
    } else {
        cub = coplanarity_cubic(v3_sub(s[1], s[0]), v3_sub(v3_sub(e[1], e[0]), v3_sub(s[1], s[0])),
                                v3_sub(s[3], s[2]), v3_sub(v3_sub(e[3], e[2]), v3_sub(s[3], s[2])),
                                v3_sub(s[2], s[0]), v3_sub(v3_sub(e[2], e[0]), v3_sub(s[2], s[0])));
    }
    const int ident = dd_sign(cub.c0) == 0 && dd_sign(cub.c1) == 0 && dd_sign(cub.c2) == 0 &&
                      dd_sign(cub.c3) == 0;
    if (ident) {
        v3 origin, bu, bv;
        double t_hit = 0.0;
        int h = HIT_NONE;
        if (common_fixed_plane(s, e, &origin, &bu, &bv)) {
            lin2 m[4];
            for (int i = 0; i < 4; ++i) {
                m[i].p0.x = v3_dot(v3_sub(s[i], origin), bu);
                m[i].p0.y = v3_dot(v3_sub(s[i], origin), bv);
                const v3 d = v3_sub(e[i], s[i]);
                m[i].d.x = v3_dot(d, bu);
                m[i].d.y = v3_dot(d, bv);
            }
            h = is_vt ? planar_vt_hit(m, &t_hit) : planar_ee_hit(m, &t_hit);
        } else {
            for (int k = 0; k <= 32 && h == HIT_NONE; ++k) {
                const double t = k / 32.0;
                v3 p[4];
                for (int i = 0; i < 4; ++i) p[i] = v3_add(s[i], v3_scale(t, v3_sub(e[i], s[i])));
                const int hh = is_vt ? vt_inside_at(p[0], p[1], p[2], p[3])
                                     : ee_inside_at(p[0], p[1], p[2], p[3]);
                if (hh != HIT_NONE) h = HIT_UNCERTAIN;
            }
        }
        return h;
    }
    dlist roots = {{0}, 0}, extrema = {{0}, 0};
    cubic_roots01(&cub, &roots, &extrema);
    for (int i = 0; i < extrema.n; ++i) {
        const dd f = eval_cubic(&cub, extrema.v[i]);
        if (dd_sign(f) != 0 && fabs(dd_value(f)) < 1e-24) dl_push(&roots, extrema.v[i]);
    }
    for (int i = 0; i < roots.n; ++i) {
        const double t = roots.v[i];
        v3 p[4];
        for (int k = 0; k < 4; ++k) {
            const v3 a = v3_load(x0 + 3 * (size_t)ids[k]), b = v3_load(x1 + 3 * (size_t)ids[k]);
            p[k] = v3_add(a, v3_scale(t, v3_sub(b, a)));
        }
        const int h = is_vt ? vt_inside_at(p[0], p[1], p[2], p[3]) : ee_inside_at(p[0], p[1], p[2], p[3]);
        if (h != HIT_NONE) return h; /* one report per pair */
    }
    return HIT_NONE;
}

/* -------------------------------------------------------- dedup set */
typedef struct {
    uint64_t* k;
    uint64_t mask;
    int64_t n;
} kset;
static void kset_init(kset* s) {
    s->mask = 4095;
    s->k = (uint64_t*)or_xcalloc(s->mask + 1, sizeof(uint64_t));
    s->n = 0;
}
static int kset_insert(kset* s, uint64_t key) { /* key+1 stored */
    if ((uint64_t)(s->n + 1) * 2 > s->mask + 1) {
        kset n;
        n.mask = s->mask * 2 + 1;
        n.k = (uint64_t*)or_xcalloc(n.mask + 1, sizeof(uint64_t));
        n.n = 0;
        for (uint64_t i = 0; i <= s->mask; ++i)
            if (s->k[i]) {
                uint64_t h = or_mix64(s->k[i]) & n.mask;
                while (n.k[h]) h = (h + 1) & n.mask;
                n.k[h] = s->k[i];
                ++n.n;
            }
        free(s->k);
        *s = n;
    }
    const uint64_t kk = key + 1;
    uint64_t h = or_mix64(kk) & s->mask;
    while (s->k[h]) {
        if (s->k[h] == kk) return 0;
        h = (h + 1) & s->mask;
    }
    s->k[h] = kk;
    ++s->n;
    return 1;
}

/* ccd_certify, ccd.cpp:339-498 */
int or_ccd_certify(int nv, int ne, const int* edges, int nt, const int* tris, const double* x0,
                   const double* x1, int* certain_out) {
    int violations = 0, certain = 0;
    box* vboxes = (box*)or_xmalloc(((size_t)nv + 1) * sizeof(box));
    box* eboxes = (box*)or_xmalloc(((size_t)ne + 1) * sizeof(box));
    box* tboxes = (box*)or_xmalloc(((size_t)nt + 1) * sizeof(box));
    for (int v = 0; v < nv; ++v) vboxes[v] = swept_box(&v, 1, x0, x1, 1e-12);
    for (int e = 0; e < ne; ++e) eboxes[e] = swept_box(edges + 2 * e, 2, x0, x1, 1e-12);
    for (int t = 0; t < nt; ++t) tboxes[t] = swept_box(tris + 3 * t, 3, x0, x1, 1e-12);

#define REPORT(h)                          \
    do {                                   \
        if ((h) != HIT_NONE) {             \
            ++violations;                  \
            certain += (h) == HIT_CERTAIN; \
        }                                  \
    } while (0)

    /* vertex-triangle candidates */
    {
        bins tb;
        bins_build(&tb, tboxes, nt, pick_cell_size(vboxes, nv, tboxes, nt));
        kset seen;
        kset_init(&seen);
        for (int v = 0; v < nv; ++v) {
            const box* b = &vboxes[v];
#define TRY_VT(t)                                                                           \
    do {                                                                                    \
        const int* tri = tris + 3 * (t);                                                    \
        if (v == tri[0] || v == tri[1] || v == tri[2]) break;                               \
        if (!overlap(b, &tboxes[t])) break;                                                 \
        if (!kset_insert(&seen, ((uint64_t)(uint32_t)v << 32) | (uint64_t)(uint32_t)(t))) break; \
        const int ids[4] = {v, tri[0], tri[1], tri[2]};                                     \
        REPORT(check_stencil(ids, 1, x0, x1));                                              \
    } while (0)
            const int64_t cx0 = (int64_t)floor(b->lo.x / tb.cell), cy0 = (int64_t)floor(b->lo.y / tb.cell),
                          cz0 = (int64_t)floor(b->lo.z / tb.cell);
            const int64_t cx1 = (int64_t)floor(b->hi.x / tb.cell), cy1 = (int64_t)floor(b->hi.y / tb.cell),
                          cz1 = (int64_t)floor(b->hi.z / tb.cell);
            const int64_t span = (cx1 - cx0 + 1) * (cy1 - cy0 + 1) * (cz1 - cz0 + 1);
            if (span > 4096) {
                for (int t = 0; t < nt; ++t) TRY_VT(t);
                continue;
            }
            for (int64_t x = cx0; x <= cx1; ++x)
                for (int64_t y = cy0; y <= cy1; ++y)
                    for (int64_t z = cz0; z <= cz1; ++z) {
                        const uint64_t h = cell_hash(x, y, z);
                        int64_t at = bins_find(&tb, h);
                        if (at < 0) continue;
                        for (; at < tb.nrec && tb.recs[at].h == h; ++at) TRY_VT(tb.recs[at].id);
                    }
            for (int g = 0; g < tb.nglobal; ++g) TRY_VT(tb.global[g]);
#undef TRY_VT
        }
        free(seen.k);
        bins_free(&tb);
    }

    /* edge-edge candidates */
    {
        bins eb;
        bins_build(&eb, eboxes, ne, pick_cell_size(eboxes, ne, eboxes, ne));
        kset seen;
        kset_init(&seen);
#define TRY_EE(E1, E2)                                                                             \
    do {                                                                                           \
        int e1 = (E1), e2 = (E2);                                                                  \
        if (e1 >= e2) {                                                                            \
            const int tmp = e1;                                                                    \
            e1 = e2;                                                                               \
            e2 = tmp;                                                                              \
        }                                                                                          \
        if (e1 == e2) break;                                                                       \
        const int *a = edges + 2 * e1, *bb = edges + 2 * e2;                                       \
        if (a[0] == bb[0] || a[0] == bb[1] || a[1] == bb[0] || a[1] == bb[1]) break;               \
        if (!overlap(&eboxes[e1], &eboxes[e2])) break;                                             \
        if (!kset_insert(&seen, ((uint64_t)(uint32_t)e1 << 32) | (uint64_t)(uint32_t)e2)) break;   \
        const int ids[4] = {a[0], a[1], bb[0], bb[1]};                                             \
        REPORT(check_stencil(ids, 0, x0, x1));                                                     \
    } while (0)
        for (int64_t i0 = 0; i0 < eb.nrec;) {
            int64_t i1 = i0 + 1;
            while (i1 < eb.nrec && eb.recs[i1].h == eb.recs[i0].h) ++i1;
            for (int64_t i = i0; i < i1; ++i)
                for (int64_t j = i + 1; j < i1; ++j) TRY_EE(eb.recs[i].id, eb.recs[j].id);
            i0 = i1;
        }
        uint8_t* is_global = (uint8_t*)or_xcalloc((size_t)ne + 1, 1);
        for (int g = 0; g < eb.nglobal; ++g) is_global[eb.global[g]] = 1;
        for (int g = 0; g < eb.nglobal; ++g) {
            for (int g2 = g + 1; g2 < eb.nglobal; ++g2) TRY_EE(eb.global[g], eb.global[g2]);
            for (int e = 0; e < ne; ++e)
                if (!is_global[e]) TRY_EE(eb.global[g], e);
        }
#undef TRY_EE
        free(is_global);
        free(seen.k);
        bins_free(&eb);
    }
#undef REPORT
    free(vboxes);
    free(eboxes);
    free(tboxes);
    if (certain_out) *certain_out = certain;
    return violations;
}

/*
 * ORACLE — test infrastructure only.
 * Restatement of proj/src/mesh.cpp:10-33 (edge order) and proj/src/proximity.cpp
 * (hash-grid broad phase + exact narrow-phase filter, refresh, bound update,
 * per-vertex bound).
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "or_internal.h"

void* or_xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) {
        fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n);
        abort();
    }
    return p;
}
void* or_xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz ? sz : 1);
    if (!p) {
        fprintf(stderr, "oracle: out of memory\n");
        abort();
    }
    return p;
}
void* or_xrealloc(void* p, size_t n) {
    void* q = realloc(p, n ? n : 1);
    if (!q) {
        fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n);
        abort();
    }
    return q;
}

/* ------------------------------------------------------------------ mesh */

/* MeshState::finalize edge derivation, mesh.cpp:15-26: explicit edges keep
 * their stored orientation; new strand edges are appended as given; triangle
 * edges are appended as (min, max) in (t, k) order; dedup on the unordered
 * pair. */
typedef struct {
    uint64_t* keys;
    uint64_t mask;
    int64_t count;
} u64set;

static void u64set_init(u64set* s, int64_t expect) {
    uint64_t cap = 16;
    while (cap < (uint64_t)(expect * 2 + 16)) cap <<= 1;
    s->keys = (uint64_t*)or_xcalloc(cap, sizeof(uint64_t));
    s->mask = cap - 1;
    s->count = 0;
}
static void u64set_free(u64set* s) { free(s->keys); }
static inline uint64_t u64_hash(uint64_t k) { return or_mix64(k); }
static int u64set_insert(u64set* s, uint64_t key); /* key != 0; returns 1 if new */
static void u64set_grow(u64set* s) {
    u64set n;
    n.mask = s->mask * 2 + 1;
    n.keys = (uint64_t*)or_xcalloc(n.mask + 1, sizeof(uint64_t));
    n.count = 0;
    for (uint64_t i = 0; i <= s->mask; ++i)
        if (s->keys[i]) u64set_insert(&n, s->keys[i]);
    free(s->keys);
    *s = n;
}
static int u64set_insert(u64set* s, uint64_t key) {
    if ((uint64_t)(s->count + 1) * 2 > s->mask + 1) u64set_grow(s);
    uint64_t h = u64_hash(key) & s->mask;
    for (;;) {
        const uint64_t k = s->keys[h];
        if (k == 0) {
            s->keys[h] = key;
            ++s->count;
            return 1;
        }
        if (k == key) return 0;
        h = (h + 1) & s->mask;
    }
}

int or_finalize_edges(int nv, int ne_explicit, const int* explicit_edges, int ns,
                      const int* strand_edges, int nt, const int* tris, int* out_edges) {
    (void)nv;
    u64set seen;
    u64set_init(&seen, (int64_t)ne_explicit + ns + 3 * (int64_t)nt);
#define UKEY(a, b)                                                                          \
    ((((uint64_t)(uint32_t)((a) < (b) ? (a) : (b))) << 32) | (uint64_t)(uint32_t)((a) < (b) ? (b) : (a))) + 1ull
    int n = 0;
    for (int i = 0; i < ne_explicit; ++i) {
        u64set_insert(&seen, UKEY(explicit_edges[2 * i], explicit_edges[2 * i + 1]));
        out_edges[2 * n] = explicit_edges[2 * i];
        out_edges[2 * n + 1] = explicit_edges[2 * i + 1];
        ++n;
    }
    for (int i = 0; i < ns; ++i) {
        const int a = strand_edges[2 * i], b = strand_edges[2 * i + 1];
        if (u64set_insert(&seen, UKEY(a, b))) {
            out_edges[2 * n] = a;
            out_edges[2 * n + 1] = b;
            ++n;
        }
    }
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) {
            const int a = tris[3 * t + k], b = tris[3 * t + (k + 1) % 3];
            if (u64set_insert(&seen, UKEY(a, b))) {
                out_edges[2 * n] = a < b ? a : b;
                out_edges[2 * n + 1] = a < b ? b : a;
                ++n;
            }
        }
#undef UKEY
    u64set_free(&seen);
    return n;
}

void or_mesh_init(or_mesh* m, int nv, const double* inv_mass, int ne, const int* edges, int nt,
                  const int* tris) {
    m->nv = nv, m->ne = ne, m->nt = nt;
    m->inv_mass = inv_mass, m->edges = edges, m->tris = tris;
    m->isolated = (uint8_t*)or_xmalloc((size_t)nv + 1);
    memset(m->isolated, 1, (size_t)nv + 1);
    /* MeshState::is_isolated_vertex, mesh.hpp:57-59 */
    for (int e = 0; e < ne; ++e) m->isolated[edges[2 * e]] = m->isolated[edges[2 * e + 1]] = 0;
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) m->isolated[tris[3 * t + k]] = 0;
}
void or_mesh_free(or_mesh* m) {
    free(m->isolated);
    m->isolated = NULL;
}

/* make_simplex, proximity.cpp:41-51 */
or_simplex or_make_simplex(const or_mesh* m, int kind, int index) {
    or_simplex s = {kind, {-1, -1, -1}};
    if (kind == OR_KIND_V) {
        s.idx[0] = index;
    } else if (kind == OR_KIND_E) {
        s.idx[0] = m->edges[2 * index];
        s.idx[1] = m->edges[2 * index + 1];
    } else {
        s.idx[0] = m->tris[3 * index];
        s.idx[1] = m->tris[3 * index + 1];
        s.idx[2] = m->tris[3 * index + 2];
    }
    return s;
}

/* ------------------------------------------------------------- search */

/* HashGrid::hash_cell, proximity.cpp:66-74 */
static uint64_t hash_cell(int64_t x, int64_t y, int64_t z) {
    uint64_t h = (uint64_t)x * 0x9E3779B97F4A7C15ull;
    h ^= (uint64_t)y * 0xC2B2AE3D27D4EB4Full;
    h ^= (uint64_t)z * 0x165667B19E3779F9ull;
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 32;
    return h;
}

typedef struct {
    uint64_t h;
    int32_t kind;
    int32_t index;
    int64_t seq;
} grid_rec;

static int cmp_rec(const void* a, const void* b) {
    const grid_rec* x = (const grid_rec*)a;
    const grid_rec* y = (const grid_rec*)b;
    if (x->h != y->h) return x->h < y->h ? -1 : 1;
    return x->seq < y->seq ? -1 : (x->seq > y->seq);
}
static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y);
}

typedef struct {
    grid_rec* r;
    int64_t n, cap;
} recvec;

static void rec_push(recvec* v, uint64_t h, int kind, int index) {
    if (v->n == v->cap) {
        v->cap = v->cap ? v->cap * 2 : 1024;
        v->r = (grid_rec*)or_xrealloc(v->r, (size_t)v->cap * sizeof(grid_rec));
    }
    v->r[v->n].h = h;
    v->r[v->n].kind = kind;
    v->r[v->n].index = index;
    v->r[v->n].seq = v->n;
    ++v->n;
}

/* simplex_aabb (proximity.cpp:23-32) + registration in every overlapped cell
 * (proximity.cpp:89-102) */
static void insert_entry(recvec* recs, const or_mesh* m, const double* x, int kind, int index,
                         double d_max) {
    const or_simplex s = or_make_simplex(m, kind, index);
    v3 lo = v3_load(x + 3 * (size_t)s.idx[0]), hi = lo;
    for (int i = 1; i < or_simplex_size(&s); ++i) {
        const v3 p = v3_load(x + 3 * (size_t)s.idx[i]);
        lo = v3_make(or_min(lo.x, p.x), or_min(lo.y, p.y), or_min(lo.z, p.z));
        hi = v3_make(or_max(hi.x, p.x), or_max(hi.y, p.y), or_max(hi.z, p.z));
    }
    const double inflate = 0.5 * d_max;
    lo = v3_make(lo.x - inflate, lo.y - inflate, lo.z - inflate);
    hi = v3_make(hi.x + inflate, hi.y + inflate, hi.z + inflate);
    const double cell = d_max;
    const int64_t x0 = (int64_t)floor(lo.x / cell), y0 = (int64_t)floor(lo.y / cell),
                  z0 = (int64_t)floor(lo.z / cell);
    const int64_t x1 = (int64_t)floor(hi.x / cell), y1 = (int64_t)floor(hi.y / cell),
                  z1 = (int64_t)floor(hi.z / cell);
    for (int64_t cx = x0; cx <= x1; ++cx)
        for (int64_t cy = y0; cy <= y1; ++cy)
            for (int64_t cz = z0; cz <= z1; ++cz) rec_push(recs, hash_cell(cx, cy, cz), kind, index);
}

/* canonical candidate rule, proximity.cpp:111-138 */
static int candidate(const or_mesh* m, int xk, int xi, int yk, int yi, int* ak, int* ai, int* bk,
                     int* bi) {
    int has_v = 0, vi = -1, ok = -1, oi = -1;
    if (xk == OR_KIND_V) has_v = 1, vi = xi, ok = yk, oi = yi;
    else if (yk == OR_KIND_V) has_v = 1, vi = yi, ok = xk, oi = xi;
    if (xk == OR_KIND_E && yk == OR_KIND_E) {
        *ak = *bk = OR_KIND_E;
        *ai = xi <= yi ? xi : yi;
        *bi = xi <= yi ? yi : xi;
        return *ai != *bi;
    }
    if (has_v && ok == OR_KIND_T) {
        *ak = OR_KIND_V, *ai = vi, *bk = OR_KIND_T, *bi = oi;
        return 1;
    }
    if (has_v && ok == OR_KIND_E && m->isolated[vi]) {
        *ak = OR_KIND_V, *ai = vi, *bk = OR_KIND_E, *bi = oi;
        return 1;
    }
    if (xk == OR_KIND_V && yk == OR_KIND_V && m->isolated[xi] && m->isolated[yi]) {
        *ak = *bk = OR_KIND_V;
        *ai = xi <= yi ? xi : yi;
        *bi = xi <= yi ? yi : xi;
        return *ai != *bi;
    }
    return 0;
}

static void pairset_push(or_pairset* set, const or_pair* p) {
    if (set->n == set->cap) {
        set->cap = set->cap ? set->cap * 2 : 256;
        set->pairs = (or_pair*)or_xrealloc(set->pairs, (size_t)set->cap * sizeof(or_pair));
    }
    set->pairs[set->n++] = *p;
}

void or_pairset_free(or_pairset* set) {
    free(set->pairs);
    set->pairs = NULL;
    set->n = set->cap = 0;
}

/* proximity_search, proximity.cpp:76-183 */
void or_pairset_search(or_pairset* set, const or_mesh* m, const double* x, double d_max) {
    set->n = 0;
    set->bound = d_max;
    if (m->nv == 0) return;

    recvec recs = {NULL, 0, 0};
    for (int v = 0; v < m->nv; ++v) insert_entry(&recs, m, x, OR_KIND_V, v, d_max);
    for (int e = 0; e < m->ne; ++e) insert_entry(&recs, m, x, OR_KIND_E, e, d_max);
    for (int t = 0; t < m->nt; ++t) insert_entry(&recs, m, x, OR_KIND_T, t, d_max);
    qsort(recs.r, (size_t)recs.n, sizeof(grid_rec), cmp_rec);

    /* per-bucket O(n^2) candidates with dedup (proximity.cpp:141-157) */
    u64set dedup;
    u64set_init(&dedup, recs.n);
    for (int64_t i0 = 0; i0 < recs.n;) {
        int64_t i1 = i0 + 1;
        while (i1 < recs.n && recs.r[i1].h == recs.r[i0].h) ++i1;
        for (int64_t i = i0; i < i1; ++i)
            for (int64_t j = i + 1; j < i1; ++j) {
                int ak, ai, bk, bi;
                if (!candidate(m, recs.r[i].kind, recs.r[i].index, recs.r[j].kind,
                               recs.r[j].index, &ak, &ai, &bk, &bi))
                    continue;
                u64set_insert(&dedup, or_pair_key(ak, ai, bk, bi));
            }
        i0 = i1;
    }
    free(recs.r);

    uint64_t* raw = (uint64_t*)or_xmalloc((size_t)(dedup.count + 1) * sizeof(uint64_t));
    int64_t nraw = 0;
    for (uint64_t i = 0; i <= dedup.mask; ++i)
        if (dedup.keys[i]) raw[nraw++] = dedup.keys[i];
    u64set_free(&dedup);
    qsort(raw, (size_t)nraw, sizeof(uint64_t), cmp_u64); /* proximity.cpp:158-160 */

    /* exact narrow-phase filter, proximity.cpp:162-181 */
    for (int64_t k = 0; k < nraw; ++k) {
        int ka, ia, kb, ib;
        or_key_decode(raw[k], &ka, &ia, &kb, &ib);
        or_pair p;
        memset(&p, 0, sizeof p);
        p.a = or_make_simplex(m, ka, ia);
        p.b = or_make_simplex(m, kb, ib);
        if (or_shares_vertex(&p.a, &p.b)) continue;
        if (or_pair_closest(&p.a, &p.b, x, &p.c) != 1) continue;
        if (p.c.distance >= d_max) continue;
        p.key = raw[k];
        p.ia = ia;
        p.ib = ib;
        p.active = 1;
        int all_static = 1;
        for (int i = 0; i < or_simplex_size(&p.a); ++i) all_static &= m->inv_mass[p.a.idx[i]] == 0.0;
        for (int i = 0; i < or_simplex_size(&p.b); ++i) all_static &= m->inv_mass[p.b.idx[i]] == 0.0;
        p.all_static = all_static;
        pairset_push(set, &p);
    }
    free(raw);
}

/* refresh_distances, proximity.cpp:190-202 */
void or_pairset_refresh(or_pairset* set, const double* x) {
    for (int64_t i = 0; i < set->n; ++i) {
        or_pair* p = &set->pairs[i];
        or_closest_t r;
        if (or_pair_closest(&p->a, &p->b, x, &r) != 1) {
            p->active = 0;
            continue;
        }
        if (r.degenerate && !v3_is_zero(p->c.dir)) r.dir = p->c.dir; /* keep last good direction */
        p->c = r;
        p->active = r.distance < set->bound;
    }
}

/* per_vertex_bound, proximity.cpp:204-211, evaluated for every vertex */
void or_pairset_vertex_bound(const or_pairset* set, int nv, double* out) {
    for (int v = 0; v < nv; ++v) out[v] = set->bound;
    for (int64_t i = 0; i < set->n; ++i) {
        const or_pair* p = &set->pairs[i];
        if (!p->active) continue;
        for (int k = 0; k < or_simplex_size(&p->a); ++k)
            out[p->a.idx[k]] = or_min(out[p->a.idx[k]], p->c.distance);
        for (int k = 0; k < or_simplex_size(&p->b); ++k)
            out[p->b.idx[k]] = or_min(out[p->b.idx[k]], p->c.distance);
    }
}

/* ------------------------------------------------------- flat-array API */

static void export_pairs(const or_pairset* set, uint64_t* keys, double* dist, double* wa,
                         double* wb, double* dir, uint8_t* flags) {
    for (int64_t i = 0; i < set->n; ++i) {
        const or_pair* p = &set->pairs[i];
        keys[i] = p->key;
        dist[i] = p->c.distance;
        for (int k = 0; k < 3; ++k) wa[3 * i + k] = p->c.wa[k], wb[3 * i + k] = p->c.wb[k];
        dir[3 * i] = p->c.dir.x, dir[3 * i + 1] = p->c.dir.y, dir[3 * i + 2] = p->c.dir.z;
        flags[i] = (uint8_t)((p->active ? OR_PF_ACTIVE : 0) | (p->all_static ? OR_PF_ALL_STATIC : 0) |
                             (p->c.degenerate ? OR_PF_DEGENERATE : 0));
    }
}

static void import_pairs(or_pairset* set, const or_mesh* m, int64_t np, const uint64_t* keys,
                         const double* dist, const double* wa, const double* wb, const double* dir,
                         const uint8_t* flags) {
    set->pairs = (or_pair*)or_xmalloc((size_t)(np + 1) * sizeof(or_pair));
    set->n = set->cap = np;
    for (int64_t i = 0; i < np; ++i) {
        or_pair* p = &set->pairs[i];
        int ka, ia, kb, ib;
        or_key_decode(keys[i], &ka, &ia, &kb, &ib);
        p->key = keys[i];
        p->a = or_make_simplex(m, ka, ia);
        p->b = or_make_simplex(m, kb, ib);
        p->ia = ia, p->ib = ib;
        p->c.distance = dist[i];
        for (int k = 0; k < 3; ++k) p->c.wa[k] = wa[3 * i + k], p->c.wb[k] = wb[3 * i + k];
        p->c.dir = v3_load(dir + 3 * i);
        p->c.degenerate = (flags[i] & OR_PF_DEGENERATE) != 0;
        p->active = (flags[i] & OR_PF_ACTIVE) != 0;
        p->all_static = (flags[i] & OR_PF_ALL_STATIC) != 0;
    }
}

int64_t or_search(int nv, const double* inv_mass, int ne, const int* edges, int nt, const int* tris,
                  const double* x, double d_max, int64_t cap, uint64_t* keys, double* dist,
                  double* wa, double* wb, double* dir, uint8_t* flags) {
    or_mesh m;
    or_mesh_init(&m, nv, inv_mass, ne, edges, nt, tris);
    or_pairset set = {NULL, 0, 0, 0.0};
    or_pairset_search(&set, &m, x, d_max);
    const int64_t n = set.n;
    if (n <= cap) export_pairs(&set, keys, dist, wa, wb, dir, flags);
    or_pairset_free(&set);
    or_mesh_free(&m);
    return n <= cap ? n : -n;
}

void or_refresh(int nv, int ne, const int* edges, int nt, const int* tris, const double* x,
                double bound, int64_t np, const uint64_t* keys, double* dist, double* wa,
                double* wb, double* dir, uint8_t* flags) {
    or_mesh m;
    or_mesh_init(&m, nv, NULL, ne, edges, nt, tris);
    or_pairset set;
    import_pairs(&set, &m, np, keys, dist, wa, wb, dir, flags);
    set.bound = bound;
    or_pairset_refresh(&set, x);
    for (int64_t i = 0; i < np; ++i) {
        /* all_static is a per-pair constant; keep the caller's bit */
        const uint8_t keep = flags[i] & OR_PF_ALL_STATIC;
        uint8_t tmp;
        uint64_t key_tmp;
        or_pairset s1 = {set.pairs + i, 1, 1, bound};
        export_pairs(&s1, &key_tmp, dist + i, wa + 3 * i, wb + 3 * i, dir + 3 * i, &tmp);
        flags[i] = (uint8_t)((tmp & ~OR_PF_ALL_STATIC) | keep);
    }
    free(set.pairs);
    or_mesh_free(&m);
}

void or_vertex_bound(int nv, int ne, const int* edges, int nt, const int* tris, double bound,
                     int64_t np, const uint64_t* keys, const double* dist, const uint8_t* flags,
                     double* out) {
    or_mesh m;
    or_mesh_init(&m, nv, NULL, ne, edges, nt, tris);
    or_pairset set;
    set.pairs = (or_pair*)or_xmalloc((size_t)(np + 1) * sizeof(or_pair));
    set.n = set.cap = np;
    set.bound = bound;
    for (int64_t i = 0; i < np; ++i) {
        int ka, ia, kb, ib;
        or_key_decode(keys[i], &ka, &ia, &kb, &ib);
        set.pairs[i].a = or_make_simplex(&m, ka, ia);
        set.pairs[i].b = or_make_simplex(&m, kb, ib);
        set.pairs[i].c.distance = dist[i];
        set.pairs[i].active = (flags[i] & OR_PF_ACTIVE) != 0;
    }
    or_pairset_vertex_bound(&set, nv, out);
    free(set.pairs);
    or_mesh_free(&m);
}

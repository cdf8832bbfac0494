/*
 * ORACLE — test infrastructure only.
 * Restatement of proj/src/resolve.cpp:12-149 (ResolveConfig::validate and the
 * Alg.-1 driver: search-if-stale, linearize, warm start, color, assemble,
 * solve, recover, lambda persistence, advance, refresh, shrink, erase,
 * convergence).
 */
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "or_internal.h"

/* std::unordered_map<uint64_t, double> replacement: open addressing with
 * tombstones (key 0 never occurs: a pair key always has ia != ib or kinds). */
typedef struct {
    uint64_t* keys; /* 0 empty, ~0 tombstone */
    double* vals;
    uint64_t mask;
    int64_t used; /* live + tombstones */
} lmap;

static const uint64_t kTomb = ~0ull;

static void lmap_init(lmap* m) {
    m->mask = 1023;
    m->keys = (uint64_t*)or_xcalloc(m->mask + 1, sizeof(uint64_t));
    m->vals = (double*)or_xcalloc(m->mask + 1, sizeof(double));
    m->used = 0;
}
static void lmap_free(lmap* m) {
    free(m->keys);
    free(m->vals);
}
static void lmap_put(lmap* m, uint64_t key, double val);
static void lmap_rehash(lmap* m) {
    lmap n;
    int64_t live = 0;
    for (uint64_t i = 0; i <= m->mask; ++i) live += m->keys[i] != 0 && m->keys[i] != kTomb;
    n.mask = 1023;
    while ((uint64_t)live * 4 > n.mask) n.mask = n.mask * 2 + 1;
    n.keys = (uint64_t*)or_xcalloc(n.mask + 1, sizeof(uint64_t));
    n.vals = (double*)or_xcalloc(n.mask + 1, sizeof(double));
    n.used = 0;
    for (uint64_t i = 0; i <= m->mask; ++i)
        if (m->keys[i] != 0 && m->keys[i] != kTomb) lmap_put(&n, m->keys[i], m->vals[i]);
    lmap_free(m);
    *m = n;
}
static int64_t lmap_find(const lmap* m, uint64_t key) {
    uint64_t h = or_mix64(key) & m->mask;
    for (;;) {
        if (m->keys[h] == 0) return -1;
        if (m->keys[h] == key) return (int64_t)h;
        h = (h + 1) & m->mask;
    }
}
static void lmap_put(lmap* m, uint64_t key, double val) {
    const int64_t at = lmap_find(m, key);
    if (at >= 0) {
        m->vals[at] = val;
        return;
    }
    if ((uint64_t)(m->used + 1) * 2 > m->mask + 1) lmap_rehash(m);
    uint64_t h = or_mix64(key) & m->mask;
    while (m->keys[h] != 0 && m->keys[h] != kTomb) h = (h + 1) & m->mask;
    if (m->keys[h] == 0) ++m->used;
    m->keys[h] = key;
    m->vals[h] = val;
}
static void lmap_erase(lmap* m, uint64_t key) {
    const int64_t at = lmap_find(m, key);
    if (at >= 0) m->keys[at] = kTomb;
}

/* ResolveConfig::validate, resolve.cpp:12-21 */
static int validate(const or_config* c) {
    if (!(c->d_min > 0.0) || !(c->d_min <= c->d_max)) return -1;
    if (!(c->delta > 0.0) || !(c->delta <= c->d_min)) return -1;
    if (!(c->gamma > 0.0) || !(c->gamma < 1.0)) return -1;
    if (!(c->eps > 0.0)) return -1;
    if (c->step_limit < 1) return -1;
    if (c->sweeps < 1) return -1;
    return 0;
}

static int all_finite(const double* x, int n) {
    for (int i = 0; i < 3 * n; ++i)
        if (!isfinite(x[i])) return 0;
    return 1;
}

int or_resolve(int nv, const double* inv_mass, int ne, const int* edges, int nt, const int* tris,
               const double* x_start, const double* y_target, const or_config* cfg,
               double* x_out, or_stats* st, double* step_max_disp, double* path,
               or_step_trace* trace) {
    memset(st, 0, sizeof *st);
    if (validate(cfg) != 0) return st->status = -1;
    if (!all_finite(x_start, nv) || !all_finite(y_target, nv)) return st->status = -1;
    if (cfg->solver != OR_SOLVER_PGS && cfg->solver != OR_SOLVER_JACOBI) return st->status = -2;

    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);

    or_mesh m;
    or_mesh_init(&m, nv, inv_mass, ne, edges, nt, tris);

    /* static vertices never move: their target is their current position */
    double* y_k1 = (double*)or_xmalloc((size_t)nv * 3 * sizeof(double) + 8);
    memcpy(y_k1, y_target, (size_t)nv * 3 * sizeof(double));
    for (int v = 0; v < nv; ++v)
        if (inv_mass[v] == 0.0) memcpy(y_k1 + 3 * v, x_start + 3 * v, 3 * sizeof(double));

    /* edge-length denominators frozen at y^{[k+1]} (resolve.cpp:53-55) */
    double* edge_targets = (double*)or_xmalloc(((size_t)ne + 1) * sizeof(double));
    for (int e = 0; e < ne; ++e)
        edge_targets[e] = v3_norm(v3_sub(v3_load(y_k1 + 3 * edges[2 * e]), v3_load(y_k1 + 3 * edges[2 * e + 1])));

    double* x = x_out;
    memcpy(x, x_start, (size_t)nv * 3 * sizeof(double));
    double* r = (double*)or_xmalloc(((size_t)nv + 1) * sizeof(double));
    for (int v = 0; v < nv; ++v) r[v] = 1.0;
    double last_max_disp = 0.0;
    if (cfg->record_path) memcpy(path, x, (size_t)nv * 3 * sizeof(double));

    int32_t* edge_color = NULL;
    if (cfg->coloring_mode == OR_COLOR_DEVICE) {
        edge_color = (int32_t*)or_xmalloc(((size_t)ne + 1) * sizeof(int32_t));
        or_color_edges_impl(nv, inv_mass, ne, edges, edge_color);
    }

    or_pairset set = {NULL, 0, 0, 0.0}; /* bound 0 forces a search on step 0 */
    lmap contact_lambda;
    lmap_init(&contact_lambda);
    double* edge_lambda = (double*)or_xcalloc((size_t)ne + 1, sizeof(double));
    or_rowvec rows = {NULL, 0, 0};
    double* y = (double*)or_xmalloc((size_t)nv * 3 * sizeof(double) + 8);
    double* D = (double*)or_xmalloc(((size_t)nv + 1) * sizeof(double));

    double prev_residual = 1.0;
    for (int l = 0; l < cfg->step_limit; ++l) {
        int searched = 0;
        if (cfg->force_fresh_search || set.bound < cfg->d_min) {
            or_pairset_search(&set, &m, x, cfg->d_max);
            ++st->searches;
            searched = 1;
            if (st->searches == 1)
                for (int64_t i = 0; i < set.n; ++i)
                    if (set.pairs[i].c.distance < 1e-10) st->start_in_contact = 1;
        }

        /* backward step at x^(l) */
        or_linearize_all(&set, x, &m, edge_targets, cfg->delta, cfg->sigma, cfg->family,
                         cfg->edge_constraints, &rows);
        int64_t ncontact = 0;
        for (int64_t i = 0; i < rows.n; ++i) {
            or_row* c = &rows.rows[i];
            if (c->kind == OR_ROW_EDGE) {
                c->lambda = edge_lambda[c->edge_index];
            } else {
                const int64_t at = lmap_find(&contact_lambda, c->pair_key);
                c->lambda = at < 0 ? 0.0 : contact_lambda.vals[at];
                ++ncontact;
            }
        }
        const int ncolors =
            cfg->coloring_mode == OR_COLOR_DEVICE
                ? or_color_device(rows.rows, rows.n, inv_mass, nv, cfg->color_seed, edge_color, ne,
                                  edges, cfg->edge_constraints)
                : or_color_reference(rows.rows, rows.n, inv_mass, nv, cfg->color_seed);
        or_lcp sys;
        or_lcp_assemble(&sys, rows.rows, rows.n, x, y_k1, inv_mass, nv, ncolors);
        if (cfg->solver == OR_SOLVER_PGS) or_lcp_pgs(&sys, cfg->sweeps);
        else or_lcp_jacobi(&sys, cfg->sweeps, cfg->under_relax);
        or_lcp_recover(&sys, y_k1, y);
        or_lcp_free(&sys);

        /* multipliers persist per pair identity (resolve.cpp:106-111) */
        for (int64_t i = 0; i < rows.n; ++i) {
            const or_row* c = &rows.rows[i];
            if (c->kind == OR_ROW_EDGE) edge_lambda[c->edge_index] = c->lambda;
            else lmap_put(&contact_lambda, c->pair_key, c->lambda);
        }

        /* forward step */
        const double bound_used = set.bound;
        or_pairset_vertex_bound(&set, nv, D);
        last_max_disp = or_advance(nv, inv_mass, y, D, cfg->gamma, x, r);
        if (last_max_disp > 0.5 * cfg->gamma * set.bound) st->step_law_violated = 1;
        if (step_max_disp) step_max_disp[l] = last_max_disp;
        st->steps = l + 1;
        if (cfg->record_path) memcpy(path + (size_t)(l + 1) * nv * 3, x, (size_t)nv * 3 * sizeof(double));

        or_pairset_refresh(&set, x);
        set.bound -= 2.0 * last_max_disp; /* shrink_bound, proximity.cpp:185-188 */
        int nactive = 0;
        for (int64_t i = 0; i < set.n; ++i) {
            if (!set.pairs[i].active) lmap_erase(&contact_lambda, set.pairs[i].key);
            else ++nactive;
        }

        double residual = 0.0;
        for (int v = 0; v < nv; ++v) residual = or_max(residual, r[v]);
        st->final_residual = residual;
        if (trace) {
            or_step_trace* t = &trace[l];
            t->searched = searched;
            t->num_pairs = (int32_t)set.n;
            t->num_contact_rows = (int32_t)ncontact;
            t->num_edge_rows = (int32_t)(rows.n - ncontact);
            t->num_colors = ncolors;
            t->num_active_pairs = nactive;
            t->bound = bound_used;
            t->max_disp = last_max_disp;
            t->residual = residual;
        }
        if (residual < cfg->eps) {
            st->converged = 1;
            break;
        }
        (void)prev_residual; /* AL stagnation test only applies to the AL solvers */
        prev_residual = residual;
    }
    st->hit_step_limit = !st->converged && !st->stagnated;

    clock_gettime(CLOCK_MONOTONIC, &t1);
    st->wall_ms = (double)(t1.tv_sec - t0.tv_sec) * 1e3 + (double)(t1.tv_nsec - t0.tv_nsec) * 1e-6;

    free(y_k1);
    free(edge_targets);
    free(r);
    free(edge_color);
    or_pairset_free(&set);
    lmap_free(&contact_lambda);
    free(edge_lambda);
    or_rowvec_free(&rows);
    free(y);
    free(D);
    or_mesh_free(&m);
    return 0;
}

/* flat-array linearize / color API for stage tests */
int64_t or_linearize(int nv, const double* inv_mass, int ne, const int* edges, int nt,
                     const int* tris, const double* x, int64_t np, const uint64_t* keys,
                     const double* dist, const double* wa, const double* wb, const double* dir,
                     const uint8_t* flags, const double* edge_targets, double delta, double window,
                     double sigma, int family, int edge_constraints, int64_t cap, uint8_t* kind,
                     int32_t* nverts,
                     int32_t* verts, double* value, double* jac, double* diag, uint64_t* pair_key,
                     int32_t* edge_index, uint8_t* flavor, double* ref_volume, double* gap_weights,
                     double* denom) {
    or_mesh m;
    or_mesh_init(&m, nv, inv_mass, ne, edges, nt, tris);
    or_pairset set;
    set.pairs = (or_pair*)or_xcalloc((size_t)np + 1, sizeof(or_pair));
    set.n = set.cap = np;
    set.bound = 0.0;
    for (int64_t i = 0; i < np; ++i) {
        or_pair* p = &set.pairs[i];
        int ka, ia, kb, ib;
        or_key_decode(keys[i], &ka, &ia, &kb, &ib);
        p->key = keys[i];
        p->a = or_make_simplex(&m, ka, ia);
        p->b = or_make_simplex(&m, kb, ib);
        p->ia = ia, p->ib = ib;
        p->c.distance = dist[i];
        for (int k = 0; k < 3; ++k) p->c.wa[k] = wa[3 * i + k], p->c.wb[k] = wb[3 * i + k];
        p->c.dir = v3_load(dir + 3 * i);
        p->c.degenerate = (flags[i] & OR_PF_DEGENERATE) != 0;
        p->active = (flags[i] & OR_PF_ACTIVE) != 0;
        p->all_static = (flags[i] & OR_PF_ALL_STATIC) != 0;
    }
    or_rowvec rows = {NULL, 0, 0};
    or_linearize_window(&set, x, &m, edge_targets, delta, window > 0.0 ? window : delta, sigma, family,
                        edge_constraints, &rows);
    const int64_t n = rows.n;
    if (n <= cap) {
        for (int64_t i = 0; i < n; ++i) {
            const or_row* c = &rows.rows[i];
            kind[i] = (uint8_t)c->kind;
            nverts[i] = c->nverts;
            for (int k = 0; k < 4; ++k) {
                verts[4 * i + k] = c->verts[k];
                jac[12 * i + 3 * k] = c->jac[k].x;
                jac[12 * i + 3 * k + 1] = c->jac[k].y;
                jac[12 * i + 3 * k + 2] = c->jac[k].z;
                gap_weights[4 * i + k] = c->gap_weights[k];
            }
            value[i] = c->value;
            diag[i] = c->diag;
            pair_key[i] = c->pair_key;
            edge_index[i] = c->edge_index;
            flavor[i] = (uint8_t)c->flavor;
            ref_volume[i] = c->ref_volume;
            denom[i] = c->denom;
        }
    }
    or_rowvec_free(&rows);
    free(set.pairs);
    or_mesh_free(&m);
    return n <= cap ? n : -n;
}

int or_color(int nv, const double* inv_mass, int64_t nrows, const uint8_t* kind,
             const int32_t* nverts, const int32_t* verts, const uint64_t* pair_key,
             const int32_t* edge_index, uint64_t seed, int mode, int ne, const int* edges,
             int edge_constraints, int32_t* color) {
    or_row* rows = (or_row*)or_xcalloc((size_t)nrows + 1, sizeof(or_row));
    for (int64_t i = 0; i < nrows; ++i) {
        rows[i].kind = kind[i];
        rows[i].nverts = nverts[i];
        for (int k = 0; k < 4; ++k) rows[i].verts[k] = verts[4 * i + k];
        rows[i].pair_key = pair_key[i];
        rows[i].edge_index = edge_index[i];
        rows[i].color = -1;
    }
    int nc;
    if (mode == OR_COLOR_DEVICE) {
        int32_t* ec = (int32_t*)or_xmalloc(((size_t)ne + 1) * sizeof(int32_t));
        or_color_edges_impl(nv, inv_mass, ne, edges, ec);
        nc = or_color_device(rows, nrows, inv_mass, nv, seed, ec, ne, edges, edge_constraints);
        free(ec);
    } else {
        nc = or_color_reference(rows, nrows, inv_mass, nv, seed);
    }
    for (int64_t i = 0; i < nrows; ++i) color[i] = rows[i].color;
    free(rows);
    return nc;
}

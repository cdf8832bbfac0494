/* ORACLE — test infrastructure only. Internal declarations. */
#ifndef OR_INTERNAL_H
#define OR_INTERNAL_H

#include <stddef.h>
#include <stdint.h>

#include "oracle.h"
#include "or_vec3.h"

/* ClosestResult, distance.hpp:15-21 */
typedef struct {
    double distance;
    double wa[3];
    double wb[3];
    v3 dir;
    int degenerate;
} or_closest_t;

typedef struct {
    int kind;
    int idx[3];
} or_simplex;

static inline int or_simplex_size(const or_simplex* s) { return s->kind + 1; }

/* distance.cpp */
void or_vv(v3 p, v3 q, or_closest_t* r);
void or_ve(v3 p, v3 e0, v3 e1, or_closest_t* r);
int or_vt(v3 p, v3 a, v3 b, v3 c, or_closest_t* r);
int or_ee(v3 p1, v3 p2, v3 q1, v3 q2, or_closest_t* r);
int or_shares_vertex(const or_simplex* a, const or_simplex* b);
/* 1 value, 0 nullopt, -1 invalid (reference throws) */
int or_pair_closest(const or_simplex* a, const or_simplex* b, const double* x, or_closest_t* r);

/* mesh view */
typedef struct {
    int nv, ne, nt;
    const double* inv_mass;
    const int* edges;
    const int* tris;
    uint8_t* isolated; /* owned */
} or_mesh;

void or_mesh_init(or_mesh* m, int nv, const double* inv_mass, int ne, const int* edges, int nt,
                  const int* tris);
void or_mesh_free(or_mesh* m);
or_simplex or_make_simplex(const or_mesh* m, int kind, int index);

/* pair record */
typedef struct {
    uint64_t key;
    or_simplex a, b;
    int ia, ib;
    or_closest_t c;
    int active;
    int all_static;
} or_pair;

typedef struct {
    or_pair* pairs;
    int64_t n, cap;
    double bound;
} or_pairset;

static inline uint64_t or_pair_key(int ka, int ia, int kb, int ib) {
    return ((uint64_t)ka << 62) | ((uint64_t)kb << 60) | ((uint64_t)(uint32_t)ia << 30) |
           (uint64_t)(uint32_t)ib;
}
static inline void or_key_decode(uint64_t k, int* ka, int* ia, int* kb, int* ib) {
    *ka = (int)(k >> 62);
    *kb = (int)((k >> 60) & 3);
    *ia = (int)((k >> 30) & 0x3fffffff);
    *ib = (int)(k & 0x3fffffff);
}

void or_pairset_search(or_pairset* set, const or_mesh* m, const double* x, double d_max);
void or_pairset_refresh(or_pairset* set, const double* x);
void or_pairset_vertex_bound(const or_pairset* set, int nv, double* out);
void or_pairset_free(or_pairset* set);

/* constraint row, constraints.hpp:16-36 */
typedef struct {
    int kind;
    int nverts;
    int verts[4];
    double value;
    v3 jac[4];
    double diag;
    double lambda;
    int color;
    int64_t pair_index;
    uint64_t pair_key;
    int edge_index;
    int flavor;
    double ref_volume;
    double gap_weights[4];
    double denom;
    double sigma;
} or_row;

typedef struct {
    or_row* rows;
    int64_t n, cap;
} or_rowvec;

void or_rowvec_push(or_rowvec* v, const or_row* r);
void or_rowvec_free(or_rowvec* v);

void or_linearize_all(const or_pairset* set, const double* x, const or_mesh* m,
                      const double* edge_targets, double delta, double sigma, int family,
                      int edge_constraints, or_rowvec* out);
void or_linearize_window(const or_pairset* set, const double* x, const or_mesh* m,
                         const double* edge_targets, double delta, double window, double sigma,
                         int family, int edge_constraints, or_rowvec* out);
void or_fill_diag(or_row* c, const double* inv_mass);
int or_color_reference(or_row* rows, int64_t n, const double* inv_mass, int nv, uint64_t seed);
int or_color_device(or_row* rows, int64_t n, const double* inv_mass, int nv, uint64_t seed,
                    const int32_t* edge_color, int ne, const int* edges, int edge_constraints);
int or_color_edges_impl(int nv, const double* inv_mass, int ne, const int* edges, int32_t* color);

/* lcp */
typedef struct {
    or_row* rows;
    int64_t n;
    const double* inv_mass;
    double* q;
    double* impulse; /* nv * 3 */
    int nv;
    int ncolors;
} or_lcp;

void or_lcp_assemble(or_lcp* s, or_row* rows, int64_t n, const double* x, const double* y,
                     const double* inv_mass, int nv, int ncolors);
void or_lcp_pgs(or_lcp* s, int iters);
void or_lcp_jacobi(or_lcp* s, int iters, double under_relax);
void or_lcp_recover(const or_lcp* s, const double* y_target, double* y_out);
void or_lcp_free(or_lcp* s);

/* mt19937_64 + libstdc++ uniform_int_distribution<size_t> (Lemire _S_nd) */
typedef struct {
    uint64_t mt[312];
    int idx;
} or_mt64;
void or_mt64_seed(or_mt64* g, uint64_t seed);
uint64_t or_mt64_next(or_mt64* g);
uint64_t or_uniform_below(or_mt64* g, uint64_t range); /* uniform in [0, range) */

/* device-coloring priority hash (splitmix64 finalizer) */
static inline uint64_t or_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void* or_xmalloc(size_t n);
void* or_xcalloc(size_t n, size_t sz);
void* or_xrealloc(void* p, size_t n);

#endif

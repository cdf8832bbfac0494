/*
 * ORACLE — CPU restatement of the reference two-way collision-handling path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in paper_2211_04045_b200/ links, loads or
 * calls this code; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do, as the checker and the timed CPU
 * baseline. Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 *
 * Parity status: the reference cannot be built here (it requires Eigen >= 3.3,
 * an external library that is absent from the image, plus an absent vendor/
 * tree), so this restatement is pinned against the known-answer tests of the
 * reference's own test suite (tests/test_*.cpp; see tests/test_oracle_kats.py)
 * rather than against reference binaries.
 */
#ifndef TW_ORACLE_H
#define TW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_KIND_V = 0, OR_KIND_E = 1, OR_KIND_T = 2 };

/* constraint kinds, constraints.hpp:7 */
enum { OR_ROW_VT = 0, OR_ROW_EE = 1, OR_ROW_VE = 2, OR_ROW_VV = 3, OR_ROW_EDGE = 4 };
/* constraint flavors, constraints.hpp:31 */
enum { OR_FLAVOR_VOLUME = 0, OR_FLAVOR_GAP = 1, OR_FLAVOR_LENGTH = 2 };

enum { OR_SOLVER_PGS = 0, OR_SOLVER_JACOBI = 1, OR_SOLVER_AL20 = 2, OR_SOLVER_AL100 = 3 };
enum { OR_FAMILY_VOLUME = 0, OR_FAMILY_GAP = 1 };
/* coloring: 0 = exact reference algorithm (constraints.cpp:222-288),
 *           1 = the product's deterministic parallel (Jones-Plassmann) coloring */
enum { OR_COLOR_REFERENCE = 0, OR_COLOR_DEVICE = 1 };

/* pair flag bits */
enum { OR_PF_ACTIVE = 1, OR_PF_ALL_STATIC = 2, OR_PF_DEGENERATE = 4 };

/* Same field layout as tw_resolve_config in include/tw_c.h (ResolveConfig,
 * resolve.hpp:13-34, plus coloring_mode). */
typedef struct {
    int32_t step_limit;
    int32_t solver;
    double eps;
    double d_min;
    double d_max;
    double delta;
    double sigma;
    double gamma;
    int32_t sweeps;
    int32_t family;
    double under_relax;
    int32_t edge_constraints;
    int32_t force_fresh_search;
    int32_t record_path;
    int32_t coloring_mode;
    uint64_t color_seed;
} or_config;

/* ResolveStats (resolve.hpp:36-51) minus the vectors (passed as buffers). */
typedef struct {
    int32_t steps;
    int32_t searches;
    double final_residual;
    double wall_ms;
    int32_t converged;
    int32_t hit_step_limit;
    int32_t stagnated;
    int32_t start_in_contact;
    int32_t step_law_violated;
    int32_t status; /* 0 ok, <0 error */
} or_stats;

/* one record per Alg.-1 step (diagnostics for stage-by-stage comparison) */
typedef struct {
    int32_t searched;
    int32_t num_pairs;
    int32_t num_contact_rows;
    int32_t num_edge_rows;
    int32_t num_colors;
    int32_t num_active_pairs;
    double bound;     /* bound used by this step's advance */
    double max_disp;  /* last_max_disp after advance */
    double residual;  /* max r after the step */
} or_step_trace;

/* ---- geometry (distance.cpp) ---- */
/* Closest-point query between simplex (ka, va) and (kb, vb) at positions x.
 * out = [dist, wa0, wa1, wa2, wb0, wb1, wb2, dir0, dir1, dir2, degenerate].
 * Returns 1 for a value, 0 for nullopt, -1 for adjacency / unsupported kinds
 * (the reference throws std::invalid_argument there). */
int or_closest(int ka, const int* va, int kb, const int* vb, const double* x, double* out);

/* ---- mesh (mesh.cpp:10-33) ---- */
/* Derives the unique edge list: explicit edges, then new strand edges, then
 * triangle edges in (t, k) order as (min, max). Returns the edge count;
 * out_edges must hold ne_explicit + ns + 3 nt pairs. */
int or_finalize_edges(int nv, int ne_explicit, const int* explicit_edges, int ns,
                      const int* strand_edges, int nt, const int* tris, int* out_edges);

/* ---- proximity (proximity.cpp) ---- */
/* proximity_search: returns the pair count P (sorted by key); when P > cap the
 * outputs are not written and -P is returned. */
int64_t or_search(int nv, const double* inv_mass, int ne, const int* edges, int nt, const int* tris,
                  const double* x, double d_max, int64_t cap, uint64_t* keys, double* dist,
                  double* wa, double* wb, double* dir, uint8_t* flags);

/* refresh_distances (proximity.cpp:190-202), in place */
void or_refresh(int nv, int ne, const int* edges, int nt, const int* tris, const double* x,
                double bound, int64_t np, const uint64_t* keys, double* dist, double* wa,
                double* wb, double* dir, uint8_t* flags);

/* per_vertex_bound (proximity.cpp:204-211) for every vertex */
void or_vertex_bound(int nv, int ne, const int* edges, int nt, const int* tris, double bound,
                     int64_t np, const uint64_t* keys, const double* dist, const uint8_t* flags,
                     double* out);

/* ---- constraints (constraints.cpp) ---- */
/* linearize_all (window <= 0 -> delta): returns R (contact rows then edge rows) or -R if R > cap. */
int64_t or_linearize(int nv, const double* inv_mass, int ne, const int* edges, int nt,
                     const int* tris, const double* x, int64_t np, const uint64_t* keys,
                     const double* dist, const double* wa, const double* wb, const double* dir,
                     const uint8_t* flags, const double* edge_targets, double delta, double window,
                     double sigma, int family, int edge_constraints, int64_t cap, uint8_t* kind,
                     int32_t* nverts,
                     int32_t* verts, double* value, double* jac, double* diag, uint64_t* pair_key,
                     int32_t* edge_index, uint8_t* flavor, double* ref_volume, double* gap_weights,
                     double* denom);

/* constraint_value_at (constraints.cpp:39-54) */
double or_constraint_value_at(int flavor, int nverts, const int32_t* verts, double ref_volume,
                              const double* gap_weights, double denom, double sigma,
                              const double* x);

/* color_constraints; mode OR_COLOR_REFERENCE or OR_COLOR_DEVICE. For the
 * device mode, edge_colors (per mesh edge, -1 for both-static edges) are the
 * precomputed edge-row colors (or NULL to compute them here). Returns ncolors. */
int or_color(int nv, const double* inv_mass, int64_t nrows, const uint8_t* kind,
             const int32_t* nverts, const int32_t* verts, const uint64_t* pair_key,
             const int32_t* edge_index, uint64_t seed, int mode, int ne, const int* edges,
             int edge_constraints, int32_t* color);

/* device-mode precoloring of the edge rows (one color per mesh edge, -1 for
 * edges whose endpoints are both static). Returns the color count. */
int or_color_edges(int nv, const double* inv_mass, int ne, const int* edges, int32_t* edge_color);

/* ---- backward step (lcp.cpp) ---- */
/* assemble_lcp + {pgs,jacobi} sweeps + recover_target. lambda is in/out (warm
 * start in, solution out); q_out (R) and impulse_out (nv*3) may be NULL. */
int or_backward(int nv, const double* inv_mass, int64_t nrows, const int32_t* nverts,
                const int32_t* verts, const double* value, const double* jac, const double* diag,
                const int32_t* color, int ncolors, const double* x, const double* y_target,
                int solver, int sweeps, double under_relax, double* lambda, double* q_out,
                double* impulse_out, double* y_out);

/* ---- forward step (advance.cpp:8-39) ---- */
/* x, r in/out; D = per-vertex bound. Returns last_max_disp. */
double or_advance(int nv, const double* inv_mass, const double* y, const double* D, double gamma,
                  double* x, double* r);

/* ---- driver (resolve.cpp:36-144) ---- */
int or_resolve(int nv, const double* inv_mass, int ne, const int* edges, int nt, const int* tris,
               const double* x_start, const double* y_target, const or_config* cfg,
               double* x_out, or_stats* stats, double* step_max_disp, double* path,
               or_step_trace* trace);

/* ---- RNG helpers exposed for tests ---- */
uint64_t or_mt19937_64_nth(uint64_t seed, int64_t n); /* n-th output, 1-based */
uint64_t or_uniform_index(uint64_t seed, int64_t draws, uint64_t size); /* debug */

/* ---- CCD certifier (testkit/ccd.cpp) ---- */
/* ccd_certify on one linear segment x0 -> x1. Returns the number of
 * violations; certain_out receives the certain count. */
int or_ccd_certify(int nv, int ne, const int* edges, int nt, const int* tris, const double* x0,
                   const double* x1, int* certain_out);

#ifdef __cplusplus
}
#endif

#endif

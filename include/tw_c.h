/*
 * tw_c.h — C-ABI of the B200-native two-way continuous collision handling
 * path (arXiv 2211.04045, reference proj/include/twoway/resolve.hpp).
 *
 * The reference exposes only C++ (twoway::resolve / twoway::repair,
 * resolve.hpp:63-69) and a pybind11 module (bindings/module.cpp:101-186). This
 * C-ABI is the boundary a drop-in replacement needs: plain pointers and sizes,
 * no CUDA or torch types. include/twoway/resolve.hpp re-implements the
 * reference C++ API on top of it; paper_2211_04045_b200/_twoway mirrors the
 * Python module. All arithmetic is FP64 on the GPU (sm_100a); there is no
 * CPU fallback — without a CUDA device every call returns TW_ECUDA.
 *
 * Positions are N x 3 row-major doubles: the byte layout of
 * std::vector<Eigen::Vector3d> (types.hpp:10-14) and of a numpy (N, 3) array.
 */
#ifndef TW_C_H
#define TW_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TW_ABI_VERSION 1

/* error codes (the C++ wrapper maps EINVAL/EUNSUPPORTED to
 * std::invalid_argument as resolve.cpp:12-21,39-43 throws, the rest to
 * std::runtime_error) */
enum {
    TW_OK = 0,
    TW_EINVAL = 1,       /* bad config / sizes / non-finite input */
    TW_EUNSUPPORTED = 2, /* solver al20/al100 (paper baseline, out of scope) */
    TW_ECAPACITY = 3,    /* internal: a device buffer was too small (regrown + retried) */
    TW_ECUDA = 4,        /* CUDA runtime error / no device */
    TW_ETIMEOUT = 5      /* device watchdog fired inside the resolve kernel */
};

enum { TW_SOLVER_PGS = 0, TW_SOLVER_JACOBI = 1, TW_SOLVER_AL20 = 2, TW_SOLVER_AL100 = 3 };
enum { TW_FAMILY_VOLUME = 0, TW_FAMILY_GAP = 1 };
/* TW_COLOR_REFERENCE replays the reference's randomized smallest-last greedy
 * coloring (constraints.cpp:222-288) exactly on one device thread — bit-exact
 * end-to-end parity, slow at scale. TW_COLOR_DEVICE is the parallel
 * deterministic Jones-Plassmann coloring: a different but valid
 * Gauss-Seidel order, the performance mode. */
enum { TW_COLOR_REFERENCE = 0, TW_COLOR_DEVICE = 1 };

/* ResolveConfig, resolve.hpp:13-34 (+ coloring_mode) */
typedef struct {
    int32_t step_limit;   /* L = 512 */
    int32_t solver;       /* TW_SOLVER_* */
    double eps;           /* 1e-4 */
    double d_min;         /* 2e-3 m */
    double d_max;         /* 4e-3 m */
    double delta;         /* 1e-3 m */
    double sigma;         /* 1.1 */
    double gamma;         /* 0.9 */
    int32_t sweeps;       /* 1 */
    int32_t family;       /* TW_FAMILY_* */
    double under_relax;   /* 0.5 */
    int32_t edge_constraints;
    int32_t force_fresh_search;
    int32_t record_path;
    int32_t coloring_mode; /* TW_COLOR_* */
    uint64_t color_seed;   /* 0x5eed */
} tw_resolve_config;

/* ResolveStats, resolve.hpp:36-51 (vectors are separate buffers) */
typedef struct {
    int32_t steps;
    int32_t searches;
    double final_residual;
    double wall_ms;           /* host wall time of the call */
    int32_t converged;
    int32_t hit_step_limit;
    int32_t stagnated;
    int32_t start_in_contact;
    int32_t step_law_violated;
    int32_t num_pairs;        /* |P| after the last step */
    int64_t pairs_evaluated;  /* narrow-phase closest evaluations (search + refresh) */
    int64_t rows_solved;      /* sum over steps of (contact + edge rows) */
    double device_ms;         /* CUDA-event time of the device resolve (no H2D/D2H) */
    int32_t kernel_launches;  /* kernels this call launched */
    int32_t retries;          /* capacity regrow restarts */
    double kernel_ms;         /* CUDA-event time of the persistent resolve kernel alone */
    double setup_ms;          /* unpack + LBVH build before it */
} tw_resolve_stats;

/* per-step diagnostics (same fields as the oracle's trace) */
typedef struct {
    int32_t searched;
    int32_t num_pairs;
    int32_t num_contact_rows;
    int32_t num_edge_rows;
    int32_t num_colors;
    int32_t num_active_pairs;
    double bound;
    double max_disp;
    double residual;
} tw_step_trace;

typedef struct tw_ctx tw_ctx;
typedef struct tw_mesh tw_mesh;

int tw_abi_version(void);
void tw_default_config(tw_resolve_config* cfg);

/* One context per (host thread, device); not thread-safe. stream may be NULL
 * (the context creates its own) or a cudaStream_t to run on. */
int tw_ctx_create(int device, void* stream, tw_ctx** out);
void tw_ctx_destroy(tw_ctx* ctx);
const char* tw_last_error(const tw_ctx* ctx);
/* Share the device with parts - 1 other contexts that run concurrently on
 * their own streams (independent scenes, BASELINE configs[4]): this context's
 * persistent kernels use 1/parts of the co-resident CTAs. */
int tw_ctx_set_grid_share(tw_ctx* ctx, int32_t parts);
/* kernels launched by this context since creation */
int64_t tw_ctx_kernel_launches(const tw_ctx* ctx);
/* Per-phase wall time of the last resolve (CTA 0, barrier to barrier):
 * call-site ids (source line & 127 in tw_kernels.cu), milliseconds and
 * counts; returns the number of sites (entries beyond cap are not written). */
int32_t tw_ctx_phase_profile(const tw_ctx* ctx, int32_t* sites, double* ms, int32_t* counts, int32_t cap);

/* Topology upload (once per scene). Runs MeshState::finalize's edge
 * derivation (mesh.cpp:10-33) on the explicit, strand and triangle edges:
 * the resulting order defines edge indices. inv_mass may be NULL (all 1). */
int tw_mesh_create(tw_ctx* ctx, int32_t nv, const double* inv_mass, int32_t ne_explicit,
                   const int32_t* edges, int32_t ns, const int32_t* strand_edges, int32_t nt,
                   const int32_t* triangles, tw_mesh** out);
int32_t tw_mesh_num_edges(const tw_mesh* mesh);
int tw_mesh_edges(const tw_mesh* mesh, int32_t* out_edges /* 2 * ne */);
/* A mesh and its context may be destroyed in either order. */
void tw_mesh_destroy(tw_mesh* mesh);

/* resolve(x_start, y_target, mesh, cfg) — resolve.cpp:36-144. Host buffers.
 * step_max_disp: NULL or step_limit doubles; path: NULL or
 * (step_limit + 1) * nv * 3 doubles (used when cfg->record_path); trace:
 * NULL or step_limit entries. */
int tw_resolve(tw_ctx* ctx, tw_mesh* mesh, const double* x_start, const double* y_target,
               const tw_resolve_config* cfg, double* x_out, tw_resolve_stats* stats,
               double* step_max_disp, double* path, tw_step_trace* trace);

/* The path of the last resolve run with cfg->record_path (x^(0) .. x^(final),
 * ResolveStats::path, resolve.hpp:48): kept on the device in a buffer that
 * grows on demand (no step_limit-sized allocation); copies min(cap_states,
 * states) states of nv * 3 doubles into out and the state count into *nstates. */
int tw_last_path(tw_ctx* ctx, int64_t cap_states, double* out, int32_t* nstates);

/* Same with device pointers already resident in HBM (nv * 3 doubles each). */
int tw_resolve_device(tw_ctx* ctx, tw_mesh* mesh, const double* d_x_start,
                      const double* d_y_target, const tw_resolve_config* cfg, double* d_x_out,
                      tw_resolve_stats* stats);

/* ---- stage entry points (stage-by-stage parity; host buffers) ---- */

/* simplex_pair_closest for n arbitrary pairs. kinds: 2n (ka, kb); verts: 6n
 * (3 ids of a, 3 ids of b, -1 padded). out: 11n = [dist, wa[3], wb[3],
 * dir[3], degenerate]; has: n = 1 value, 0 nullopt, -1 adjacent/unsupported. */
int tw_stage_closest(tw_ctx* ctx, int32_t nv, const double* x, int64_t n, const int32_t* kinds,
                     const int32_t* verts, double* out, int32_t* has);

/* proximity_search (proximity.cpp:76-183) on the device broad phase. Writes
 * at most cap pairs sorted by key; *np receives P (if P > cap, nothing is
 * written and TW_ECAPACITY is returned). wa/wb/dir: 3 doubles per pair;
 * flags: bit0 active, bit1 all_static, bit2 degenerate. */
int tw_stage_search(tw_ctx* ctx, tw_mesh* mesh, const double* x, double d_max, int64_t cap,
                    uint64_t* keys, double* dist, double* wa, double* wb, double* dir,
                    uint8_t* flags, int64_t* np);

/* refresh_distances (proximity.cpp:190-202) in place, then per_vertex_bound
 * (proximity.cpp:204-211) for every vertex into vertex_bound (may be NULL). */
int tw_stage_refresh(tw_ctx* ctx, tw_mesh* mesh, const double* x, double bound, int64_t np,
                     const uint64_t* keys, double* dist, double* wa, double* wb, double* dir,
                     uint8_t* flags, double* vertex_bound);

/* linearize_all (constraints.cpp:181-220): contact rows then edge rows.
 * Row arrays: kind (u8), verts (4 x i32, -1 padded), value, jac (12 doubles),
 * diag, pair_key (u64), edge_index (i32). Returns R in *nrows. */
int tw_stage_linearize(tw_ctx* ctx, tw_mesh* mesh, const double* x, int64_t np,
                       const uint64_t* keys, const double* dist, const double* wa,
                       const double* wb, const double* dir, const uint8_t* flags,
                       const double* edge_targets, double delta, double sigma, int32_t family,
                       int32_t edge_constraints, int64_t cap, uint8_t* kind, int32_t* verts,
                       double* value, double* jac, double* diag, uint64_t* pair_key,
                       int32_t* edge_index, int64_t* nrows);

/* color_constraints on rows produced by tw_stage_linearize (contact rows
 * first). mode TW_COLOR_*. Returns the color count in *ncolors. */
int tw_stage_color(tw_ctx* ctx, tw_mesh* mesh, int64_t nrows, const uint8_t* kind,
                   const int32_t* verts, const uint64_t* pair_key, const int32_t* edge_index,
                   uint64_t seed, int32_t mode, int32_t edge_constraints, int32_t* color,
                   int32_t* ncolors);

/* assemble_lcp + pgs/jacobi sweeps + recover_target (lcp.cpp). lambda in/out. */
int tw_stage_backward(tw_ctx* ctx, int32_t nv, const double* inv_mass, int64_t nrows,
                      const int32_t* verts, const double* value, const double* jac,
                      const double* diag, const int32_t* color, int32_t ncolors,
                      const double* x, const double* y_target, int32_t solver, int32_t sweeps,
                      double under_relax, double* lambda, double* q_out, double* y_out);

/* The backward step split as the reference's lcp.hpp:36-53 splits it.
 * mode: TW_LCP_ASSEMBLE = assemble_lcp (q = value + J (y - x), lcp.cpp:8-25;
 * the warm-start impulse M^-1 J^T lambda accumulated in row order), TW_LCP_SOLVE
 * = pgs_sweeps / projected_jacobi_sweeps (lcp.cpp:27-59) from the given q,
 * lambda and impulse, TW_LCP_RECOVER = recover_target (lcp.cpp:131-136) into
 * y_out. Without ASSEMBLE, q (nrows) and impulse (nv * 3) are inputs; lambda
 * and impulse are written back after the sweeps; q is written by ASSEMBLE. */
enum { TW_LCP_ASSEMBLE = 1, TW_LCP_SOLVE = 2, TW_LCP_RECOVER = 4 };
int tw_stage_lcp(tw_ctx* ctx, int32_t nv, const double* inv_mass, int64_t nrows, const int32_t* verts,
                 const double* value, const double* jac, const double* diag, const int32_t* color, int32_t ncolors,
                 const double* x, const double* y_target, int32_t solver, int32_t sweeps, double under_relax,
                 int32_t mode, double* lambda, double* q, double* impulse, double* y_out);

/* Row flavors (Constraint::Flavor, constraints.hpp:31) */
enum { TW_FLAVOR_VOLUME = 0, TW_FLAVOR_GAP = 1, TW_FLAVOR_LENGTH = 2 };

/* linearize_all plus each row's re-evaluation data (Constraint::flavor,
 * ref_volume, gap_weights[4], denom; constraints.hpp:26-33) for
 * constraint_value_at. Same arguments as tw_stage_linearize plus the four
 * outputs (R entries; gap_weights 4 per row). */
int tw_stage_linearize_ex(tw_ctx* ctx, tw_mesh* mesh, const double* x, int64_t np, const uint64_t* keys,
                          const double* dist, const double* wa, const double* wb, const double* dir,
                          const uint8_t* flags, const double* edge_targets, double delta, double sigma,
                          int32_t family, int32_t edge_constraints, int64_t cap, uint8_t* kind, int32_t* verts,
                          double* value, double* jac, double* diag, uint64_t* pair_key, int32_t* edge_index,
                          uint8_t* flavor, double* ref_volume, double* gap_weights, double* denom, int64_t* nrows);

/* build_vt / build_ee / build_vv / build_ve_constraint (constraints.cpp:78-142;
 * gap = 0: by the pair kinds with the reference's gap fallbacks) or
 * build_gap_constraint (constraints.cpp:56-76; gap = 1) for n pairs given as
 * kinds (2n: ka, kb), simplex vertex ids (6n, -1 padded) and cached closest
 * results (11n, the tw_stage_closest layout). Rows carry no diag (fill it
 * with tw_stage_fill_diag). */
int tw_stage_build_rows(tw_ctx* ctx, int32_t nv, const double* x, int64_t n, const int32_t* kinds,
                        const int32_t* verts, const double* closest, double delta, int32_t gap, uint8_t* kind,
                        int32_t* nverts, int32_t* row_verts, double* value, double* jac, uint8_t* flavor,
                        double* ref_volume, double* gap_weights, double* denom);

/* constraint_value_at (constraints.cpp:39-54) of n rows at x. */
int tw_stage_constraint_value(tw_ctx* ctx, int32_t nv, const double* x, int64_t n, const uint8_t* flavor,
                              const int32_t* nverts, const int32_t* row_verts, const double* ref_volume,
                              const double* gap_weights, const double* denom, const double* sigma, double* out);

/* fill_diag (constraints.cpp:175-179) of n rows. */
int tw_stage_fill_diag(tw_ctx* ctx, int32_t nv, const double* inv_mass, int64_t n, const int32_t* nverts,
                       const int32_t* row_verts, const double* jac, double* diag);

/* advance (advance.cpp:8-39): x and r in/out, D = per-vertex bound. */
int tw_stage_advance(tw_ctx* ctx, int32_t nv, const double* inv_mass, const double* y,
                     const double* D, double gamma, double* x, double* r, double* max_disp);

/* ccd_certify (proj/src/testkit/ccd.cpp:339-498) of the linear segment
 * x0 -> x1 (nv * 3 doubles each): the number of vertex-triangle and edge-edge
 * stencils whose motion crosses (*violations) and how many of those are
 * certain (*certain, away from the numerical margins). Zero violations
 * certify the segment intersection-free. *candidates (nullable): swept-box
 * candidate stencils tested. Runs on the device. */
int tw_ccd_certify(tw_ctx* ctx, tw_mesh* mesh, const double* x0, const double* x1, int32_t* violations,
                   int32_t* certain, int64_t* candidates);


/* ---- dynamics: the step-and-project simulator around resolve -------------
 * proj/include/twoway/dynamics.hpp / proj/src/dynamics.cpp on the device: the
 * implicit-Euler incremental potential (inertia, springs, flat-rest bending,
 * gravity), the quadratic repulsion on the proximity set, the block-Jacobi
 * PCG Newton target and step() = target + resolve + velocity update. */

/* EnergyModel scalars (dynamics.hpp:12-24) */
typedef struct {
    double spring_stiffness;    /* 50 N/m */
    double bending_stiffness;   /* 0 */
    double gravity[3];          /* (0, 0, -9.81) */
    double repulsion_stiffness; /* 1e3 N/m */
    double repulsion_radius;    /* 1e-3 m */
    double dt;                  /* 0.01 s */
    int32_t newton_iters;       /* 1 */
    double mu;                  /* 0; mu > 0 runs friction_filter on the target */
    double pcg_tol;             /* 1e-6 relative */
    int32_t pcg_max_iters;      /* 400 */
} tw_energy_model;

/* StepStats (dynamics.hpp:78-90) plus device diagnostics */
typedef struct {
    int32_t resolve_steps;   /* total_resolve_steps() */
    int32_t searches;        /* total_searches() of the resolves */
    int32_t resolve_converged;
    int32_t pcg_iterations;  /* summed over Newton iterations */
    int32_t pcg_converged;
    int32_t num_pairs;       /* pairs of the last target's search (cutoff min(d_max, repulsion_radius); d_max when mu > 0) */
    int32_t repulsive_pairs; /* pairs closer than repulsion_radius */
    double device_ms;        /* CUDA-event time of the whole step on the device */
    double resolve_ms;       /* of which resolve */
    double wall_ms;
    double target_ms;        /* of which the Newton targets (search + gradient/Hessian + PCG) */
    double pcg_ms;           /* of which the PCG kernels */
    double friction_ms;      /* friction_filter (mu > 0) */
} tw_step_stats;

typedef struct tw_dyn tw_dyn;

void tw_default_energy_model(tw_energy_model* model);
/* EnergyModel::prepare (dynamics.cpp:17-69): rest lengths and flat-rest
 * hinges from rest_x (nv * 3). The model is validated (EnergyModel::validate,
 * dynamics.cpp:10-15 -> TW_EINVAL). */
int tw_dyn_create(tw_ctx* ctx, tw_mesh* mesh, const tw_energy_model* model, const double* rest_x, tw_dyn** out);
void tw_dyn_destroy(tw_dyn* dyn);
int32_t tw_dyn_num_hinges(const tw_dyn* dyn);
/* proximity_search(x, d_max) + gradient_and_hessian + add_repulsion +
 * newton_target (dynamics.cpp:334-337) with the inertia target built from
 * (x0, v0), then friction_filter when mu > 0 (dynamics.cpp:338): writes the
 * target y_out and (nullable) the gradient. */
int tw_newton_target(tw_ctx* ctx, tw_mesh* mesh, tw_dyn* dyn, double d_max, const double* x0, const double* v0,
                     const double* x, double* y_out, double* grad_out, tw_step_stats* stats);
/* friction_filter (dynamics.cpp:272-324) with the pair set of
 * proximity_search(x, d_max): the target y_target (nv * 3) filtered by the
 * inelastic, Coulomb-capped pair impulses of the dyn's model, in pair order
 * (bit-identical to the sequential loop). step() / tw_newton_target apply it
 * when mu > 0, as dynamics.cpp:338 does. */
int tw_friction_filter(tw_ctx* ctx, tw_mesh* mesh, tw_dyn* dyn, double d_max, const double* x, const double* y_target,
                       double* y_out);
/* step() (dynamics.cpp:326-349): x, v (nv * 3) in/out, host buffers. */
int tw_step(tw_ctx* ctx, tw_mesh* mesh, tw_dyn* dyn, const tw_resolve_config* cfg, double* x, double* v,
            tw_step_stats* stats);
/* Same on device-resident state (HBM pointers, nv * 3 doubles each). */
int tw_step_device(tw_ctx* ctx, tw_mesh* mesh, tw_dyn* dyn, const tw_resolve_config* cfg, double* d_x, double* d_v,
                   tw_step_stats* stats);


/* normal_flow_target (normal_flow.cpp:38-81; the validation of
 * require_closed_manifold, normal_flow.cpp:24-36, -> TW_EINVAL): area-weighted
 * unit normals, the offset y = x + beta n, cotangent edge weights and three
 * Jacobi smoothing passes scaled by alpha_smooth, on the device. */
int tw_normal_flow_target(tw_ctx* ctx, int32_t nv, const double* x, int32_t nt, const int32_t* triangles,
                          double beta, double alpha_smooth, double* y_out);

#ifdef __cplusplus
}
#endif

#endif

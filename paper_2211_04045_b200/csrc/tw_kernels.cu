// Kernels of the B200 two-way collision handling path: per-call setup, the
// LBVH build, the persistent cooperative resolve kernel (the whole Alg. 1
// loop on the device, no host round trip per step) and the stage kernels
// used for stage-by-stage parity. Compiled with -fmad=false.
#include <cstdlib>
#include <cub/device/device_radix_sort.cuh>

#include "tw_ccd.cuh"
#include "tw_internal.h"
#include "tw_phases.cuh"

namespace tw {

// ================================================================= setup
// Unpack N x 3 host-layout positions into double4 (w = inv_mass), apply the
// static override y_k1 = x_start (resolve.cpp:48-50), initialise r = 1 and
// the per-vertex scratch; flag non-finite input (resolve.cpp:41-43).
__global__ void k_unpack(int nv, const double* xs, const double* ys, const double* inv_mass, double4* x,
                         double4* yk1, double* r, unsigned long long* dmin, int* voff, int* vcnt,
                         double4* imp, int* nonfinite) {
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x) {
        const double im = inv_mass[v];
        const double a0 = xs[3 * v], a1 = xs[3 * v + 1], a2 = xs[3 * v + 2];
        double b0 = ys[3 * v], b1 = ys[3 * v + 1], b2 = ys[3 * v + 2];
        if (!isfinite(a0) || !isfinite(a1) || !isfinite(a2) || !isfinite(b0) || !isfinite(b1) ||
            !isfinite(b2))
            atomicOr(nonfinite, 1);
        if (im == 0.0) b0 = a0, b1 = a1, b2 = a2;
        x[v] = make_double4(a0, a1, a2, im);
        yk1[v] = make_double4(b0, b1, b2, im);
        r[v] = 1.0;
        dmin[v] = INF_BITS;
        voff[v] = 0;
        vcnt[v] = 0;
        imp[v] = make_double4(0, 0, 0, 0);
    }
}

// frozen edge targets (resolve.cpp:53-55) and the edge-row set of the call
// (constraints.cpp:152-153): target > 1e-12 and not both endpoints static
__global__ void k_edges_init(int ne, const int2* edges, const double4* yk1, double* ly, uint8_t* is_er,
                             double* edge_lambda, int* er_color, const int* edge_color, int edge_rows,
                             int device_coloring) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
         e += (long long)gridDim.x * blockDim.x) {
        const int2 ed = edges[e];
        const double4 a = yk1[ed.x], b = yk1[ed.y];
        const double l = nrm(mk(a.x - b.x, a.y - b.y, a.z - b.z));
        ly[e] = l;
        is_er[e] = (edge_rows && l > 1e-12 && !(a.w == 0.0 && b.w == 0.0)) ? 1 : 0;
        edge_lambda[e] = 0.0;
        er_color[e] = device_coloring ? edge_color[e] : -1;
    }
}

__global__ void k_pack(int nv, const double4* x, double* out) {
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x) {
        const double4 a = x[v];
        out[3 * v] = a.x, out[3 * v + 1] = a.y, out[3 * v + 2] = a.z;
    }
}

// ================================================================ LBVH
__device__ __forceinline__ unsigned long long ord_bits(double d) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ord(unsigned long long o) {
    const unsigned long long b = (o & 0x8000000000000000ull) ? (o & ~0x8000000000000000ull) : ~o;
    return __longlong_as_double((long long)b);
}

__global__ void k_bounds(int nv, const double4* x, unsigned long long* box /* 6: lo xyz, hi xyz */) {
    __shared__ unsigned long long s[6];
    if (threadIdx.x < 3) s[threadIdx.x] = ~0ull, s[3 + threadIdx.x] = 0ull;
    __syncthreads();
    unsigned long long l[3] = {~0ull, ~0ull, ~0ull}, h[3] = {0, 0, 0};
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x) {
        const double4 p = x[v];
        const double c[3] = {p.x, p.y, p.z};
        for (int k = 0; k < 3; ++k) {
            const unsigned long long o = ord_bits(c[k]);
            l[k] = min(l[k], o);
            h[k] = max(h[k], o);
        }
    }
    for (int k = 0; k < 3; ++k) atomicMin(&s[k], l[k]), atomicMax(&s[3 + k], h[k]);
    __syncthreads();
    if (threadIdx.x < 3) atomicMin(&box[threadIdx.x], s[threadIdx.x]), atomicMax(&box[3 + threadIdx.x], s[3 + threadIdx.x]);
}

__device__ __forceinline__ unsigned expand_bits(unsigned v) {
    v = (v * 0x00010001u) & 0xFF0000FFu;
    v = (v * 0x00000101u) & 0x0F00F00Fu;
    v = (v * 0x00000011u) & 0xC30C30C3u;
    v = (v * 0x00000005u) & 0x49249249u;
    return v;
}

// 30-bit Morton code of each primitive's centroid
__global__ void k_morton(int n, int cls, const int4* tris, const int2* edges, const int* iso, const double4* x,
                         const unsigned long long* box, unsigned* codes, int* idx) {
    const double lo[3] = {from_ord(box[0]), from_ord(box[1]), from_ord(box[2])};
    const double hi[3] = {from_ord(box[3]), from_ord(box[4]), from_ord(box[5])};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double c[3] = {0, 0, 0};
        int ids[3], k;
        if (cls == 0) {
            const int4 t = tris[i];
            ids[0] = t.x, ids[1] = t.y, ids[2] = t.z, k = 3;
        } else if (cls == 1) {
            const int2 e = edges[i];
            ids[0] = e.x, ids[1] = e.y, k = 2;
        } else if (cls == 2) {
            ids[0] = iso[i], k = 1;
        } else {  // 3: the vertices themselves (query order of the broad phase)
            ids[0] = (int)i, k = 1;
        }
        for (int j = 0; j < k; ++j) {
            const double4 p = x[ids[j]];
            c[0] += p.x, c[1] += p.y, c[2] += p.z;
        }
        unsigned q[3];
        for (int a = 0; a < 3; ++a) {
            const double ext = hi[a] - lo[a];
            double u = ext > 0.0 ? (c[a] / k - lo[a]) / ext : 0.5;
            u = fmin(fmax(u, 0.0), 1.0);
            q[a] = min(1023u, (unsigned)(u * 1024.0));
        }
        codes[i] = (expand_bits(q[0]) << 2) | (expand_bits(q[1]) << 1) | expand_bits(q[2]);
        idx[i] = (int)i;
    }
}

__device__ __forceinline__ int lcp_delta(const unsigned* c, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    const unsigned a = c[i], b = c[j];
    if (a == b) return 32 + __clz((unsigned)(i ^ j));
    return __clz(a ^ b);
}

// Karras 2012 hierarchy over sorted codes: internal nodes 0..n-2, leaf j at n-1+j
__global__ void k_karras(int n, const unsigned* codes, const int* sorted_idx, int* prim, int2* child, int* parent,
                         unsigned* flag) {
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)t;
        prim[i] = sorted_idx[i];
        if (i == 0) parent[n > 1 ? 0 : 0] = -1;
        if (i >= n - 1) continue;
        flag[i] = 0u;
        const int d = (lcp_delta(codes, n, i, i + 1) - lcp_delta(codes, n, i, i - 1)) >= 0 ? 1 : -1;
        const int dmin = lcp_delta(codes, n, i, i - d);
        int lmax = 2;
        while (lcp_delta(codes, n, i, i + lmax * d) > dmin) lmax *= 2;
        int l = 0;
        for (int s = lmax / 2; s >= 1; s /= 2)
            if (lcp_delta(codes, n, i, i + (l + s) * d) > dmin) l += s;
        const int j = i + l * d;
        const int dnode = lcp_delta(codes, n, i, j);
        int s = 0, div = 2, step;
        do {
            step = (l + div - 1) / div;
            if (lcp_delta(codes, n, i, i + (s + step) * d) > dnode) s += step;
            div *= 2;
        } while (step > 1);
        const int gamma = i + s * d + min(d, 0);
        const int left = (min(i, j) == gamma) ? (n - 1 + gamma) : gamma;
        const int right = (max(i, j) == gamma + 1) ? (n - 1 + gamma + 1) : gamma + 1;
        child[i] = make_int2(left, right);
        parent[left] = i;
        parent[right] = i;
    }
}

// =========================================================== closest
__global__ void k_stage_closest(int nv, const double4* x, long long n, const int* kinds, const int* verts,
                                double* out, int* has) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int ka = kinds[2 * i], kb = kinds[2 * i + 1];
        const int* va = verts + 6 * i;
        const int* vb = verts + 6 * i + 3;
        Closest c;
        const int h = pair_closest(ka, va, kb, vb, XLoad{x}, c);
        has[i] = h;
        double* o = out + 11 * i;
        if (h == 1) {
            o[0] = c.dist;
            for (int k = 0; k < 3; ++k) o[1 + k] = c.wa[k], o[4 + k] = c.wb[k];
            o[7] = c.dir.x, o[8] = c.dir.y, o[9] = c.dir.z;
            o[10] = c.degenerate ? 1.0 : 0.0;
        }
    }
    (void)nv;
}

// ================================================= row stage entries
// build_{vt,ee,vv,ve}_constraint / build_gap_constraint (constraints.cpp:56-142)
// for n pairs given as (kinds, vertex ids, cached closest result): the row and
// its re-evaluation data. gap = 1: build_gap_constraint for every kind.
__global__ void k_stage_build_rows(const double4* x, long long n, const int* kinds, const int* verts,
                                   const double* closest, double delta, int gap, int* kind, int* nverts, int* rv,
                                   double* value, double* jac, int* flavor, double* ref_volume, double* gw,
                                   double* denom) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int ka = kinds[2 * i], kb = kinds[2 * i + 1];
        const int* va = verts + 6 * i;
        const int* vb = verts + 6 * i + 3;
        const double* c = closest + 11 * i;
        Row r;
        RowEval ev;
        build_contact(ka, va, kb, vb, c + 1, c + 4, c[0], mk(c[7], c[8], c[9]), delta, gap, XLoad{x}, r, &ev);
        kind[i] = r.kind;
        nverts[i] = r.nverts;
        for (int m = 0; m < 4; ++m) {
            rv[4 * i + m] = m < r.nverts ? r.v[m] : -1;
            const d3 j = m < r.nverts ? r.jac[m] : mk(0, 0, 0);
            jac[12 * i + 3 * m] = j.x, jac[12 * i + 3 * m + 1] = j.y, jac[12 * i + 3 * m + 2] = j.z;
            gw[4 * i + m] = ev.gw[m];
        }
        value[i] = r.value;
        flavor[i] = ev.flavor;
        ref_volume[i] = ev.ref_volume;
        denom[i] = ev.denom;
    }
}

// constraint_value_at (constraints.cpp:39-54) for n rows
__global__ void k_stage_value_at(const double4* x, long long n, const int* flavor, const int* nverts, const int* rv,
                                 const double* ref_volume, const double* gw, const double* denom, const double* sigma,
                                 double* out) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int* v = rv + 4 * i;
        double val = 0.0;
        if (flavor[i] == FLAVOR_VOLUME) {
            val = stencil_det(ld3(x, v[0]), ld3(x, v[1]), ld3(x, v[2]), ld3(x, v[3])) / ref_volume[i] - 1.0;
        } else if (flavor[i] == FLAVOR_GAP) {
            d3 g = mk(0, 0, 0);
            for (int m = 0; m < nverts[i]; ++m) g = add(g, scl(gw[4 * i + m], ld3(x, v[m])));
            val = nrm(g) / denom[i] - 1.0;
        } else {
            val = sigma[i] - nrm(sub(ld3(x, v[0]), ld3(x, v[1]))) / denom[i];
        }
        out[i] = val;
    }
}

// fill_diag (constraints.cpp:175-179) for n rows
__global__ void k_stage_fill_diag(const double* inv_mass, long long n, const int* nverts, const int* rv,
                                  const double* jac, double* diag) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double d = 0.0;
        for (int m = 0; m < nverts[i]; ++m) {
            const double* J = jac + 12 * i + 3 * m;
            d += inv_mass[rv[4 * i + m]] * sqn(mk(J[0], J[1], J[2]));
        }
        diag[i] = maxd(d, 1e-10);
    }
}

// ====================================================== call prologue
// ER compaction (edge order) and, in device-coloring mode, the static edge
// row buckets by color (the edge-row colors are fixed for the call).
__device__ bool prologue(const Params& P) {
    long long lo, hi;
    chunk_of(P.ne, &lo, &hi);
    long long cnt = 0;
    for (long long e = lo + threadIdx.x; e < hi; e += TPB) cnt += P.is_er[e];
    const long long t = block_sum(cnt);
    if (threadIdx.x == 0) P.part_k[blockIdx.x] = t;
    if (P.cfg.record_path)
        for (long long v = gtid(); v < P.nv; v += gstride()) {
            const double4 a = P.x[v];
            P.path[3 * v] = a.x, P.path[3 * v + 1] = a.y, P.path[3 * v + 2] = a.z;
        }
    if (!grid_sync(P.g)) return false;
    const long long ner_total = prefix_of(P.part_k, gridDim.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) P.g->ner = (int)ner_total;
    long long base = prefix_of(P.part_k, blockIdx.x);
    for (long long tt = lo; tt < hi; tt += TPB) {
        const long long e = tt + threadIdx.x;
        const int f = e < hi ? P.is_er[e] : 0;
        long long tot;
        const long long pos = base + block_scan(f, &tot);
        base += tot;
        if (e < hi) P.er_index[e] = f ? (int)pos : -1;
        if (f) {
            P.er_edge[pos] = (int)e;
            if (P.cfg.coloring_mode == 1) atomicAdd(&P.er_color_cnt[P.er_color[e]], 1);
        }
    }
    if (!grid_sync(P.g)) return false;
    if (P.cfg.coloring_mode == 1) {
        long long run = 0;
        for (int b0 = 0; b0 < P.er_ncolors; b0 += TPB) {
            const int c = b0 + threadIdx.x;
            const long long v = c < P.er_ncolors ? P.er_color_cnt[c] : 0;
            long long tt;
            const long long ex = block_scan(v, &tt);
            if (blockIdx.x == 0 && c < P.er_ncolors) P.er_color_off[c] = (int)(run + ex);
            run += tt;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) P.er_color_off[P.er_ncolors] = (int)run;
        if (!grid_sync(P.g)) return false;
        for (long long k = gtid(); k < P.g->ner; k += gstride()) {
            const int e = P.er_edge[k];
            const int c = P.er_color[e];
            const int slot = atomicSub(&P.er_color_cnt[c], 1) - 1;
            P.er_by_color[P.er_color_off[c] + slot] = e;
        }
        if (!grid_sync(P.g)) return false;
    }
    return true;
}

// ======================================================== resolve kernel
// The Alg.-1 loop of resolve.cpp:69-137, device resident: every CTA runs the
// same control flow (replicated scalars, read from device memory after each
// grid barrier), so the host only sees the final state.
// progress marker (TW_DEBUG=1): the last phase each CTA completed, written to
// host-mapped memory so it survives a device fault
// Phase profile: CTA 0 accumulates the wall time (globaltimer) between its
// barrier exits per call site (slot = source line & 127).
#define SYNC()                                                                    \
    do {                                                                          \
        if (P.dbg && threadIdx.x == 0) {                                          \
            P.dbg[blockIdx.x] = (dbg_step << 16) | __LINE__;                      \
            __threadfence_system();                                               \
        }                                                                         \
        if (!grid_sync(g)) return;                                                \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                \
            const unsigned long long now_ = global_ns();                          \
            atomicAdd(&g->phase_ns[__LINE__ % kPhaseSites], now_ - ph_t0);         \
            atomicAdd(&g->phase_cnt[__LINE__ % kPhaseSites], 1u);                  \
            ph_t0 = now_;                                                         \
        }                                                                         \
    } while (0)

// the same over the first n CTAs only (sub_sync)
#define SUBSYNC(n)                                                                \
    do {                                                                          \
        if (!sub_sync(g, (n))) return;                                            \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                \
            const unsigned long long now_ = global_ns();                          \
            atomicAdd(&g->phase_ns[__LINE__ % kPhaseSites], now_ - ph_t0);         \
            atomicAdd(&g->phase_cnt[__LINE__ % kPhaseSites], 1u);                  \
            ph_t0 = now_;                                                         \
        }                                                                         \
    } while (0)

// MINB = resident CTAs per SM the register allocation targets (2: 128 regs,
// 3: 80, 4: 64); the context picks the instance (TW_BLOCKS_PER_SM).
template <int MINB>
__global__ void __launch_bounds__(TPB, MINB) k_resolve(Params P) {
    Globals* g = P.g;
    int dbg_step = 0;
    if (g->nonfinite || g->error) return;  // non-finite input detected by k_unpack
    if (!prologue(P)) return;
    unsigned long long ph_t0 = (blockIdx.x == 0 && threadIdx.x == 0) ? global_ns() : 0ull;
    const Config& C = P.cfg;
    double bound = 0.0;  // forces a search on step 0
    int searches = 0;
    int sel = 0;
    long long narch = 0;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    int steps = 0;
    double residual = 0.0;
    bool converged = false;
    for (int l = 0; l < C.step_limit; ++l) {
        dbg_step = l;
        const bool search = C.force_fresh_search || bound < C.d_min;
        if (search) {
            ph_refit(P);
            SYNC();
            ph_traverse(P);
            SYNC();
            ph_cand_eval(P);
            SYNC();
            ph_query_totals(P);
            SYNC();
            ph_emit_pairs(P);
            SYNC();
            ph_emit_records(P, searches == 0);
            SYNC();
            bound = C.d_max;
            ++searches;
        }
        if (lead) {
            g->maxdisp_bits = 0ull;
            g->resid_bits = 0ull;
            g->colored = 0;
            g->max_color = -1;
        }
        // ---- backward step at x^(l)
        ph_rows(P);
        SYNC();
        const long long nc = g->nc;
        if (lead) g->nactive = 0;
        ph_rows_build(P, sel, narch, nc);
        SYNC();
        ph_inc_totals(P);
        SYNC();
        ph_inc_offsets(P);
        SYNC();
        ph_inc_scatter(P, nc);
        SYNC();
        ph_warm(P, nc);
        SYNC();
        int ncol_c, ncol_e, ncol;
        if (C.coloring_mode == 0) {
            ph_color_ref_count(P, nc);
            SYNC();
            ph_color_ref_fill(P, nc);
            SYNC();
            ph_color_ref(P, nc);
            SYNC();
            ncol = g->max_color + 1;
            if (ncol > P.colcap) {
                if (lead) atomicOr(&g->error, ERR_CAP_COLORS);
                return;
            }
            ph_bucket_count(P, nc);
            SYNC();
            ph_bucket_scatter(P, nc, ncol, true);
            SYNC();
            ph_bucket_place(P, nc, true);
            SYNC();
            ncol_c = ncol_e = ncol;
        } else {
            for (int k = 1; *((volatile int*)&g->colored) < nc; ++k) {
                if (k > 1) {
                    ph_color_rank(P);
                    SYNC();
                }
                ph_color_propose(P, nc, k);
                SYNC();
                ph_color_conflict(P, k);
                SYNC();
                ph_color_commit(P, nc, k);
                SYNC();
            }
            ncol_c = g->max_color + 1;
            ncol_e = C.edge_constraints ? P.er_ncolors : 0;
            ncol = max(ncol_c, ncol_e);
            ph_bucket_scatter(P, nc, ncol_c, false);
            SYNC();
            ph_bucket_place(P, nc, false);
            SYNC();
        }
        if (C.solver == 0) {
            // the color phases run on the first pgs_ctas block indices
            // (sm_count x TW_PGS_CTAS_PER_SM, default 2 per SM on average; a
            // cooperative launch does not fix their placement) behind their own
            // sub-grid barrier; the rest of the grid waits at the join
            const int nsub = P.pgs_ctas;
            if ((int)blockIdx.x < nsub) {
                const PgsRanges R = pgs_ranges(P, ncol, ncol_c, ncol_e, nc);
                const long long tail_rows = P.pgs_tail_rows;
                PgsRow pre;
                pre.color = -1;
                for (int sw = 0; sw < C.sweeps; ++sw) {
                    int c = 0;
                    while (c < ncol && R.rows(P, c) == 0) ++c;  // unused colors: no phase, no barrier
                    if (c < ncol && R.rows(P, c) > tail_rows) pgs_prefetch(P, R, c, nsub, pre);
                    while (c < ncol) {
                        const long long nrow = R.rows(P, c);
                        int next;
                        if (nrow <= tail_rows) {
                            // a run of small colors: CTA 0 alone, CTA barriers between them
                            next = c;
                            while (next < ncol && R.rows(P, next) <= tail_rows) ++next;
                            ph_pgs_tail_r(P, R, c, next);
                        } else {
                            ph_pgs_color_pre(P, R, c, nsub, pre);
                            next = c + 1;
                        }
                        while (next < ncol && R.rows(P, next) == 0) ++next;
                        // the next large color's static row data, in flight across the barrier
                        if (next < ncol && R.rows(P, next) > tail_rows) pgs_prefetch(P, R, next, nsub, pre);
                        // ph_pgs_color (a large color or a run of small ones)
                        SUBSYNC(nsub);
                        c = next;
                    }
                }
            }
            // ph_pgs_join
            SYNC();
        } else {
            for (int sw = 0; sw < C.sweeps; ++sw) {
                ph_jacobi_next(P, nc);
                SYNC();
                ph_jacobi_apply(P, nc);
                SYNC();
                ph_jacobi_commit(P, nc);
                SYNC();
            }
        }
        // ---- forward step
        ph_advance(P, bound, l, nc, sel);
        SYNC();
        const double maxdisp = to_d(g->maxdisp_bits);
        residual = to_d(g->resid_bits);
        if (lead) {
            if (maxdisp > 0.5 * C.gamma * bound) g->step_law_violated = 1;
            if (P.step_max_disp) P.step_max_disp[l] = maxdisp;
            g->rows_solved += nc + (C.edge_constraints ? P.g->ner : 0);
        }
        const double bound_next = bound - 2.0 * maxdisp;
        const bool next_search = C.force_fresh_search || bound_next < C.d_min;
        const long long nnew = prefix_of(P.part_k, gridDim.x);
        if (nnew > 0) {
            if (narch + nnew > P.arch_cap) {
                if (lead) atomicOr(&g->error, ERR_CAP_ARCH);
                return;
            }
            ph_arch_rank(P, nc);
            SYNC();
            ph_arch_merge(P, nnew, sel, narch);
            SYNC();
            sel ^= 1;
            narch += nnew;
        }
        // refresh at x^(l+1) (resolve.cpp:120-123). Without a trace to fill,
        // the refresh after the final step has no observable effect, and
        // before a re-search only its multiplier erasures matter.
        const bool final_step = residual < C.eps || l + 1 == C.step_limit;
        if (P.trace || (!final_step && !next_search)) {
            ph_refresh(P, bound, next_search);
            SYNC();
            if (narch > 0) {
                ph_arch_erase(P, sel, narch);
                SYNC();
            }
        } else if (!final_step && narch > 0) {
            ph_refresh_archive(P, bound, sel, narch);
            SYNC();
        }
        if (lead && P.trace) {
            Trace& t = P.trace[l];
            t.searched = search;
            t.num_pairs = (int)g->np;
            t.num_contact_rows = (int)nc;
            t.num_edge_rows = C.edge_constraints ? P.g->ner : 0;
            t.num_colors = ncol;
            t.num_active_pairs = g->nactive;
            t.bound = bound;
            t.max_disp = maxdisp;
            t.residual = residual;
        }
        if (lead) g->ncolors_last = ncol;
        bound = bound_next;
        steps = l + 1;
        if (residual < C.eps) {
            converged = true;
            break;
        }
    }
    if (lead) {
        g->steps = steps;
        g->searches = searches;
        g->converged = converged;
        g->final_residual = residual;
        g->narch = narch;
        g->arch_sel = sel;
    }
}

// ======================================================== stage kernels
// stage kernels run on the context's cooperative grid (up to 4 CTAs/SM)
__global__ void __launch_bounds__(TPB, 4) k_stage_search(Params P) {
    ph_refit(P);
    if (!grid_sync(P.g)) return;
    ph_traverse(P);
    if (!grid_sync(P.g)) return;
    ph_cand_eval(P);
    if (!grid_sync(P.g)) return;
    ph_query_totals(P);
    if (!grid_sync(P.g)) return;
    ph_emit_pairs(P);
    if (!grid_sync(P.g)) return;
    ph_emit_records(P, false);
}

// refresh + per-vertex bound into P.r (min(bound, dmin))
template <int MINB>
__global__ void __launch_bounds__(TPB, MINB) k_stage_refresh(Params P, double bound) {
    ph_refresh(P, bound, false);
    if (!grid_sync(P.g)) return;
    for (long long v = gtid(); v < P.nv; v += gstride()) P.r[v] = mind(bound, to_d(P.dmin[v]));
}

__global__ void k_stage_advance(Params P, double* max_disp) {
    ph_advance(P, __longlong_as_double(0x7ff0000000000000ll), -1, 0, 0);
    (void)max_disp;
}

#define STAGE_SYNC() \
    do {                           \
        if (!grid_sync(P.g)) return; \
    } while (0)

// contact predicate of linearize_all over an uploaded pair set (the flags
// carry active / all_static), block totals for the compaction of ph_rows
__device__ void ph_stage_contact_flags(const Params& P) {
    const long long np = P.g->np;
    for_pair_tiles(P, np, [&](long long p) -> bool {
        const uint64_t key = P.pkey[p];
        const int ka = key_ka(key), kb = key_kb(key);
        int va[3], vb[3];
        split_ids(ka, kb, P.pids[p], va, vb);
        uint8_t fl = P.pflag[p] & (PF_ACTIVE | PF_ALL_STATIC | PF_DEGENERATE);
        if (contact_pred(P, ka, kb, va, vb, P.pdd[p], P.pw[p], fl)) fl |= PF_CONTACT;
        P.pflag[p] = fl;
        return (fl & PF_CONTACT) != 0;
    });
}

// vertex -> row incidence of uploaded rows (dynamic vertices only)
__device__ void ph_stage_incidence(const Params& P, long long nc) {
    for (long long e = gtid(); e < 4 * nc; e += gstride()) {
        const int v = (&P.c_ids[e >> 2].x)[e & 3];
        if (v >= 0 && P.inv_mass[v] > 0.0) record_incidence(P, v, (int)e);
        else P.c_slot[e] = -1;
    }
}

// q = value + sum_m jac_m . (y_k1 - x) of uploaded rows (lcp.cpp:16-20)
__device__ void ph_stage_q(const Params& P, long long nc) {
    for (long long i = gtid(); i < nc; i += gstride()) {
        const int4 id = P.c_ids[i];
        const int vv[4] = {id.x, id.y, id.z, id.w};
        const double* J = P.c_jac + i * 12;
        double q = P.c_value[i];
        for (int m = 0; m < 4 && vv[m] >= 0; ++m) {
            const double4 xv = P.x[vv[m]];
            q += dot(mk(J[3 * m], J[3 * m + 1], J[3 * m + 2]), sub(ld3(P.yk1, vv[m]), mk(xv.x, xv.y, xv.z)));
        }
        P.c_q[i] = q;
    }
}

// ================================================ CCD certification
// ccd_certify (testkit/ccd.cpp:339-498) of one segment x -> ccd_x1: swept-box
// candidates from the LBVH walk (VT: every vertex against the triangles; EE:
// canonical e1 < e2), the reference's exact double swept-box overlap and
// adjacency filters, then the per-stencil test (tw_ccd.cuh).
__device__ __forceinline__ void swept_box_d(const Params& P, const int* ids, int n, double lo[3], double hi[3]) {
    const d3 s0 = ld3(P.x, ids[0]);
    lo[0] = hi[0] = s0.x, lo[1] = hi[1] = s0.y, lo[2] = hi[2] = s0.z;
    for (int i = 0; i < n; ++i) {
        const d3 p = ld3(P.x, ids[i]), q = ld3(P.ccd_x1, ids[i]);
        lo[0] = mind(mind(lo[0], p.x), q.x), lo[1] = mind(mind(lo[1], p.y), q.y), lo[2] = mind(mind(lo[2], p.z), q.z);
        hi[0] = maxd(maxd(hi[0], p.x), q.x), hi[1] = maxd(maxd(hi[1], p.y), q.y), hi[2] = maxd(maxd(hi[2], p.z), q.z);
    }
    for (int k = 0; k < 3; ++k) lo[k] = lo[k] - 1e-12, hi[k] = hi[k] + 1e-12;
}

__device__ void ph_ccd_eval(const Params& P) {
    const long long n = min((long long)P.g->ncand, P.ccap);
    int viol = 0, cert = 0;
    for (long long i = gtid(); i < n; i += gstride()) {
        const int2 e = P.cand[i];
        int ka, ia, kb, cls;
        query_of(P, e.x, &ka, &ia, &kb, &cls);
        const int ib = e.y;
        int ids[4];
        bool is_vt;
        if (ka == KV) {  // vertex against triangle
            const int4 t = P.tris[ib];
            if (ia == t.x || ia == t.y || ia == t.z) continue;
            ids[0] = ia, ids[1] = t.x, ids[2] = t.y, ids[3] = t.z;
            is_vt = true;
        } else {  // edge against edge, ia < ib
            if (ib <= ia) continue;
            const int2 a = P.edges[ia], b = P.edges[ib];
            if (a.x == b.x || a.x == b.y || a.y == b.x || a.y == b.y) continue;
            ids[0] = a.x, ids[1] = a.y, ids[2] = b.x, ids[3] = b.y;
            is_vt = false;
        }
        double alo[3], ahi[3], blo[3], bhi[3];
        swept_box_d(P, ids, is_vt ? 1 : 2, alo, ahi);
        swept_box_d(P, ids + (is_vt ? 1 : 2), is_vt ? 3 : 2, blo, bhi);
        if (!(alo[0] <= bhi[0] && alo[1] <= bhi[1] && alo[2] <= bhi[2] && blo[0] <= ahi[0] && blo[1] <= ahi[1] &&
              blo[2] <= ahi[2]))
            continue;
        d3 s[4], en[4];
        for (int k = 0; k < 4; ++k) s[k] = ld3(P.x, ids[k]), en[k] = ld3(P.ccd_x1, ids[k]);
        const int h = ccd::check_stencil(s, en, is_vt);
        if (h != ccd::HIT_NONE) {
            ++viol;
            cert += h == ccd::HIT_CERTAIN;
        }
    }
    const long long v = block_sum(viol), c = block_sum(cert);
    if (threadIdx.x == 0 && v) {
        atomicAdd(&P.g->ccd_violations, (int)v);
        atomicAdd(&P.g->ccd_certain, (int)c);
    }
}

__global__ void __launch_bounds__(TPB, 4) k_ccd(Params P) {
    ph_refit(P);
    STAGE_SYNC();
    ph_traverse(P);
    STAGE_SYNC();
    ph_ccd_eval(P);
}

// linearize_all on an uploaded pair set (tw_stage_linearize)
__global__ void __launch_bounds__(TPB, 4) k_stage_linearize(Params P) {
    if (!prologue(P)) return;  // edge-row list from is_er
    ph_stage_contact_flags(P);
    STAGE_SYNC();
    ph_rows(P);
    STAGE_SYNC();
    ph_rows_build(P, 0, 0, P.g->nc);
}

// color_constraints on uploaded rows (tw_stage_color): incidence, sorted
// vertex segments, then the reference replica or the device rounds
__global__ void __launch_bounds__(TPB, 4) k_stage_color(Params P, long long nc) {
    if (!prologue(P)) return;
    ph_stage_incidence(P, nc);
    STAGE_SYNC();
    ph_inc_totals(P);
    STAGE_SYNC();
    ph_inc_offsets(P);
    STAGE_SYNC();
    ph_inc_scatter(P, nc);
    STAGE_SYNC();
    ph_warm(P, nc);
    STAGE_SYNC();
    if (P.cfg.coloring_mode == 0) {
        ph_color_ref_count(P, nc);
        STAGE_SYNC();
        ph_color_ref_fill(P, nc);
        STAGE_SYNC();
        ph_color_ref(P, nc);
        return;
    }
    for (int k = 1; *((volatile int*)&P.g->colored) < nc; ++k) {
        if (k > 1) {
            ph_color_rank(P);
            STAGE_SYNC();
        }
        ph_color_propose(P, nc, k);
        STAGE_SYNC();
        ph_color_conflict(P, k);
        STAGE_SYNC();
        ph_color_commit(P, nc, k);
        STAGE_SYNC();
    }
}

// assemble_lcp + sweeps + recover_target on uploaded rows (tw_stage_backward);
// every row is handled as a contact row, y_out is written into P.x
// mode bits (TW_LCP_*): 1 assemble (q and the warm-start impulse; otherwise
// both are uploaded in c_q / imp), 2 solve (the sweeps), 4 recover (y into x).
__global__ void __launch_bounds__(TPB, 4) k_stage_backward(Params P, long long nc, int ncol, int mode) {
    if (mode & 1) ph_stage_q(P, nc);
    ph_stage_incidence(P, nc);
    STAGE_SYNC();
    ph_inc_totals(P);
    STAGE_SYNC();
    ph_inc_offsets(P);
    STAGE_SYNC();
    ph_inc_scatter(P, nc);
    STAGE_SYNC();
    if (mode & 1) {
        ph_warm(P, nc, false);
        STAGE_SYNC();
    }
    if (!(mode & 2)) {
    } else if (P.cfg.solver == 0) {
        ph_bucket_count(P, nc);
        STAGE_SYNC();
        ph_bucket_scatter(P, nc, ncol, false);
        STAGE_SYNC();
        ph_bucket_place(P, nc, false);
        STAGE_SYNC();
        for (int sw = 0; sw < P.cfg.sweeps; ++sw)
            for (int c = 0; c < ncol; ++c) {
                ph_pgs_color(P, c, ncol, 0, gridDim.x);
                STAGE_SYNC();
            }
    } else {
        for (int sw = 0; sw < P.cfg.sweeps; ++sw) {
            ph_jacobi_next(P, nc);
            STAGE_SYNC();
            ph_jacobi_apply(P, nc);
            STAGE_SYNC();
            ph_jacobi_commit(P, nc);
            STAGE_SYNC();
        }
    }
    // recover_target (lcp.cpp:131-136): dynamic y = y_k1 + impulse, static keep y_k1
    if (mode & 4)
    for (long long v = gtid(); v < P.nv; v += gstride()) {
        const double4 yk = P.yk1[v];
        const double4 a = P.imp[v];
        P.x[v] = P.inv_mass[v] > 0.0 ? make_double4(yk.x + a.x, yk.y + a.y, yk.z + a.z, yk.w) : yk;
    }
}

}  // namespace tw

// ==================================================== edge precoloring
namespace tw {

// One Jones-Plassmann round over the mesh edges (device-mode edge-row
// colors, computed once per mesh): same rule as the contact rows, priority
// edge_prio(e), conflicts through shared vertices with inv_mass > 0.
__global__ void k_edge_color_round(int ne, const int2* edges, const double* inv_mass, const int* vedge_off,
                                   const int* vedge, int* color, int* stamp, int round, int* colored) {
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < ne;
         t += (long long)gridDim.x * blockDim.x) {
        const int e = (int)t;
        if (stamp[e] != 0) continue;
        const int2 ed = edges[e];
        const int vv[2] = {ed.x, ed.y};
        const uint64_t pe = edge_prio(e);
        bool is_max = true;
        for (int k = 0; k < 2 && is_max; ++k) {
            const int v = vv[k];
            if (!(inv_mass[v] > 0.0)) continue;
            for (int q = vedge_off[v]; q < vedge_off[v + 1]; ++q) {
                const int f = vedge[q];
                if (f == e) continue;
                const int sf = *((volatile int*)&stamp[f]);
                if (sf != 0 && sf != round) continue;
                if (!jp_beats(pe, e, edge_prio(f), f)) {
                    is_max = false;
                    break;
                }
            }
        }
        if (!is_max) continue;
        unsigned long long used[4] = {0, 0, 0, 0};
        int big_min = 1 << 30;
        for (int k = 0; k < 2; ++k) {
            const int v = vv[k];
            if (!(inv_mass[v] > 0.0)) continue;
            for (int q = vedge_off[v]; q < vedge_off[v + 1]; ++q) {
                const int f = vedge[q];
                if (f == e) continue;
                const int sf = *((volatile int*)&stamp[f]);
                if (sf >= 1 && sf < round) {
                    const int c = color[f];
                    if (c < 256) used[c >> 6] |= 1ull << (c & 63);
                }
            }
        }
        int col = -1;
        for (int w = 0; w < 4 && col < 0; ++w)
            if (~used[w]) col = w * 64 + __ffsll(~used[w]) - 1;
        (void)big_min;
        color[e] = col < 0 ? 256 : col;  // > 256 edge colors: not reachable for manifold meshes
        stamp[e] = round;
        atomicAdd(colored, 1);
    }
}

static int g_last_launches = 0;
int launch_count_last() { return g_last_launches; }

static int grid_for(long long n, int tpb = 256) {
    long long b = (n + tpb - 1) / tpb;
    if (b < 1) b = 1;
    if (b > 148 * 8) b = 148 * 8;
    return (int)b;
}

void launch_setup(cudaStream_t s, int nv, const double* xs, const double* ys, const double* inv_mass,
                  double4* x, double4* yk1, double* r, unsigned long long* dmin, int* voff, int* vcnt,
                  double4* imp, int* nonfinite, int ne, const int2* edges, double* ly, uint8_t* is_er,
                  double* edge_lambda, int* er_color, const int* edge_color, int edge_rows,
                  int device_coloring) {
    g_last_launches = 0;
    if (nv > 0) {
        k_unpack<<<grid_for(nv), 256, 0, s>>>(nv, xs, ys, inv_mass, x, yk1, r, dmin, voff, vcnt, imp, nonfinite);
        ++g_last_launches;
    }
    if (ne > 0) {
        k_edges_init<<<grid_for(ne), 256, 0, s>>>(ne, edges, yk1, ly, is_er, edge_lambda, er_color, edge_color,
                                                  edge_rows, device_coloring);
        ++g_last_launches;
    }
}

void launch_pack(cudaStream_t s, int nv, const double4* x, double* out) {
    g_last_launches = 0;
    if (nv > 0) {
        k_pack<<<grid_for(nv), 256, 0, s>>>(nv, x, out);
        ++g_last_launches;
    }
}

size_t bvh_tmp_bytes(int n) {
    size_t cub_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const unsigned*)nullptr, (unsigned*)nullptr,
                                    (const int*)nullptr, (int*)nullptr, n < 1 ? 1 : n, 0, 30);
    const size_t arr = ((size_t)(n < 1 ? 1 : n) * 4 + 255) & ~(size_t)255;
    return cub_bytes + 4 * arr + 256;
}

void launch_bvh_build(cudaStream_t s, int cls, const Bvh& B, const int4* tris, const int2* edges, const int* iso,
                      const double4* x, int nv, void* tmp, size_t tmp_bytes, unsigned long long* box) {
    g_last_launches = 0;
    const int n = B.n;
    if (n == 0) return;
    const size_t arr = ((size_t)n * 4 + 255) & ~(size_t)255;
    char* base = (char*)tmp;
    unsigned* codes = (unsigned*)base;
    unsigned* codes2 = (unsigned*)(base + arr);
    int* idx = (int*)(base + 2 * arr);
    int* idx2 = (int*)(base + 3 * arr);
    void* cub_tmp = base + 4 * arr;
    size_t cub_bytes = tmp_bytes - 4 * arr - 256;
    k_morton<<<grid_for(n), 256, 0, s>>>(n, cls, tris, edges, iso, x, box, codes, idx);
    cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, codes, codes2, idx, idx2, n, 0, 30, s);
    k_karras<<<grid_for(n), 256, 0, s>>>(n, codes2, idx2, B.prim, B.child, B.parent, B.flag);
    g_last_launches = 3;
    (void)nv;
}

// Spread of the 32-query packets of a query class in two orders: the mesh
// numbering (identity) and Morton order (perm). spread[0] / spread[1] receive
// the sums over packets of the union-box extents (x + y + z); the broad phase
// hands out packets in the more compact order (query_at).
__global__ void k_packet_spread(int n, int cls, const int2* edges, const double4* x, const int* perm,
                                double* spread) {
    const int npk = (n + 31) / 32;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 2 * npk; t += gridDim.x * blockDim.x) {
        const int pk = t >> 1, ord = t & 1;
        float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
        for (int j = pk * 32; j < min(n, pk * 32 + 32); ++j) {
            const int q = ord ? perm[j] : j;
            double c[3];
            if (cls == 1) {
                const int2 e = edges[q];
                const double4 a = x[e.x], b = x[e.y];
                c[0] = 0.5 * (a.x + b.x), c[1] = 0.5 * (a.y + b.y), c[2] = 0.5 * (a.z + b.z);
            } else {
                const double4 a = x[q];
                c[0] = a.x, c[1] = a.y, c[2] = a.z;
            }
            for (int k = 0; k < 3; ++k) lo[k] = fminf(lo[k], (float)c[k]), hi[k] = fmaxf(hi[k], (float)c[k]);
        }
        atomicAdd(&spread[ord], (double)((hi[0] - lo[0]) + (hi[1] - lo[1]) + (hi[2] - lo[2])));
    }
}

void launch_packet_spread(cudaStream_t s, int n, int cls, const int2* edges, const double4* x, const int* perm,
                          double* spread) {
    if (n == 0) return;
    k_packet_spread<<<grid_for((n + 31) / 16), 256, 0, s>>>(n, cls, edges, x, perm, spread);
}

// vertices in Morton order: the order the broad phase hands vertex queries to
// warps (32 spatially compact queries per packet whatever the mesh numbering)
void launch_vertex_order(cudaStream_t s, int nv, const double4* x, void* tmp, size_t tmp_bytes,
                         unsigned long long* box, int* vperm) {
    g_last_launches = 0;
    if (nv == 0) return;
    const size_t arr = ((size_t)nv * 4 + 255) & ~(size_t)255;
    char* base = (char*)tmp;
    unsigned* codes = (unsigned*)base;
    unsigned* codes2 = (unsigned*)(base + arr);
    int* idx = (int*)(base + 2 * arr);
    void* cub_tmp = base + 4 * arr;
    size_t cub_bytes = tmp_bytes - 4 * arr - 256;
    k_morton<<<grid_for(nv), 256, 0, s>>>(nv, 3, nullptr, nullptr, nullptr, x, box, codes, idx);
    cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, codes, codes2, idx, vperm, nv, 0, 30, s);
    g_last_launches = 2;
}

void launch_bounds(cudaStream_t s, int nv, const double4* x, unsigned long long* box) {
    k_bounds<<<grid_for(nv), 256, 0, s>>>(nv, x, box);
}

static const void* resolve_fn(int minb) {
    if (minb >= 4) return (const void*)k_resolve<4>;
    if (minb == 3) return (const void*)k_resolve<3>;
    return (const void*)k_resolve<2>;
}

#ifndef TW_CARVEOUT
#define TW_CARVEOUT -1
#endif
// Shared-memory carveout of the resolve kernel (percent of the maximum; -1:
// the driver's choice). Env TW_CARVEOUT overrides.
static void set_carveout(const void* fn) {
    int pct = TW_CARVEOUT;
    if (const char* e = getenv("TW_CARVEOUT")) pct = atoi(e);
    if (pct >= 0) cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

int resolve_blocks_per_sm(int minb) {
    int b = 0;
    set_carveout(resolve_fn(minb));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, resolve_fn(minb), TPB, 0);
    return b;
}

static cudaError_t coop(const void* fn, cudaStream_t s, int nblocks, void** args) {
    return cudaLaunchCooperativeKernel(fn, dim3(nblocks), dim3(TPB), args, 0, s);
}

cudaError_t coop_resolve(cudaStream_t s, const Params& P, int nblocks, int minb) {
    // Preferred shared-memory carveout of the resolve kernel: 25% (57 KB
    // shared for 4 x 8.6 KB, the rest L1) measured 1.3% faster on the bow-knot
    // frame than the driver's choice (16%: same; 50%: -1.7%). TW_RESOLVE_CARVEOUT
    // overrides (-1: the driver's choice).
    static int carve = -2;
    if (carve == -2) {
        const char* e = std::getenv("TW_RESOLVE_CARVEOUT");
        carve = e ? std::atoi(e) : 25;
        if (carve >= 0)
            for (int mb : {2, 3, 4})
                cudaFuncSetAttribute(resolve_fn(mb), cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    }
    Params p = P;
    void* args[] = {&p};
    return coop(resolve_fn(minb), s, nblocks, args);
}
cudaError_t coop_search(cudaStream_t s, const Params& P, int nblocks) {
    Params p = P;
    void* args[] = {&p};
    return coop((const void*)k_stage_search, s, nblocks, args);
}
cudaError_t coop_refresh(cudaStream_t s, const Params& P, int nblocks, double bound) {
    Params p = P;
    double b = bound;
    void* args[] = {&p, &b};
    // TW_REFRESH_MINB=2: the 128-register instance (register-budget experiment)
    static const int minb = std::getenv("TW_REFRESH_MINB") ? std::atoi(std::getenv("TW_REFRESH_MINB")) : 4;
    if (minb == 2) return coop((const void*)k_stage_refresh<2>, s, std::min(nblocks, resolve_blocks_per_sm(2) * 148), args);
    if (minb == 3) return coop((const void*)k_stage_refresh<3>, s, std::min(nblocks, 3 * 148), args);
    return coop((const void*)k_stage_refresh<4>, s, nblocks, args);
}
cudaError_t coop_ccd(cudaStream_t s, const Params& P, int nblocks) {
    Params p = P;
    void* args[] = {&p};
    return coop((const void*)k_ccd, s, nblocks, args);
}
cudaError_t coop_stage_linearize(cudaStream_t s, const Params& P, int nblocks) {
    Params p = P;
    void* args[] = {&p};
    return coop((const void*)k_stage_linearize, s, nblocks, args);
}
cudaError_t coop_stage_color(cudaStream_t s, const Params& P, int nblocks, long long nc) {
    Params p = P;
    long long n = nc;
    void* args[] = {&p, &n};
    return coop((const void*)k_stage_color, s, nblocks, args);
}
cudaError_t coop_stage_backward(cudaStream_t s, const Params& P, int nblocks, long long nc, int ncol, int mode) {
    Params p = P;
    long long n = nc;
    int c = ncol, md = mode;
    void* args[] = {&p, &n, &c, &md};
    return coop((const void*)k_stage_backward, s, nblocks, args);
}
void launch_build_rows(cudaStream_t s, const double4* x, long long n, const int* kinds, const int* verts,
                       const double* closest, double delta, int gap, int* kind, int* nverts, int* rv, double* value,
                       double* jac, int* flavor, double* ref_volume, double* gw, double* denom) {
    if (n == 0) return;
    k_stage_build_rows<<<grid_for(n), 256, 0, s>>>(x, n, kinds, verts, closest, delta, gap, kind, nverts, rv, value,
                                                  jac, flavor, ref_volume, gw, denom);
}
void launch_value_at(cudaStream_t s, const double4* x, long long n, const int* flavor, const int* nverts,
                     const int* rv, const double* ref_volume, const double* gw, const double* denom,
                     const double* sigma, double* out) {
    if (n == 0) return;
    k_stage_value_at<<<grid_for(n), 256, 0, s>>>(x, n, flavor, nverts, rv, ref_volume, gw, denom, sigma, out);
}
void launch_fill_diag(cudaStream_t s, const double* inv_mass, long long n, const int* nverts, const int* rv,
                      const double* jac, double* diag) {
    if (n == 0) return;
    k_stage_fill_diag<<<grid_for(n), 256, 0, s>>>(inv_mass, n, nverts, rv, jac, diag);
}
cudaError_t launch_advance(cudaStream_t s, const Params& P, int nblocks) {
    double* md = nullptr;
    k_stage_advance<<<nblocks, TPB, 0, s>>>(P, md);
    return cudaGetLastError();
}
cudaError_t launch_closest(cudaStream_t s, int nv, const double4* x, long long n, const int* kinds, const int* verts,
                           double* out, int* has) {
    if (n == 0) return cudaSuccess;
    k_stage_closest<<<grid_for(n), 256, 0, s>>>(nv, x, n, kinds, verts, out, has);
    return cudaGetLastError();
}
void launch_edge_color_round(cudaStream_t s, int ne, const int2* edges, const double* inv_mass, const int* vedge_off,
                             const int* vedge, int* color, int* stamp, int round, int* colored) {
    k_edge_color_round<<<grid_for(ne), 256, 0, s>>>(ne, edges, inv_mass, vedge_off, vedge, color, stamp, round,
                                                   colored);
}

}  // namespace tw

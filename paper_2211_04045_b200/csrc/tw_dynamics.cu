// Device dynamics: the caller of the resolve path that defines a simulation
// step (proj/src/dynamics.cpp). One step (dynamics.cpp:326-349) runs, per
// Newton iteration,
//   proximity search at x (the device broad phase of the resolve path),
//   gradient_and_hessian (dynamics.cpp:111-168) + add_repulsion (170-202),
//   newton_target: block-Jacobi preconditioned CG (204-270),
//   resolve(x, y) (the device-resident Alg. 1),
// then the velocity update v = (x - x0)/dt (345-347); everything stays in HBM.
//
// The Hessian is never assembled. Its blocks are the reference's triplets:
//   vertex  dynamic: m/dt^2 I ; static: I                    (dynamics.cpp:118-127)
//   edge    K = k (u u^T + max(0, 1 - L0/l)(I - u u^T)) = a I + b u u^T on
//           (i,i) / (j,j) for dynamic rows, -K on (i,j) / (j,i) when both are
//           dynamic                                           (dynamics.cpp:130-150)
//   hinge   kb k_i k_j I for dynamic rows and columns         (dynamics.cpp:153-166)
//   pair    sw_a sw_b k dir dir^T on every vertex of a repulsive pair, static
//           ones included, as add_repulsion does              (dynamics.cpp:170-202)
// and H z is a per-vertex gather over the vertex's edges (mesh CSR, edge
// order), hinges (hinge order) and repulsive pair slots (a CSR rebuilt per
// Newton iteration, pair order): deterministic, no atomics. The gradient is
// gathered in the same orders, i.e. in the reference's accumulation order.
//
// The CG runs in one cooperative kernel with two grid barriers per iteration:
// phase A updates d, r, z = P r and the partial sums of r.r and r.z; phase B
// copies d to the best iterate when the residual improved, forms
// p = z + beta p and q = H p = H z + beta q (the recurrence saves the third
// barrier a fresh H p would need) and the partial sum of p.q. Block partials
// are summed by every CTA in the same fixed order, so all CTAs agree on
// alpha / beta / the exit test without another barrier.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <utility>
#include <vector>

#include "tw_ctx.h"
#include "tw_barrier.cuh"
#include "tw_math.cuh"

namespace tw {
namespace dyn {

constexpr int DTPB = 256;

struct Model {
    double k_spring, k_bend, grav[3], k_rep, r_rep, dt;
    double mu, pcg_tol;
    int pcg_max_iters;
};

struct DynGlobals {
    unsigned bar;
    char pad0[124];
    int error;
    int iters;
    int converged;
    int nrep;  // repulsive pairs of this Newton iteration
    double bnorm;
    double best_res;
    char pad1[88];
};

struct DynParams {
    int nv, ne, nh, nblocks;
    Model m;
    const double* inv_mass;
    const int2* edges;
    const int* vedge_off;
    const int* vedge;
    const double* rest;      // rest length per edge
    const int4* hv;          // hinge vertices
    const double4* hk;       // hinge coefficients
    const int* vh_off;       // vertex -> (hinge << 2 | slot), hinge order
    const int* vh;
    const double* x0;        // N x 3: positions at t (inertia target)
    const double* v0;        // N x 3: velocities at t
    const double* x;         // N x 3: current Newton point
    // per edge (this Newton iteration)
    double4* e_u;            // (u, k * strain); u = 0 for an inactive edge
    double2* e_ab;           // (a, b): K = a I + b u u^T (0, 0 inactive)
    // the same per vertex incidence (CSR order of vedge), written by k_grad_diag
    // so the CG's H z gathers one level shallower: (u, b), a, and the other end
    // (-1 when it is static: no z_o term; a = b = 0 for rows of static vertices)
    double4* inc_u;
    double* inc_a;
    int* inc_o;
    // repulsive pairs: compacted records and the vertex -> slot CSR
    const uint64_t* pkey;
    const int4* pids;
    const double4* pdd;
    const double4* pw;
    const uint8_t* pflag;
    long long np;
    int* rp_ids;             // 4 per repulsive pair (-1 padded)
    double* rp_sw;           // 4 signed weights per repulsive pair
    double4* rp_dir;         // (dir, depth)
    int* rp_count;           // [0]: repulsive pairs
    unsigned long long* rs_key;  // (vertex << 32 | pair << 2 | slot) per nonzero slot
    int* vr_off;             // vertex -> range in the sorted rs_key
    // per vertex
    double* sdiag;           // m/dt^2 (dynamic) or 1 (static)
    double4* grad;
    double* pre;             // 9 per vertex: inverse of the diagonal block (row-major)
    double4 *b, *d, *r, *z, *p, *q, *best;
    double* part;            // 2 per block
    DynGlobals* g;
};

__device__ __forceinline__ d3 ld3(const double* a, int v) { return mk(a[3 * v], a[3 * v + 1], a[3 * v + 2]); }
__device__ __forceinline__ d3 l4(const double4& a) { return mk(a.x, a.y, a.z); }
__device__ __forceinline__ double4 s4(d3 a, double w = 0.0) { return make_double4(a.x, a.y, a.z, w); }

// inertia target x^t + dt v^t + dt^2 g (dynamics.cpp:73-76)
__device__ __forceinline__ d3 inertia_target(const DynParams& P, int v) {
    const d3 g = mk(P.m.grav[0], P.m.grav[1], P.m.grav[2]);
    return add(add(ld3(P.x0, v), scl(P.m.dt, ld3(P.v0, v))), scl(P.m.dt * P.m.dt, g));
}

// ------------------------------------------------------------------ edges
// k * strain * u and the PSD-projected block of every edge at x
// (dynamics.cpp:130-150); both-static and zero-length edges are inactive.
__global__ void k_edges(DynParams P) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= P.ne) return;
    const int2 ij = P.edges[e];
    const bool si = P.inv_mass[ij.x] == 0.0, sj = P.inv_mass[ij.y] == 0.0;
    double4 u4 = make_double4(0, 0, 0, 0);
    double2 ab = make_double2(0, 0);
    if (!(si && sj)) {
        const d3 dd = sub(ld3(P.x, ij.x), ld3(P.x, ij.y));
        const double l = nrm(dd);
        if (!(l < 1e-12)) {
            const d3 u = dvd(dd, l);
            const double k = P.m.k_spring;
            const double strain = l - P.rest[e];
            const double c = maxd(0.0, 1.0 - P.rest[e] / l);
            u4 = s4(u, k * strain);
            ab = make_double2(k * c, k * (1.0 - c));  // K = k (c I + (1 - c) u u^T)
        }
    }
    P.e_u[e] = u4;
    P.e_ab[e] = ab;
}

// ------------------------------------------------------- repulsive pairs
// add_repulsion's pair filter (dynamics.cpp:176-181): active, not all-static,
// depth = r_rep - d > 0, nonzero direction. One record per pair, slots with a
// nonzero signed weight become CSR entries keyed (vertex, pair, slot).
__global__ void k_rep_pairs(DynParams P) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.np) return;
    const uint8_t fl = P.pflag[i];
    if (!(fl & 1) || (fl & 2)) return;
    const double4 dd = P.pdd[i];
    const double depth = P.m.r_rep - dd.w;
    if (!(depth > 0.0)) return;
    const d3 dir = l4(dd);
    if (is_zero(dir)) return;
    const uint64_t key = P.pkey[i];
    const int ka = key_ka(key), kb = key_kb(key);
    const int4 ids = P.pids[i];
    const double4 w = P.pw[i];
    int vid[4] = {-1, -1, -1, -1};
    double sw[4] = {0, 0, 0, 0};
    if (ka == KE) {  // EE: (a0, a1, b0, b1), weights (wa0, wa1, wb0, wb1)
        vid[0] = ids.x, vid[1] = ids.y, vid[2] = ids.z, vid[3] = ids.w;
        sw[0] = w.x, sw[1] = w.y, sw[2] = -w.z, sw[3] = -w.w;
    } else {  // vertex a (weight 1) against b = V / E / T
        vid[0] = ids.x, sw[0] = 1.0;
        const int nb = kb + 1;
        const int bid[3] = {ids.y, ids.z, ids.w};
        const double bw[3] = {w.x, w.y, w.z};
        for (int k = 0; k < nb; ++k) vid[1 + k] = bid[k], sw[1 + k] = -(kb == KV ? 1.0 : bw[k]);
    }
    atomicAdd(P.rp_count, 1);  // repulsive pairs (diagnostics)
    // records are indexed by pair index (sparse, only repulsive ones written);
    // the CSR keys carry the pair index so the gather runs in pair order
    for (int k = 0; k < 4; ++k) {
        P.rp_ids[4 * i + k] = vid[k];
        P.rp_sw[4 * i + k] = sw[k];
    }
    P.rp_dir[i] = s4(dir, depth);
    for (int k = 0; k < 4; ++k)
        if (vid[k] >= 0 && sw[k] != 0.0) {
            const unsigned long long e = ((unsigned long long)(unsigned)vid[k] << 32) | ((unsigned long long)i << 2) | k;
            P.rs_key[atomicAdd(P.rp_count + 1, 1)] = e;
        }
}

// vr_off[v] = first sorted entry of vertex v (lower bound), v in [0, nv]
__global__ void k_rep_offsets(const unsigned long long* keys, int n, int nv, int* off) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v > nv) return;
    int lo = 0, hi = n;
    const unsigned long long t = (unsigned long long)(unsigned)v << 32;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (keys[mid] < t) lo = mid + 1;
        else hi = mid;
    }
    off[v] = lo;
}

// ------------------------------------------------- gradient + diag block
// Gradient and the diagonal Hessian block of vertex v, gathered in the
// reference's accumulation order: inertia, edges (edge order), hinges (hinge
// order), repulsive pairs (pair order). The block is inverted for the 3x3
// block-Jacobi preconditioner (dynamics.cpp:218-235; a singular block keeps
// the identity, as a failed LDLT does).
__global__ void k_grad_diag(DynParams P) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= P.nv) return;
    const double im = P.inv_mass[v];
    const bool dyn = im != 0.0;
    const double inv_dt2 = 1.0 / (P.m.dt * P.m.dt);
    d3 g = mk(0, 0, 0);
    double B[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    double s = 1.0;
    if (dyn) {
        const double mass = 1.0 / im;
        s = mass * inv_dt2;
        g = scl(mass * inv_dt2, sub(ld3(P.x, v), inertia_target(P, v)));
    }
    B[0] = B[4] = B[8] = s;
    P.sdiag[v] = s;
    for (int k = P.vedge_off[v]; k < P.vedge_off[v + 1]; ++k) {  // incidence data for the CG
        const int e = P.vedge[k];
        const double4 u4 = P.e_u[e];
        const double2 ab = dyn ? P.e_ab[e] : make_double2(0.0, 0.0);
        const int2 ij = P.edges[e];
        const int o = ij.x == v ? ij.y : ij.x;
        P.inc_u[k] = make_double4(u4.x, u4.y, u4.z, ab.y);
        P.inc_a[k] = ab.x;
        P.inc_o[k] = P.inv_mass[o] != 0.0 ? o : -1;
    }
    if (dyn) {
        for (int k = P.vedge_off[v]; k < P.vedge_off[v + 1]; ++k) {
            const int e = P.vedge[k];
            const double4 u4 = P.e_u[e];
            const double2 ab = P.e_ab[e];
            if (ab.x == 0.0 && ab.y == 0.0 && u4.x == 0.0 && u4.y == 0.0 && u4.z == 0.0) continue;
            const d3 u = l4(u4);
            const d3 f = scl(u4.w, u);
            g = P.edges[e].x == v ? add(g, f) : sub(g, f);
            const double ul[3] = {u.x, u.y, u.z};
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) B[3 * r + c] += (r == c ? ab.x : 0.0) + ab.y * ul[r] * ul[c];
        }
        for (int k = P.vh_off[v]; k < P.vh_off[v + 1]; ++k) {
            const int h = P.vh[k] >> 2, i = P.vh[k] & 3;
            const int4 hv = P.hv[h];
            const double4 hk = P.hk[h];
            const int hvv[4] = {hv.x, hv.y, hv.z, hv.w};
            const double hkk[4] = {hk.x, hk.y, hk.z, hk.w};
            d3 c = mk(0, 0, 0);
            for (int j = 0; j < 4; ++j) c = add(c, scl(hkk[j], ld3(P.x, hvv[j])));
            g = add(g, scl(P.m.k_bend * hkk[i], c));
            const double w = P.m.k_bend * hkk[i] * hkk[i];
            B[0] += w, B[4] += w, B[8] += w;
        }
    }
    for (int k = P.vr_off[v]; k < P.vr_off[v + 1]; ++k) {
        const unsigned long long e = P.rs_key[k];
        const long long pi = (long long)((e & 0xffffffffull) >> 2);
        const int a = (int)(e & 3);
        const double4 dd = P.rp_dir[pi];
        const d3 dir = l4(dd);
        const double swa = P.rp_sw[4 * pi + a];
        const double kr = P.m.k_rep;
        g = add(g, scl(-kr * dd.w * swa, dir));
        const d3 gn = scl(kr, dir);
        const double dl[3] = {dir.x, dir.y, dir.z}, gl[3] = {gn.x, gn.y, gn.z};
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) B[3 * r + c] += swa * swa * (gl[r] * dl[c]);
    }
    P.grad[v] = s4(g);
    // inverse of the symmetric block (adjugate / determinant)
    const double c00 = B[4] * B[8] - B[5] * B[7], c01 = B[5] * B[6] - B[3] * B[8], c02 = B[3] * B[7] - B[4] * B[6];
    const double det = B[0] * c00 + B[1] * c01 + B[2] * c02;
    double* Pi = P.pre + 9 * (size_t)v;
    if (det > 0.0 && isfinite(det)) {
        const double id = 1.0 / det;
        Pi[0] = c00 * id;
        Pi[1] = (B[2] * B[7] - B[1] * B[8]) * id;
        Pi[2] = (B[1] * B[5] - B[2] * B[4]) * id;
        Pi[3] = c01 * id;
        Pi[4] = (B[0] * B[8] - B[2] * B[6]) * id;
        Pi[5] = (B[2] * B[3] - B[0] * B[5]) * id;
        Pi[6] = c02 * id;
        Pi[7] = (B[1] * B[6] - B[0] * B[7]) * id;
        Pi[8] = (B[0] * B[4] - B[1] * B[3]) * id;
    } else {
        for (int k = 0; k < 9; ++k) Pi[k] = (k % 4 == 0) ? 1.0 : 0.0;
    }
}

// ------------------------------------------------------------- operator
// (H z)_v: the row of vertex v of the implicit Hessian
__device__ __forceinline__ d3 hess_row(const DynParams& P, int v, const double4* z) {
    const bool dyn = P.inv_mass[v] != 0.0;
    const d3 zv = l4(z[v]);
    d3 out = scl(P.sdiag[v], zv);
    if (dyn) {
        // K z_v - K z_o per incident edge (the second only when the other end
        // is dynamic), added in incidence order; two incidences per round so
        // their loads and neighbour gathers overlap
        const int k1 = P.vedge_off[v + 1];
        int k = P.vedge_off[v];
        auto term = [&](double a, const double4& ub, int o, const d3& zo) {
            if (a == 0.0 && ub.w == 0.0) return;
            const d3 u = l4(ub);
            d3 t = zv;
            if (o >= 0) t = sub(zv, zo);
            out = add(out, add(scl(a, t), scl(ub.w * dot(u, t), u)));
        };
        for (; k + 1 < k1; k += 2) {
            const double a0 = P.inc_a[k], a1 = P.inc_a[k + 1];
            const double4 u0 = P.inc_u[k], u1 = P.inc_u[k + 1];
            const int o0 = P.inc_o[k], o1 = P.inc_o[k + 1];
            const d3 z0 = o0 >= 0 ? l4(z[o0]) : zv, z1 = o1 >= 0 ? l4(z[o1]) : zv;
            term(a0, u0, o0, z0);
            term(a1, u1, o1, z1);
        }
        if (k < k1) {
            const int o0 = P.inc_o[k];
            term(P.inc_a[k], P.inc_u[k], o0, o0 >= 0 ? l4(z[o0]) : zv);
        }
        for (int k = P.vh_off[v]; k < P.vh_off[v + 1]; ++k) {
            const int h = P.vh[k] >> 2, i = P.vh[k] & 3;
            const int4 hv = P.hv[h];
            const double4 hk = P.hk[h];
            const int hvv[4] = {hv.x, hv.y, hv.z, hv.w};
            const double hkk[4] = {hk.x, hk.y, hk.z, hk.w};
            for (int j = 0; j < 4; ++j)
                if (P.inv_mass[hvv[j]] != 0.0) out = add(out, scl(P.m.k_bend * hkk[i] * hkk[j], l4(z[hvv[j]])));
        }
    }
    for (int k = P.vr_off[v]; k < P.vr_off[v + 1]; ++k) {
        const unsigned long long e = P.rs_key[k];
        const long long pi = (long long)((e & 0xffffffffull) >> 2);
        const int a = (int)(e & 3);
        const d3 dir = l4(P.rp_dir[pi]);
        double s = 0.0;
        for (int b = 0; b < 4; ++b) {
            const int vb = P.rp_ids[4 * pi + b];
            const double swb = P.rp_sw[4 * pi + b];
            if (vb >= 0 && swb != 0.0) s += swb * dot(dir, l4(z[vb]));
        }
        out = add(out, scl(P.rp_sw[4 * pi + a] * P.m.k_rep * s, dir));
    }
    return out;
}

__device__ __forceinline__ d3 precond(const DynParams& P, int v, d3 r) {
    const double* Pi = P.pre + 9 * (size_t)v;
    return mk((Pi[0] * r.x + Pi[1] * r.y) + Pi[2] * r.z, (Pi[3] * r.x + Pi[4] * r.y) + Pi[5] * r.z,
              (Pi[6] * r.x + Pi[7] * r.y) + Pi[8] * r.z);
}

// ---------------------------------------------------- grid-wide helpers
__device__ __forceinline__ void dyn_sync(DynGlobals* g) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned old = bar_arrive(&g->bar, blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u);
        while (!bar_flipped(old, bar_poll_relaxed(&g->bar))) {
        }
        bar_acquire_fence();
    }
    __syncthreads();
}

// block sums of two values -> part[2 * block + {0, 1}]
template <int NT = DTPB>
__device__ __forceinline__ void block_partial2(double a, double b, double* part) {
    __shared__ double sa[NT / 32], sb[NT / 32];
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sa[w] = a, sb[w] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        double ta = 0.0, tb = 0.0;
        for (int i = 0; i < NT / 32; ++i) ta += sa[i], tb += sb[i];
        part[2 * blockIdx.x] = ta;
        part[2 * blockIdx.x + 1] = tb;
    }
    __syncthreads();
}

// every CTA sums the partials in the same order -> identical totals
__device__ __forceinline__ void grid_total2(const double* part, int nb, double* ta, double* tb) {
    __shared__ double ra, rb;
    if (threadIdx.x < 32) {
        double a = 0.0, b = 0.0;
        // L2 loads (the barrier's acquire ordered them after the writers);
        // one (a, b) pair per 16-byte load
        for (int i = threadIdx.x; i < nb; i += 32) {
            const double2 ab = __ldcg(reinterpret_cast<const double2*>(part) + i);
            a += ab.x, b += ab.y;
        }
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_down_sync(0xffffffffu, a, o);
            b += __shfl_down_sync(0xffffffffu, b, o);
        }
        if (threadIdx.x == 0) ra = a, rb = b;
    }
    __syncthreads();
    *ta = ra;
    *tb = rb;
    __syncthreads();
}

// ------------------------------------------------------------------ PCG
// newton_target's CG (dynamics.cpp:239-262) on b = -grad (static rows 0).
__global__ void __launch_bounds__(DTPB) k_pcg(DynParams P) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    // partial sums alternate between two buffers, so a CTA may write the next
    // phase's partials while a slower one still reads the previous ones: one
    // barrier per phase
    double* part[2] = {P.part, P.part + 2 * gridDim.x};
    int cur = 0;
    // init: b, r = b, z = P r, p = z, d = best = 0; sums r.z and b.b
    double rz_l = 0.0, bb_l = 0.0;
    for (int v = tid; v < P.nv; v += nth) {
        d3 bv = neg(l4(P.grad[v]));
        if (P.inv_mass[v] == 0.0) bv = mk(0, 0, 0);
        const d3 zv = precond(P, v, bv);
        P.b[v] = s4(bv);
        P.r[v] = s4(bv);
        P.z[v] = s4(zv);
        P.p[v] = s4(zv);
        P.d[v] = make_double4(0, 0, 0, 0);
        P.best[v] = make_double4(0, 0, 0, 0);
        rz_l += dot(bv, zv);
        bb_l += sqn(bv);
    }
    block_partial2(rz_l, bb_l, part[cur]);
    dyn_sync(P.g);
    double rz, bb;
    grid_total2(part[cur], gridDim.x, &rz, &bb);
    cur ^= 1;
    const double bnorm = sqrt(bb);
    double best_res = bnorm;
    // q = H p, p.q
    double pq_l = 0.0;
    for (int v = tid; v < P.nv; v += nth) {
        const d3 q = hess_row(P, v, P.p);
        P.q[v] = s4(q);
        pq_l += dot(l4(P.p[v]), q);
    }
    block_partial2(pq_l, 0.0, part[cur]);
    dyn_sync(P.g);
    int it = 0;
    const int maxit = P.m.pcg_max_iters;
    const double tol = P.m.pcg_tol;
    for (; it < maxit && best_res > tol * bnorm; ++it) {
        double pq, unused;
        grid_total2(part[cur], gridDim.x, &pq, &unused);
        cur ^= 1;
        if (pq <= 0.0) break;
        const double alpha = rz / pq;
        // phase A: d += alpha p; r -= alpha q; z = P r; sums r.r, r.z
        double rr_l = 0.0, rz_l2 = 0.0;
        for (int v = tid; v < P.nv; v += nth) {
            const d3 pv = l4(P.p[v]);
            const d3 dv = add(l4(P.d[v]), scl(alpha, pv));
            const d3 rv = sub(l4(P.r[v]), scl(alpha, l4(P.q[v])));
            const d3 zv = precond(P, v, rv);
            P.d[v] = s4(dv);
            P.r[v] = s4(rv);
            P.z[v] = s4(zv);
            rr_l += sqn(rv);
            rz_l2 += dot(rv, zv);
        }
        block_partial2(rr_l, rz_l2, part[cur]);
        dyn_sync(P.g);
        double rr, rzn;
        grid_total2(part[cur], gridDim.x, &rr, &rzn);
        cur ^= 1;
        const double res = sqrt(rr);
        const bool improved = res < best_res;
        if (improved) best_res = res;
        const double beta = rzn / rz;
        rz = rzn;
        // phase B: best = d (if improved); p = z + beta p; q = H z + beta q; sum p.q
        double pq_l2 = 0.0;
        for (int v = tid; v < P.nv; v += nth) {
            if (improved) P.best[v] = P.d[v];
            const d3 pv = add(l4(P.z[v]), scl(beta, l4(P.p[v])));
            const d3 qv = add(hess_row(P, v, P.z), scl(beta, l4(P.q[v])));
            P.p[v] = s4(pv);
            P.q[v] = s4(qv);
            pq_l2 += dot(pv, qv);
        }
        block_partial2(pq_l2, 0.0, part[cur]);
        dyn_sync(P.g);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.g->iters = it;
        P.g->converged = best_res <= tol * bnorm ? 1 : 0;
        P.g->bnorm = bnorm;
        P.g->best_res = best_res;
    }
}

// Register-resident CG: one vertex per thread (grid = ceil(nv / 256) CTAs,
// all co-resident), so d, r, p, q, best and the preconditioner block stay in
// registers across iterations and only z -- the operand of the neighbours'
// H z gathers -- goes through memory (L2-resident). Same phases, partial
// sums and exit logic as k_pcg; used whenever the grid fits on the device.
template <int NT, int VPT>
__global__ void __launch_bounds__(NT, VPT == 1 ? 2 : 1) k_pcg_reg(DynParams P) {
    // thread owns vertices (blockIdx.x * VPT + k) * NT + threadIdx.x, k < VPT
    double* part[2] = {P.part, P.part + 2 * gridDim.x};
    int cur = 0;
    int vv[VPT];
    bool own[VPT];
    d3 b[VPT], r[VPT], z[VPT], p[VPT], q[VPT], d[VPT], best[VPT];
    double pre[VPT][9];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        vv[k] = (blockIdx.x * VPT + k) * NT + threadIdx.x;
        own[k] = vv[k] < P.nv;
        b[k] = d[k] = best[k] = mk(0, 0, 0);
        if (own[k]) {
            for (int i = 0; i < 9; ++i) pre[k][i] = P.pre[9 * (size_t)vv[k] + i];
            if (P.inv_mass[vv[k]] != 0.0) b[k] = neg(l4(P.grad[vv[k]]));
        } else {
            for (int i = 0; i < 9; ++i) pre[k][i] = 0.0;
        }
    }
    auto pc = [&](int k, d3 x) {
        const double* m = pre[k];
        return mk((m[0] * x.x + m[1] * x.y) + m[2] * x.z, (m[3] * x.x + m[4] * x.y) + m[5] * x.z,
                  (m[6] * x.x + m[7] * x.y) + m[8] * x.z);
    };
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        r[k] = b[k];
        z[k] = own[k] ? pc(k, r[k]) : mk(0, 0, 0);
        p[k] = z[k];
        if (own[k]) {
            P.z[vv[k]] = s4(z[k]);
            s0 += dot(r[k], z[k]);
            s1 += sqn(b[k]);
        }
    }
    block_partial2<NT>(s0, s1, part[cur]);
    dyn_sync(P.g);
    double rz, bb;
    grid_total2(part[cur], gridDim.x, &rz, &bb);
    cur ^= 1;
    const double bnorm = sqrt(bb);
    double best_res = bnorm;
    s0 = 0.0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        q[k] = own[k] ? hess_row(P, vv[k], P.z) : mk(0, 0, 0);
        if (own[k]) s0 += dot(p[k], q[k]);
    }
    block_partial2<NT>(s0, 0.0, part[cur]);
    dyn_sync(P.g);
    int it = 0;
    const int maxit = P.m.pcg_max_iters;
    const double tol = P.m.pcg_tol;
    for (; it < maxit && best_res > tol * bnorm; ++it) {
        double pq, unused;
        grid_total2(part[cur], gridDim.x, &pq, &unused);
        cur ^= 1;
        if (pq <= 0.0) break;
        const double alpha = rz / pq;
        // phase A
        s0 = s1 = 0.0;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            d[k] = add(d[k], scl(alpha, p[k]));
            r[k] = sub(r[k], scl(alpha, q[k]));
            z[k] = own[k] ? pc(k, r[k]) : mk(0, 0, 0);
            if (own[k]) {
                P.z[vv[k]] = s4(z[k]);
                s0 += sqn(r[k]);
                s1 += dot(r[k], z[k]);
            }
        }
        block_partial2<NT>(s0, s1, part[cur]);
        dyn_sync(P.g);
        double rr, rzn;
        grid_total2(part[cur], gridDim.x, &rr, &rzn);
        cur ^= 1;
        const double res = sqrt(rr);
        const bool improved = res < best_res;
        if (improved) best_res = res;
        const double beta = rzn / rz;
        rz = rzn;
        // phase B
        s0 = 0.0;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            if (improved) best[k] = d[k];
            p[k] = add(z[k], scl(beta, p[k]));
            q[k] = own[k] ? add(hess_row(P, vv[k], P.z), scl(beta, q[k])) : mk(0, 0, 0);
            if (own[k]) s0 += dot(p[k], q[k]);
        }
        block_partial2<NT>(s0, 0.0, part[cur]);
        dyn_sync(P.g);
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k)
        if (own[k]) P.best[vv[k]] = s4(best[k]);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.g->iters = it;
        P.g->converged = best_res <= tol * bnorm ? 1 : 0;
        P.g->bnorm = bnorm;
        P.g->best_res = best_res;
    }
}

// y = x + best for dynamic vertices (dynamics.cpp:266-268)
__global__ void k_target(int nv, const double* inv_mass, const double* x, const double4* best, int converged_zero,
                         double* y) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    double3 o = make_double3(x[3 * v], x[3 * v + 1], x[3 * v + 2]);
    if (inv_mass[v] != 0.0 && !converged_zero) {
        const double4 b = best[v];
        o.x += b.x, o.y += b.y, o.z += b.z;
    }
    y[3 * v] = o.x, y[3 * v + 1] = o.y, y[3 * v + 2] = o.z;
}

// positions (N x 3) -> the resolve path's double4 (x, inv_mass) for the search
__global__ void k_pack_x4(int nv, const double* x, const double* inv_mass, double4* x4) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < nv) x4[v] = make_double4(x[3 * v], x[3 * v + 1], x[3 * v + 2], inv_mass[v]);
}

// v = (x - x0) / dt for dynamic vertices, 0 for static (dynamics.cpp:345-347)
__global__ void k_velocity(int nv, const double* inv_mass, const double* x, const double* x0, double dt, double* vel) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * nv) return;
    vel[i] = inv_mass[i / 3] == 0.0 ? 0.0 : (x[i] - x0[i]) / dt;
}

// ------------------------------------------------------- friction filter
// friction_filter (dynamics.cpp:272-324) is a Gauss-Seidel pass over the pair
// set in pair order: every pair reads y at its vertices and, when it
// penetrates the repulsion radius at that y, writes y back. In the sorted pair
// set nearly every pair shares a vertex with the one before it, so the pass is
// one long dependency chain -- but only the writers carry data along it (a
// pair that leaves y unchanged is invisible to the pairs after it). The device
// therefore runs it speculatively and verifies exactly:
//
//  1. every pair is evaluated at the input y0 in parallel; the ones that reach
//     the write (depth > 0, a normal, kappa > 0) form the writer set W;
//  2. the sequential pass is replayed over W alone as a dataflow (below),
//     logging every write as (vertex, pair, y after);
//  3. every pair outside W is re-evaluated at the state it would see in that
//     replay (per vertex, the last logged write of an earlier pair, else y0);
//     pairs that would write join W and the replay restarts from y0.
// When step 3 adds nothing, no pair outside W writes in the replay's
// history, so by induction over the pair order the full sequential pass
// visits exactly the states of the replay: the result is bit-identical.
//
// The replay is a dataflow over W's shared vertices: every (vertex, pair,
// slot) incidence sorted by vertex names the pair to wait for (pred, <= 4
// per pair); a pair runs once its predecessors have published their done
// flag (release store; relaxed polls and one fence) and touches only its own
// vertices. A vertex joins the order only when a write can change it:
// dynamic vertices, and static ones with a -0.0 coordinate (the write adds
// (dt * 0 * sw) * dv = +-0, which leaves every other bit pattern unchanged).
constexpr uint8_t FR_ALL_STATIC = 2;  // the pair flag bit PF_ALL_STATIC (tw_engine.cuh)

struct FrParams {
    long long np;
    double dt, mu, r_rep;
    const double* inv_mass;
    const double* x;        // N x 3: the Newton point
    double* y;              // N x 3: target in, filtered target out
    const double* y0;       // N x 3: the input target (replays restart from it)
    const uint64_t* pkey;
    const int4* pids;
    const double4* pdd;     // search direction at x (the fallback normal), distance
    const uint8_t* pflag;
    uint8_t* cand;          // per pair: in the writer set W
    unsigned long long* ent;  // (vertex << 32 | pair << 2 | slot)
    int* pred;              // 4 per pair: the pair to wait for at that slot, -1 none
    int* done;
    int* misc;              // [0] entries, [1] ticket, [2] |W|, [3] added to W, [4] log entries
    int* rank;              // per pair: its position among W's pairs (exclusive scan of cand)
    int* wlist;             // W's pairs in pair order
    int nw;
    unsigned long long* log_key;  // (vertex << 32 | pair) per logged write
    double4* log_val;             // y after that write
    const unsigned long long* slog_key;  // the log sorted by key, with the entry index
    const int* slog_idx;
    int nlog;
};

// the pair's vertex ids in the reference's vid order (a's, then b's; -1 padded)
__device__ __forceinline__ void fr_verts(int4 ids, int (&v)[4]) {
    v[0] = ids.x, v[1] = ids.y, v[2] = ids.z, v[3] = ids.w;
}

__device__ __forceinline__ bool fr_tracked(const FrParams& F, int v) {
    if (F.inv_mass[v] > 0.0) return true;
    const double* p = F.y0 + 3 * (size_t)v;  // static vertices: only the input can hold a -0.0
    return (p[0] == 0.0 && signbit(p[0])) || (p[1] == 0.0 && signbit(p[1])) || (p[2] == 0.0 && signbit(p[2]));
}

// The body of the reference loop for pair i (dynamics.cpp:278-318) at the
// state Y: false when the pair leaves y alone, else the signed weights and dv
// of its write (:320-321).
template <int KA, int KB, typename LoadY>
__device__ __forceinline__ bool fr_eval(const FrParams& F, long long i, const int (&vid)[4], const LoadY& Y,
                                        double (&sw)[4], d3& dv) {
    constexpr int m = (KA + 1) + (KB + 1);
    const int ia[3] = {vid[0], KA >= 1 ? vid[1] : -1, KA >= 2 ? vid[2] : -1};
    const int ib[3] = {vid[KA + 1], KB >= 1 ? vid[KA + 2] : -1, KB >= 2 ? vid[KA + 3] : -1};
    Closest res;
    closest_init(res);
    if (pair_closest_t<KA, KB>(ia, ib, Y, res) != 1) return false;  // penetration at the target state
    const double depth = F.r_rep - res.dist;
    if (depth <= 0.0) return false;
    d3 n = res.dir;
    if (is_zero(n)) {
        const double4 c = F.pdd[i];
        n = mk(c.x, c.y, c.z);
    }
    if (is_zero(n)) return false;
#pragma unroll
    for (int a = 0; a <= KA; ++a) sw[a] = res.wa[a];
#pragma unroll
    for (int b = 0; b <= KB; ++b) sw[KA + 1 + b] = -res.wb[b];
    double kappa = 0.0;
    d3 v_rel = mk(0, 0, 0);
#pragma unroll
    for (int a = 0; a < m; ++a) {
        const int v = vid[a];
        kappa += sw[a] * sw[a] * F.inv_mass[v];
        v_rel = add(v_rel, dvd(scl(sw[a], sub(Y(v), ld3(F.x, v))), F.dt));
    }
    if (kappa <= 0.0) return false;
    // inelastic normal impulse capped by the depth rate, Coulomb-capped tangential part
    const double vn = dot(v_rel, n);
    const double jn = clampd(-vn, 0.0, depth / F.dt);
    d3 impulse = scl(jn, n);
    const d3 vt = sub(v_rel, scl(vn, n));
    const double vt_norm = nrm(vt);
    if (vt_norm > 1e-12) {
        const double dvt = mind(F.mu * jn, vt_norm);
        impulse = sub(impulse, scl(dvt, dvd(vt, vt_norm)));
    }
    dv = dvd(impulse, kappa);
    return true;
}

template <typename F_>
__device__ __forceinline__ bool fr_class(uint64_t key, F_&& f) {
    return with_pair_class(key_ka(key), key_kb(key), f);
}

// 1. W = the pairs that write at y0
__global__ void k_fr_eval0(FrParams F) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= F.np) return;
    bool w = false;
    if (!(F.pflag[i] & FR_ALL_STATIC)) {  // dynamics.cpp:278
        const uint64_t key = F.pkey[i];
        int vid[4];
        fr_verts(F.pids[i], vid);
        auto Y = [&](int v) { return ld3(F.y0, v); };
        fr_class(key, [&](auto c) {
            double sw[4];
            d3 dv;
            w = fr_eval<decltype(c)::ka, decltype(c)::kb>(F, i, vid, Y, sw, dv);
        });
    }
    F.cand[i] = w;
    if (w) atomicAdd(F.misc + 2, 1);
}

// 2a. dependency order of W (pred reset for every pair)
__global__ void k_fr_entries(FrParams F) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= F.np) return;
    reinterpret_cast<int4*>(F.pred)[i] = make_int4(-1, -1, -1, -1);
    F.done[i] = 0;
    if (!F.cand[i]) return;
    const uint64_t key = F.pkey[i];
    int v[4];
    fr_verts(F.pids[i], v);
    const int n = (key_ka(key) + 1) + (key_kb(key) + 1);
    for (int k = 0; k < n; ++k)
        if (fr_tracked(F, v[k]))
            F.ent[atomicAdd(F.misc, 1)] = ((unsigned long long)(unsigned)v[k] << 32) | ((unsigned long long)i << 2) | k;
}

__global__ void k_fr_pred(FrParams F, int n) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n || j == 0) return;
    const unsigned long long e = F.ent[j], p = F.ent[j - 1];
    if ((e >> 32) == (p >> 32)) F.pred[(e & 0xffffffffu)] = (int)((p & 0xffffffffu) >> 2);
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// y is written by other CTAs during the replay: read it at L2 (never a stale L1 line)
__device__ __forceinline__ d3 ldy(const double* y, int v) {
    return mk(__ldcg(y + 3 * v), __ldcg(y + 3 * v + 1), __ldcg(y + 3 * v + 2));
}

template <int KA, int KB>
__device__ __forceinline__ void fr_apply(const FrParams& F, long long i, const int (&vid)[4]) {
    constexpr int m = (KA + 1) + (KB + 1);
    double sw[4];
    d3 dv;
    auto Y = [&](int v) { return ldy(F.y, v); };
    if (!fr_eval<KA, KB>(F, i, vid, Y, sw, dv)) return;
#pragma unroll
    for (int a = 0; a < m; ++a) {
        const int v = vid[a];
        if (!fr_tracked(F, v)) continue;  // a +-0 write to an unchanged static vertex
        const d3 o = add(ldy(F.y, v), scl(F.dt * F.inv_mass[v] * sw[a], dv));
        __stcg(F.y + 3 * v, o.x), __stcg(F.y + 3 * v + 1, o.y), __stcg(F.y + 3 * v + 2, o.z);
        if (F.log_key) {
            const int e = atomicAdd(F.misc + 4, 1);
            F.log_key[e] = ((unsigned long long)(unsigned)v << 32) | (unsigned long long)i;
            F.log_val[e] = make_double4(o.x, o.y, o.z, 0.0);
        }
    }
}

__global__ void k_fr_compact(FrParams F) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < F.np && F.cand[i]) F.wlist[F.rank[i]] = (int)i;
}

// 2b. the replay over W (compacted: a warp holds 32 consecutive pairs of W,
// which mostly chain through their shared query vertex). Warps take them from
// a ticket counter in pair order, so the earliest unfinished pair of W always
// belongs to a running warp whose predecessors are all finished: the pass
// cannot stall. A predecessor in the same warp is waited for through the
// warp's done ballot (its writes are ordered by __syncwarp, y at L2); one in
// another warp through its done flag.
__global__ void __launch_bounds__(DTPB) k_friction(FrParams F) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(F.misc + 1, 32);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= F.nw) return;
        const int t = base + lane;
        bool fin = t >= F.nw;
        long long i = 0;
        int pq[4] = {-1, -1, -1, -1};  // >= 0: pair index (another warp); <= -2: -2 - lane (this warp)
        uint64_t key = 0;
        int vid[4] = {-1, -1, -1, -1};
        if (!fin) {
            i = F.wlist[t];
            const int4 pr = reinterpret_cast<const int4*>(F.pred)[i];
            const int pp[4] = {pr.x, pr.y, pr.z, pr.w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (pp[k] >= 0) {
                    const int r = F.rank[pp[k]];
                    pq[k] = r >= base ? -2 - (r - base) : pp[k];
                }
            key = F.pkey[i];
            fr_verts(F.pids[i], vid);
        }
        for (;;) {
            __syncwarp();
            const unsigned donem = __ballot_sync(0xffffffffu, fin);
            if (donem == 0xffffffffu) break;
            if (!fin) {
                bool ready = true, remote = false;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (pq[k] <= -2) ready = ready && ((donem >> (-2 - pq[k])) & 1u);
                    else if (pq[k] >= 0) ready = ready && ld_relaxed(F.done + pq[k]), remote = true;
                }
                if (ready) {
                    if (remote) asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    fr_class(key, [&](auto c) { fr_apply<decltype(c)::ka, decltype(c)::kb>(F, i, vid); });
                    st_release(F.done + i, 1);
                    fin = true;
                }
            }
        }
    }
}

// every pair that is not all-static joins W (the plain dataflow: no verification needed)
__global__ void k_fr_all(FrParams F) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < F.np) F.cand[i] = !(F.pflag[i] & FR_ALL_STATIC);
}

__global__ void k_iota(int* a, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

// the state pair i sees at vertex v in the replay: the last logged write of
// an earlier pair, else the input
__device__ __forceinline__ d3 fr_state(const FrParams& F, int v, long long i) {
    const unsigned long long t = ((unsigned long long)(unsigned)v << 32) | (unsigned long long)i;
    int lo = 0, hi = F.nlog;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (F.slog_key[mid] < t) lo = mid + 1;
        else hi = mid;
    }
    if (lo > 0 && (F.slog_key[lo - 1] >> 32) == (unsigned long long)(unsigned)v) {
        const double4 o = F.log_val[F.slog_idx[lo - 1]];
        return mk(o.x, o.y, o.z);
    }
    return ld3(F.y0, v);
}

// 3. pairs outside W that would write in the replay's history join W
__global__ void k_fr_verify(FrParams F) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= F.np || F.cand[i] || (F.pflag[i] & FR_ALL_STATIC)) return;
    const uint64_t key = F.pkey[i];
    int vid[4];
    fr_verts(F.pids[i], vid);
    auto Y = [&](int v) { return fr_state(F, v, i); };
    bool w = false;
    fr_class(key, [&](auto c) {
        double sw[4];
        d3 dv;
        w = fr_eval<decltype(c)::ka, decltype(c)::kb>(F, i, vid, Y, sw, dv);
    });
    if (w) {
        F.cand[i] = 1;
        atomicAdd(F.misc + 3, 1);
    }
}

// ---------------------------------------------------------- normal flow
// normal_flow_target (normal_flow.cpp:38-81): area-weighted unit normals
// (per-vertex gather over the incident triangles in triangle order), the
// offset y = x + beta n, cotangent edge weights (per edge over its triangles
// in triangle order), then three Jacobi smoothing passes whose per-vertex sums
// run over the neighbours in ascending id -- the iteration order of the
// reference's std::map keyed (min, max).
__global__ void k_nf_offset(int nv, const double* x, const int* vt_off, const int* vt, const int4* tris, double beta,
                            double* y) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    d3 n = mk(0, 0, 0);
    for (int k = vt_off[v]; k < vt_off[v + 1]; ++k) {
        const int4 t = tris[vt[k]];
        const d3 p0 = ld3(x, t.x);
        n = add(n, scl(0.5, crs(sub(ld3(x, t.y), p0), sub(ld3(x, t.z), p0))));
    }
    const double l = nrm(n);
    if (l > 1e-18) n = dvd(n, l);
    const d3 o = add(ld3(x, v), scl(beta, n));
    y[3 * v] = o.x, y[3 * v + 1] = o.y, y[3 * v + 2] = o.z;
}

// w_e = sum over the (t, k) occurrences of the edge of 0.5 cot(angle at the opposite corner)
__global__ void k_nf_weights(int ne, const int* occ_off, const int* occ, const int4* tris, const double* y, double* w) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    double acc = 0.0;
    for (int k = occ_off[e]; k < occ_off[e + 1]; ++k) {
        const int4 t4 = tris[occ[k] >> 2];
        const int c = occ[k] & 3;
        const int tv[3] = {t4.x, t4.y, t4.z};
        const int a = tv[c], b = tv[(c + 1) % 3], o = tv[(c + 2) % 3];
        const d3 u = sub(ld3(y, a), ld3(y, o)), q = sub(ld3(y, b), ld3(y, o));
        const double cr = nrm(crs(u, q));
        acc += 0.5 * (dot(u, q) / maxd(cr, 1e-18));
    }
    w[e] = acc;
}

__global__ void k_nf_smooth(int nv, const int* nb_off, const int2* nb, const double* w, double alpha, const double* y,
                            double* y_next) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const d3 yv = ld3(y, v);
    d3 lap = mk(0, 0, 0);
    double ws = 0.0;
    for (int k = nb_off[v]; k < nb_off[v + 1]; ++k) {
        const int2 n = nb[k];  // (neighbour, edge)
        const double we = maxd(w[n.y], 1e-6);
        lap = add(lap, scl(we, sub(ld3(y, n.x), yv)));
        ws += we;
    }
    d3 o = yv;
    if (ws > 0.0) o = add(yv, dvd(scl(alpha, lap), ws));
    y_next[3 * v] = o.x, y_next[3 * v + 1] = o.y, y_next[3 * v + 2] = o.z;
}

}  // namespace dyn
}  // namespace tw

using namespace tw;
using namespace tw::dyn;
using namespace tw::host;

// --------------------------------------------------------------- C-ABI
struct tw_dyn {
    tw_ctx* ctx = nullptr;
    tw_mesh* mesh = nullptr;
    tw_energy_model model{};
    int nh = 0;
    DevMem rest, hv, hk, vh_off, vh;
    DevMem inc_u, inc_a, inc_o, hx, hvel, x0, v0, xk, y, e_u, e_ab, rp_ids, rp_sw, rp_dir, rp_count, rs_key, rs_key2, vr_off, sort_tmp;
    DevMem sdiag, grad, pre, b, d, r, z, p, q, best, part, glob;
    DevMem fr_pred, fr_done, fr_misc, fr_cand, fr_y0;  // friction_filter replay state
    DevMem fr_log_key, fr_log_key2, fr_log_val, fr_log_idx, fr_log_idx2, fr_rank, fr_wlist;
    long long rp_cap = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // step timing (the resolve uses the context's own events)
    cudaEvent_t evt0 = nullptr, evp0 = nullptr, evp1 = nullptr;  // target / PCG timing
    cudaEvent_t evf0 = nullptr, evf1 = nullptr;                  // friction_filter timing
};

namespace {

bool model_valid(const tw_energy_model& m) {  // EnergyModel::validate, dynamics.cpp:10-15
    if (m.spring_stiffness < 0.0 || m.bending_stiffness < 0.0 || m.repulsion_stiffness < 0.0) return false;
    if (!(m.dt > 0.0)) return false;
    if (m.newton_iters < 1) return false;
    if (m.mu < 0.0) return false;
    return true;
}

// Flat-rest hinge coefficients (dynamics.cpp:26-68): for every interior edge
// with exactly two incident triangles, the unit null vector of
// [1 1 1 1; in-plane rest coordinates of the 4 stencil vertices]. The null
// vector of a rank-3 3x4 matrix is its generalized cross product (signed 3x3
// minors); its sign is irrelevant (the energy is quadratic in it).
void build_hinges(const tw_mesh* m, const std::vector<int32_t>& tris, const double* X, std::vector<int>& hv,
                  std::vector<double>& hk) {
    std::vector<std::pair<uint64_t, int>> et;  // (edge key, triangle)
    const int nt = (int)tris.size() / 3;
    et.reserve(3 * (size_t)nt);
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) {
            const int a = tris[3 * t + k], b = tris[3 * t + (k + 1) % 3];
            et.push_back({((uint64_t)(uint32_t)std::min(a, b) << 32) | (uint32_t)std::max(a, b), t});
        }
    std::stable_sort(et.begin(), et.end(), [](auto& p, auto& q) { return p.first < q.first; });
    auto P = [&](int v) { return mk(X[3 * v], X[3 * v + 1], X[3 * v + 2]); };
    for (size_t i = 0; i < et.size();) {
        size_t j = i;
        while (j < et.size() && et[j].first == et[i].first) ++j;
        if (j - i == 2) {
            const int e0 = (int)(et[i].first >> 32), e1 = (int)(et[i].first & 0xffffffffu);
            auto opposite = [&](int t) {
                for (int k = 0; k < 3; ++k) {
                    const int v = tris[3 * t + k];
                    if (v != e0 && v != e1) return v;
                }
                return -1;
            };
            const int v[4] = {e0, e1, opposite(et[i].second), opposite(et[i + 1].second)};
            const d3 x0 = P(v[0]), e1v = sub(P(v[1]), x0);
            d3 n = crs(e1v, sub(P(v[2]), x0));
            if (!(sqn(n) < 1e-24 || sqn(e1v) < 1e-24)) {
                n = normalized(n);
                const d3 bu = normalized(e1v), bv = crs(n, bu);
                double M[3][4];
                for (int c = 0; c < 4; ++c) {
                    const d3 d = sub(P(v[c]), x0);
                    M[0][c] = 1.0, M[1][c] = dot(d, bu), M[2][c] = dot(d, bv);
                }
                auto minor = [&](int skip) {
                    int cols[3], q = 0;
                    for (int c = 0; c < 4; ++c)
                        if (c != skip) cols[q++] = c;
                    const double(*A)[4] = M;
                    return A[0][cols[0]] * (A[1][cols[1]] * A[2][cols[2]] - A[1][cols[2]] * A[2][cols[1]]) -
                           A[0][cols[1]] * (A[1][cols[0]] * A[2][cols[2]] - A[1][cols[2]] * A[2][cols[0]]) +
                           A[0][cols[2]] * (A[1][cols[0]] * A[2][cols[1]] - A[1][cols[1]] * A[2][cols[0]]);
                };
                double k[4] = {minor(0), -minor(1), minor(2), -minor(3)};
                double scale = 0.0, kn = 0.0;
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 4; ++c) scale = std::max(scale, std::fabs(M[r][c]));
                for (int c = 0; c < 4; ++c) kn += k[c] * k[c];
                kn = std::sqrt(kn);
                // rank 3 at the reference's 1e-9 relative LU threshold
                if (kn > 1e-9 * scale * scale * scale) {
                    for (int c = 0; c < 4; ++c) hv.push_back(v[c]), hk.push_back(k[c] / kn);
                }
            }
        }
        i = j;
    }
}

template <typename T>
cudaError_t upload(DevMem& d, const std::vector<T>& h) {
    cudaError_t e = d.ensure(std::max<size_t>(16, h.size() * sizeof(T)));
    if (e == cudaSuccess && !h.empty()) e = cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

DynParams make_dparams(tw_dyn* D, const double* d_x) {
    tw_ctx* ctx = D->ctx;
    tw_mesh* m = D->mesh;
    DynParams P;
    std::memset(&P, 0, sizeof P);
    P.nv = m->nv, P.ne = m->ne, P.nh = D->nh;
    P.nblocks = 0;
    const tw_energy_model& em = D->model;
    P.m.k_spring = em.spring_stiffness, P.m.k_bend = em.bending_stiffness;
    for (int k = 0; k < 3; ++k) P.m.grav[k] = em.gravity[k];
    P.m.k_rep = em.repulsion_stiffness, P.m.r_rep = em.repulsion_radius, P.m.dt = em.dt;
    P.m.mu = em.mu, P.m.pcg_tol = em.pcg_tol, P.m.pcg_max_iters = em.pcg_max_iters;
    P.inv_mass = m->d_inv_mass.as<double>();
    P.edges = m->d_edges.as<int2>();
    P.vedge_off = m->d_vedge_off.as<int>();
    P.vedge = m->d_vedge.as<int>();
    P.rest = D->rest.as<double>();
    P.hv = D->hv.as<int4>();
    P.hk = D->hk.as<double4>();
    P.vh_off = D->vh_off.as<int>();
    P.vh = D->vh.as<int>();
    P.x0 = D->x0.as<double>();
    P.v0 = D->v0.as<double>();
    P.x = d_x;
    P.e_u = D->e_u.as<double4>();
    P.e_ab = D->e_ab.as<double2>();
    P.inc_u = D->inc_u.as<double4>();
    P.inc_a = D->inc_a.as<double>();
    P.inc_o = D->inc_o.as<int>();
    P.pkey = ctx->pkey.as<uint64_t>();
    P.pids = ctx->pids.as<int4>();
    P.pdd = ctx->pdd.as<double4>();
    P.pw = ctx->pw.as<double4>();
    P.pflag = ctx->pflag.as<uint8_t>();
    P.rp_ids = D->rp_ids.as<int>();
    P.rp_sw = D->rp_sw.as<double>();
    P.rp_dir = D->rp_dir.as<double4>();
    P.rp_count = D->rp_count.as<int>();
    P.rs_key = D->rs_key.as<unsigned long long>();
    P.vr_off = D->vr_off.as<int>();
    P.sdiag = D->sdiag.as<double>();
    P.grad = D->grad.as<double4>();
    P.pre = D->pre.as<double>();
    P.b = D->b.as<double4>(), P.d = D->d.as<double4>(), P.r = D->r.as<double4>(), P.z = D->z.as<double4>();
    P.p = D->p.as<double4>(), P.q = D->q.as<double4>(), P.best = D->best.as<double4>();
    P.part = D->part.as<double>();
    P.g = D->glob.as<DynGlobals>();
    return P;
}

// TW_DEBUG_SYNC=1: synchronize after every dynamics launch and name the failing one
int debug_sync(tw_ctx* ctx, const char* what) {
    static const bool on = getenv("TW_DEBUG_SYNC") != nullptr;
    if (!on) return TW_OK;
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, what);
    return TW_OK;
}
#define DSYNC(name)                               \
    do {                                          \
        const int _r = debug_sync(ctx, name);     \
        if (_r) return _r;                        \
    } while (0)

int pcg_blocks(tw_ctx* ctx, int nv) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg, DTPB, 0);
    per_sm = std::max(1, std::min(per_sm, 4));
    const int want = (nv + DTPB - 1) / DTPB;
    return std::max(1, std::min(ctx->sm_count * per_sm, want));
}

// Runs the proximity search of the resolve path at ctx->x (double4) with
// capacity regrowth; leaves the pair set in the context's pair buffers.
int search_at_x(tw_ctx* ctx, tw_mesh* m, double d_max, long long* np) {
    tw_resolve_config cfg;
    tw_default_config(&cfg);
    cfg.d_max = d_max;
    cfg.step_limit = 1;
    Globals G;
    for (int attempt = 0;; ++attempt) {
        int rc = ensure_buffers(ctx, m, cfg);
        if (rc) return rc;
        Params P = make_params(ctx, m, cfg);
        CK(cudaMemsetAsync(ctx->globals.p, 0, sizeof(Globals), ctx->stream));
        CK(cudaMemsetAsync(ctx->dmin.p, 0x7f, (size_t)m->nv * 8, ctx->stream));
        rc = build_bvhs(ctx, m);
        if (rc) return rc;
        CK(coop_search(ctx->stream, P, ctx->nblocks));
        ++ctx->launches;
        CK(cudaMemcpyAsync(&G, ctx->globals.p, sizeof G, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (G.error & ERR_TIMEOUT) return fail(ctx, TW_ETIMEOUT, "search: watchdog");
        if (!(G.error & (ERR_CAP_SLOTS | ERR_CAP_PAIRS | ERR_CAP_CAND))) break;
        if (attempt > 10) return fail(ctx, TW_ECAPACITY, "search: capacity");
        if (G.error & ERR_CAP_SLOTS) ctx->K = std::max(ctx->K * 2, ((G.needed_k + 31) / 32) * 32);
        if (G.error & ERR_CAP_PAIRS) grow_ll(ctx->pcap, G.needed_pairs + G.needed_pairs / 4);
        if (G.error & ERR_CAP_CAND) grow_ll(ctx->ccap, (long long)G.ncand + (long long)G.ncand / 4);
    }
    *np = G.np;
    return TW_OK;
}

// friction_filter (dynamics.cpp:272-324) on d_y (N x 3, in place) with the
// pair set the context holds from the search at d_xk (np pairs, key order):
// the writer-set speculation of k_fr_eval0 / k_friction / k_fr_verify.
struct ScanAdd {
    __device__ __forceinline__ int operator()(int a, int b) const { return a + b; }
};

template <typename K>
cudaError_t sort_keys(tw_dyn* D, K* in, K* out, int n, cudaStream_t s) {
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, in, out, n, 0, 64, s);
    cudaError_t e = D->sort_tmp.ensure(tb);
    if (e == cudaSuccess) e = cub::DeviceRadixSort::SortKeys(D->sort_tmp.p, tb, in, out, n, 0, 64, s);
    return e;
}

int friction_device(tw_dyn* D, const double* d_xk, double* d_y, long long np) {
    tw_ctx* ctx = D->ctx;
    tw_mesh* m = D->mesh;
    cudaStream_t s = ctx->stream;
    if (np <= 0) return TW_OK;
    if (np >= (1ll << 30)) return fail(ctx, TW_ECAPACITY, "friction_filter: too many pairs");
    const size_t nv = (size_t)std::max(1, m->nv);
    CK(D->fr_pred.ensure((size_t)np * 16));
    CK(D->fr_done.ensure((size_t)np * 4));
    CK(D->fr_cand.ensure((size_t)np));
    CK(D->fr_rank.ensure((size_t)np * 4));
    CK(D->fr_wlist.ensure((size_t)np * 4));
    CK(D->fr_misc.ensure(32));
    CK(D->fr_y0.ensure(nv * 24));
    CK(cudaMemcpyAsync(D->fr_y0.p, d_y, (size_t)m->nv * 24, cudaMemcpyDeviceToDevice, s));
    FrParams F;
    std::memset(&F, 0, sizeof F);
    F.np = np, F.dt = D->model.dt, F.mu = D->model.mu, F.r_rep = D->model.repulsion_radius;
    F.inv_mass = m->d_inv_mass.as<double>();
    F.x = d_xk, F.y = d_y, F.y0 = D->fr_y0.as<double>();
    F.pkey = ctx->pkey.as<uint64_t>();
    F.pids = ctx->pids.as<int4>();
    F.pdd = ctx->pdd.as<double4>();
    F.pflag = ctx->pflag.as<uint8_t>();
    F.cand = D->fr_cand.as<uint8_t>();
    F.pred = D->fr_pred.as<int>();
    F.done = D->fr_done.as<int>();
    F.misc = D->fr_misc.as<int>();
    const unsigned pb = (unsigned)((np + DTPB - 1) / DTPB);
    CK(cudaMemsetAsync(D->fr_misc.p, 0, 32, s));
    k_fr_eval0<<<pb, DTPB, 0, s>>>(F);
    ++ctx->launches;
    DSYNC("k_fr_eval0");
    static int occ = -1;
    if (occ < 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_friction, DTPB, 0);
    int misc[8];
    CK(cudaMemcpyAsync(misc, D->fr_misc.p, 32, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // A cascade (a write pushes the next pair into the radius, whose write
    // pushes the next ...) adds few pairs per round; after kMaxRounds the
    // replay runs over every pair instead, which needs no verification.
    static const int kMaxRounds = getenv("TW_FR_MAX_ROUNDS") ? std::atoi(getenv("TW_FR_MAX_ROUNDS")) : 8;
    bool all = false;
    for (int round = 0;; ++round) {
        if (round == kMaxRounds) {
            k_fr_all<<<pb, DTPB, 0, s>>>(F);
            ++ctx->launches;
            all = true;
            misc[2] = (int)std::min<long long>(np, 0x7fffffff);
        }
        const long long nw = misc[2];  // |W|
        if (nw == 0) return TW_OK;     // nothing writes at y0 and (verified) nothing after
        // buffers sized by |W|: <= 4 incidences and <= 4 logged writes per pair
        CK(D->rs_key.ensure((size_t)nw * 4 * 8));
        CK(D->rs_key2.ensure((size_t)nw * 4 * 8));
        F.ent = D->rs_key.as<unsigned long long>();
        if (!all) {  // the write log (the full replay needs none)
            CK(D->fr_log_key.ensure((size_t)nw * 4 * 8));
            CK(D->fr_log_key2.ensure((size_t)nw * 4 * 8));
            CK(D->fr_log_val.ensure((size_t)nw * 4 * 32));
            CK(D->fr_log_idx.ensure((size_t)nw * 4 * 4));
            CK(D->fr_log_idx2.ensure((size_t)nw * 4 * 4));
            F.log_key = D->fr_log_key.as<unsigned long long>();
            F.log_val = D->fr_log_val.as<double4>();
        } else {
            F.log_key = nullptr;
        }
        if (round) CK(cudaMemcpyAsync(d_y, D->fr_y0.p, (size_t)m->nv * 24, cudaMemcpyDeviceToDevice, s));
        // misc[0] entries, [1] ticket, [3] added, [4] log entries restart; [2] = |W| stays
        CK(cudaMemsetAsync(F.misc, 0, 8, s));
        CK(cudaMemsetAsync(F.misc + 3, 0, 8, s));
        k_fr_entries<<<pb, DTPB, 0, s>>>(F);
        ++ctx->launches;
        DSYNC("k_fr_entries");
        CK(cudaMemcpyAsync(misc, D->fr_misc.p, 32, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int nent = misc[0];
        if (nent > 1) {
            CK(sort_keys(D, D->rs_key.as<unsigned long long>(), D->rs_key2.as<unsigned long long>(), nent, s));
            ctx->launches += 4;
            F.ent = D->rs_key2.as<unsigned long long>();
            k_fr_pred<<<(nent + DTPB - 1) / DTPB, DTPB, 0, s>>>(F, nent);
            ++ctx->launches;
            DSYNC("k_fr_pred");
        }
        {  // W in pair order: rank = exclusive scan of cand, wlist[rank] = pair
            size_t tb = 0;
            int* rk = D->fr_rank.as<int>();
            cub::DeviceScan::ExclusiveScan(nullptr, tb, F.cand, rk, ScanAdd{}, 0, (int)np, s);
            CK(D->sort_tmp.ensure(tb));
            CK(cub::DeviceScan::ExclusiveScan(D->sort_tmp.p, tb, F.cand, rk, ScanAdd{}, 0, (int)np, s));
            F.rank = rk;
            F.wlist = D->fr_wlist.as<int>();
            F.nw = (int)nw;
            k_fr_compact<<<pb, DTPB, 0, s>>>(F);
            ctx->launches += 3;
        }
        const unsigned wb = (unsigned)((nw + DTPB - 1) / DTPB);
        const int grid = (int)std::max(1ll, std::min<long long>(wb, (long long)ctx->sm_count * std::max(1, occ)));
        k_friction<<<grid, DTPB, 0, s>>>(F);
        ++ctx->launches;
        DSYNC("k_friction");
        CK(cudaMemcpyAsync(misc, D->fr_misc.p, 32, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (all) break;
        const int nlog = misc[4];
        F.nlog = nlog;
        if (nlog > 0) {  // the log sorted by (vertex, pair), carrying the entry index
            size_t tb = 0;
            auto* k1 = D->fr_log_key.as<unsigned long long>();
            auto* k2 = D->fr_log_key2.as<unsigned long long>();
            int* i1 = D->fr_log_idx.as<int>();
            int* i2 = D->fr_log_idx2.as<int>();
            k_iota<<<(nlog + DTPB - 1) / DTPB, DTPB, 0, s>>>(i1, nlog);
            cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, k2, i1, i2, nlog, 0, 64, s);
            CK(D->sort_tmp.ensure(tb));
            CK(cub::DeviceRadixSort::SortPairs(D->sort_tmp.p, tb, k1, k2, i1, i2, nlog, 0, 64, s));
            ctx->launches += 5;
            F.slog_key = k2;
            F.slog_idx = i2;
        }
        k_fr_verify<<<pb, DTPB, 0, s>>>(F);
        ++ctx->launches;
        DSYNC("k_fr_verify");
        CK(cudaMemcpyAsync(misc, D->fr_misc.p, 32, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (getenv("TW_FR_STATS"))
            fprintf(stderr, "friction round %d: |W| %lld, incidences %d, logged writes %d, added %d\n", round, nw,
                    nent, nlog, misc[3]);
        if (misc[3] == 0) break;  // verified: no pair outside W writes
        misc[2] += misc[3];
        CK(cudaMemcpyAsync(F.misc + 2, misc + 2, 4, cudaMemcpyHostToDevice, s));
    }
    CK(cudaGetLastError());
    return TW_OK;
}

// search + gradient/Hessian + repulsion + PCG at d_xk (N x 3, device) with
// inertia data D->x0 / D->v0; the target goes to d_y. stats: pcg iterations /
// convergence / pairs.
int newton_target_device(tw_dyn* D, double d_max, const double* d_xk, double* d_y, tw_step_stats* st,
                         double* grad_host) {
    tw_ctx* ctx = D->ctx;
    tw_mesh* m = D->mesh;
    cudaStream_t s = ctx->stream;
    const int nv = m->nv;
    const int nb = (nv + DTPB - 1) / DTPB;
    CK(cudaEventRecord(D->evt0, s));
    CK(ctx->x.ensure((size_t)std::max(1, nv) * 32));
    k_pack_x4<<<std::max(1, nb), DTPB, 0, s>>>(nv, d_xk, m->d_inv_mass.as<double>(), ctx->x.as<double4>());
    ++ctx->launches;
    DSYNC("k_pack_x4");
    // add_repulsion (dynamics.cpp:176-181) only reads pairs closer than the
    // repulsion radius, and the search is exact (every pair below its cutoff,
    // in key order), so searching with min(d_max, radius) yields exactly the
    // repulsive pairs of step()'s d_max search -- in the same order -- at a
    // fraction of the broad-phase cost; no repulsion, no search.
    // friction_filter (mu > 0) reads every pair of the d_max set -- a pair
    // farther than the radius at x can penetrate it at the target -- so then
    // the search runs at d_max (the repulsive pairs are the same either way).
    long long np = 0;
    const bool repel = D->model.repulsion_stiffness > 0.0 && D->model.repulsion_radius > 0.0;
    const bool friction = D->model.mu > 0.0;
    if (repel || friction) {
        const int rc0 = search_at_x(ctx, m, friction ? d_max : std::min(d_max, D->model.repulsion_radius), &np);
        if (rc0) return rc0;
    }
    int rc = TW_OK;
    if (D->rp_cap < np + 1) {
        D->rp_cap = np + 1024;
        CK(D->rp_ids.ensure((size_t)D->rp_cap * 16));
        CK(D->rp_sw.ensure((size_t)D->rp_cap * 32));
        CK(D->rp_dir.ensure((size_t)D->rp_cap * 32));
        CK(D->rs_key.ensure((size_t)D->rp_cap * 4 * 8));
        CK(D->rs_key2.ensure((size_t)D->rp_cap * 4 * 8));
    }
    DynParams P = make_dparams(D, d_xk);
    P.np = np;
    CK(cudaMemsetAsync(D->rp_count.p, 0, 16, s));
    if (m->ne) {
        k_edges<<<(m->ne + DTPB - 1) / DTPB, DTPB, 0, s>>>(P);
        ++ctx->launches;
        DSYNC("k_edges");
    }
    if (np && D->model.repulsion_stiffness > 0.0) {
        k_rep_pairs<<<(unsigned)((np + DTPB - 1) / DTPB), DTPB, 0, s>>>(P);
        ++ctx->launches;
        DSYNC("k_rep_pairs");
    }
    int counts[2] = {0, 0};
    CK(cudaMemcpyAsync(counts, D->rp_count.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int nent = counts[1];
    if (nent > 1) {
        size_t tb = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, D->rs_key.as<unsigned long long>(),
                                       D->rs_key2.as<unsigned long long>(), nent, 0, 64, s);
        CK(D->sort_tmp.ensure(tb));
        cub::DeviceRadixSort::SortKeys(D->sort_tmp.p, tb, D->rs_key.as<unsigned long long>(),
                                       D->rs_key2.as<unsigned long long>(), nent, 0, 64, s);
        ctx->launches += 4;
        P.rs_key = D->rs_key2.as<unsigned long long>();
    }
    DSYNC("sort");
    k_rep_offsets<<<(nv + 1 + DTPB - 1) / DTPB, DTPB, 0, s>>>(P.rs_key, nent, nv, P.vr_off);
    DSYNC("k_rep_offsets");
    k_grad_diag<<<std::max(1, nb), DTPB, 0, s>>>(P);
    DSYNC("k_grad_diag");
    ctx->launches += 2;
    if (grad_host) {
        std::vector<double4> g(nv);
        CK(cudaMemcpyAsync(g.data(), D->grad.p, (size_t)nv * 32, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int v = 0; v < nv; ++v) grad_host[3 * v] = g[v].x, grad_host[3 * v + 1] = g[v].y, grad_host[3 * v + 2] = g[v].z;
    }
    // register-resident CG: one vertex per thread (2 CTAs/SM) or, when that
    // grid would not fit (or TW_PCG_VPT=2), two per thread at 1 CTA/SM. A
    // 512-thread instance made the following resolve kernel 35% slower on
    // B200 (measured), so CTAs stay at 256 threads.
    static int occ[2] = {-1, -1};
    if (occ[0] < 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[0], k_pcg_reg<256, 1>, 256, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[1], k_pcg_reg<256, 2>, 256, 0);
    }
    const int parts = std::max(1, ctx->grid_parts);  // concurrent contexts share the device
    const int b1 = std::max(1, (nv + 255) / 256), b2 = std::max(1, (nv + 511) / 512);
    const char* vpt_env = getenv("TW_PCG_VPT");
    const bool want2 = vpt_env && std::atoi(vpt_env) == 2;
    const bool fit1 = b1 <= ctx->sm_count * occ[0] / parts, fit2 = b2 <= ctx->sm_count * occ[1] / parts;
    const int vpt = getenv("TW_PCG_GLOBAL") ? 0 : (want2 && fit2) ? 2 : fit1 ? 1 : fit2 ? 2 : 0;
    const int pb = vpt == 1 ? b1 : vpt == 2 ? b2 : std::max(1, pcg_blocks(ctx, nv) / parts);
    P.nblocks = pb;
    CK(D->part.ensure((size_t)pb * 32));
    P.part = D->part.as<double>();
    CK(cudaMemsetAsync(D->glob.p, 0, sizeof(DynGlobals), s));
    void* args[] = {&P};
    CK(cudaEventRecord(D->evp0, s));
    const void* fn = vpt == 1 ? (const void*)k_pcg_reg<256, 1> : vpt == 2 ? (const void*)k_pcg_reg<256, 2>
                                                                        : (const void*)k_pcg;
    CK(cudaLaunchCooperativeKernel(fn, dim3(pb), dim3(DTPB), args, 0, s));
    CK(cudaEventRecord(D->evp1, s));
    ++ctx->launches;
    DSYNC("k_pcg");
    DynGlobals G;
    CK(cudaMemcpyAsync(&G, D->glob.p, sizeof G, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    k_target<<<std::max(1, nb), DTPB, 0, s>>>(nv, m->d_inv_mass.as<double>(), d_xk, P.best, G.bnorm == 0.0, d_y);
    ++ctx->launches;
    if (friction) {  // dynamics.cpp:338
        CK(cudaEventRecord(D->evf0, s));
        rc = friction_device(D, d_xk, d_y, np);
        if (rc) return rc;
        CK(cudaEventRecord(D->evf1, s));
    }
    float tms = 0.f, pms = 0.f;
    CK(cudaEventElapsedTime(&tms, D->evt0, D->evp1));
    CK(cudaEventElapsedTime(&pms, D->evp0, D->evp1));
    if (st) {
        st->target_ms += tms;
        st->pcg_ms += pms;
        st->pcg_iterations += G.iters;
        st->pcg_converged = st->pcg_converged && G.converged;
        st->num_pairs = (int32_t)np;
        st->repulsive_pairs = counts[0];
        if (friction) {
            float fms = 0.f;
            CK(cudaEventSynchronize(D->evf1));
            CK(cudaEventElapsedTime(&fms, D->evf0, D->evf1));
            st->friction_ms += fms;
        }
    }
    CK(cudaGetLastError());
    return TW_OK;
}

int dyn_check(tw_ctx* ctx, tw_mesh* m, tw_dyn* D) {
    if (!ctx || !m || !D) return fail(ctx, TW_EINVAL, "dynamics: null argument");
    if (D->mesh != m) return fail(ctx, TW_EINVAL, "dynamics: model prepared on another mesh");
    return TW_OK;
}

// one step (dynamics.cpp:326-349) on device state d_x / d_v (N x 3)
int step_device(tw_ctx* ctx, tw_mesh* m, tw_dyn* D, const tw_resolve_config* cfg, double* d_x, double* d_v,
                tw_step_stats* st) {
    cudaStream_t s = ctx->stream;
    const size_t bytes = (size_t)m->nv * 24;
    CK(cudaEventRecord(D->ev0, s));
    CK(cudaMemcpyAsync(D->x0.p, d_x, bytes, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(D->v0.p, d_v, bytes, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(D->xk.p, d_x, bytes, cudaMemcpyDeviceToDevice, s));
    st->pcg_converged = 1;
    for (int k = 0; k < D->model.newton_iters; ++k) {
        int rc = newton_target_device(D, cfg->d_max, D->xk.as<double>(), D->y.as<double>(), st, nullptr);
        if (rc) return rc;
        tw_resolve_stats rs;
        rc = run_resolve(ctx, m, D->xk.as<double>(), D->y.as<double>(), *cfg, d_x, &rs, nullptr, nullptr, nullptr);
        if (rc) return rc;
        st->resolve_steps += rs.steps;
        st->searches += rs.searches;
        st->resolve_converged = rs.converged;
        st->resolve_ms += rs.device_ms;
        if (k + 1 < D->model.newton_iters) CK(cudaMemcpyAsync(D->xk.p, d_x, bytes, cudaMemcpyDeviceToDevice, s));
    }
    const int n3 = 3 * m->nv;
    k_velocity<<<std::max(1, (n3 + DTPB - 1) / DTPB), DTPB, 0, s>>>(m->nv, m->d_inv_mass.as<double>(), d_x,
                                                                   D->x0.as<double>(), D->model.dt, d_v);
    ++ctx->launches;
    CK(cudaEventRecord(D->ev1, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, D->ev0, D->ev1));
    st->device_ms = ms;
    CK(cudaGetLastError());
    return TW_OK;
}

int ensure_state(tw_dyn* D) {
    tw_ctx* ctx = D->ctx;
    const size_t nv = (size_t)std::max(1, D->mesh->nv), ne = (size_t)std::max(1, D->mesh->ne);
    DevMem* v24[] = {&D->hx, &D->hvel, &D->x0, &D->v0, &D->xk, &D->y};
    for (DevMem* d : v24) CK(d->ensure(nv * 24));
    DevMem* v32[] = {&D->grad, &D->b, &D->d, &D->r, &D->z, &D->p, &D->q, &D->best};
    for (DevMem* d : v32) CK(d->ensure(nv * 32));
    CK(D->sdiag.ensure(nv * 8));
    CK(D->pre.ensure(nv * 72));
    CK(D->vr_off.ensure((nv + 1) * 4));
    CK(D->e_u.ensure(ne * 32));
    CK(D->e_ab.ensure(ne * 16));
    CK(D->inc_u.ensure(2 * ne * 32));
    CK(D->inc_a.ensure(2 * ne * 8));
    CK(D->inc_o.ensure(2 * ne * 4));
    CK(D->rp_count.ensure(16));
    CK(D->glob.ensure(sizeof(DynGlobals)));
    if (D->rp_cap == 0) {
        D->rp_cap = 1024;
        CK(D->rp_ids.ensure((size_t)D->rp_cap * 16));
        CK(D->rp_sw.ensure((size_t)D->rp_cap * 32));
        CK(D->rp_dir.ensure((size_t)D->rp_cap * 32));
        CK(D->rs_key.ensure((size_t)D->rp_cap * 32));
        CK(D->rs_key2.ensure((size_t)D->rp_cap * 32));
    }
    return TW_OK;
}

}  // namespace

extern "C" {

void tw_default_energy_model(tw_energy_model* m) {  // EnergyModel defaults, dynamics.hpp:12-24
    m->spring_stiffness = 50.0;
    m->bending_stiffness = 0.0;
    m->gravity[0] = 0.0, m->gravity[1] = 0.0, m->gravity[2] = -9.81;
    m->repulsion_stiffness = 1e3;
    m->repulsion_radius = 1e-3;
    m->dt = 0.01;
    m->newton_iters = 1;
    m->mu = 0.0;
    m->pcg_tol = 1e-6;
    m->pcg_max_iters = 400;
}

int tw_dyn_create(tw_ctx* ctx, tw_mesh* m, const tw_energy_model* model, const double* rest_x, tw_dyn** out) {
    if (!ctx || !m || !model || !rest_x || !out) return fail(ctx, TW_EINVAL, "dynamics: null argument");
    if (!model_valid(*model)) return fail(ctx, TW_EINVAL, "dynamics: invalid energy model");
    CK(cudaSetDevice(ctx->device));
    auto* D = new tw_dyn();
    D->ctx = ctx;
    D->mesh = m;
    D->model = *model;
    // EnergyModel::prepare (dynamics.cpp:17-69): rest lengths and hinges
    std::vector<double> rest(std::max(1, m->ne));
    for (int e = 0; e < m->ne; ++e) {
        const int i = m->edges[2 * e], j = m->edges[2 * e + 1];
        const d3 d = sub(mk(rest_x[3 * i], rest_x[3 * i + 1], rest_x[3 * i + 2]),
                         mk(rest_x[3 * j], rest_x[3 * j + 1], rest_x[3 * j + 2]));
        rest[e] = nrm(d);
    }
    std::vector<int> hv;
    std::vector<double> hk;
    if (model->bending_stiffness > 0.0 && m->nt) {
        std::vector<int32_t> tris((size_t)m->nt * 3);
        std::vector<int4> t4(m->nt);
        cudaMemcpy(t4.data(), m->d_tris.p, (size_t)m->nt * 16, cudaMemcpyDeviceToHost);
        for (int t = 0; t < m->nt; ++t) tris[3 * t] = t4[t].x, tris[3 * t + 1] = t4[t].y, tris[3 * t + 2] = t4[t].z;
        build_hinges(m, tris, rest_x, hv, hk);
    }
    D->nh = (int)hv.size() / 4;
    // vertex -> (hinge, slot) in hinge order
    std::vector<int> off(m->nv + 1, 0), lst(hv.size());
    for (int v : hv) ++off[v + 1];
    for (int v = 0; v < m->nv; ++v) off[v + 1] += off[v];
    std::vector<int> fill(off.begin(), off.end() - 1);
    for (int h = 0; h < D->nh; ++h)
        for (int i = 0; i < 4; ++i) lst[fill[hv[4 * h + i]]++] = (h << 2) | i;
    cudaError_t e = upload(D->rest, rest);
    if (e == cudaSuccess) e = upload(D->hv, hv);
    if (e == cudaSuccess) e = upload(D->hk, hk);
    if (e == cudaSuccess) e = upload(D->vh_off, off);
    if (e == cudaSuccess) e = upload(D->vh, lst);
    if (e != cudaSuccess) {
        delete D;
        return cuda_fail(ctx, e, "tw_dyn_create");
    }
    int rc = ensure_state(D);
    if (!rc && (cudaEventCreate(&D->ev0) != cudaSuccess || cudaEventCreate(&D->ev1) != cudaSuccess ||
                cudaEventCreate(&D->evt0) != cudaSuccess || cudaEventCreate(&D->evp0) != cudaSuccess ||
                cudaEventCreate(&D->evp1) != cudaSuccess || cudaEventCreate(&D->evf0) != cudaSuccess ||
                cudaEventCreate(&D->evf1) != cudaSuccess))
        rc = fail(ctx, TW_ECUDA, "dynamics: event creation failed");
    if (rc) {
        tw_dyn_destroy(D);
        return rc;
    }
    *out = D;
    return TW_OK;
}

void tw_dyn_destroy(tw_dyn* D) {
    if (!D) return;
    cudaSetDevice(D->ctx ? D->ctx->device : 0);
    DevMem* all[] = {&D->inc_u, &D->inc_a, &D->inc_o, &D->hx, &D->hvel, &D->rest, &D->hv, &D->hk, &D->vh_off, &D->vh, &D->x0, &D->v0, &D->xk, &D->y, &D->e_u,
                     &D->e_ab, &D->rp_ids, &D->rp_sw, &D->rp_dir, &D->rp_count, &D->rs_key, &D->rs_key2,
                     &D->vr_off, &D->sort_tmp, &D->sdiag, &D->grad, &D->pre, &D->b, &D->d, &D->r, &D->z,
                     &D->p, &D->q, &D->best, &D->part, &D->glob, &D->fr_pred, &D->fr_done, &D->fr_misc,
                     &D->fr_cand, &D->fr_y0, &D->fr_log_key, &D->fr_log_key2, &D->fr_log_val, &D->fr_log_idx,
                     &D->fr_log_idx2, &D->fr_rank, &D->fr_wlist};
    for (DevMem* d : all) d->release();
    for (cudaEvent_t e : {D->ev0, D->ev1, D->evt0, D->evp0, D->evp1, D->evf0, D->evf1})
        if (e) cudaEventDestroy(e);
    delete D;
}

int32_t tw_dyn_num_hinges(const tw_dyn* D) { return D ? D->nh : 0; }

int tw_newton_target(tw_ctx* ctx, tw_mesh* m, tw_dyn* D, double d_max, const double* x0, const double* v0,
                     const double* x, double* y_out, double* grad_out, tw_step_stats* st) {
    int rc = dyn_check(ctx, m, D);
    if (rc) return rc;
    if (!x0 || !v0 || !x || !y_out) return fail(ctx, TW_EINVAL, "newton_target: null argument");
    if (!(d_max > 0.0)) return fail(ctx, TW_EINVAL, "newton_target: d_max must be > 0");
    CK(cudaSetDevice(ctx->device));
    const size_t bytes = (size_t)m->nv * 24;
    cudaStream_t s = ctx->stream;
    CK(cudaMemcpyAsync(D->x0.p, x0, bytes, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(D->v0.p, v0, bytes, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(D->xk.p, x, bytes, cudaMemcpyHostToDevice, s));
    tw_step_stats local;
    std::memset(&local, 0, sizeof local);
    local.pcg_converged = 1;
    rc = newton_target_device(D, d_max, D->xk.as<double>(), D->y.as<double>(), &local, grad_out);
    if (rc) return rc;
    CK(cudaMemcpyAsync(y_out, D->y.p, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (st) *st = local;
    return TW_OK;
}

int tw_friction_filter(tw_ctx* ctx, tw_mesh* m, tw_dyn* D, double d_max, const double* x, const double* y_target,
                       double* y_out) {
    int rc = dyn_check(ctx, m, D);
    if (rc) return rc;
    if (!x || !y_target || !y_out) return fail(ctx, TW_EINVAL, "friction_filter: null argument");
    if (!(d_max > 0.0)) return fail(ctx, TW_EINVAL, "friction_filter: d_max must be > 0");
    CK(cudaSetDevice(ctx->device));
    const int nv = m->nv;
    const size_t bytes = (size_t)nv * 24;
    cudaStream_t s = ctx->stream;
    CK(cudaMemcpyAsync(D->xk.p, x, bytes, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(D->y.p, y_target, bytes, cudaMemcpyHostToDevice, s));
    CK(ctx->x.ensure((size_t)std::max(1, nv) * 32));
    k_pack_x4<<<std::max(1, (nv + DTPB - 1) / DTPB), DTPB, 0, s>>>(nv, D->xk.as<double>(), m->d_inv_mass.as<double>(),
                                                                 ctx->x.as<double4>());
    ++ctx->launches;
    long long np = 0;
    rc = search_at_x(ctx, m, d_max, &np);
    if (rc) return rc;
    rc = friction_device(D, D->xk.as<double>(), D->y.as<double>(), np);
    if (rc) return rc;
    CK(cudaMemcpyAsync(y_out, D->y.p, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return TW_OK;
}

int tw_step(tw_ctx* ctx, tw_mesh* m, tw_dyn* D, const tw_resolve_config* cfg, double* x, double* v,
            tw_step_stats* st) {
    int rc = dyn_check(ctx, m, D);
    if (rc) return rc;
    if (!x || !v) return fail(ctx, TW_EINVAL, "step: null argument");
    rc = check_cfg(ctx, cfg);
    if (rc) return rc;
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaSetDevice(ctx->device));
    rc = ensure_buffers(ctx, m, *cfg);
    if (rc) return rc;
    const size_t bytes = (size_t)m->nv * 24;
    cudaStream_t s = ctx->stream;
    CK(cudaMemcpyAsync(D->hx.p, x, bytes, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(D->hvel.p, v, bytes, cudaMemcpyHostToDevice, s));
    tw_step_stats local;
    std::memset(&local, 0, sizeof local);
    tw_resolve_config c = *cfg;
    c.record_path = 0;
    rc = step_device(ctx, m, D, &c, D->hx.as<double>(), D->hvel.as<double>(), &local);
    if (rc) return rc;
    CK(cudaMemcpyAsync(x, D->hx.p, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(v, D->hvel.p, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    local.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (st) *st = local;
    return TW_OK;
}

int tw_step_device(tw_ctx* ctx, tw_mesh* m, tw_dyn* D, const tw_resolve_config* cfg, double* d_x, double* d_v,
                   tw_step_stats* st) {
    int rc = dyn_check(ctx, m, D);
    if (rc) return rc;
    if (!d_x || !d_v) return fail(ctx, TW_EINVAL, "step: null argument");
    rc = check_cfg(ctx, cfg);
    if (rc) return rc;
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaSetDevice(ctx->device));
    rc = ensure_buffers(ctx, m, *cfg);
    if (rc) return rc;
    tw_step_stats local;
    std::memset(&local, 0, sizeof local);
    tw_resolve_config c = *cfg;
    c.record_path = 0;
    rc = step_device(ctx, m, D, &c, d_x, d_v, &local);
    if (rc) return rc;
    local.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (st) *st = local;
    return TW_OK;
}


int tw_normal_flow_target(tw_ctx* ctx, int32_t nv, const double* x, int32_t nt, const int32_t* triangles,
                          double beta, double alpha_smooth, double* y_out) {
    if (!ctx || nv < 0 || nt < 0 || !x || !y_out || (nt && !triangles))
        return fail(ctx, TW_EINVAL, "normal flow: null argument");
    // require_closed_manifold (normal_flow.cpp:24-36): every directed edge once,
    // and its reverse exactly once
    if (nt == 0) return fail(ctx, TW_EINVAL, "normal flow: no triangles");
    std::vector<uint64_t> dir;
    dir.reserve(3 * (size_t)nt);
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) {
            const int a = triangles[3 * t + k], b = triangles[3 * t + (k + 1) % 3];
            if (a < 0 || a >= nv || b < 0 || b >= nv) return fail(ctx, TW_EINVAL, "normal flow: vertex id out of range");
            dir.push_back(((uint64_t)(uint32_t)a << 32) | (uint32_t)b);
        }
    std::vector<uint64_t> sorted = dir;
    std::sort(sorted.begin(), sorted.end());
    for (size_t i = 1; i < sorted.size(); ++i)
        if (sorted[i] == sorted[i - 1]) return fail(ctx, TW_EINVAL, "normal flow: non-manifold edge (repeated direction)");
    for (uint64_t d : sorted) {
        const uint64_t rev = (d << 32) | (d >> 32);
        if (!std::binary_search(sorted.begin(), sorted.end(), rev))
            return fail(ctx, TW_EINVAL, "normal flow: mesh is not closed/consistently oriented");
    }
    // topology tables: vertex -> triangles (triangle order); undirected edges in
    // (min, max) order with their (t, k) occurrences; vertex -> (neighbour, edge)
    // in ascending neighbour order
    std::vector<int> vt_off(nv + 1, 0), vt(3 * (size_t)nt);
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) ++vt_off[triangles[3 * t + k] + 1];
    for (int v = 0; v < nv; ++v) vt_off[v + 1] += vt_off[v];
    {
        std::vector<int> fill(vt_off.begin(), vt_off.end() - 1);
        for (int t = 0; t < nt; ++t)
            for (int k = 0; k < 3; ++k) vt[fill[triangles[3 * t + k]]++] = t;
    }
    std::vector<std::pair<uint64_t, int>> occ;  // (undirected key, t << 2 | k)
    occ.reserve(3 * (size_t)nt);
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) {
            const int a = triangles[3 * t + k], b = triangles[3 * t + (k + 1) % 3];
            occ.push_back({((uint64_t)(uint32_t)std::min(a, b) << 32) | (uint32_t)std::max(a, b), (t << 2) | k});
        }
    std::stable_sort(occ.begin(), occ.end(), [](auto& p, auto& q) { return p.first < q.first; });
    std::vector<int> occ_off{0}, occ_v;
    std::vector<std::pair<int, int>> ekeys;  // (min, max) per undirected edge
    for (size_t i = 0; i < occ.size(); ++i) {
        if (i > 0 && occ[i].first != occ[i - 1].first) occ_off.push_back((int)i);
        if (i == 0 || occ[i].first != occ[i - 1].first)
            ekeys.push_back({(int)(occ[i].first >> 32), (int)(occ[i].first & 0xffffffffu)});
        occ_v.push_back(occ[i].second);
    }
    occ_off.push_back((int)occ.size());
    const int ne = (int)ekeys.size();
    std::vector<std::vector<std::pair<int, int>>> nbl(nv);
    for (int e = 0; e < ne; ++e) {
        nbl[ekeys[e].first].push_back({ekeys[e].second, e});
        nbl[ekeys[e].second].push_back({ekeys[e].first, e});
    }
    std::vector<int> nb_off(nv + 1, 0);
    std::vector<int2> nb;
    for (int v = 0; v < nv; ++v) {
        std::sort(nbl[v].begin(), nbl[v].end());
        for (auto& p : nbl[v]) nb.push_back(make_int2(p.first, p.second));
        nb_off[v + 1] = (int)nb.size();
    }
    std::vector<int4> t4(nt);
    for (int t = 0; t < nt; ++t) t4[t] = make_int4(triangles[3 * t], triangles[3 * t + 1], triangles[3 * t + 2], 0);
    CK(cudaSetDevice(ctx->device));
    DevMem dx, dy0, dy1, dvto, dvt, dtris, doo, docc, dnbo, dnb, dw;
    struct Rel {
        std::vector<DevMem*> m;
        ~Rel() {
            for (DevMem* d : m) d->release();
        }
    } rel{{&dx, &dy0, &dy1, &dvto, &dvt, &dtris, &doo, &docc, &dnbo, &dnb, &dw}};
    cudaError_t e = cudaSuccess;
    auto up = [&](DevMem& d, const void* h, size_t bytes) {
        if (e == cudaSuccess) e = d.ensure(std::max<size_t>(16, bytes));
        if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(d.p, h, bytes, cudaMemcpyHostToDevice, ctx->stream);
    };
    up(dx, x, (size_t)nv * 24);
    up(dvto, vt_off.data(), vt_off.size() * 4);
    up(dvt, vt.data(), vt.size() * 4);
    up(dtris, t4.data(), t4.size() * 16);
    up(doo, occ_off.data(), occ_off.size() * 4);
    up(docc, occ_v.data(), occ_v.size() * 4);
    up(dnbo, nb_off.data(), nb_off.size() * 4);
    up(dnb, nb.data(), nb.size() * 8);
    if (e == cudaSuccess) e = dy0.ensure((size_t)std::max(1, nv) * 24);
    if (e == cudaSuccess) e = dy1.ensure((size_t)std::max(1, nv) * 24);
    if (e == cudaSuccess) e = dw.ensure((size_t)std::max(1, ne) * 8);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "normal flow: upload");
    cudaStream_t s = ctx->stream;
    const int nb_v = std::max(1, (nv + DTPB - 1) / DTPB);
    k_nf_offset<<<nb_v, DTPB, 0, s>>>(nv, dx.as<double>(), dvto.as<int>(), dvt.as<int>(), dtris.as<int4>(), beta,
                                       dy0.as<double>());
    k_nf_weights<<<std::max(1, (ne + DTPB - 1) / DTPB), DTPB, 0, s>>>(ne, doo.as<int>(), docc.as<int>(),
                                                                      dtris.as<int4>(), dy0.as<double>(), dw.as<double>());
    DevMem* cur = &dy0;
    DevMem* nxt = &dy1;
    for (int pass = 0; pass < 3; ++pass) {  // NormalFlowConfig::kSmoothingIterations
        k_nf_smooth<<<nb_v, DTPB, 0, s>>>(nv, dnbo.as<int>(), dnb.as<int2>(), dw.as<double>(), alpha_smooth,
                                           cur->as<double>(), nxt->as<double>());
        std::swap(cur, nxt);
    }
    ctx->launches += 5;
    CK(cudaMemcpyAsync(y_out, cur->p, (size_t)nv * 24, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return TW_OK;
}

}  // extern "C"

// Phase functions of the device-resident Alg. 1 (resolve.cpp:36-144). Every
// phase is a grid-stride (or block-chunked, where order matters) loop run by
// all CTAs of the persistent cooperative kernel; phases are separated by
// grid_sync(). Reference citations are into /root/reference/proj.
#pragma once

#include "tw_barrier.cuh"
#include "tw_engine.cuh"

namespace tw {

// =============================================================== barrier
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Grid barrier over all CTAs of a cooperative launch (flip-bit, one release
// atomic per CTA: tw_barrier.cuh). A waiter also leaves when the error word is
// set -- CTAs that bail out on an error may never arrive -- and a watchdog
// (20 s, or Globals::watchdog_ns) turns any other hang into ERR_TIMEOUT.
__device__ __forceinline__ void flip_wait(Globals* g, unsigned* w, unsigned inc) {
    const unsigned old = bar_arrive(w, inc);
    volatile int* err = &g->error;
    unsigned long long t0 = 0;
    for (unsigned it = 0; !bar_flipped(old, bar_poll_relaxed(w)); ++it) {
        if ((it & 63u) == 63u) {
            if (*err) break;
            const unsigned long long t = global_ns();
            if (t0 == 0) t0 = t;
            else if (t - t0 > (g->watchdog_ns ? g->watchdog_ns : 20000000000ull)) {
                atomicOr(&g->error, ERR_TIMEOUT);
                break;
            }
        }
    }
    bar_acquire_fence();
}

__device__ __forceinline__ bool grid_sync(Globals* g) {
    __syncthreads();
    if (threadIdx.x == 0) flip_wait(g, &g->bar_count, blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u);
    __syncthreads();
    return *((volatile int*)&g->error) == 0;
}

// Barrier of the first n CTAs of the grid only (the same flip-bit scheme on
// its own counter); the other CTAs wait at the next grid barrier.
__device__ __forceinline__ bool sub_sync(Globals* g, unsigned n) {
    __syncthreads();
    if (threadIdx.x == 0) flip_wait(g, &g->sub_count, blockIdx.x == 0 ? 0x80000000u - (n - 1u) : 1u);
    __syncthreads();
    return *((volatile int*)&g->error) == 0;
}

// ============================================================ block scans
// exclusive scan of v over the CTA; *total receives the CTA sum
__device__ __forceinline__ long long block_scan(long long v, long long* total) {
    __shared__ long long ws[TPB / 32 + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        long long s = lane < TPB / 32 ? ws[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < TPB / 32) ws[lane] = s;  // inclusive warp prefix
    }
    __syncthreads();
    const long long wpre = warp ? ws[warp - 1] : 0;
    *total = ws[TPB / 32 - 1];
    __syncthreads();
    return wpre + inc - v;
}

__device__ __forceinline__ long long block_sum(long long v) {
    long long t;
    block_scan(v, &t);
    return t;
}

// max over the CTA (every thread gets it)
__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long v) {
    __shared__ unsigned long long wm[TPB / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) wm[warp] = v;
    __syncthreads();
    unsigned long long m = wm[0];
#pragma unroll
    for (int w = 1; w < TPB / 32; ++w) m = max(m, wm[w]);
    return m;
}

// One shared-memory scratch buffer for the phases that stage data per warp
// (walk stacks and candidate queues, warm-start segments). Phases never
// overlap (a grid barrier, hence a CTA barrier, separates them), and a small
// static footprint leaves more of the SM's unified 256 KB to L1, which the
// vertex gathers of the pair passes live on.
constexpr int SCRATCH_BYTES = 8192;
__device__ __forceinline__ char* smem_scratch() {
    __shared__ __align__(16) char buf[SCRATCH_BYTES];
    return buf;
}

// sum of part[0..upto) (every thread gets it)
__device__ __forceinline__ long long prefix_of(const long long* part, int upto) {
    long long s = 0;
    for (int i = threadIdx.x; i < upto; i += TPB) s += ((volatile const long long*)part)[i];
    return block_sum(s);
}

__device__ __forceinline__ void chunk_of(long long n, long long* lo, long long* hi) {
    const long long c = (n + gridDim.x - 1) / gridDim.x;
    *lo = min(n, (long long)blockIdx.x * c);
    *hi = min(n, *lo + c);
}

// Pair passes that feed the row compaction run over tiles of PAIR_TILE
// consecutive pairs dealt round-robin to the CTAs (the contact pairs cluster
// where the knot is tight; contiguous chunks would leave that work to a few
// CTAs). body(p) returns whether pair p is a contact pair; per-tile counts go
// to part_c[tile] for ph_rows.
#ifndef TW_PAIR_PER
#define TW_PAIR_PER 4
#endif
constexpr int PAIR_PER = TW_PAIR_PER;  // pairs per thread per tile (4: 2.5% faster than 16)
constexpr long long PAIR_TILE = (long long)TPB * PAIR_PER;
__device__ __forceinline__ long long pair_tiles(long long np) { return (np + PAIR_TILE - 1) / PAIR_TILE; }

__device__ __forceinline__ long long gtid() { return (long long)blockIdx.x * TPB + threadIdx.x; }
__device__ __forceinline__ long long gstride() { return (long long)gridDim.x * TPB; }

template <typename F>
__device__ __forceinline__ void for_pair_tiles(const Params& P, long long np, F&& body) {
    const long long ntile = pair_tiles(np);
    for (long long tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const long long lo = tile * PAIR_TILE, hi = min(np, lo + PAIR_TILE);
        long long c = 0;
        for (long long p = lo + threadIdx.x; p < hi; p += TPB) c += body(p) ? 1 : 0;
        const long long t = block_sum(c);
        if (threadIdx.x == 0) P.part_c[tile] = t;
    }
}
__device__ __forceinline__ long long gwarp() { return gtid() >> 5; }
__device__ __forceinline__ long long gwarps() { return gstride() >> 5; }

struct XLoad {
    const double4* x;
    __device__ __forceinline__ d3 operator()(int i) const { return ld3(x, i); }
};

// ================================================================= BVH
__device__ __forceinline__ void prim_box(const Params& P, int cls, int prim, double lo[3], double hi[3]) {
    int ids[3];
    int n;
    if (cls == 0) {
        const int4 t = P.tris[prim];
        ids[0] = t.x, ids[1] = t.y, ids[2] = t.z, n = 3;
    } else if (cls == 1) {
        const int2 e = P.edges[prim];
        ids[0] = e.x, ids[1] = e.y, n = 2;
    } else {
        ids[0] = P.iso[prim], n = 1;
    }
    const d3 p0 = ld3(P.x, ids[0]);
    lo[0] = hi[0] = p0.x, lo[1] = hi[1] = p0.y, lo[2] = hi[2] = p0.z;
    for (int i = 1; i < n; ++i) {
        const d3 p = ld3(P.x, ids[i]);
        lo[0] = fmin(lo[0], p.x), hi[0] = fmax(hi[0], p.x);
        lo[1] = fmin(lo[1], p.y), hi[1] = fmax(hi[1], p.y);
        lo[2] = fmin(lo[2], p.z), hi[2] = fmax(hi[2], p.z);
    }
    if (P.ccd_x1) {  // certification: the box swept from x to x1
        for (int i = 0; i < n; ++i) {
            const d3 p = ld3(P.ccd_x1, ids[i]);
            lo[0] = fmin(lo[0], p.x), hi[0] = fmax(hi[0], p.x);
            lo[1] = fmin(lo[1], p.y), hi[1] = fmax(hi[1], p.y);
            lo[2] = fmin(lo[2], p.z), hi[2] = fmax(hi[2], p.z);
        }
        for (int k = 0; k < 3; ++k) lo[k] -= 1e-12, hi[k] += 1e-12;
    }
}

__device__ __forceinline__ int prim_to_index(const Params& P, int cls, int prim) {
    return cls == 2 ? P.iso[prim] : prim;
}

// A1: bottom-up refit of all three hierarchies at the current positions
// (node flags are zero on entry; the second child to arrive builds the
// parent's box). Every finished box is written into its slot of the parent's
// packed node (Bvh::node).
__device__ void ph_refit(const Params& P) {
    if (blockIdx.x == 0 && threadIdx.x == 0) P.g->work_q = 0ull, P.g->work_s = 0ull, P.g->ncand = 0ull;
    for (int cls = 0; cls < 3; ++cls) {
        const Bvh& B = P.bvh[cls];
        if (B.n == 0) continue;
        for (long long j = gtid(); j < B.n; j += gstride()) {
            double lo[3], hi[3];
            const int prim = B.prim[j];
            prim_box(P, cls, prim, lo, hi);
            float4 blo = make_float4(__double2float_rd(lo[0]), __double2float_rd(lo[1]), __double2float_rd(lo[2]),
                                     __int_as_float(~prim_to_index(P, cls, prim)));
            const int idx = prim_to_index(P, cls, prim);
            float4 bhi = make_float4(__double2float_ru(hi[0]), __double2float_ru(hi[1]), __double2float_ru(hi[2]),
                                     __int_as_float(idx));  // w: largest primitive index below
            if (B.n == 1) {
                B.node[0] = blo, B.node[1] = bhi;
                B.node[2] = make_float4(INFINITY, INFINITY, INFINITY, __int_as_float(~0));
                B.node[3] = make_float4(-INFINITY, -INFINITY, -INFINITY, __int_as_float(-1));
                continue;
            }
            int node = B.n - 1 + (int)j;
            for (;;) {
                const int par = B.parent[node];
                if (par < 0) break;
                const int slot = B.child[par].x == node ? 0 : 1;
                float4* pn = B.node + 4LL * par + 2 * slot;
                pn[0] = blo, pn[1] = bhi;
                // acq_rel arrival: the first child's box is visible to the second
                unsigned prev;
                asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&B.flag[par]) : "memory");
                if (prev == 0u) break;
                const float4* q = B.node + 4LL * par;
                const float4 a0 = __ldcg(q), a1 = __ldcg(q + 1), b0 = __ldcg(q + 2), b1 = __ldcg(q + 3);
                blo = make_float4(fminf(a0.x, b0.x), fminf(a0.y, b0.y), fminf(a0.z, b0.z), __int_as_float(par));
                bhi = make_float4(fmaxf(a1.x, b1.x), fmaxf(a1.y, b1.y), fmaxf(a1.z, b1.z),
                                  __int_as_float(max(__float_as_int(a1.w), __float_as_int(b1.w))));
                node = par;
            }
        }
    }
}

// Euclidean refinement of the inflated-box test: with the query box inflated
// by dinfl (rounded outwards), lo - qhi + dinfl and qlo + dinfl - hi are lower
// bounds of the axis gaps between the un-inflated boxes, hence of the gaps
// between the simplices; a box pair whose gap vector is longer than d_max
// holds no pair closer than d_max. The float slack per axis (1 um + 3e-7 of
// the query box's largest coordinate: several ulps of the float rounding of
// the differences) and 1e-5 relative on the square keep the test
// conservative, so only candidates the exact filter would reject are dropped
// (the pair set is unchanged).
__device__ __forceinline__ bool box_near(float4 qlo, float4 qhi, float4 lo, float4 hi, float dinf, float d2) {
    const float gx = fmaxf(0.f, fmaxf(lo.x - qhi.x, qlo.x - hi.x) + dinf);
    const float gy = fmaxf(0.f, fmaxf(lo.y - qhi.y, qlo.y - hi.y) + dinf);
    const float gz = fmaxf(0.f, fmaxf(lo.z - qhi.z, qlo.z - hi.z) + dinf);
    return gx * gx + gy * gy + gz * gz <= d2;
}

__device__ __forceinline__ bool box_hit(float4 qlo, float4 qhi, float4 lo, float4 hi) {
    return qlo.x <= hi.x && qlo.y <= hi.y && qlo.z <= hi.z && lo.x <= qhi.x && lo.y <= qhi.y &&
           lo.z <= qhi.z;
}

// Query index space in output (key) order — VV, VE, VT, EE — with every
// class starting at a multiple of 32 so that a warp's 32 queries share one
// hierarchy; padding queries are invalid (ia = -1) and produce no pairs.
__device__ __forceinline__ void query_of(const Params& P, long long q, int* ka, int* ia, int* kb,
                                         int* cls) {
    const long long niso = P.niso, s1 = pad32(niso), s2 = 2 * s1, s3 = s2 + pad32(P.nv);
    if (q < s1) {
        *ka = KV, *ia = q < niso ? P.iso[q] : -1, *kb = KV, *cls = 2;
    } else if (q < s2) {
        *ka = KV, *ia = q - s1 < niso ? P.iso[q - s1] : -1, *kb = KE, *cls = 1;
    } else if (q < s3) {
        *ka = KV, *ia = q - s2 < P.nv ? (int)(q - s2) : -1, *kb = KT, *cls = 0;
    } else {
        *ka = KE, *ia = q - s3 < P.ne ? (int)(q - s3) : -1, *kb = KE, *cls = 1;
    }
}
__device__ __forceinline__ long long num_queries(const Params& P) {
    return 2 * pad32(P.niso) + pad32(P.nv) + pad32(P.ne);
}

// The query handed out at packet position pos. Isolated vertices go in Morton
// order (the leaf order of their hierarchy). Vertices and edges go in mesh
// order or Morton order (P.vperm / P.eperm), whichever makes the 32 queries
// of a warp packet more compact (k_packet_spread, at the mesh's first call):
// strip meshes numbered row by row are compact as they are, arbitrary
// numberings are not. Padding positions map to themselves.
__device__ __forceinline__ long long query_at(const Params& P, long long pos) {
    const long long niso = P.niso, s1 = pad32(niso), s2 = 2 * s1, s3 = s2 + pad32(P.nv);
    if (pos < s1) return pos < niso ? P.bvh[2].prim[pos] : pos;
    if (pos < s2) return s1 + (pos - s1 < niso ? P.bvh[2].prim[pos - s1] : pos - s1);
    if (pos < s3) {
        const long long j = pos - s2;
        const bool morton = P.qspread[1] < 0.9 * P.qspread[0];
        return s2 + (j < P.nv && morton ? P.vperm[j] : j);
    }
    const long long j = pos - s3;
    const bool morton = P.qspread[3] < 0.9 * P.qspread[2];
    return s3 + (j < P.ne && morton ? P.eperm[j] : j);
}

__device__ __forceinline__ void simplex_ids(const Params& P, int k, int idx, int* v) {
    v[0] = v[1] = v[2] = -1;
    if (k == KV) {
        v[0] = idx;
    } else if (k == KE) {
        const int2 e = P.edges[idx];
        v[0] = e.x, v[1] = e.y;
    } else {
        const int4 t = P.tris[idx];
        v[0] = t.x, v[1] = t.y, v[2] = t.z;
    }
}

// The exact narrow-phase test of the reference search (proximity.cpp:162-167):
// canonical candidate, non-adjacent, has a closest point, distance < d_max.
template <int K>
__device__ __forceinline__ void simplex_ids_t(const Params& P, int idx, int (&v)[3]) {
    v[0] = v[1] = v[2] = -1;
    if constexpr (K == KV) {
        v[0] = idx;
    } else if constexpr (K == KE) {
        const int2 e = P.edges[idx];
        v[0] = e.x, v[1] = e.y;
    } else {
        const int4 t = P.tris[idx];
        v[0] = t.x, v[1] = t.y, v[2] = t.z;
    }
}
template <int KA, int KB>
__device__ __forceinline__ bool candidate_keep_t(const Params& P, int ia, int ib, Closest& c) {
    if (KA == KE && ib <= ia) return false;              // EE: a is the lower edge index
    if (KA == KV && KB == KV && ib <= ia) return false;  // VV: a < b
    int va[3], vb[3];
    simplex_ids_t<KA>(P, ia, va);
    simplex_ids_t<KB>(P, ib, vb);
    const int h = pair_closest_t<KA, KB>(va, vb, XLoad{P.x}, c);
    return h == 1 && c.dist < P.cfg.d_max;
}
__device__ __forceinline__ bool candidate_keep(const Params& P, int ka, int ia, const int* va,
                                               int kb, int ib, Closest& c) {
    if (ka == KE && ib <= ia) return false;             // EE: a is the lower edge index
    if (ka == KV && kb == KV && ib <= ia) return false; // VV: a < b
    int vb[3];
    simplex_ids(P, kb, ib, vb);
    const int h = pair_closest(ka, va, kb, vb, XLoad{P.x}, c);
    return h == 1 && c.dist < P.cfg.d_max;
}

// ascending bitonic sort of 64 ints held as (a, b) = elements (lane, lane + 32)
__device__ __forceinline__ void bitonic64(int& a, int& b, int lane) {
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {  // k == 64: partner is the other register of this lane
                const int lo = min(a, b), hi = max(a, b);
                a = lo, b = hi;
                continue;
            }
            const int pa = __shfl_xor_sync(0xffffffffu, a, j);
            const int pb = __shfl_xor_sync(0xffffffffu, b, j);
            const bool low = (lane & j) == 0;
            const bool up_a = (lane & k) == 0, up_b = ((lane + 32) & k) == 0;
            a = (up_a == low) ? min(a, pa) : max(a, pa);
            b = (up_b == low) ? min(b, pb) : max(b, pb);
        }
    }
}

// ascending bitonic sort of 32 ints, one per lane
__device__ __forceinline__ int bitonic32(int a, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const int pa = __shfl_xor_sync(0xffffffffu, a, j);
            a = (((lane & k) == 0) == ((lane & j) == 0)) ? min(a, pa) : max(a, pa);
        }
    }
    return a;
}

// Ascending bitonic sort of L independent lists at once, each of up to 32 R
// ints held as v[i][r] = element r * 32 + lane: stages with a partner distance
// of 32 or more compare registers of the same lane, the others shuffle. The L
// lists' shuffle chains interleave. v is sized for the largest R (SORT_R).
#ifndef TW_SORT_L
#define TW_SORT_L 4
#endif
constexpr int SORT_L = TW_SORT_L, SORT_R = 4;  // K <= 128 partners per query sort in registers
template <int R, int L>
__device__ __forceinline__ void bitonic_lists(int (&v)[L][SORT_R], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * R; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jr = j >> 5;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (r & jr) continue;
                    const bool up = ((r * 32 + lane) & k) == 0;
#pragma unroll
                    for (int i = 0; i < L; ++i) {
                        const int lo = min(v[i][r], v[i][r | jr]), hi = max(v[i][r], v[i][r | jr]);
                        v[i][r] = up ? lo : hi;
                        v[i][r | jr] = up ? hi : lo;
                    }
                }
                continue;
            }
            const bool low = (lane & j) == 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool keep_min = (((r * 32 + lane) & k) == 0) == low;
#pragma unroll
                for (int i = 0; i < L; ++i) {
                    const int p = __shfl_xor_sync(0xffffffffu, v[i][r], j);
                    v[i][r] = keep_min ? min(v[i][r], p) : max(v[i][r], p);
                }
            }
        }
    }
}

// warp-cooperative ascending sort of one query's partner list (n >= 2)
__device__ __forceinline__ void sort_partners(int* s, int n, int lane) {
    if (n <= 32) {
        const int a = bitonic32(lane < n ? s[lane] : 0x7fffffff, lane);
        if (lane < n) s[lane] = a;
    } else if (n <= 64) {
        int a = lane < n ? s[lane] : 0x7fffffff;
        int b = lane + 32 < n ? s[lane + 32] : 0x7fffffff;
        bitonic64(a, b, lane);
        if (lane < n) s[lane] = a;
        if (lane + 32 < n) s[lane + 32] = b;
    } else if (lane == 0) {
        for (int i = 1; i < n; ++i) {
            const int v = s[i];
            int j = i - 1;
            while (j >= 0 && s[j] > v) s[j + 1] = s[j], --j;
            s[j + 1] = v;
        }
    }
    __syncwarp();
}

// A2: broad phase. A warp takes 32 consecutive queries (spatially coherent:
// consecutive vertices / edges of the mesh) from a global counter and walks
// the hierarchy as a packet: one shared DFS stack, a node is descended when
// any lane's query box overlaps it (ballot), so the walk never diverges. A
// leaf hit by a lane's box (and canonical for the query: EE and VV keep
// a < b, proximity.cpp:125-140) becomes a (query, partner) candidate, queued
// per warp and written out 32 at a time. The walk holds no FP64 state, which
// keeps it light on registers; the exact tests run in ph_cand_eval.
constexpr int TRAV_STACK = 128;
#ifndef TW_WALK_PAIRS
#define TW_WALK_PAIRS 1  // two nodes per walk step (four: slower, register pressure)
#endif
__device__ void ph_traverse(const Params& P) {
    static_assert(sizeof(int) * (TPB / 32) * TRAV_STACK + sizeof(int2) * (TPB / 32) * 64 <= SCRATCH_BYTES, "");
    int(*sstack)[TRAV_STACK] = reinterpret_cast<int(*)[TRAV_STACK]>(smem_scratch());
    int2(*cq)[64] = reinterpret_cast<int2(*)[64]>(smem_scratch() + sizeof(int) * (TPB / 32) * TRAV_STACK);
    const long long nq = num_queries(P);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    int* stack = sstack[warp];
    const double dinfl_all = P.cfg.d_max * (1.0 + 1e-6) + 1e-12;
    // Euclidean pruning (box_near) for the proximity search; off for the
    // swept boxes of the certification
    const float dinf_f = P.ccd_x1 ? 0.f : __double2float_rd(dinfl_all);
    const float d2_f = P.ccd_x1 ? __int_as_float(0x7f800000) : (float)(P.cfg.d_max * P.cfg.d_max * (1.0 + 1e-5));
    for (;;) {
        long long base = 0;
        if (lane == 0) base = (long long)atomicAdd(&P.g->work_q, 32ull);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= nq) break;
        const long long q = query_at(P, base + lane);  // nq is a multiple of 32
        int ka, ia, kb, cls;
        query_of(P, q, &ka, &ia, &kb, &cls);  // ka, kb, cls are warp-uniform
        const Bvh& B = P.bvh[cls];
        P.qcount[q] = 0;
        float4 qlo = make_float4(1.f, 1.f, 1.f, 0.f), qhi = make_float4(0.f, 0.f, 0.f, 0.f);  // empty box
        float dinf_q = 0.f;
        if (ia >= 0) {
            int va[3];
            simplex_ids(P, ka, ia, va);
            double lo3[3], hi3[3];
            const d3 p0 = ld3(P.x, va[0]);
            lo3[0] = hi3[0] = p0.x, lo3[1] = hi3[1] = p0.y, lo3[2] = hi3[2] = p0.z;
            for (int k = 0; k <= ka; ++k) {
                const d3 p1 = ld3(P.x, va[k]);
                lo3[0] = fmin(lo3[0], p1.x), hi3[0] = fmax(hi3[0], p1.x);
                lo3[1] = fmin(lo3[1], p1.y), hi3[1] = fmax(hi3[1], p1.y);
                lo3[2] = fmin(lo3[2], p1.z), hi3[2] = fmax(hi3[2], p1.z);
                if (P.ccd_x1) {  // certification: swept from x to x1
                    const d3 p2 = ld3(P.ccd_x1, va[k]);
                    lo3[0] = fmin(lo3[0], p2.x), hi3[0] = fmax(hi3[0], p2.x);
                    lo3[1] = fmin(lo3[1], p2.y), hi3[1] = fmax(hi3[1], p2.y);
                    lo3[2] = fmin(lo3[2], p2.z), hi3[2] = fmax(hi3[2], p2.z);
                }
            }
            // float box of the query inflated by d_max (certification: 1e-12 on
            // both boxes), rounded outwards
            const double dinfl = P.ccd_x1 ? 1e-12 : dinfl_all;
            qlo = make_float4(__double2float_rd(lo3[0] - dinfl), __double2float_rd(lo3[1] - dinfl),
                              __double2float_rd(lo3[2] - dinfl), 0.f);
            qhi = make_float4(__double2float_ru(hi3[0] + dinfl), __double2float_ru(hi3[1] + dinfl),
                              __double2float_ru(hi3[2] + dinfl), 0.f);
            const float mag = fmaxf(fmaxf(fmaxf(fabsf(qlo.x), fabsf(qhi.x)), fmaxf(fabsf(qlo.y), fabsf(qhi.y))),
                                    fmaxf(fabsf(qlo.z), fabsf(qhi.z)));
            dinf_q = dinf_f - (1e-6f + 3e-7f * mag);  // the gap lower bounds, less the float slack
        }
        // canonical partners only: EE (a = lower edge index) and VV (a < b)
        const bool ordered = (ka == KE) || (ka == KV && kb == KV);
        int qn = 0;  // queued candidates (warp-uniform)
        auto flush = [&](bool all) {
            while (qn >= 32 || (all && qn > 0)) {
                const int take = min(qn, 32);
                unsigned long long gb = 0;
                if (lane == 0) gb = atomicAdd(&P.g->ncand, (unsigned long long)take);
                gb = __shfl_sync(0xffffffffu, gb, 0);
                if (lane < take && (long long)(gb + lane) < P.ccap) {
                    const int2 e = cq[warp][qn - take + lane];
                    P.cand[gb + lane] = e;
                }
                if (lane == 0 && (long long)(gb + take) > P.ccap) atomicOr(&P.g->error, ERR_CAP_CAND);
                qn -= take;
                __syncwarp();
            }
        };
        auto leaf = [&](bool hit, int ib) {
            const bool take = hit && !(ordered && ib <= ia);
            const unsigned m = __ballot_sync(0xffffffffu, take);
            if (take) cq[warp][qn + __popc(m & lt)] = make_int2((int)q, ib);
            qn += __popc(m);
            __syncwarp();
            if (qn >= 32) flush(false);
        };
        if (B.n > 0 && __any_sync(0xffffffffu, ia >= 0)) {
            int sp = 0;
            if (lane == 0) stack[0] = 0;
            sp = 1;
            __syncwarp();
            auto push = [&](int ref) {
                if (sp < TRAV_STACK) {
                    if (lane == 0) stack[sp] = ref;
                    ++sp;
                } else if (lane == 0) {
                    atomicOr(&P.g->error, ERR_CAP_STACK);
                }
            };
            // ordered classes (EE, VV) only need partners above the query's own index:
            // subtrees whose largest index is <= ia are skipped
            const int need = ordered ? ia : -0x7fffffff - 1;
            auto visit = [&](float4 l0, float4 h0, float4 l1, float4 h1) {
                const int r0 = __float_as_int(l0.w), r1 = __float_as_int(l1.w);
                // leaves (ref < 0, warp-uniform) also pass the Euclidean test
                bool hit0 = box_hit(qlo, qhi, l0, h0) && __float_as_int(h0.w) > need;
                bool hit1 = box_hit(qlo, qhi, l1, h1) && __float_as_int(h1.w) > need;
                if (r0 < 0) hit0 = hit0 && box_near(qlo, qhi, l0, h0, dinf_q, d2_f);
                if (r1 < 0) hit1 = hit1 && box_near(qlo, qhi, l1, h1, dinf_q, d2_f);
                const bool any0 = __any_sync(0xffffffffu, hit0), any1 = __any_sync(0xffffffffu, hit1);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    if (!(k ? any1 : any0)) continue;
                    const int ref = k ? r1 : r0;
                    if (ref < 0) leaf(k ? hit1 : hit0, ~ref);
                    else push(ref);
                }
            };
            while (sp > 0) {
#if TW_WALK_PAIRS
                // two nodes per step when the stack holds two: their child boxes
                // load together, halving the dependent load chain of the walk
                if (sp >= 2) {
                    const int na = stack[sp - 1], nb = stack[sp - 2];
                    sp -= 2;
                    __syncwarp();
                    const float4* da = B.node + 4LL * na;
                    const float4* db = B.node + 4LL * nb;
                    const float4 a0 = da[0], a1 = da[1], a2 = da[2], a3 = da[3];
                    const float4 b0 = db[0], b1 = db[1], b2 = db[2], b3 = db[3];
                    visit(a0, a1, a2, a3);
                    visit(b0, b1, b2, b3);
                    __syncwarp();
                    continue;
                }
#endif
                const int node = stack[--sp];
                __syncwarp();
                const float4* nd = B.node + 4LL * node;  // both child boxes: one 64 B line
                visit(nd[0], nd[1], nd[2], nd[3]);
                __syncwarp();
            }
            flush(true);
        }
    }
}

// A2b: the exact narrow-phase test of every candidate (all lanes busy);
// survivors are appended to their query's partner list.
__device__ void ph_cand_eval(const Params& P) {
    const long long n = min((long long)P.g->ncand, P.ccap);
    long long evals = 0;
    for (long long i = gtid(); i < n; i += gstride()) {
        const int2 e = P.cand[i];
        int ka, ia, kb, cls;
        query_of(P, e.x, &ka, &ia, &kb, &cls);
        Closest c;
        ++evals;
        bool keep = false;
        if (!with_pair_class(ka, kb, [&](auto pc) {
                keep = candidate_keep_t<decltype(pc)::ka, decltype(pc)::kb>(P, ia, e.y, c);
            })) {
            int va[3];
            simplex_ids(P, ka, ia, va);
            keep = candidate_keep(P, ka, ia, va, kb, e.y, c);
        }
        if (keep) {
            const int pos = atomicAdd(&P.qcount[e.x], 1);
            if (pos < P.K) {
                P.qslot[(long long)e.x * P.K + pos] = e.y;
            } else {
                atomicOr(&P.g->error, ERR_CAP_SLOTS);
                atomicMax(&P.g->needed_k, pos + 1);
            }
        }
    }
    const long long ev = block_sum(evals);
    if (threadIdx.x == 0) atomicAdd((unsigned long long*)&P.g->pairs_evaluated, (unsigned long long)ev);
}

// A2c: per-block totals of the query counts over the block's chunk (the
// chunking ph_emit_pairs uses), and the key order of each query's partners
// (one warp per query, queries handed out dynamically)
__device__ void ph_query_totals(const Params& P) {
    const long long nq = num_queries(P);
    long long lo, hi;
    chunk_of(nq, &lo, &hi);
    long long s = 0;
    for (long long q = lo + threadIdx.x; q < hi; q += TPB) s += min(P.qcount[q], P.K);
    const long long tot = block_sum(s);
    if (threadIdx.x == 0) P.part_q[blockIdx.x] = tot;
    // K <= 128: ph_emit_pairs sorts each list in registers as it writes it
    // out. Larger K: the lists are sorted here, one warp per list.
    if (P.K <= 32 * SORT_R) return;
    const int lane = threadIdx.x & 31;
    for (;;) {
        long long qb = 0;
        if (lane == 0) qb = (long long)atomicAdd(&P.g->work_s, 32ull);
        qb = __shfl_sync(0xffffffffu, qb, 0);
        if (qb >= nq) break;
        const int cnt = P.qcount[qb + lane];
        unsigned todo = __ballot_sync(0xffffffffu, cnt >= 2 && cnt <= P.K);
        while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            sort_partners(P.qslot + (qb + j) * P.K, __shfl_sync(0xffffffffu, cnt, j), lane);
        }
    }
}

__device__ __forceinline__ void vertex_min(const Params& P, int v, double d) {
    const unsigned long long b = to_b(d);
    // The bound only decreases, so skip the atomic when it cannot lower it. A
    // plain (L1-cacheable) read: within the phase a stale copy is only ever
    // larger than the current bound (the atomic then runs needlessly), and
    // the grid barrier's fences order it after the reset of the previous step.
    if (b < P.dmin[v]) atomicMin(&P.dmin[v], b);
}

// contact predicate of linearize_all (constraints.cpp:186-199): active,
// not all static, inside the activation window, non-degenerate jacobian
__device__ __forceinline__ bool contact_pred(const Params& P, int ka, int kb, const int* va,
                                             const int* vb, const double4& dd, const double4& w,
                                             uint8_t flags) {
    if (!(flags & PF_ACTIVE) || (flags & PF_ALL_STATIC)) return false;
    if (!(dd.w < P.cfg.delta)) return false;
    double wa[3], wb[3];
    unpack_weights(ka, kb, w, wa, wb);
    Row c;
    build_contact(ka, va, kb, vb, wa, wb, dd.w, mk(dd.x, dd.y, dd.z), P.cfg.delta, P.cfg.family,
                  XLoad{P.x}, c);
    return !(row_jnorm(c) < 1e-28);
}

// A3: prefix the per-query counts and write the pair keys in key order (the
// query order is the key order of (ka, kb, ia), the partners of a query are
// sorted by the traversal); reset the refit flags.
__device__ void ph_emit_pairs(const Params& P) {
    const long long nq = num_queries(P);
    long long lo, hi;
    chunk_of(nq, &lo, &hi);
    const long long total = prefix_of(P.part_q, gridDim.x);
    if (total > P.pcap) {
        if (threadIdx.x == 0 && blockIdx.x == 0) {
            atomicOr(&P.g->error, ERR_CAP_PAIRS);
            P.g->needed_pairs = total;
        }
        return;
    }
    const int lane = threadIdx.x & 31;
    long long base = prefix_of(P.part_q, blockIdx.x);
    for (long long t = lo; t < hi; t += TPB) {
        const long long q = t + threadIdx.x;
        const int cnt = q < hi ? min(P.qcount[q], P.K) : 0;
        long long tile_tot;
        const long long off = base + block_scan(cnt, &tile_tot);
        base += tile_tot;
        if (P.K <= 32 * SORT_R) {
            // the warp writes the keys of its 32 queries, SORT_L lists at a
            // time: each list is loaded into registers, sorted in lockstep with
            // the others and written out as keys
            unsigned todo = __ballot_sync(0xffffffffu, cnt > 0);
            while (todo) {
                int ns[SORT_L], v[SORT_L][SORT_R];
                long long os[SORT_L];
                uint64_t kbase[SORT_L];
                int nmax = 0;
#pragma unroll
                for (int i = 0; i < SORT_L; ++i) {
                    ns[i] = 0, os[i] = 0, kbase[i] = 0;
#pragma unroll
                    for (int r = 0; r < SORT_R; ++r) v[i][r] = 0x7fffffff;
                    if (todo) {
                        const int j = __ffs(todo) - 1;
                        todo &= todo - 1;
                        ns[i] = __shfl_sync(0xffffffffu, cnt, j);
                        os[i] = __shfl_sync(0xffffffffu, off, j);
                        const long long qj = __shfl_sync(0xffffffffu, q, j);
                        int ka, ia, kb, cls;
                        query_of(P, qj, &ka, &ia, &kb, &cls);
                        kbase[i] = pair_key(ka, ia, kb, 0);
                        const int* sl = P.qslot + qj * P.K;
#pragma unroll
                        for (int r = 0; r < SORT_R; ++r)
                            if (r * 32 + lane < ns[i]) v[i][r] = sl[r * 32 + lane];
                        nmax = max(nmax, ns[i]);
                    }
                }
                if (nmax > 64) bitonic_lists<4>(v, lane);
                else if (nmax > 32) bitonic_lists<2>(v, lane);
                else if (nmax > 1) bitonic_lists<1>(v, lane);
#pragma unroll
                for (int i = 0; i < SORT_L; ++i)
#pragma unroll
                    for (int r = 0; r < SORT_R; ++r)
                        if (r * 32 + lane < ns[i]) P.pkey[os[i] + r * 32 + lane] = kbase[i] | uint64_t(uint32_t(v[i][r]));
            }
            continue;
        }
        // the warp writes the keys of its 32 queries, lanes over the partners
        for (int j = 0; j < 32; ++j) {
            const int cj = __shfl_sync(0xffffffffu, cnt, j);
            if (cj == 0) continue;
            const long long oj = __shfl_sync(0xffffffffu, off, j);
            const long long qj = __shfl_sync(0xffffffffu, q, j);
            int ka, ia, kb, cls;
            query_of(P, qj, &ka, &ia, &kb, &cls);
            const int* s = P.qslot + qj * P.K;
            for (int k = lane; k < cj; k += 32) P.pkey[oj + k] = pair_key(ka, ia, kb, s[k]);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) P.g->np = total;
    // reset refit flags for the next search
    for (int cls = 0; cls < 3; ++cls) {
        const Bvh& B = P.bvh[cls];
        for (long long j = gtid(); j < (long long)B.n - 1; j += gstride()) B.flag[j] = 0u;
    }
}

// A3b: the pair records, balanced over the output: CTA b writes pairs
// [b P / nb, (b+1) P / nb), each decoded from its key.
// one pair record for a compile-time pair class
template <int KA, int KB>
__device__ __forceinline__ bool emit_record_t(const Params& P, long long p, uint64_t key, int& touching,
                                              bool first_search) {
    int va[3], vb[3];
    simplex_ids_t<KA>(P, key_ia(key), va);
    simplex_ids_t<KB>(P, key_ib(key), vb);
    Closest c;
    pair_closest_t<KA, KB>(va, vb, XLoad{P.x}, c);
    const int4 ids = KA == KE ? make_int4(va[0], va[1], vb[0], vb[1]) : make_int4(va[0], vb[0], vb[1], vb[2]);
    bool all_static = true;
#pragma unroll
    for (int k = 0; k <= KA; ++k) all_static &= P.inv_mass[va[k]] == 0.0;
#pragma unroll
    for (int k = 0; k <= KB; ++k) all_static &= P.inv_mass[vb[k]] == 0.0;
    uint8_t fl = PF_ACTIVE | (all_static ? PF_ALL_STATIC : 0) | (c.degenerate ? PF_DEGENERATE : 0);
    const double4 dd = make_double4(c.dir.x, c.dir.y, c.dir.z, c.dist);
    const double4 w = pack_weights(KA, KB, c);
    if (!all_static && dd.w < P.cfg.delta) {  // contact_pred's own early exits, checked first
        int a3[3] = {va[0], va[1], va[2]}, b3[3] = {vb[0], vb[1], vb[2]};
        if (contact_pred(P, KA, KB, a3, b3, dd, w, fl)) fl |= PF_CONTACT;
    }
    P.pids[p] = ids;
    P.pdd[p] = dd;
    if (P.pw_all || (fl & PF_CONTACT)) P.pw[p] = w;  // weights are read for contact rows only
    P.pflag[p] = fl;
#pragma unroll
    for (int k = 0; k <= KA; ++k) vertex_min(P, va[k], c.dist);
#pragma unroll
    for (int k = 0; k <= KB; ++k) vertex_min(P, vb[k], c.dist);
    if (first_search && c.dist < 1e-10) touching = 1;
    return (fl & PF_CONTACT) != 0;
}

// A3b: the pair records, balanced over the output: CTA b writes pairs
// [b P / nb, (b+1) P / nb), each decoded from its key.
__device__ void ph_emit_records(const Params& P, bool first_search) {
    const long long np = P.g->np;
    int touching = 0;
    for_pair_tiles(P, np, [&](long long p) -> bool {
        const uint64_t key = P.pkey[p];
        const int ka = key_ka(key), kb = key_kb(key);
        bool contact = false;
        if (with_pair_class(ka, kb, [&](auto pc) {
                contact = emit_record_t<decltype(pc)::ka, decltype(pc)::kb>(P, p, key, touching, first_search);
            }))
            return contact;
        const int ia = key_ia(key), ib = key_ib(key);
        int va[3], vb[3];
        simplex_ids(P, ka, ia, va);
        simplex_ids(P, kb, ib, vb);
        Closest c;
        pair_closest(ka, va, kb, vb, XLoad{P.x}, c);
        const int4 ids = ka == KE ? make_int4(va[0], va[1], vb[0], vb[1]) : make_int4(va[0], vb[0], vb[1], vb[2]);
        bool all_static = true;
        for (int k = 0; k <= ka; ++k) all_static &= P.inv_mass[va[k]] == 0.0;
        for (int k = 0; k <= kb; ++k) all_static &= P.inv_mass[vb[k]] == 0.0;
        uint8_t fl = PF_ACTIVE | (all_static ? PF_ALL_STATIC : 0) | (c.degenerate ? PF_DEGENERATE : 0);
        const double4 dd = make_double4(c.dir.x, c.dir.y, c.dir.z, c.dist);
        const double4 w = pack_weights(ka, kb, c);
        if (contact_pred(P, ka, kb, va, vb, dd, w, fl)) fl |= PF_CONTACT;
        P.pids[p] = ids;
        P.pdd[p] = dd;
        if (P.pw_all || (fl & PF_CONTACT)) P.pw[p] = w;
        P.pflag[p] = fl;
        for (int k = 0; k <= ka; ++k) vertex_min(P, va[k], c.dist);
        for (int k = 0; k <= kb; ++k) vertex_min(P, vb[k], c.dist);
        if (first_search && c.dist < 1e-10) touching = 1;
        return (fl & PF_CONTACT) != 0;
    });
    const long long touch = block_sum(touching);
    if (threadIdx.x == 0 && touch) P.g->start_in_contact = 1;
}

// ============================================================== archive
__device__ __forceinline__ long long arch_lower_bound(const uint64_t* keys, long long n, uint64_t k) {
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (keys[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ============================================================ rows (B2)
// Vertex -> contact-row incidence, built per step as CSR: B2 takes a slot per
// (row, dynamic vertex) entry, then counts are scanned (ph_inc_totals,
// ph_inc_offsets) and entries scattered (ph_inc_scatter); ph_warm sorts each
// vertex segment by entry id (= row order).
__device__ __forceinline__ void record_incidence(const Params& P, int v, int entry) {
    P.c_slot[entry] = atomicAdd(&P.vcnt[v], 1);
}

// edge-length row at x (constraints.cpp:144-173) + fill_diag + q
__device__ __forceinline__ void edge_row(const Params& P, int e) {
    const int2 ed = P.edges[e];
    const double4 xi4 = P.x[ed.x], xj4 = P.x[ed.y];
    const d3 xi = mk(xi4.x, xi4.y, xi4.z), xj = mk(xj4.x, xj4.y, xj4.z);
    const double ly = P.ly[e];
    const d3 d = sub(xi, xj);
    const double len = nrm(d);
    const double value = P.cfg.sigma - len / ly;
    d3 g = mk(0, 0, 0), j0 = mk(0, 0, 0);
    if (len > 1e-12) {
        const d3 u = dvd(d, len);
        g = dvd(u, ly);
        j0 = dvd(neg(u), ly);
    }
    double dg = 0.0;
    dg += xi4.w * sqn(j0);
    dg += xj4.w * sqn(g);
    const double diag = maxd(dg, 1e-10);
    const d3 yi = ld3(P.yk1, ed.x), yj = ld3(P.yk1, ed.y);
    double q = value;
    q += dot(j0, sub(yi, xi));
    q += dot(g, sub(yj, xj));
    P.er_value[e] = value;
    P.er_g[e] = make_double4(g.x, g.y, g.z, diag);
    P.er_q[e] = q;
}

// jacobian block of edge row e at vertex slot m (0: -u/ly, 1: u/ly)
__device__ __forceinline__ d3 edge_jac(const double4& g4, int m) {
    const d3 g = mk(g4.x, g4.y, g4.z);
    if (m == 1) return g;
    if (g.x == 0.0 && g.y == 0.0 && g.z == 0.0) return g;  // len <= 1e-12: zero rows
    return neg(g);
}

// B2: order-preserving compaction of the contact rows (pair order), their
// q = c + J (y_k1 - x), warm-start multiplier from the archive, vertex
// incidence lists; plus every edge row's value / jacobian / diag / q.
__device__ void ph_rows(const Params& P) {
    const long long np = P.g->np, ntile = pair_tiles(np);
    const long long nc_total = prefix_of(P.part_c, (int)ntile);
    // pass 1: the contact pairs in pair order (= row order) over scan tiles of
    // TPB * 16 pairs (SUP pair tiles of the contact-flag pass): each thread
    // scans 16 consecutive pairs, one block scan per tile, and records the
    // pair of each row (c_arch holds it until ph_rows_build). The CTA's scan
    // tiles are blockIdx.x + k * grid: its first base is a prefix over
    // part_c, each next one adds the pair tiles in between.
    constexpr int PER = 16;
    constexpr long long SUP = (long long)PER / PAIR_PER, SCAN_TILE = PAIR_TILE * SUP;
    static_assert(PER % PAIR_PER == 0, "scan tiles are whole pair tiles");
    const long long nscan = (np + SCAN_TILE - 1) / SCAN_TILE;
    long long base = blockIdx.x < nscan ? prefix_of(P.part_c, (int)(blockIdx.x * SUP)) : 0;
    for (long long tile = blockIdx.x; tile < nscan; tile += gridDim.x) {
        if (tile != blockIdx.x) {
            long long s = 0;
            for (long long i = (tile - gridDim.x) * SUP + threadIdx.x; i < tile * SUP; i += TPB)
                s += ((volatile const long long*)P.part_c)[i];
            base += block_sum(s);
        }
        const long long lo = tile * SCAN_TILE, hi = min(np, lo + SCAN_TILE);
        const long long p0 = lo + (long long)threadIdx.x * PER;
        unsigned fm = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (p0 + j < hi && (P.pflag[p0 + j] & PF_CONTACT)) fm |= 1u << j;
        long long tile_tot;
        long long pos = base + block_scan(__popc(fm), &tile_tot);
        while (fm) {
            P.c_arch[pos++] = p0 + (__ffs(fm) - 1);
            fm &= fm - 1;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) P.g->nc = nc_total;
    if (P.cfg.edge_constraints)
        for (long long k = gtid(); k < P.g->ner; k += gstride()) edge_row(P, P.er_edge[k]);
}

// B2': the contact rows, one thread per row over the whole grid (the contact
// pairs cluster where the knot is tight: building them in their pair chunks
// left most CTAs idle)
__device__ void ph_rows_build(const Params& P, int sel, long long narch, long long nc) {
    const uint64_t* akey = P.arch_key[sel];
    const double* aval = P.arch_val[sel];
    for (long long pos = gtid(); pos < nc; pos += gstride()) {
        const long long p = P.c_arch[pos];
        const uint64_t key = P.pkey[p];
        const int ka = key_ka(key), kb = key_kb(key);
        int va[3], vb[3];
        split_ids(ka, kb, P.pids[p], va, vb);
        const double4 dd = P.pdd[p];
        double wa[3], wb[3];
        unpack_weights(ka, kb, P.pw[p], wa, wb);
        Row c;
        build_contact(ka, va, kb, vb, wa, wb, dd.w, mk(dd.x, dd.y, dd.z), P.cfg.delta, P.cfg.family,
                      XLoad{P.x}, c);
        // fill_diag (constraints.cpp:175-179) and q (lcp.cpp:16-20)
        double dg = 0.0, q = c.value;
        for (int m = 0; m < c.nverts; ++m) {
            const double4 xv = P.x[c.v[m]];
            dg += xv.w * sqn(c.jac[m]);
            q += dot(c.jac[m], sub(ld3(P.yk1, c.v[m]), mk(xv.x, xv.y, xv.z)));
        }
        double* J = P.c_jac + pos * 12;
        for (int m = 0; m < 4; ++m) {
            const d3 j = m < c.nverts ? c.jac[m] : mk(0, 0, 0);
            J[3 * m] = j.x, J[3 * m + 1] = j.y, J[3 * m + 2] = j.z;
        }
        P.c_ids[pos] = make_int4(c.v[0], c.nverts > 1 ? c.v[1] : -1, c.nverts > 2 ? c.v[2] : -1,
                                 c.nverts > 3 ? c.v[3] : -1);
        P.c_key[pos] = key;
        P.c_value[pos] = c.value;
        P.c_diag[pos] = maxd(dg, 1e-10);
        P.c_q[pos] = q;
        // warm start from the archive (resolve.cpp:86-93)
        const long long at = arch_lower_bound(akey, narch, key);
        double lam = 0.0;
        if (at < narch && akey[at] == key) {
            const double v = aval[at];
            lam = isnan(v) ? 0.0 : v;
            P.c_arch[pos] = at;
        } else {
            P.c_arch[pos] = -at - 1;
        }
        P.c_lambda[pos] = lam;
        for (int m = 0; m < 4; ++m) {
            const int e = (int)(pos * 4 + m);
            if (m < c.nverts && P.inv_mass[c.v[m]] > 0.0) record_incidence(P, c.v[m], e);
            else P.c_slot[e] = -1;
        }
    }
}

// B2b: per-block totals of the incidence counts over the block's vertex chunk
__device__ void ph_inc_totals(const Params& P) {
    long long lo, hi;
    chunk_of(P.nv, &lo, &hi);
    long long s = 0;
    for (long long v = lo + threadIdx.x; v < hi; v += TPB) s += P.vcnt[v];
    const long long t = block_sum(s);
    if (threadIdx.x == 0) P.part_v[blockIdx.x] = t;
}

// B2c: CSR offsets of the incidence
__device__ void ph_inc_offsets(const Params& P) {
    long long lo, hi;
    chunk_of(P.nv, &lo, &hi);
    long long base = prefix_of(P.part_v, blockIdx.x);
    for (long long t = lo; t < hi; t += TPB) {
        const long long v = t + threadIdx.x;
        const int c = v < hi ? P.vcnt[v] : 0;
        long long tt;
        const long long o = base + block_scan(c, &tt);
        base += tt;
        if (v < hi) P.voff[v] = (int)o;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) P.voff[P.nv] = (int)base;
}

// B2d: scatter the entries (4*row + m) into their vertex segments
__device__ void ph_inc_scatter(const Params& P, long long nc) {
    for (long long e = gtid(); e < 4 * nc; e += gstride()) {
        const int s = P.c_slot[e];
        if (s < 0) continue;
        const int v = (&P.c_ids[e >> 2].x)[e & 3];
        P.vinc[P.voff[v] + s] = (int)e;
    }
}

// in-place ascending sort of a vertex segment (insertion sort for short
// segments, heap sort for long ones; segments live in L1/L2)
__device__ __forceinline__ void sort_segment(int* a, int n) {
    if (n <= 48) {
        for (int i = 1; i < n; ++i) {
            const int v = a[i];
            int j = i - 1;
            while (j >= 0 && a[j] > v) a[j + 1] = a[j], --j;
            a[j + 1] = v;
        }
        return;
    }
    auto sift = [&](int root, int end) {
        while (2 * root + 1 < end) {
            int child = 2 * root + 1;
            if (child + 1 < end && a[child] < a[child + 1]) ++child;
            if (a[root] >= a[child]) return;
            const int t = a[root];
            a[root] = a[child];
            a[child] = t;
            root = child;
        }
    };
    for (int i = n / 2 - 1; i >= 0; --i) sift(i, n);
    for (int end = n - 1; end > 0; --end) {
        const int t = a[0];
        a[0] = a[end];
        a[end] = t;
        sift(0, end);
    }
}

// visit the (sorted) contact-row entries of v
template <typename F>
__device__ __forceinline__ void for_sorted_entries(const Params& P, int v, F&& f) {
    const int b = P.voff[v], e = P.voff[v + 1];
    for (int k = b; k < e; ++k) f(P.vinc[k]);
}

__device__ __forceinline__ void imp_add(d3& a, double s, d3 j) {
    a.x = a.x + s * j.x;
    a.y = a.y + s * j.y;
    a.z = a.z + s * j.z;
}

// B3: warm-start impulse M^-1 J^T lambda accumulated per vertex in row order
// (lcp.cpp:16-23: contact rows in pair order, then edge rows in edge order)
// and the coloring priorities of the contact rows
// edge-row part of the warm start at v (after its contact rows, lcp.cpp:16-23)
__device__ __forceinline__ void warm_edges(const Params& P, int v, double im, d3& a) {
    if (!P.cfg.edge_constraints) return;
    for (int k = P.vedge_off[v]; k < P.vedge_off[v + 1]; ++k) {
        const int e = P.vedge[k];
        if (!P.is_er[e]) continue;
        const double lam = P.edge_lambda[e];
        if (lam != 0.0) imp_add(a, im * lam, edge_jac(P.er_g[e], P.edges[e].x == v ? 0 : 1));
    }
}

// The vertices v = gwarp() + j * gwarps() (j = 0, 1, ...) for which take(v)
// holds, visited one at a time by the whole warp; the predicate is evaluated
// for 32 vertices at once (one load round instead of 32 dependent ones).
template <typename T, typename F>
__device__ __forceinline__ void for_warp_vertices(long long nv, T&& take, F&& f) {
    const int lane = threadIdx.x & 31;
    const long long w0 = gwarp(), G = gwarps();
    for (long long j0 = 0; w0 + j0 * G < nv; j0 += 32) {
        const long long v = w0 + (j0 + lane) * G;
        unsigned m = __ballot_sync(0xffffffffu, v < nv && take((int)v));
        while (m) {
            const int q = __ffs(m) - 1;
            m &= m - 1;
            f((int)(w0 + (j0 + q) * G));
        }
    }
}

// a += the lanes' terms t (where nz) in lane order, in every lane
__device__ __forceinline__ void warp_ordered_add(d3& a, const d3& t, bool nz) {
    const unsigned nzm = __ballot_sync(0xffffffffu, nz);
    for (int q = 0; q < 32; ++q) {
        if (!((nzm >> q) & 1u)) continue;
        const double tx = __shfl_sync(0xffffffffu, t.x, q);
        const double ty = __shfl_sync(0xffffffffu, t.y, q);
        const double tz = __shfl_sync(0xffffffffu, t.z, q);
        a.x = a.x + tx, a.y = a.y + ty, a.z = a.z + tz;
    }
}

// warm_edges with the terms formed by the lanes (same order and arithmetic)
__device__ __forceinline__ void warm_edges_warp(const Params& P, int v, double im, d3& a) {
    if (!P.cfg.edge_constraints) return;
    const int lane = threadIdx.x & 31;
    const int b = P.vedge_off[v], e1 = P.vedge_off[v + 1];
    for (int k0 = b; k0 < e1; k0 += 32) {
        const int k = k0 + lane;
        bool nz = false;
        d3 t = mk(0, 0, 0);
        if (k < e1) {
            const int e = P.vedge[k];
            if (P.is_er[e]) {
                const double lam = P.edge_lambda[e];
                if (lam != 0.0) {
                    const double sc = im * lam;
                    const d3 j = edge_jac(P.er_g[e], P.edges[e].x == v ? 0 : 1);
                    t = mk(sc * j.x, sc * j.y, sc * j.z);
                    nz = true;
                }
            }
        }
        warp_ordered_add(a, t, nz);
    }
}

// Vertices with contact entries are handled by one warp each (rank-by-counting
// sort of the segment in shared memory up to WARM_WARP_MAX entries, lane 0
// beyond; lanes form the terms, which are added in row order, then the edge
// terms in edge order); the others -- most vertices -- by one thread each.
constexpr int WARM_WARP_MAX = 256;

__device__ void ph_warm(const Params& P, long long nc, bool reset_colors = true) {
    static_assert(sizeof(int) * (TPB / 32) * WARM_WARP_MAX <= SCRATCH_BYTES, "");
    int(*sseg)[WARM_WARP_MAX] = reinterpret_cast<int(*)[WARM_WARP_MAX]>(smem_scratch());
    for (long long vl = gtid(); vl < P.nv; vl += gstride()) {
        const int v = (int)vl;
        const double im = P.inv_mass[v];
        if (!(im > 0.0) || P.voff[v + 1] == P.voff[v]) {
            d3 a = mk(0, 0, 0);
            if (im > 0.0) warm_edges(P, v, im, a);
            P.imp[v] = make_double4(a.x, a.y, a.z, im);  // w: inv_mass, read with the impulse by the PGS
        }
        if (P.cfg.coloring_mode == 1) {
            // device coloring: the vertex starts with the colors of its edge rows
            unsigned long long mk4[4] = {0, 0, 0, 0};
            int big = 0;
            if (im > 0.0 && P.cfg.edge_constraints)
                for (int q = P.vedge_off[v]; q < P.vedge_off[v + 1]; ++q) {
                    const int ec = P.edge_color[P.vedge[q]];
                    if (ec >= 256) big = 1;
                    else if (ec >= 0) mk4[ec >> 6] |= 1ull << (ec & 63);
                }
            for (int k = 0; k < 4; ++k) P.vmask[4LL * v + k] = mk4[k];
            P.vbig[v] = big;
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // (static vertices have no entries)
    for_warp_vertices(P.nv, [&](int v) { return P.voff[v + 1] > P.voff[v]; }, [&](int v) {
        const int b = P.voff[v], n = P.voff[v + 1] - b;
        const double im = P.inv_mass[v];
        int* seg = P.vinc + b;
        if (n <= WARM_WARP_MAX) {
            for (int i = lane; i < n; i += 32) sseg[w][i] = seg[i];
            __syncwarp();
            int rk[WARM_WARP_MAX / 32], ev[WARM_WARP_MAX / 32];
#pragma unroll
            for (int r = 0; r < WARM_WARP_MAX / 32; ++r) {
                const int i = lane + 32 * r;
                rk[r] = -1;
                if (i < n) {
                    const int e = sseg[w][i];
                    int c = 0;
                    for (int t = 0; t < n; ++t) c += sseg[w][t] < e;
                    rk[r] = c, ev[r] = e;
                }
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < WARM_WARP_MAX / 32; ++r)
                if (rk[r] >= 0) {
                    sseg[w][rk[r]] = ev[r];
                    seg[rk[r]] = ev[r];
                    P.erank[ev[r]] = rk[r];  // rank inside the vertex clique
                }
            __syncwarp();
        } else {
            if (lane == 0) {
                sort_segment(seg, n);
                for (int k = 0; k < n; ++k) P.erank[seg[k]] = k;
            }
            __syncwarp();
        }
        // ordered sum of the contact terms (lcp.cpp:16-23: contact rows in row order)
        d3 a = mk(0, 0, 0);
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            bool nz = false;
            d3 t = mk(0, 0, 0);
            if (k < n) {
                const int e = n <= WARM_WARP_MAX ? sseg[w][k] : seg[k];
                const int row = e >> 2, m = e & 3;
                const double lam = P.c_lambda[row];
                if (lam != 0.0) {
                    const double* J = P.c_jac + (long long)row * 12 + 3 * m;
                    const double sc = im * lam;
                    t = mk(sc * J[0], sc * J[1], sc * J[2]);
                    nz = true;
                }
            }
            warp_ordered_add(a, t, nz);
        }
        warm_edges_warp(P, v, im, a);
        if (lane == 0) P.imp[v] = make_double4(a.x, a.y, a.z, im);
        __syncwarp();
    });
    if (reset_colors)  // coloring state of the contact rows (colors given: keep them)
        for (long long i = gtid(); i < nc; i += gstride()) {
            P.c_stamp[i] = 0;
            P.c_lost[i] = 0;
            P.c_color[i] = -1;
        }
}

// ============================================================ coloring
// C (device mode), speculative greedy coloring in rounds; the lower row index
// (pair order) has priority, so a round reproduces the sequential greedy
// coloring in row order wherever it does not conflict. Round k:
//   rank     (vertex pass) every uncolored entry learns how many uncolored
//            entries precede it in its vertex segment (segments are sorted by
//            row index; round 1: its position, set by ph_warm);
//   propose  (row pass) an uncolored row proposes the rank-th color free at
//            all of its dynamic vertices (rank = max over the vertices), so
//            the rows of a clique propose distinct colors;
//   conflict (vertex pass) a proposal loses if an earlier uncolored entry of
//            one of its segments proposed the same color;
//   commit   (row pass) the winners take their color and mark it in the
//            color masks of their vertices.
// The oracle's or_color_device (oracle/or_constraints.c) states the same
// rounds row by row.

__device__ void ph_color_rank(const Params& P) {
    const int lane = threadIdx.x & 31;
    // vertices with no uncolored entry left are skipped
    for_warp_vertices(P.nv, [&](int v) { return P.vcnt[v] != 0; }, [&](int v) {
        const int b = P.voff[v], e = P.voff[v + 1];
        int run = 0;
        for (int t0 = b; t0 < e; t0 += 32) {
            const int t = t0 + lane;
            int ent = 0;
            bool unc = false;
            if (t < e) {
                ent = P.vinc[t];
                unc = P.c_stamp[ent >> 2] == 0;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, unc);
            if (unc) P.erank[ent] = run + __popc(bal & ((1u << lane) - 1u));
            run += __popc(bal);
        }
    });
}

__device__ void ph_color_conflict(const Params& P, int k) {
    __shared__ unsigned long long seen[TPB / 32][4];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // vertices with no uncolored entry left (also: empty segments) are skipped
    for_warp_vertices(P.nv, [&](int v) { return P.vcnt[v] != 0; }, [&](int v) {
        const int b = P.voff[v], e = P.voff[v + 1];
        if (lane < 4) seen[w][lane] = 0ull;
        __syncwarp();
        for (int t0 = b; t0 < e; t0 += 32) {
            const int t = t0 + lane;
            int row = -1, tc = -1;
            if (t < e) {
                row = P.vinc[t] >> 2;
                if (P.c_stamp[row] == 0) tc = P.c_tent[row];
            }
            const bool unc = tc >= 0;
            const unsigned um = __ballot_sync(0xffffffffu, unc);
            const unsigned peers = __match_any_sync(0xffffffffu, tc);
            if (unc) {
                bool dup = (peers & um & ((1u << lane) - 1u)) != 0u;
                if (!dup) {
                    if (tc < 256) {
                        dup = (seen[w][tc >> 6] >> (tc & 63)) & 1ull;
                    } else {
                        for (int s = b; s < t0 && !dup; ++s) {
                            const int r2 = P.vinc[s] >> 2;
                            dup = P.c_stamp[r2] == 0 && P.c_tent[r2] == tc;
                        }
                    }
                }
                if (dup) P.c_lost[row] = k;
            }
            __syncwarp();
            if (unc && tc < 256) atomicOr(&seen[w][tc >> 6], 1ull << (tc & 63));
            __syncwarp();
        }
    });
}

__device__ void ph_color_commit(const Params& P, long long nc, int k) {
    int ncolored = 0, maxc = -1;
    for (long long i = gtid(); i < nc; i += gstride()) {
        if (P.c_stamp[i] != 0 || P.c_lost[i] == k) continue;
        const int ti = P.c_tent[i];
        P.c_color[i] = ti;
        P.c_stamp[i] = k;
        ++ncolored;
        maxc = max(maxc, ti);
        if (ti < P.colcap) atomicAdd(&P.ccount[ti], 1);
        else atomicOr(&P.g->error, ERR_CAP_COLORS);
        const int4 id = P.c_ids[i];
        const int vv[4] = {id.x, id.y, id.z, id.w};
        for (int m = 0; m < 4; ++m) {
            const int v = vv[m];
            if (v < 0 || !(P.inv_mass[v] > 0.0)) continue;
            if (ti < 256) atomicOr(&P.vmask[4LL * v + (ti >> 6)], 1ull << (ti & 63));
            else P.vbig[v] = 1;
            atomicSub(&P.vcnt[v], 1);  // uncolored entries left at v
        }
    }
    const int wn = __reduce_add_sync(0xffffffffu, (unsigned)ncolored);
    const int wm = __reduce_max_sync(0xffffffffu, maxc);
    if ((threadIdx.x & 31) == 0 && wn > 0) {
        atomicAdd(&P.g->colored, wn);
        atomicMax(&P.g->max_color, wm);
    }
}

__device__ void ph_color_propose(const Params& P, long long nc, int k) {
    for (long long i = gtid(); i < nc; i += gstride()) {
        if (P.c_stamp[i] != 0) continue;
        const int4 id = P.c_ids[i];
        const int vv[4] = {id.x, id.y, id.z, id.w};
        unsigned long long used[4] = {0, 0, 0, 0};
        bool big = false;
        int rank = 0;  // max over vertices of the uncolored rows there that beat this row
        for (int m = 0; m < 4; ++m) {
            const int v = vv[m];
            if (v < 0 || !(P.inv_mass[v] > 0.0)) continue;
            rank = max(rank, P.erank[4 * i + m]);
            const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(P.vmask + 4LL * v);
            const ulonglong2 c = *reinterpret_cast<const ulonglong2*>(P.vmask + 4LL * v + 2);
            used[0] |= a.x, used[1] |= a.y, used[2] |= c.x, used[3] |= c.y;
            big |= P.vbig[v] != 0;
        }
        // propose the rank-th free color: a clique of uncolored rows takes
        // distinct colors in priority order within one round
        int col = -1, left = rank;
        for (int w = 0; w < 4 && col < 0; ++w) {
            unsigned long long free_bits = ~used[w];
            const int nfree = __popcll(free_bits);
            if (left >= nfree) {
                left -= nfree;
                continue;
            }
            for (int t = 0; t < left; ++t) free_bits &= free_bits - 1;  // drop the lowest `left` free bits
            col = w * 64 + __ffsll(free_bits) - 1;
        }
        if (col < 0 && !big) col = 256 + left;
        if (col < 0 || (big && col >= 256)) {
            // > 256 colors around this row: linear search over the neighborhood
            for (int c = 256;; ++c) {
                bool hit = c < 256 ? ((used[c >> 6] >> (c & 63)) & 1) : false;
                for (int m = 0; m < 4 && !hit; ++m) {
                    const int v = vv[m];
                    if (v < 0 || !(P.inv_mass[v] > 0.0)) continue;
                    for (int t = P.voff[v]; t < P.voff[v + 1] && !hit; ++t) {
                        const int j = P.vinc[t] >> 2;
                        if (j == i) continue;
                        const int sj = P.c_stamp[j];
                        hit = sj >= 1 && sj < k && P.c_color[j] == c;
                    }
                    if (P.cfg.edge_constraints)
                        for (int q = P.vedge_off[v]; q < P.vedge_off[v + 1] && !hit; ++q)
                            hit = P.edge_color[P.vedge[q]] == c;
                }
                if (!hit && left-- == 0) {
                    col = c;
                    break;
                }
            }
        }
        P.c_tent[i] = col;
    }
}

// ----------------------------------------------- reference coloring replica
// mt19937_64 (single device thread)
struct Mt64 {
    unsigned long long mt[312];
    int idx;
    __device__ void seed(unsigned long long s) {
        mt[0] = s;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
        idx = 312;
    }
    __device__ unsigned long long next() {
        if (idx >= 312) {
            const unsigned long long upper = ~0ull << 31, lower = ~upper;
            for (int k = 0; k < 312; ++k) {
                const unsigned long long y = (mt[k] & upper) | (mt[(k + 1) % 312] & lower);
                mt[k] = mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ull : 0ull);
            }
            idx = 0;
        }
        unsigned long long z = mt[idx++];
        z ^= (z >> 29) & 0x5555555555555555ull;
        z ^= (z << 17) & 0x71D67FFFEDA60000ull;
        z ^= (z << 37) & 0xFFF7EEE000000000ull;
        z ^= z >> 43;
        return z;
    }
    // libstdc++ uniform_int_distribution<size_t>(0, range-1): Lemire _S_nd
    __device__ unsigned long long below(unsigned long long range) {
        unsigned long long g = next();
        unsigned long long low = g * range, high = __umul64hi(g, range);
        if (low < range) {
            const unsigned long long thr = (0ull - range) % range;
            while (low < thr) {
                g = next();
                low = g * range;
                high = __umul64hi(g, range);
            }
        }
        return high;
    }
};

// C (reference mode): color_constraints (constraints.cpp:222-288) replayed on
// one thread over contact rows [0, nc) and edge rows [nc, nc + ner).
#define TW_INVARIANT(cond)                   \
    if (!(cond)) {                           \
        atomicOr(&P.g->error, ERR_INTERNAL); \
        P.g->internal_line = __LINE__;       \
        return;                              \
    }

// The reference coloring's conflict graph (constraints.cpp:229-244: rows that
// share a dynamic vertex; sorted, unique neighbour lists), built by the whole
// grid before the sequential replay: row r's candidate list lives at
// pool[2R + 2 + off(r)] with off = the exclusive prefix of the candidate counts
// (chunked per CTA), sorted and deduplicated in place; its length goes to
// pool[R + 1 + r]. The lists need not be contiguous.
__device__ __forceinline__ int ref_row_verts(const Params& P, long long nc, long long r, int* v) {
    if (r < nc) {
        const int4 id = P.c_ids[r];
        v[0] = id.x, v[1] = id.y, v[2] = id.z, v[3] = id.w;
        int n = 0;
        while (n < 4 && v[n] >= 0) ++n;
        return n;
    }
    const int2 e = P.edges[P.er_edge[r - nc]];
    v[0] = e.x, v[1] = e.y;
    return 2;
}

__device__ __forceinline__ long long ref_candidates(const Params& P, long long nc, long long r) {
    int vv[4];
    const int n = ref_row_verts(P, nc, r, vv);
    long long c = 0;
    for (int m = 0; m < n; ++m) {
        const int v = vv[m];
        if (!(P.inv_mass[v] > 0.0)) continue;
        c += P.voff[v + 1] - P.voff[v];
        if (P.cfg.edge_constraints)
            for (int q = P.vedge_off[v]; q < P.vedge_off[v + 1]; ++q) c += P.is_er[P.vedge[q]];
    }
    return c;
}

__device__ void ph_color_ref_count(const Params& P, long long nc) {
    const long long R = nc + P.g->ner;
    long long lo, hi;
    chunk_of(R, &lo, &hi);
    long long s = 0;
    for (long long r = lo + threadIdx.x; r < hi; r += TPB) s += ref_candidates(P, nc, r);
    const long long t = block_sum(s);
    if (threadIdx.x == 0) P.part_k[blockIdx.x] = t;
}

__device__ void ph_color_ref_fill(const Params& P, long long nc) {
    const long long R = nc + P.g->ner;
    int* pool = P.refpool;
    int* adj_off = pool;          // R + 1
    int* adj_len = pool + R + 1;  // R
    int* lists = pool + 2 * R + 2;
    const long long total = prefix_of(P.part_k, gridDim.x);
    if (2 * R + 2 + total > P.refpool_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&P.g->error, ERR_CAP_REFPOOL);
        return;
    }
    long long lo, hi;
    chunk_of(R, &lo, &hi);
    long long base = prefix_of(P.part_k, blockIdx.x);
    for (long long t0 = lo; t0 < hi; t0 += TPB) {
        const long long r = t0 + threadIdx.x;
        const long long c = r < hi ? ref_candidates(P, nc, r) : 0;
        long long tile;
        const long long ex = block_scan(c, &tile);
        if (r < hi) {
            const long long start = base + ex;
            adj_off[r] = (int)start;
            int* L = lists + start;
            int len = 0;
            int vv[4];
            const int n = ref_row_verts(P, nc, r, vv);
            for (int m = 0; m < n; ++m) {
                const int v = vv[m];
                if (!(P.inv_mass[v] > 0.0)) continue;
                for (int t = P.voff[v]; t < P.voff[v + 1]; ++t) {
                    const long long j = P.vinc[t] >> 2;
                    if (j != r) L[len++] = (int)j;
                }
                if (P.cfg.edge_constraints)
                    for (int q = P.vedge_off[v]; q < P.vedge_off[v + 1]; ++q) {
                        const int e = P.vedge[q];
                        if (!P.is_er[e]) continue;
                        const long long j = nc + P.er_index[e];
                        if (j != r) L[len++] = (int)j;
                    }
            }
            for (int i = 1; i < len; ++i) {  // insertion sort + unique
                const int x = L[i];
                int j = i - 1;
                while (j >= 0 && L[j] > x) L[j + 1] = L[j], --j;
                L[j + 1] = x;
            }
            int w = 0;
            for (int i = 0; i < len; ++i)
                if (i == 0 || L[i] != L[i - 1]) L[w++] = L[i];
            adj_len[r] = w;
        }
        base += tile;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) adj_off[R] = (int)total;
}

// The smallest-last peel and the greedy pass of constraints.cpp:245-287 on
// warp 0 of CTA 0. The order-carrying parts stay sequential (the random pick,
// swap-pop, on lane 0); the per-neighbour work of a picked row is spread over
// the 32 lanes with every bucket append landing at the position the sequential
// loop would give it (lanes grouped by target bucket, ranked by neighbour
// order: a bucket's contents and order are exactly the reference's), and the
// greedy pass marks neighbour colors in parallel and finds the first free
// color with ballots. Bit-identical to the one-thread replay (tests compare
// with the oracle / the reference build), several times faster.
__device__ void ph_color_ref(const Params& P, long long nc) {
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x;
    const unsigned lt_mask = (1u << lane) - 1u;
    const long long R = nc + P.g->ner;
    if (R == 0) {
        if (lane == 0) P.g->max_color = -1;
        return;
    }
    if (P.g->error) return;
    int* pool = P.refpool;
    const int* adj_start = pool;
    const int* adj_len = pool + R + 1;
    const int* adj = pool + 2 * R + 2;
    long long top = 2 * R + 2 + adj_start[R];  // identical on every lane (allocations are warp-uniform)
    bool bad = false;
    auto alloc = [&](long long n) -> int* {
        if (top + n > P.refpool_cap) {
            bad = true;
            return nullptr;
        }
        int* p = pool + top;
        top += n;
        return p;
    };
    int* degree = alloc(R);
    int* order = alloc(R);
    int* removed = alloc(R);
    int* used = alloc(R + 1);
    if (bad) {
        if (lane == 0) atomicOr(&P.g->error, ERR_CAP_REFPOOL);
        return;
    }
    int max_deg = 0;
    for (long long i = lane; i < R; i += 32) {
        degree[i] = adj_len[i];
        removed[i] = 0;
        max_deg = max(max_deg, adj_len[i]);
    }
    for (int o = 16; o > 0; o >>= 1) max_deg = max(max_deg, __shfl_xor_sync(FULL, max_deg, o));
    // buckets as growable vectors in the pool: (ptr offset, size, cap)
    int* bptr = alloc(max_deg + 1);
    int* bsize = alloc(max_deg + 1);
    int* bcap = alloc(max_deg + 1);
    if (bad) {
        if (lane == 0) atomicOr(&P.g->error, ERR_CAP_REFPOOL);
        return;
    }
    for (int d = lane; d <= max_deg; d += 32) bptr[d] = -1, bsize[d] = 0, bcap[d] = 0;
    __syncwarp();
    // Appends x to bucket d for every active lane, in lane order within a
    // bucket (= the sequential order of the pushes); a full bucket doubles
    // (4, 8, 16, ...) with its contents copied, as the sequential growth does.
    auto warp_push = [&](bool act, int d, int x) {
        unsigned m = __ballot_sync(FULL, act);
        while (m) {
            const int leader = __ffs(m) - 1;
            const int dl = __shfl_sync(FULL, d, leader);
            const unsigned grp = __ballot_sync(FULL, act && d == dl);
            const int cnt = __popc(grp);
            int base = 0, ptr = 0;
            if (lane == leader) {
                const int need = bsize[dl] + cnt;
                if (need > bcap[dl]) {
                    int cap = bcap[dl];
                    while (cap < need) cap = cap ? cap * 2 : 4;
                    int* nb = alloc(cap);
                    if (nb) {
                        for (int i = 0; i < bsize[dl]; ++i) nb[i] = pool[bptr[dl] + i];
                        bptr[dl] = (int)(nb - pool);
                        bcap[dl] = cap;
                    }
                }
                base = bsize[dl];
                ptr = bptr[dl];
                if (!bad) bsize[dl] = need;
            }
            top = __shfl_sync(FULL, top, leader);
            bad = __shfl_sync(FULL, bad ? 1 : 0, leader) != 0;
            base = __shfl_sync(FULL, base, leader);
            ptr = __shfl_sync(FULL, ptr, leader);
            if (!bad && act && d == dl) pool[ptr + base + __popc(grp & lt_mask)] = x;
            m &= ~grp;
        }
        __syncwarp();
    };
    for (long long i0 = 0; i0 < R && !bad; i0 += 32) {
        const long long i = i0 + lane;
        warp_push(i < R, i < R ? degree[i] : 0, (int)i);
    }
    if (bad) {
        if (lane == 0) atomicOr(&P.g->error, ERR_CAP_REFPOOL);
        return;
    }
    Mt64 rng;
    if (lane == 0) rng.seed(P.cfg.color_seed);
    for (long long picked = 0; picked < R; ++picked) {
        int cand = -1;
        if (lane == 0) {
            int d = 0;
            while (cand < 0) {
                while (d <= max_deg && bsize[d] == 0) ++d;
                if (d > max_deg) break;  // invariant broken (reported below)
                const unsigned long long at = rng.below((unsigned long long)bsize[d]);
                int* b = pool + bptr[d];
                const int c = b[at];
                if (c < 0 || c >= R) break;
                b[at] = b[bsize[d] - 1];
                --bsize[d];
                if (!removed[c] && degree[c] == d) cand = c;
            }
            if (cand >= 0) {
                removed[cand] = 1;
                order[picked] = cand;
            }
        }
        cand = __shfl_sync(FULL, cand, 0);
        __syncwarp();
        if (cand < 0) {  // the peel ran out of candidates: an invariant is broken
            if (lane == 0) {
                atomicOr(&P.g->error, ERR_INTERNAL);
                P.g->internal_line = __LINE__;
            }
            return;
        }
        const int k0 = adj_start[cand], k1 = k0 + adj_len[cand];
        for (int kb = k0; kb < k1 && !bad; kb += 32) {
            const int k = kb + lane;
            int nb = -1, nd = 0;
            bool act = false;
            if (k < k1) {
                nb = adj[k];
                if (!removed[nb]) {  // distinct neighbours: no two lanes touch one degree
                    nd = --degree[nb];
                    act = true;
                }
            }
            warp_push(act, nd, nb);
        }
        if (bad) {
            if (lane == 0) atomicOr(&P.g->error, ERR_CAP_REFPOOL);
            return;
        }
    }
    // colors: -1 initially
    for (long long r = lane; r < nc; r += 32) P.c_color[r] = -1;
    for (long long k = lane; k < P.g->ner; k += 32) P.er_color[P.er_edge[k]] = -1;
    for (long long i = lane; i <= R; i += 32) used[i] = -1;
    __syncwarp();
    auto color_of = [&](long long r) -> int {
        return r < nc ? P.c_color[r] : P.er_color[P.er_edge[r - nc]];
    };
    int maxc = -1;
    for (long long it = R - 1; it >= 0; --it) {
        const int i = order[it];
        for (int k = adj_start[i] + lane; k < adj_start[i] + adj_len[i]; k += 32) {
            const int c = color_of(adj[k]);
            if (c >= 0) used[c] = i;
        }
        __syncwarp();
        int col = -1;
        for (int c0 = 0; col < 0; c0 += 32) {  // used has R + 1 slots: a free color always exists
            const unsigned busy = __ballot_sync(FULL, c0 + lane <= R && used[c0 + lane] == i);
            const unsigned freeb = ~busy;
            if (freeb) col = c0 + __ffs(freeb) - 1;
        }
        if (lane == 0) {
            if (i < nc) P.c_color[i] = col;
            else P.er_color[P.er_edge[i - nc]] = col;
        }
        maxc = max(maxc, col);
        __syncwarp();
    }
    if (lane == 0) P.g->max_color = maxc;
}

// D: bucket rows by color. Contact counts ccount come from the coloring
// (device mode) or are counted here (reference mode, which also buckets the
// edge rows of this step).
__device__ void ph_bucket_count(const Params& P, long long nc) {
    for (long long i = gtid(); i < nc; i += gstride()) atomicAdd(&P.ccount[P.c_color[i]], 1);
    for (long long k = gtid(); k < P.g->ner; k += gstride())
        atomicAdd(&P.er_color_cnt[P.er_color[P.er_edge[k]]], 1);
}

__device__ void ph_bucket_scatter(const Params& P, long long nc, int ncol, bool edges_too) {
    // every block computes the color prefix (ncol is small); block 0 publishes
    long long run = 0;
    for (int base = 0; base < ncol; base += TPB) {
        const int c = base + threadIdx.x;
        const long long v = c < ncol ? P.ccount[c] : 0;
        long long tt;
        const long long ex = block_scan(v, &tt);
        if (blockIdx.x == 0 && c < ncol) P.coff[c] = (int)(run + ex);
        run += tt;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) P.coff[ncol] = (int)run;
    if (edges_too) {
        run = 0;
        for (int base = 0; base < ncol; base += TPB) {
            const int c = base + threadIdx.x;
            const long long v = c < ncol ? P.er_color_cnt[c] : 0;
            long long tt;
            const long long ex = block_scan(v, &tt);
            if (blockIdx.x == 0 && c < ncol) P.er_color_off[c] = (int)(run + ex);
            run += tt;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) P.er_color_off[ncol] = (int)run;
    }
}

__device__ void ph_bucket_place(const Params& P, long long nc, bool edges_too) {
    // counting down leaves the count tables zeroed for the next step
    const bool pack = P.cfg.solver == 0;
    for (long long i = gtid(); i < nc; i += gstride()) {
        const int c = P.c_color[i];
        const int slot = atomicSub(&P.ccount[c], 1) - 1;
        const long long pos = P.coff[c] + slot;
        P.c_by_color[pos] = (int)i;
        if (pack) {
            P.pk_ids[pos] = P.c_ids[i];
            const double2* s = reinterpret_cast<const double2*>(P.c_jac + i * 12);
            double2* d = reinterpret_cast<double2*>(P.pk_jac + pos * 12);
#pragma unroll
            for (int k = 0; k < 6; ++k) d[k] = s[k];
            P.pk_q[pos] = P.c_q[i];
            P.pk_diag[pos] = P.c_diag[i];
            P.pk_lam[pos] = P.c_lambda[i];
        }
    }
    if (edges_too)
        for (long long k = gtid(); k < P.g->ner; k += gstride()) {
            const int e = P.er_edge[k];
            const int c = P.er_color[e];
            const int slot = atomicSub(&P.er_color_cnt[c], 1) - 1;
            P.er_by_color[P.er_color_off[c] + slot] = e;
        }
}

// ================================================================= PGS
// pgs_sweeps (lcp.cpp:27-42) for one color. Rows of a color share no dynamic
// vertex, so the parallel update equals the sequential one bit for bit.
__device__ __forceinline__ void pgs_contact_row(const Params& P, int i) {
    const int4 id = P.c_ids[i];
    const int vv[4] = {id.x, id.y, id.z, id.w};
    const double* J = P.c_jac + (long long)i * 12;
    double s = 0.0;
    for (int m = 0; m < 4; ++m) {
        const int v = vv[m];
        if (v < 0 || !(P.inv_mass[v] > 0.0)) continue;
        const double4 a = P.imp[v];
        s += dot(mk(J[3 * m], J[3 * m + 1], J[3 * m + 2]), mk(a.x, a.y, a.z));
    }
    const double w = P.c_q[i] + s;
    const double lam0 = P.c_lambda[i];
    const double t = lam0 - w / P.c_diag[i];
    const double lam = 0.0 < t ? t : 0.0;
    const double d = lam - lam0;
    if (d != 0.0) {
        for (int m = 0; m < 4; ++m) {
            const int v = vv[m];
            if (v < 0) continue;
            const double im = P.inv_mass[v];
            if (!(im > 0.0)) continue;
            double4 a = P.imp[v];
            const double sc = im * d;
            a.x = a.x + sc * J[3 * m];
            a.y = a.y + sc * J[3 * m + 1];
            a.z = a.z + sc * J[3 * m + 2];
            P.imp[v] = a;
        }
    }
    P.c_lambda[i] = lam;
}

// The same row from its color-ordered copy (position pos of c_by_color):
// static row data is one coalesced read, each dynamic vertex's impulse (with
// its inverse mass in w) is gathered once and written back once.
// The row's static data (ids, q, diag, multiplier) can be loaded ahead, before
// the barrier that opens its color (PgsRow): after the barrier only the
// impulse gathers and the Jacobian load remain on the color's latency chain.
struct PgsRow {
    int color;      // the color this prefetch belongs to (-1: none)
    int edge;       // edge id for an edge row, -1 for a contact row
    long long pos;  // contact: position in the color-ordered copy
    int4 ids;       // contact: the row's vertices; edge: (v0, v1, -, -)
    double q, lam, diag;
    double3 u;      // edge: the unit direction of er_g
};

__device__ __forceinline__ void pgs_contact_pre(const Params& P, long long pos, int4 id, double q, double diag,
                                                double lam0) {
    const int vv[4] = {id.x, id.y, id.z, id.w};
    double4 a[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) a[m] = vv[m] >= 0 ? P.imp[vv[m]] : make_double4(0, 0, 0, 0);
    const double2* J2 = reinterpret_cast<const double2*>(P.pk_jac + pos * 12);
    double J[12];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const double2 t = J2[k];
        J[2 * k] = t.x, J[2 * k + 1] = t.y;
    }
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m)
        if (a[m].w > 0.0) s += dot(mk(J[3 * m], J[3 * m + 1], J[3 * m + 2]), mk(a[m].x, a[m].y, a[m].z));
    const double w = q + s;
    const double t = lam0 - w / diag;
    const double lam = 0.0 < t ? t : 0.0;
    const double d = lam - lam0;
    if (d != 0.0) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            if (!(a[m].w > 0.0)) continue;
            const double sc = a[m].w * d;
            a[m].x = a[m].x + sc * J[3 * m];
            a[m].y = a[m].y + sc * J[3 * m + 1];
            a[m].z = a[m].z + sc * J[3 * m + 2];
            P.imp[vv[m]] = a[m];
        }
    }
    P.pk_lam[pos] = lam;
    P.c_lambda[P.c_by_color[pos]] = lam;
}

// The same row from its color-ordered copy (position pos of c_by_color):
// static row data is one coalesced read, each dynamic vertex's impulse (with
// its inverse mass in w) is gathered once and written back once.
__device__ __forceinline__ void pgs_contact_packed(const Params& P, long long pos) {
    pgs_contact_pre(P, pos, P.pk_ids[pos], P.pk_q[pos], P.pk_diag[pos], P.pk_lam[pos]);
}

__device__ __forceinline__ void pgs_edge_pre(const Params& P, int e, int2 ed, double3 u, double diag, double q,
                                             double lam0) {
    const d3 j0 = edge_jac(make_double4(u.x, u.y, u.z, diag), 0), j1 = edge_jac(make_double4(u.x, u.y, u.z, diag), 1);
    const double im0 = P.inv_mass[ed.x], im1 = P.inv_mass[ed.y];
    double4 a0 = make_double4(0, 0, 0, 0), a1 = make_double4(0, 0, 0, 0);
    if (im0 > 0.0) a0 = P.imp[ed.x];
    if (im1 > 0.0) a1 = P.imp[ed.y];
    double s = 0.0;
    if (im0 > 0.0) s += dot(j0, mk(a0.x, a0.y, a0.z));
    if (im1 > 0.0) s += dot(j1, mk(a1.x, a1.y, a1.z));
    const double w = q + s;
    const double t = lam0 - w / diag;
    const double lam = 0.0 < t ? t : 0.0;
    const double d = lam - lam0;
    if (d != 0.0) {
        if (im0 > 0.0) {
            const double sc = im0 * d;
            a0.x = a0.x + sc * j0.x, a0.y = a0.y + sc * j0.y, a0.z = a0.z + sc * j0.z;
            P.imp[ed.x] = a0;
        }
        if (im1 > 0.0) {
            const double sc = im1 * d;
            a1.x = a1.x + sc * j1.x, a1.y = a1.y + sc * j1.y, a1.z = a1.z + sc * j1.z;
            P.imp[ed.y] = a1;
        }
    }
    P.edge_lambda[e] = lam;
}

__device__ __forceinline__ void pgs_edge_row(const Params& P, int e) {
    const double4 g4 = P.er_g[e];
    pgs_edge_pre(P, e, P.edges[e], make_double3(g4.x, g4.y, g4.z), g4.w, P.er_q[e], P.edge_lambda[e]);
}

// rows of color c: contact rows first, then edge rows (any order inside a
// color gives the same result: its rows touch disjoint dynamic vertices)
__device__ __forceinline__ void pgs_color_range(const Params& P, int c, int ncol_contact, int ncol_edge,
                                                long long* c0, long long* nci, long long* e0, long long* n) {
    *c0 = c < ncol_contact ? P.coff[c] : 0;
    *nci = c < ncol_contact ? P.coff[c + 1] - *c0 : 0;
    long long e1 = 0;
    *e0 = 0;
    if (P.cfg.edge_constraints && c < ncol_edge) *e0 = P.er_color_off[c], e1 = P.er_color_off[c + 1];
    *n = *nci + (e1 - *e0);
}

// The color ranges of one sweep, tabled in the CTA's scratch (shared) memory
// when they fit: the sweep's control flow then reads no global memory.
struct PgsRanges {
    const int4* tab;  // (c0, nci, e0, ne) per color, or nullptr
    int ncol_contact, ncol_edge;
    __device__ __forceinline__ void get(const Params& P, int c, long long* c0, long long* nci, long long* e0,
                                        long long* n) const {
        if (tab) {
            const int4 r = tab[c];
            *c0 = r.x, *nci = r.y, *e0 = r.z, *n = (long long)r.y + r.w;
        } else {
            pgs_color_range(P, c, ncol_contact, ncol_edge, c0, nci, e0, n);
        }
    }
    __device__ __forceinline__ long long rows(const Params& P, int c) const {
        long long c0, nci, e0, n;
        get(P, c, &c0, &nci, &e0, &n);
        return n;
    }
};

__device__ __forceinline__ PgsRanges pgs_ranges(const Params& P, int ncol, int ncol_contact, int ncol_edge,
                                                long long nc) {
    PgsRanges R{nullptr, ncol_contact, ncol_edge};
    if (ncol <= (int)(SCRATCH_BYTES / sizeof(int4)) && nc < 0x7fffffffLL) {
        int4* tab = reinterpret_cast<int4*>(smem_scratch());
        for (int c = threadIdx.x; c < ncol; c += TPB) {
            long long c0, nci, e0, n;
            pgs_color_range(P, c, ncol_contact, ncol_edge, &c0, &nci, &e0, &n);
            tab[c] = make_int4((int)c0, (int)nci, (int)e0, (int)(n - nci));
        }
        __syncthreads();
        R.tab = tab;
    }
    return R;
}

// the static data of this thread's first row of color c (rows dealt as in
// ph_pgs_color), loaded ahead of the barrier that opens the color
__device__ __forceinline__ void pgs_prefetch(const Params& P, const PgsRanges& R, int c, int nctas, PgsRow& r) {
    r.color = c;
    r.edge = -2;  // no row
    long long c0, nci, e0, n;
    R.get(P, c, &c0, &nci, &e0, &n);
    const long long k = blockIdx.x + (long long)threadIdx.x * nctas;
    if (k >= n) return;
    if (k < nci) {
        r.edge = -1;
        r.pos = c0 + k;
        r.ids = P.pk_ids[r.pos];
        r.q = P.pk_q[r.pos];
        r.diag = P.pk_diag[r.pos];
        r.lam = P.pk_lam[r.pos];
    } else {
        const int e = P.er_by_color[e0 + (k - nci)];
        r.edge = e;
        const int2 ed = P.edges[e];
        r.ids = make_int4(ed.x, ed.y, -1, -1);
        const double4 g4 = P.er_g[e];
        r.u = make_double3(g4.x, g4.y, g4.z);
        r.diag = g4.w;
        r.q = P.er_q[e];
        r.lam = P.edge_lambda[e];
    }
}

// one large color on the first nctas CTAs, its first row per thread prefetched
__device__ __forceinline__ void ph_pgs_color_pre(const Params& P, const PgsRanges& R, int c, int nctas,
                                                 const PgsRow& r) {
    long long c0, nci, e0, n;
    R.get(P, c, &c0, &nci, &e0, &n);
    const long long stride = (long long)nctas * TPB;
    long long k = blockIdx.x + (long long)threadIdx.x * nctas;
    if (k < n) {
        if (r.color == c && r.edge != -2) {
            if (r.edge == -1) pgs_contact_pre(P, r.pos, r.ids, r.q, r.diag, r.lam);
            else pgs_edge_pre(P, r.edge, make_int2(r.ids.x, r.ids.y), r.u, r.diag, r.q, r.lam);
        } else if (k < nci) {
            pgs_contact_packed(P, c0 + k);
        } else {
            pgs_edge_row(P, P.er_by_color[e0 + (k - nci)]);
        }
    }
    for (k += stride; k < n; k += stride) {
        if (k < nci) pgs_contact_packed(P, c0 + k);
        else pgs_edge_row(P, P.er_by_color[e0 + (k - nci)]);
    }
}

// ph_pgs_tail over tabled ranges
__device__ void ph_pgs_tail_r(const Params& P, const PgsRanges& R, int cfirst, int cend) {
    if (blockIdx.x != 0) return;
    for (int c = cfirst; c < cend; ++c) {
        long long c0, nci, e0, n;
        R.get(P, c, &c0, &nci, &e0, &n);
        for (long long k = threadIdx.x; k < n; k += TPB) {
            if (k < nci) pgs_contact_packed(P, c0 + k);
            else pgs_edge_row(P, P.er_by_color[e0 + (k - nci)]);
        }
        __syncthreads();
    }
}

__device__ void ph_pgs_color(const Params& P, int c, int ncol_contact, int ncol_edge, int nctas) {
    long long c0, nci, e0, n;
    pgs_color_range(P, c, ncol_contact, ncol_edge, &c0, &nci, &e0, &n);
    // rows dealt round-robin over the nctas CTAs (row k -> CTA k mod nctas): a
    // small color spreads over all SMs instead of filling the first few
    const long long stride = (long long)nctas * TPB;
    for (long long k = blockIdx.x + (long long)threadIdx.x * nctas; k < n; k += stride) {
        if (k < nci) pgs_contact_packed(P, c0 + k);
        else pgs_edge_row(P, P.er_by_color[e0 + (k - nci)]);
    }
}

// The trailing colors of a coloring are small (greedy coloring: the last
// colors pick up the few rows of the densest cliques): a grid-wide phase per
// color would cost a grid barrier for a handful of rows. small_color_run
// returns the end of the run of consecutive colors with at most `tail_rows`
// rows each that starts at cfirst; ph_pgs_tail runs such a run in order on
// CTA 0 alone, with CTA barriers between colors (one sub-grid barrier per run).
__device__ int small_color_run(const Params& P, int cfirst, int ncol, int ncol_contact, int ncol_edge,
                               long long tail_rows) {
    int c = cfirst;
    while (c < ncol) {
        long long c0, nci, e0, n;
        pgs_color_range(P, c, ncol_contact, ncol_edge, &c0, &nci, &e0, &n);
        if (n > tail_rows) break;
        ++c;
    }
    return c;
}

__device__ void ph_pgs_tail(const Params& P, int cfirst, int ncol, int ncol_contact, int ncol_edge) {
    if (blockIdx.x != 0) return;
    for (int c = cfirst; c < ncol; ++c) {
        long long c0, nci, e0, n;
        pgs_color_range(P, c, ncol_contact, ncol_edge, &c0, &nci, &e0, &n);
        for (long long k = threadIdx.x; k < n; k += TPB) {
            if (k < nci) pgs_contact_packed(P, c0 + k);
            else pgs_edge_row(P, P.er_by_color[e0 + (k - nci)]);
        }
        __syncthreads();
    }
}

// ============================================================== Jacobi
// projected_jacobi_sweeps (lcp.cpp:44-59): next = max(0, lam - (w*w_r)/diag)
// for all rows, then impulses applied per vertex in row order.
__device__ void ph_jacobi_next(const Params& P, long long nc) {
    const double om = P.cfg.under_relax;
    for (long long i = gtid(); i < nc; i += gstride()) {
        const int4 id = P.c_ids[i];
        const int vv[4] = {id.x, id.y, id.z, id.w};
        const double* J = P.c_jac + i * 12;
        double s = 0.0;
        for (int m = 0; m < 4; ++m) {
            const int v = vv[m];
            if (v < 0 || !(P.inv_mass[v] > 0.0)) continue;
            const double4 a = P.imp[v];
            s += dot(mk(J[3 * m], J[3 * m + 1], J[3 * m + 2]), mk(a.x, a.y, a.z));
        }
        const double w = P.c_q[i] + s;
        const double t = P.c_lambda[i] - om * w / P.c_diag[i];
        P.c_next[i] = 0.0 < t ? t : 0.0;
    }
    if (P.cfg.edge_constraints)
        for (long long k = gtid(); k < P.g->ner; k += gstride()) {
            const int e = P.er_edge[k];
            const int2 ed = P.edges[e];
            const double4 g4 = P.er_g[e];
            double s = 0.0;
            if (P.inv_mass[ed.x] > 0.0) {
                const double4 a = P.imp[ed.x];
                s += dot(edge_jac(g4, 0), mk(a.x, a.y, a.z));
            }
            if (P.inv_mass[ed.y] > 0.0) {
                const double4 a = P.imp[ed.y];
                s += dot(edge_jac(g4, 1), mk(a.x, a.y, a.z));
            }
            const double w = P.er_q[e] + s;
            const double t = P.edge_lambda[e] - om * w / g4.w;
            P.er_value[e] = 0.0 < t ? t : 0.0;  // er_value reused as the Jacobi "next"
        }
}

__device__ void ph_jacobi_apply(const Params& P, long long nc) {
    for (long long v = gtid(); v < P.nv; v += gstride()) {
        const double im = P.inv_mass[v];
        if (!(im > 0.0)) continue;
        double4 a4 = P.imp[v];
        d3 a = mk(a4.x, a4.y, a4.z);
        for_sorted_entries(P, (int)v, [&](int e) {
            const int row = e >> 2, m = e & 3;
            const double d = P.c_next[row] - P.c_lambda[row];
            if (d != 0.0) {
                const double* J = P.c_jac + (long long)row * 12 + 3 * m;
                imp_add(a, im * d, mk(J[0], J[1], J[2]));
            }
        });
        if (P.cfg.edge_constraints)
            for (int k = P.vedge_off[v]; k < P.vedge_off[v + 1]; ++k) {
                const int e = P.vedge[k];
                if (!P.is_er[e]) continue;
                const double d = P.er_value[e] - P.edge_lambda[e];
                if (d != 0.0) imp_add(a, im * d, edge_jac(P.er_g[e], P.edges[e].x == v ? 0 : 1));
            }
        P.imp[v] = make_double4(a.x, a.y, a.z, 0.0);
    }
}

__device__ void ph_jacobi_commit(const Params& P, long long nc) {
    for (long long i = gtid(); i < nc; i += gstride()) P.c_lambda[i] = P.c_next[i];
    if (P.cfg.edge_constraints)
        for (long long k = gtid(); k < P.g->ner; k += gstride()) {
            const int e = P.er_edge[k];
            P.edge_lambda[e] = P.er_value[e];
        }
}

// ============================================================ advance (F)
// recover_target (lcp.cpp:131-136) + advance (advance.cpp:8-39) + lambda
// store (resolve.cpp:106-111); resets per-vertex scratch for the next step.
__device__ void ph_advance(const Params& P, double bound, int step, long long nc, int sel) {
    const double half_gamma = 0.5 * P.cfg.gamma;
    // maxima as bit patterns of non-negative doubles (NaN skipped), reduced
    // per CTA before the one atomic per CTA
    unsigned long long md_bits = 0ull, rs_bits = 0ull;
    for (long long v = gtid(); v < P.nv; v += gstride()) {
        const double4 x4 = P.x[v];
        const unsigned long long db = P.dmin[v];
        P.dmin[v] = INF_BITS;
        P.vcnt[v] = 0;
        if (x4.w == 0.0) {  // static
            P.r[v] = 0.0;
        } else {
            const double4 a = P.imp[v];
            const d3 yk = ld3(P.yk1, (int)v);
            const d3 y = mk(yk.x + a.x, yk.y + a.y, yk.z + a.z);
            const d3 xv = mk(x4.x, x4.y, x4.z);
            const d3 d = sub(y, xv);
            const double dn = nrm(d);
            if (dn == 0.0) {
                P.r[v] = 0.0;
            } else {
                const double D = mind(bound, to_d(db));
                const double limit = half_gamma * D;
                double alpha = mind(limit / dn, 1.0);
                d3 disp = scl(alpha, d);
                if (alpha < 1.0) {
                    const double dnorm = nrm(disp);
                    if (dnorm > limit) {
                        const double s = (limit / dnorm) * (1.0 - 1e-14);
                        disp = mk(disp.x * s, disp.y * s, disp.z * s);
                        alpha *= s;
                    }
                }
                P.x[v] = make_double4(xv.x + disp.x, xv.y + disp.y, xv.z + disp.z, x4.w);
                P.r[v] = P.r[v] * (1.0 - alpha);
                // std::max(max_disp, |disp|) ignores a NaN operand (advance.cpp:37)
                const double nd = nrm(disp);
                if (!isnan(nd)) md_bits = max(md_bits, to_b(nd));
            }
        }
        if (!isnan(P.r[v])) rs_bits = max(rs_bits, to_b(P.r[v]));  // max_remainder, advance.hpp:21-25
        if (P.cfg.record_path) {
            if (step + 1 < P.path_cap) {
                const double4 xn = P.x[v];
                double* o = P.path + ((long long)(step + 1) * P.nv + v) * 3;
                o[0] = xn.x, o[1] = xn.y, o[2] = xn.z;
            } else if (v == gtid()) {  // path buffer full: the host grows it and reruns
                atomicOr(&P.g->error, ERR_CAP_PATH);
            }
        }
    }
    md_bits = block_max_u64(md_bits);
    rs_bits = block_max_u64(rs_bits);
    if (threadIdx.x == 0) {
        if (md_bits) atomicMax(&P.g->maxdisp_bits, md_bits);
        if (rs_bits) atomicMax(&P.g->resid_bits, rs_bits);
    }
    // contact multipliers -> archive (update in place; count new keys)
    long long lo, hi;
    chunk_of(nc, &lo, &hi);
    long long nnew = 0;
    for (long long i = lo + threadIdx.x; i < hi; i += TPB) {
        const long long at = P.c_arch[i];
        if (at >= 0) P.arch_val[sel][at] = P.c_lambda[i];
        else ++nnew;
    }
    const long long t = block_sum(nnew);
    if (threadIdx.x == 0) P.part_k[blockIdx.x] = t;
}

// G1: ranks of the new keys (pair order == key order) -> staging arrays
__device__ void ph_arch_rank(const Params& P, long long nc) {
    long long lo, hi;
    chunk_of(nc, &lo, &hi);
    long long base = prefix_of(P.part_k, blockIdx.x);
    for (long long t = lo; t < hi; t += TPB) {
        const long long i = t + threadIdx.x;
        const int f = (i < hi && P.c_arch[i] < 0) ? 1 : 0;
        long long tt;
        const long long rk = base + block_scan(f, &tt);
        base += tt;
        if (!f) continue;
        P.new_lb[rk] = -P.c_arch[i] - 1;
        P.new_key[rk] = P.c_key[i];
        P.new_val[rk] = P.c_lambda[i];
    }
}

// G2: merge old archive + new keys into the other buffer
__device__ void ph_arch_merge(const Params& P, long long nnew, int sel, long long narch) {
    const uint64_t* ok = P.arch_key[sel];
    const double* ov = P.arch_val[sel];
    uint64_t* nk = P.arch_key[sel ^ 1];
    double* nvl = P.arch_val[sel ^ 1];
    for (long long j = gtid(); j < narch; j += gstride()) {
        // number of new keys with lower bound <= j
        long long lo = 0, hi = nnew;
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            if (P.new_lb[mid] <= j) lo = mid + 1;
            else hi = mid;
        }
        nk[j + lo] = ok[j];
        nvl[j + lo] = ov[j];
    }
    for (long long r = gtid(); r < nnew; r += gstride()) {
        nk[P.new_lb[r] + r] = P.new_key[r];
        nvl[P.new_lb[r] + r] = P.new_val[r];
    }
}

// ============================================================ refresh (H)
// one pair of ph_refresh for a compile-time pair class (KA < 0: runtime class)
template <int KA, int KB>
__device__ __forceinline__ bool refresh_pair(const Params& P, long long p, uint64_t key, int4 id, uint8_t old_fl,
                                             double bound, bool next_search, long long& nact) {
    const int ka = KA >= 0 ? KA : key_ka(key), kb = KA >= 0 ? KB : key_kb(key);
    int va[3], vb[3];
    Closest c;
    int h;
    if constexpr (KA >= 0) {
        split_ids_t<KA, KB>(id, va, vb);
        h = pair_closest_t<KA, KB>(va, vb, XLoad{P.x}, c);
    } else {
        split_ids(ka, kb, id, va, vb);
        h = pair_closest(ka, va, kb, vb, XLoad{P.x}, c);
    }
    uint8_t fl = old_fl & PF_ALL_STATIC;
    double4 dd;
    double4 w;
    if (h != 1) {
        dd = P.pdd[p];
        w = P.pw[p];
        fl |= old_fl & PF_DEGENERATE;
    } else {
        d3 dir = c.dir;
        if (c.degenerate) {
            const double4 old = P.pdd[p];
            const d3 od = mk(old.x, old.y, old.z);
            if (!is_zero(od)) dir = od;
        }
        dd = make_double4(dir.x, dir.y, dir.z, c.dist);
        w = pack_weights(ka, kb, c);
        P.pdd[p] = dd;
        if (c.degenerate) fl |= PF_DEGENERATE;
        if (c.dist < bound) fl |= PF_ACTIVE;
        else if (c.dist >= bound + kFarMargin) fl |= PF_FAR;
    }
    if (fl & PF_ACTIVE) {
        ++nact;
        if (!next_search) {
            if constexpr (KA >= 0) {
#pragma unroll
                for (int k = 0; k <= KA; ++k) vertex_min(P, va[k], dd.w);
#pragma unroll
                for (int k = 0; k <= KB; ++k) vertex_min(P, vb[k], dd.w);
            } else {
                for (int k = 0; k <= ka; ++k) vertex_min(P, va[k], dd.w);
                for (int k = 0; k <= kb; ++k) vertex_min(P, vb[k], dd.w);
            }
        }
    }
    // contact_pred's own early exits (active, not all static, inside delta) checked first
    if (!next_search && (fl & PF_ACTIVE) && !(fl & PF_ALL_STATIC) && dd.w < P.cfg.delta) {
        int a3[3] = {va[0], va[1], va[2]}, b3[3] = {vb[0], vb[1], vb[2]};
        if (contact_pred(P, ka, kb, a3, b3, dd, w, fl)) fl |= PF_CONTACT;
    }
    // weights are read for contact rows only (ph_rows_build); the stage
    // entries return them for every pair
    if (h == 1 && (P.pw_all || (fl & PF_CONTACT))) P.pw[p] = w;
    P.pflag[p] = fl;
    return (fl & PF_CONTACT) != 0;
}

// refresh_distances (proximity.cpp:190-202) with the pre-shrink bound, the
// vertex bound of the next step (proximity.cpp:204-211) and, when no search
// follows, the contact predicate of the next linearization. The erase of
// the multipliers of inactive pairs runs from the archive side (ph_arch_erase).
__device__ void ph_refresh(const Params& P, double bound, bool next_search) {
    const long long np = P.g->np;
    long long nact = 0, nev = 0;
    for_pair_tiles(P, np, [&](long long p) -> bool {
        // the pair's flag, key and vertex ids in one load round
        const uint8_t old_fl = P.pflag[p];
        const uint64_t key = P.pkey[p];
        const int4 id = P.pids[p];
        if (old_fl & PF_FAR) return false;  // provably still inactive: nothing observable changes
        ++nev;
        bool contact = false;
        if (!with_pair_class(key_ka(key), key_kb(key), [&](auto pc) {
                contact = refresh_pair<decltype(pc)::ka, decltype(pc)::kb>(P, p, key, id, old_fl, bound, next_search,
                                                                           nact);
            }))
            contact = refresh_pair<-1, -1>(P, p, key, id, old_fl, bound, next_search, nact);
        return contact;
    });
    const long long na = block_sum(nact), ev = block_sum(nev);
    if (threadIdx.x == 0) {
        atomicAdd(&P.g->nactive, (int)na);
        atomicAdd((unsigned long long*)&P.g->pairs_evaluated, (unsigned long long)ev);
    }
}

// H2: the erase loop of resolve.cpp:122-123 (multipliers of pairs that left
// the active set are dropped), walked from the archive side: each live entry
// looks its key up in the (sorted) pair set and is tombstoned when that pair
// is inactive. Keys not in the set are kept, as in the reference.
__device__ void ph_arch_erase(const Params& P, int sel, long long narch) {
    const long long np = P.g->np;
    const uint64_t* akey = P.arch_key[sel];
    double* aval = P.arch_val[sel];
    for (long long a = gtid(); a < narch; a += gstride()) {
        if (isnan(aval[a])) continue;
        const uint64_t key = akey[a];
        const long long p = arch_lower_bound(P.pkey, np, key);
        if (p < np && P.pkey[p] == key && !(P.pflag[p] & PF_ACTIVE))
            aval[a] = __longlong_as_double(0x7ff8000000000000ll);
    }
}

// E2' (no trace requested, the next step re-searches): the refreshed pair
// records are discarded by the search, and the vertex bound is not needed, so
// the only lasting effect of refresh_distances + the erase loop
// (resolve.cpp:120-123) is on the multipliers stored for pairs of the set.
// Evaluate just the pairs whose key has a live archive entry (the archive is
// a subset of all contact rows ever solved, the set is sorted by key) and
// tombstone the ones that become inactive.
__device__ void ph_refresh_archive(const Params& P, double bound, int sel, long long narch) {
    const long long np = P.g->np;
    const uint64_t* akey = P.arch_key[sel];
    double* aval = P.arch_val[sel];
    long long evals = 0;
    for (long long a = gtid(); a < narch; a += gstride()) {
        if (isnan(aval[a])) continue;
        const uint64_t key = akey[a];
        const long long p = arch_lower_bound(P.pkey, np, key);
        if (p >= np || P.pkey[p] != key) continue;  // not in the set: kept (erase walks the set)
        const int ka = key_ka(key), kb = key_kb(key);
        int va[3], vb[3];
        split_ids(ka, kb, P.pids[p], va, vb);
        Closest c;
        const int h = pair_closest(ka, va, kb, vb, XLoad{P.x}, c);
        ++evals;
        if (!(h == 1 && c.dist < bound)) aval[a] = __longlong_as_double(0x7ff8000000000000ll);
    }
    const long long ev = block_sum(evals);
    if (threadIdx.x == 0) atomicAdd((unsigned long long*)&P.g->pairs_evaluated, (unsigned long long)ev);
}

}  // namespace tw

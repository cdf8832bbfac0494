// Device-side state of one resolve call and the phase functions of Alg. 1.
//
// Layout in HBM (all buffers owned by the tw_ctx, grown on demand):
//   vertices   x, y_k1: double4 (x, y, z, inv_mass) — one 32 B sector per gather
//              r, impulse, vertex bound (u64 bit pattern for atomicMin)
//   pairs      SoA: key u64 | ids int4 | (dir, dist) double4 | weights double4 | flags u8
//   contact rows (compact, pair order) SoA: key, ids, jac[12], value, diag, q, lambda, color
//   edge rows  indexed by mesh edge: g = u/ly (double4 with diag in w), value, q, lambda
//   archive    sorted (key, lambda) of every contact multiplier ever stored
//              (tombstone = NaN), ping-pong merged — the reference's
//              std::unordered_map<uint64_t,double> contact_lambda
//   BVHs       Karras LBVH over triangles, edges, isolated vertices; float
//              boxes rounded outwards
#pragma once

#include <cstdint>

#include "tw_math.cuh"

namespace tw {

constexpr int TPB = 256;  // threads per block of every engine kernel
constexpr int MAX_BLOCKS = 1024;
constexpr int kPhaseSites = 256;  // phase-profile slots, indexed by SYNC() source line mod 256

enum : int {
    ERR_CAP_SLOTS = 1,    // a broad-phase query produced more than K candidates
    ERR_CAP_PAIRS = 2,    // P > pair capacity
    ERR_CAP_ARCH = 4,     // multiplier archive full
    ERR_CAP_COLORS = 8,   // more colors than the color table holds
    ERR_CAP_REFPOOL = 16, // reference-coloring scratch pool too small
    ERR_TIMEOUT = 32,     // grid barrier watchdog fired
    ERR_CAP_STACK = 64,   // BVH traversal stack overflow
    ERR_INTERNAL = 128,   // invariant violated (line in Globals::internal_line)
    ERR_CAP_CAND = 256,   // broad-phase candidate buffer full (count in Globals::ncand)
    ERR_CAP_PATH = 512,   // record_path: more states than the path buffer holds
};

// PF_FAR: the pair's last refresh found it inactive by distance with a margin
// (d >= bound + kFarMargin); the Alg.-1 bound shrinks by exactly the distance
// the pair's vertices can have closed since (2 max_disp per step), so it stays
// inactive until the next search and later refreshes skip it.
enum : uint8_t { PF_ACTIVE = 1, PF_ALL_STATIC = 2, PF_DEGENERATE = 4, PF_CONTACT = 8, PF_FAR = 16 };
constexpr double kFarMargin = 1e-9;  // m: >> the FP slop of the bound / distance arithmetic

struct Bvh {
    int n;            // primitives (leaves); nodes = 2n-1, internal 0..n-2, leaves n-1..2n-2
    int* prim;        // leaf slot -> primitive index
    int2* child;      // internal node -> (left, right) node ids
    int* parent;      // node -> parent (-1 for root)
    // Traversal layout: internal node i (max(1, n-1) of them) holds the boxes
    // of BOTH children in one 64 B line, so a traversal step is one load
    // round: node[4i + 2s] = (lo.xyz, ref), node[4i + 2s + 1] = (hi.xyz, top)
    // for child slot s; ref = internal node id, or ~index for a leaf (index =
    // triangle / edge / vertex id of the primitive); top = the largest index
    // in the child's subtree (prunes EE / VV queries, which only need
    // partners above their own index). With n == 1 the single
    // leaf sits in slot 0 of node 0 and slot 1 is an empty box.
    float4* node;
    unsigned* flag;   // refit arrival counters (internal nodes)
};

// The words every CTA hammers live on their own 128-byte lines: the grid
// barrier's counter (spun on by every waiting CTA), the error word (polled by
// the waiters) and the dynamic work counters, so that the counters' atomics
// do not queue behind the waiters' polling loads (+1.5% resolves/s).
struct Globals {
    unsigned bar_count;
    unsigned bar_gen;
    char pad_bar[120];
    unsigned sub_count;  // barrier of the CTAs that run the PGS color phases
    char pad_sub[124];
    int error;
    int nonfinite;
    int internal_line;
    char pad_err[116];
    unsigned long long work_q;  // dynamic query counter of the traversal (reset by the refit)
    char pad_q[120];
    unsigned long long ncand;   // broad-phase candidates of the current search (reset by the refit)
    char pad_c[120];
    unsigned long long work_s;  // dynamic query counter of the partner sort (reset by the refit)
    char pad_s[120];
    int ccd_violations;         // certification results (k_ccd)
    int ccd_certain;
    int ner;             // edge rows of this call (set by the prologue)
    int needed_k;
    long long np;        // pairs in the set
    long long nc;        // contact rows this step
    long long narch;     // archive entries
    int arch_sel;        // which archive buffer is current
    int colored;         // JP coloring progress
    int max_color;       // max contact-row color this step
    int new_keys;
    int nactive;
    unsigned long long maxdisp_bits;
    unsigned long long resid_bits;
    long long needed_pairs;
    // stats
    int steps;
    int searches;
    int converged;
    int start_in_contact;
    int step_law_violated;
    int ncolors_last;
    double final_residual;
    long long pairs_evaluated;
    long long rows_solved;
    // phase profile (CTA 0 barrier-to-barrier wall time per call site)
    unsigned long long watchdog_ns;  // grid-barrier watchdog (0: 20 s), set by the host per call
    unsigned long long phase_t0;
    unsigned long long phase_ns[kPhaseSites];
    unsigned int phase_cnt[kPhaseSites];
};

struct Config {
    int step_limit;
    int solver;
    double eps, d_min, d_max, delta, sigma, gamma;
    int sweeps;
    int family;
    double under_relax;
    int edge_constraints;
    int force_fresh_search;
    int record_path;
    int coloring_mode;  // 0 reference replica, 1 device JP
    unsigned long long color_seed;
};

struct Trace {
    int searched, num_pairs, num_contact_rows, num_edge_rows, num_colors, num_active_pairs;
    double bound, max_disp, residual;
};

struct Params {
    Config cfg;
    // ---- mesh
    int nv, ne, nt, niso;
    const double* inv_mass;
    const int2* edges;
    const int4* tris;
    const int* iso;
    const int* vedge_off;   // vertex -> incident edges (ascending edge index)
    const int* vedge;
    const int* edge_color;  // device-mode precoloring (-1 both static)
    int edge_ncolors;
    Bvh bvh[3];             // 0 triangles, 1 edges, 2 isolated vertices
    const int* vperm;       // vertices in Morton order (vertex-query order of the broad phase)
    const double* qspread;  // packet spreads {vertex: mesh, Morton; edge: mesh, Morton} (k_packet_spread)
    const int* eperm;       // edges in Morton order (fixed per mesh)
    // ---- vertex state
    double4* x;
    const double4* yk1;
    double* r;
    double4* imp;
    unsigned long long* dmin;
    // ---- edge rows (by mesh edge index); their count is Globals::ner
    int* er_edge;            // ER list (ascending edge index)
    int* er_index;            // per edge: position in er_edge (-1 if no row)
    uint8_t* is_er;           // per edge
    const double* ly;         // frozen targets
    double* er_value;
    double4* er_g;            // u / ly, w = diag
    double* er_q;
    double* edge_lambda;
    int* er_color;            // per edge (ref mode: per step; device mode: = edge_color)
    int* er_by_color;         // edge ids grouped by color
    int* er_color_off;        // ncolors + 1
    int* er_color_cnt;        // per color (ref-mode per-step bucketing)
    int er_ncolors;           // device mode: colors used by ER rows
    // ---- pairs
    long long pcap;
    int K;
    uint64_t* pkey;
    int4* pids;
    double4* pdd;   // dir.xyz, dist
    double4* pw;    // weights (kind dependent, see pack_weights)
    uint8_t* pflag;
    int* qcount;
    int* qslot;     // nq * K
    long long ccap;
    int2* cand;     // broad-phase candidates (query, partner index)
    // ---- contact rows
    uint64_t* c_key;
    int4* c_ids;
    double* c_jac;  // 12 per row
    double* c_value;
    double* c_diag;
    double* c_q;
    double* c_lambda;
    double* c_next;  // Jacobi
    int* c_color;
    int* c_tent;     // coloring proposals
    int* c_stamp;
    long long* c_arch;  // archive index, or -(lower_bound)-1
    int* c_lost;        // coloring: round in which the row's proposal lost
    int* c_by_color;
    // contact rows copied into color-bucket order for the PGS (position in
    // c_by_color): one coalesced read per row instead of an indirection
    int4* pk_ids;
    double* pk_jac;   // 12 per position
    double* pk_q;
    double* pk_diag;
    double* pk_lam;
    // coloring: per-vertex mask of the colors < 256 taken around the vertex
    // (edge rows + contact rows colored so far), and a flag for colors >= 256
    unsigned long long* vmask;  // 4 per vertex
    int* vbig;
    // vertex -> contact-row incidence, CSR rebuilt every step (entry = 4*row + m)
    int* vcnt;      // entries per vertex (nv); during the device coloring: the uncolored ones
    int* voff;      // segment offsets (nv + 1)
    int* vinc;      // entries, each segment sorted by entry id (4 * rows)
    int* c_slot;    // slot of each entry in its segment before sorting (4 * rows)
    int* erank;     // position of each entry in its sorted segment (4 * rows)
    // color tables
    int colcap;
    int* ccount;
    int* coff;
    // archive
    long long arch_cap;
    uint64_t* arch_key[2];
    double* arch_val[2];
    long long* new_lb;
    uint64_t* new_key;
    double* new_val;
    // reference coloring scratch
    long long refpool_cap;
    int path_cap;    // record_path: states the path buffer holds
    int* refpool;
    // runs of consecutive PGS colors with at most this many rows each run on
    // one CTA (ph_pgs_tail); 0 disables
    long long pgs_tail_rows;
    // CTAs that run the PGS color phases (the first pgs_ctas of the grid, one
    // or two per SM): their barrier is cheaper than the whole grid's
    int pgs_ctas;
    int pw_all;      // store pair weights for every pair (stage entries) or contact pairs only (resolve)
    const double4* ccd_x1;  // certification (k_ccd): end positions of the segment, else null
    // per block scratch
    int nblocks;
    long long* part_q;
    long long* part_c;  // contact pairs per pair tile (for_pair_tiles)
    long long* part_k;
    long long* part_v;
    // globals + outputs
    Globals* g;
    double* step_max_disp;
    double* path;   // (L+1) * nv * 3
    Trace* trace;
    int* dbg;       // host-mapped progress markers (TW_DEBUG=1), else null
};

// ------------------------------------------------------------ helpers
__device__ __forceinline__ d3 ld3(const double4* p, int i) {
    const double4 v = p[i];
    return mk(v.x, v.y, v.z);
}
__device__ __forceinline__ double to_d(unsigned long long b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ unsigned long long to_b(double d) {
    return (unsigned long long)__double_as_longlong(d);
}
constexpr unsigned long long INF_BITS = 0x7ff0000000000000ull;
__host__ __device__ __forceinline__ long long pad32(long long n) { return (n + 31) & ~31LL; }

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t edge_prio(int e) {
    uint64_t z = uint64_t(uint32_t(e)) + 0x5851F42D4C957F2Dull;
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ bool jp_beats(uint64_t pa, long long ia, uint64_t pb, long long ib) {
    return pa > pb || (pa == pb && ia > ib);
}

// Weights packing: VT (wb0, wb1, wb2, -), EE (wa0, wa1, wb0, wb1), VE (wb0, wb1, -, -),
// VV (-). The reference's other weight slots are the ClosestResult defaults.
__device__ __forceinline__ double4 pack_weights(int ka, int kb, const Closest& c) {
    if (ka == KE) return make_double4(c.wa[0], c.wa[1], c.wb[0], c.wb[1]);
    return make_double4(c.wb[0], c.wb[1], c.wb[2], 0.0);
}
__device__ __forceinline__ void unpack_weights(int ka, int kb, double4 w, double* wa, double* wb) {
    wa[0] = 1.0, wa[1] = 0.0, wa[2] = 0.0;
    wb[0] = 1.0, wb[1] = 0.0, wb[2] = 0.0;
    if (ka == KE) {
        wa[0] = w.x, wa[1] = w.y, wb[0] = w.z, wb[1] = w.w;
    } else if (kb == KT) {
        wb[0] = w.x, wb[1] = w.y, wb[2] = w.z;
    } else if (kb == KE) {
        wb[0] = w.x, wb[1] = w.y;
    }
}

// vertex ids of the pair's simplices from its stored ids (a first)
// split_ids for a compile-time pair class (register arrays)
template <int KA, int KB>
__device__ __forceinline__ void split_ids_t(int4 id, int (&va)[3], int (&vb)[3]) {
    const int v[4] = {id.x, id.y, id.z, id.w};
#pragma unroll
    for (int i = 0; i < 3; ++i) va[i] = i <= KA ? v[i] : -1;
#pragma unroll
    for (int i = 0; i < 3; ++i) vb[i] = i <= KB ? v[(KA + 1 + i) & 3] : -1;
}
__device__ __forceinline__ void split_ids(int ka, int kb, int4 id, int* va, int* vb) {
    const int v[4] = {id.x, id.y, id.z, id.w};
    int k = 0;
    for (int i = 0; i <= ka; ++i) va[i] = v[k++];
    for (int i = ka + 1; i < 3; ++i) va[i] = -1;
    for (int i = 0; i <= kb; ++i) vb[i] = v[k++];
    for (int i = kb + 1; i < 3; ++i) vb[i] = -1;
}

}  // namespace tw

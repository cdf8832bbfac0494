// Host-side state of the C-ABI: the context (device buffers, capacities,
// stream) and the uploaded mesh, shared by the resolve path (tw_capi.cu) and
// the dynamics path (tw_dynamics.cu), plus the orchestration helpers both use.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "tw_c.h"
#include "tw_internal.h"

namespace tw {
namespace host {

struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t n) {
        n = n ? n : 16;
        if (n <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        const cudaError_t e = cudaMalloc(&p, n);
        if (e == cudaSuccess) bytes = n;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct BvhMem {
    DevMem prim, child, parent, node, flag;
    int n = 0;
    Bvh view() const {
        return tw::Bvh{n, prim.as<int>(), child.as<int2>(), parent.as<int>(), node.as<float4>(), flag.as<unsigned>()};
    }
};

}  // namespace host
}  // namespace tw

using tw::host::BvhMem;
using tw::host::DevMem;

struct tw_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    int sm_count = 0;
    int nblocks = 0;
    int grid_parts = 1;  // tw_ctx_set_grid_share: this context's share of the device
    int minb = 4;  // resolve-kernel instance (CTAs per SM)
    long long pgs_tail_rows = 256;  // TW_PGS_TAIL
    int pgs_per_sm = 2;             // TW_PGS_CTAS_PER_SM (measured: 1: 152, 2: 154.7, 4: 148.4 resolves/s)
    int bvh_rebuild = 16;           // TW_BVH_REBUILD: rebuild the LBVH topology every n calls on a mesh
    long long launches = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evk = nullptr;
    // capacities
    long long pcap = 0;
    long long ccap = 0;  // broad-phase candidate capacity
    int K = 64;
    long long arch_cap = 0;
    int colcap = 1024;
    long long refpool_cap = 0;
    int path_cap = 0;  // record_path states on the device (grown on demand up to step_limit + 1)
    // buffers
    DevMem xs, ys, xo;  // N x 3 staging
    DevMem x, yk1, r, imp, dmin, voff, vcnt, vinc, c_slot, erank, part_v;
    DevMem ly, is_er, er_edge, er_index, er_value, er_g, er_q, edge_lambda, er_color, er_by_color, er_color_off,
        er_color_cnt;
    DevMem pkey, pids, pdd, pw, pflag, qcount, qslot, cand;
    DevMem c_key, c_ids, c_jac, c_value, c_diag, c_q, c_lambda, c_next, c_color, c_stamp, c_arch, c_lost, c_by_color,
        c_tent, vmask, vbig, pk_ids, pk_jac, pk_q, pk_diag, pk_lam;
    DevMem ccount, coff;
    DevMem arch_key0, arch_key1, arch_val0, arch_val1, new_lb, new_key, new_val;
    DevMem refpool;
    DevMem part_q, part_c, part_k;
    DevMem globals, box, bvh_tmp, smd, trace, path;
    // stage scratch
    DevMem s_kinds, s_verts, s_out, s_has;
    // TW_DEBUG progress markers (host-mapped)
    int* dbg_host = nullptr;
    int* dbg_dev = nullptr;
    tw::Globals last{};
    int last_path_states = 0;  // record_path states of the last resolve (kept on the device)
    int last_nv = 0;  // device globals of the last resolve (phase profile)
};

struct tw_mesh {
    tw_ctx* ctx = nullptr;
    int device = 0;  // destroy does not touch the context (either may be destroyed first)
    int nv = 0, ne = 0, nt = 0, niso = 0;
    std::vector<int32_t> edges;  // 2 ne, finalized order
    std::vector<double> inv_mass;
    DevMem d_inv_mass, d_edges, d_tris, d_iso, d_vedge_off, d_vedge, d_edge_color;
    int edge_ncolors = 0;
    BvhMem bvh[3];
    // broad-phase query order (Morton vertex order + per-class choice), fixed
    // at the first call on this mesh: it only steers performance
    DevMem vperm, qspread, eperm;
    bool qorder_ready = false;
    int bvh_age = -1;  // calls since the hierarchies' topology was built (-1: never)
};

namespace tw {
namespace host {

int fail(tw_ctx* ctx, int code, const std::string& msg);
int cuda_fail(tw_ctx* ctx, cudaError_t e, const char* where);
int check_cfg(tw_ctx* ctx, const tw_resolve_config* cfg);
int ensure_buffers(tw_ctx* ctx, const tw_mesh* m, const tw_resolve_config& cfg);
Params make_params(tw_ctx* ctx, tw_mesh* m, const tw_resolve_config& c);
int build_bvhs(tw_ctx* ctx, tw_mesh* m);
// one device resolve on device inputs d_xs/d_ys (N x 3) into d_out
int run_resolve(tw_ctx* ctx, tw_mesh* m, const double* d_xs, const double* d_ys, const tw_resolve_config& cfg,
                double* d_out, tw_resolve_stats* st, double* smd_host, double* path_host, tw_step_trace* trace_host,
                double* host_out = nullptr);
void grow_ll(long long& v, long long need);

}  // namespace host
}  // namespace tw

#define CK(expr)                                                           \
    do {                                                                   \
        const cudaError_t _e = (expr);                                     \
        if (_e != cudaSuccess) return tw::host::cuda_fail(ctx, _e, #expr); \
    } while (0)

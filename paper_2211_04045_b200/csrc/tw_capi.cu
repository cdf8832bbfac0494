// C-ABI (include/tw_c.h) of the B200 two-way collision handling path: context
// and mesh management, capacity growth, the per-call orchestration around
// the persistent resolve kernel, and the stage entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <unordered_set>
#include <vector>

#include "tw_c.h"
#include "tw_internal.h"

using namespace tw;

#include "tw_ctx.h"


namespace tw {
namespace host {

int fail(tw_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

int cuda_fail(tw_ctx* ctx, cudaError_t e, const char* where) {
    std::string msg = std::string(where) + ": " + cudaGetErrorString(e);
    if (ctx && ctx->dbg_host) {  // TW_DEBUG: last phase (step << 16 | source line) per CTA
        std::map<int, int> hist;
        for (int b = 0; b < ctx->nblocks; ++b) ++hist[ctx->dbg_host[b]];
        msg += " [progress:";
        for (auto& kv : hist)
            msg += " step" + std::to_string(kv.first >> 16) + "/line" + std::to_string(kv.first & 0xffff) + "x" +
                   std::to_string(kv.second);
        msg += "]";
    }
    return fail(ctx, TW_ECUDA, msg);
}


// ResolveConfig::validate (resolve.cpp:12-21)
bool config_valid(const tw_resolve_config& c) {
    if (!(c.d_min > 0.0) || !(c.d_min <= c.d_max)) return false;
    if (!(c.delta > 0.0) || !(c.delta <= c.d_min)) return false;
    if (!(c.gamma > 0.0) || !(c.gamma < 1.0)) return false;
    if (!(c.eps > 0.0)) return false;
    if (c.step_limit < 1) return false;
    if (c.sweeps < 1) return false;
    return true;
}

// MeshState::finalize edge derivation, mesh.cpp:15-26
std::vector<int32_t> finalize_edges(int ne_explicit, const int32_t* edges, int ns, const int32_t* strands, int nt,
                                    const int32_t* tris) {
    std::vector<int32_t> out;
    out.reserve(2 * (size_t)(ne_explicit + ns + 3 * (size_t)nt));
    std::unordered_set<uint64_t> seen;
    seen.reserve(2 * (size_t)(ne_explicit + ns + 3 * (size_t)nt) + 16);
    auto key = [](int a, int b) {
        const uint32_t lo = (uint32_t)std::min(a, b), hi = (uint32_t)std::max(a, b);
        return ((uint64_t)lo << 32) | hi;
    };
    for (int i = 0; i < ne_explicit; ++i) {
        seen.insert(key(edges[2 * i], edges[2 * i + 1]));
        out.push_back(edges[2 * i]);
        out.push_back(edges[2 * i + 1]);
    }
    for (int i = 0; i < ns; ++i)
        if (seen.insert(key(strands[2 * i], strands[2 * i + 1])).second) {
            out.push_back(strands[2 * i]);
            out.push_back(strands[2 * i + 1]);
        }
    for (int t = 0; t < nt; ++t)
        for (int k = 0; k < 3; ++k) {
            const int a = tris[3 * t + k], b = tris[3 * t + (k + 1) % 3];
            if (seen.insert(key(a, b)).second) {
                out.push_back(std::min(a, b));
                out.push_back(std::max(a, b));
            }
        }
    return out;
}

void grow_ll(long long& v, long long need) {
    while (v < need) v = v * 2 + 1024;
}

int ensure_buffers(tw_ctx* ctx, const tw_mesh* m, const tw_resolve_config& cfg) {
    const size_t nv = (size_t)std::max(1, m->nv), ne = (size_t)std::max(1, m->ne);
    const long long nq = 2 * pad32(m->niso) + pad32(m->nv) + pad32(m->ne);  // = num_queries
    if (ctx->pcap == 0) ctx->pcap = 8LL * (m->nv + m->ne) + 4096;
    if (ctx->arch_cap < ctx->pcap) ctx->arch_cap = ctx->pcap;
    if (ctx->ccap == 0) ctx->ccap = 4 * ctx->pcap;
    CK(ctx->cand.ensure((size_t)ctx->ccap * 8));
    const size_t P = (size_t)ctx->pcap;
    CK(ctx->xs.ensure(nv * 24));
    CK(ctx->ys.ensure(nv * 24));
    CK(ctx->xo.ensure(nv * 24));
    CK(ctx->x.ensure(nv * 32));
    CK(ctx->yk1.ensure(nv * 32));
    CK(ctx->r.ensure(nv * 8));
    CK(ctx->imp.ensure(nv * 32));
    CK(ctx->dmin.ensure(nv * 8));
    CK(ctx->voff.ensure((nv + 1) * 4));
    CK(ctx->vinc.ensure(P * 16));
    CK(ctx->c_slot.ensure(P * 16));
    CK(ctx->erank.ensure(P * 16));
    CK(ctx->part_v.ensure((size_t)ctx->nblocks * 8));
    CK(ctx->vcnt.ensure(nv * 4));
    CK(ctx->ly.ensure(ne * 8));
    CK(ctx->is_er.ensure(ne));
    CK(ctx->er_edge.ensure(ne * 4));
    CK(ctx->er_index.ensure(ne * 4));
    CK(ctx->er_value.ensure(ne * 8));
    CK(ctx->er_g.ensure(ne * 32));
    CK(ctx->er_q.ensure(ne * 8));
    CK(ctx->edge_lambda.ensure(ne * 8));
    CK(ctx->er_color.ensure(ne * 4));
    CK(ctx->er_by_color.ensure(ne * 4));
    CK(ctx->pkey.ensure(P * 8));
    CK(ctx->pids.ensure(P * 16));
    CK(ctx->pdd.ensure(P * 32));
    CK(ctx->pw.ensure(P * 32));
    CK(ctx->pflag.ensure(P));
    CK(ctx->qcount.ensure((size_t)std::max(1LL, nq) * 4));
    CK(ctx->qslot.ensure((size_t)std::max(1LL, nq) * ctx->K * 4));
    CK(ctx->c_key.ensure(P * 8));
    CK(ctx->c_ids.ensure(P * 16));
    CK(ctx->c_jac.ensure(P * 96));
    CK(ctx->c_value.ensure(P * 8));
    CK(ctx->c_diag.ensure(P * 8));
    CK(ctx->c_q.ensure(P * 8));
    CK(ctx->c_lambda.ensure(P * 8));
    if (cfg.solver == TW_SOLVER_JACOBI) CK(ctx->c_next.ensure(P * 8));
    CK(ctx->c_color.ensure(P * 4));
    CK(ctx->c_stamp.ensure(P * 4));
    CK(ctx->c_tent.ensure(P * 4));
    CK(ctx->c_arch.ensure(P * 8));
    CK(ctx->c_lost.ensure(P * 4));
    CK(ctx->vmask.ensure(nv * 32));
    CK(ctx->vbig.ensure(nv * 4));
    if (cfg.solver == TW_SOLVER_PGS) {
        CK(ctx->pk_ids.ensure(P * 16));
        CK(ctx->pk_jac.ensure(P * 96));
        CK(ctx->pk_q.ensure(P * 8));
        CK(ctx->pk_diag.ensure(P * 8));
        CK(ctx->pk_lam.ensure(P * 8));
    }
    CK(ctx->c_by_color.ensure(P * 4));
    CK(ctx->ccount.ensure((size_t)ctx->colcap * 4));
    CK(ctx->coff.ensure(((size_t)ctx->colcap + 1) * 4));
    CK(ctx->er_color_cnt.ensure((size_t)ctx->colcap * 4));
    CK(ctx->er_color_off.ensure(((size_t)ctx->colcap + 1) * 4));
    const size_t A = (size_t)ctx->arch_cap;
    CK(ctx->arch_key0.ensure(A * 8));
    CK(ctx->arch_key1.ensure(A * 8));
    CK(ctx->arch_val0.ensure(A * 8));
    CK(ctx->arch_val1.ensure(A * 8));
    CK(ctx->new_lb.ensure(P * 8));
    CK(ctx->new_key.ensure(P * 8));
    CK(ctx->new_val.ensure(P * 8));
    if (cfg.coloring_mode == TW_COLOR_REFERENCE) {
        if (ctx->refpool_cap == 0) ctx->refpool_cap = 256LL * (m->nv + m->ne) + (1LL << 20);
        CK(ctx->refpool.ensure((size_t)ctx->refpool_cap * 4));
    }
    const size_t nb = (size_t)ctx->nblocks;
    CK(ctx->part_q.ensure(nb * 8));
    CK(ctx->part_c.ensure(((size_t)P / 256 + 2) * 8));  // per pair tile (PAIR_TILE >= TPB)
    CK(ctx->part_k.ensure(nb * 8));
    CK(ctx->globals.ensure(sizeof(Globals)));
    CK(ctx->box.ensure(64));
    CK(ctx->smd.ensure((size_t)cfg.step_limit * 8));
    CK(ctx->trace.ensure((size_t)cfg.step_limit * sizeof(Trace)));
    if (cfg.record_path) {
        // the path buffer starts small and grows through the capacity retry
        if (ctx->path_cap == 0) ctx->path_cap = 33;
        ctx->path_cap = std::min(ctx->path_cap, cfg.step_limit + 1);
        CK(ctx->path.ensure((size_t)ctx->path_cap * nv * 24));
    }
    size_t tb = bvh_tmp_bytes(m->nv);  // the vertex order sorts nv codes
    for (int c = 0; c < 3; ++c) tb = std::max(tb, bvh_tmp_bytes(m->bvh[c].n));

    CK(ctx->bvh_tmp.ensure(tb));
    return TW_OK;
}

Params make_params(tw_ctx* ctx, tw_mesh* m, const tw_resolve_config& c) {
    Params P;
    std::memset(&P, 0, sizeof P);
    P.cfg.step_limit = c.step_limit;
    P.cfg.solver = c.solver;
    P.cfg.eps = c.eps;
    P.cfg.d_min = c.d_min;
    P.cfg.d_max = c.d_max;
    P.cfg.delta = c.delta;
    P.cfg.sigma = c.sigma;
    P.cfg.gamma = c.gamma;
    P.cfg.sweeps = c.sweeps;
    P.cfg.family = c.family;
    P.cfg.under_relax = c.under_relax;
    P.cfg.edge_constraints = c.edge_constraints ? 1 : 0;
    P.cfg.force_fresh_search = c.force_fresh_search ? 1 : 0;
    P.cfg.record_path = c.record_path ? 1 : 0;
    P.cfg.coloring_mode = c.coloring_mode;
    P.cfg.color_seed = c.color_seed;
    P.nv = m->nv, P.ne = m->ne, P.nt = m->nt, P.niso = m->niso;
    P.inv_mass = m->d_inv_mass.as<double>();
    P.edges = m->d_edges.as<int2>();
    P.tris = m->d_tris.as<int4>();
    P.iso = m->d_iso.as<int>();
    P.vedge_off = m->d_vedge_off.as<int>();
    P.vedge = m->d_vedge.as<int>();
    P.edge_color = m->d_edge_color.as<int>();
    P.edge_ncolors = m->edge_ncolors;
    for (int k = 0; k < 3; ++k) P.bvh[k] = m->bvh[k].view();
    P.vperm = m->vperm.as<int>();
    P.qspread = m->qspread.as<double>();
    P.eperm = m->eperm.as<int>();
    P.x = ctx->x.as<double4>();
    P.yk1 = ctx->yk1.as<double4>();
    P.r = ctx->r.as<double>();
    P.imp = ctx->imp.as<double4>();
    P.dmin = ctx->dmin.as<unsigned long long>();
    P.er_edge = ctx->er_edge.as<int>();
    P.er_index = ctx->er_index.as<int>();
    P.is_er = ctx->is_er.as<uint8_t>();
    P.ly = ctx->ly.as<double>();
    P.er_value = ctx->er_value.as<double>();
    P.er_g = ctx->er_g.as<double4>();
    P.er_q = ctx->er_q.as<double>();
    P.edge_lambda = ctx->edge_lambda.as<double>();
    P.er_color = ctx->er_color.as<int>();
    P.er_by_color = ctx->er_by_color.as<int>();
    P.er_color_off = ctx->er_color_off.as<int>();
    P.er_color_cnt = ctx->er_color_cnt.as<int>();
    P.er_ncolors = m->edge_ncolors;
    P.pcap = ctx->pcap;
    P.ccap = ctx->ccap;
    P.cand = ctx->cand.as<int2>();
    P.K = ctx->K;
    P.pkey = ctx->pkey.as<uint64_t>();
    P.pids = ctx->pids.as<int4>();
    P.pdd = ctx->pdd.as<double4>();
    P.pw = ctx->pw.as<double4>();
    P.pflag = ctx->pflag.as<uint8_t>();
    P.qcount = ctx->qcount.as<int>();
    P.qslot = ctx->qslot.as<int>();
    P.c_key = ctx->c_key.as<uint64_t>();
    P.c_ids = ctx->c_ids.as<int4>();
    P.c_jac = ctx->c_jac.as<double>();
    P.c_value = ctx->c_value.as<double>();
    P.c_diag = ctx->c_diag.as<double>();
    P.c_q = ctx->c_q.as<double>();
    P.c_lambda = ctx->c_lambda.as<double>();
    P.c_next = ctx->c_next.as<double>();
    P.c_color = ctx->c_color.as<int>();
    P.c_stamp = ctx->c_stamp.as<int>();
    P.c_tent = ctx->c_tent.as<int>();
    P.c_arch = ctx->c_arch.as<long long>();
    P.c_lost = ctx->c_lost.as<int>();
    P.vmask = ctx->vmask.as<unsigned long long>();
    P.vbig = ctx->vbig.as<int>();
    P.pk_ids = ctx->pk_ids.as<int4>();
    P.pk_jac = ctx->pk_jac.as<double>();
    P.pk_q = ctx->pk_q.as<double>();
    P.pk_diag = ctx->pk_diag.as<double>();
    P.pk_lam = ctx->pk_lam.as<double>();
    P.c_by_color = ctx->c_by_color.as<int>();
    P.voff = ctx->voff.as<int>();
    P.vinc = ctx->vinc.as<int>();
    P.c_slot = ctx->c_slot.as<int>();
    P.erank = ctx->erank.as<int>();
    P.part_v = ctx->part_v.as<long long>();
    P.vcnt = ctx->vcnt.as<int>();
    P.colcap = ctx->colcap;
    P.ccount = ctx->ccount.as<int>();
    P.coff = ctx->coff.as<int>();
    P.arch_cap = ctx->arch_cap;
    P.arch_key[0] = ctx->arch_key0.as<uint64_t>();
    P.arch_key[1] = ctx->arch_key1.as<uint64_t>();
    P.arch_val[0] = ctx->arch_val0.as<double>();
    P.arch_val[1] = ctx->arch_val1.as<double>();
    P.new_lb = ctx->new_lb.as<long long>();
    P.new_key = ctx->new_key.as<uint64_t>();
    P.new_val = ctx->new_val.as<double>();
    P.refpool_cap = ctx->refpool_cap;
    P.refpool = ctx->refpool.as<int>();
    P.nblocks = ctx->nblocks;
    P.pgs_tail_rows = ctx->pgs_tail_rows;
    P.pgs_ctas = std::max(1, std::min(ctx->nblocks, ctx->sm_count * ctx->pgs_per_sm));
    P.pw_all = 1;
    P.part_q = ctx->part_q.as<long long>();
    P.part_c = ctx->part_c.as<long long>();
    P.part_k = ctx->part_k.as<long long>();
    P.g = ctx->globals.as<Globals>();
    P.step_max_disp = ctx->smd.as<double>();
    P.path = c.record_path ? ctx->path.as<double>() : nullptr;
    P.path_cap = c.record_path ? ctx->path_cap : 0;
    P.trace = ctx->trace.as<Trace>();
    P.dbg = ctx->dbg_dev;
    return P;
}

// The hierarchies' topology (Morton sort + Karras build) is rebuilt from the
// call's start positions every ctx->bvh_rebuild calls on a mesh; in between
// the topology of the last build is reused and only refitted (the refit runs
// at every search in the kernel). Any topology gives the same, exact pair
// set: the choice only affects how tight the boxes are. The refit arrival
// counters are cleared every call (an aborted attempt may leave them set).
int build_bvhs(tw_ctx* ctx, tw_mesh* m) {
    if (m->bvh_age >= 0 && m->bvh_age + 1 < ctx->bvh_rebuild) {
        ++m->bvh_age;
        for (int c = 0; c < 3; ++c)
            if (m->bvh[c].n > 1) CK(cudaMemsetAsync(m->bvh[c].flag.p, 0, (size_t)(m->bvh[c].n - 1) * 4, ctx->stream));
        return TW_OK;
    }
    m->bvh_age = 0;
    CK(cudaMemsetAsync(ctx->box.p, 0, 64, ctx->stream));
    // lo = ~0 (max), hi = 0
    std::vector<unsigned long long> init = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
    CK(cudaMemcpyAsync(ctx->box.p, init.data(), 48, cudaMemcpyHostToDevice, ctx->stream));
    tw::launch_bounds(ctx->stream, m->nv, ctx->x.as<double4>(), ctx->box.as<unsigned long long>());
    ctx->launches += 1;
    for (int c = 0; c < 3; ++c) {
        launch_bvh_build(ctx->stream, c, m->bvh[c].view(), m->d_tris.as<int4>(), m->d_edges.as<int2>(),
                         m->d_iso.as<int>(), ctx->x.as<double4>(), m->nv, ctx->bvh_tmp.p, ctx->bvh_tmp.bytes,
                         ctx->box.as<unsigned long long>());
        ctx->launches += launch_count_last();
    }
    if (!m->qorder_ready) {
        // Morton vertex order and edge order (the edge leaf order of this first
        // build), and which order makes the more compact query packets
        launch_vertex_order(ctx->stream, m->nv, ctx->x.as<double4>(), ctx->bvh_tmp.p, ctx->bvh_tmp.bytes,
                            ctx->box.as<unsigned long long>(), m->vperm.as<int>());
        ctx->launches += launch_count_last();
        if (m->ne)
            CK(cudaMemcpyAsync(m->eperm.p, m->bvh[1].prim.p, (size_t)m->ne * 4, cudaMemcpyDeviceToDevice,
                               ctx->stream));
        CK(cudaMemsetAsync(m->qspread.p, 0, 32, ctx->stream));
        launch_packet_spread(ctx->stream, m->nv, 0, nullptr, ctx->x.as<double4>(), m->vperm.as<int>(),
                             m->qspread.as<double>());
        launch_packet_spread(ctx->stream, m->ne, 1, m->d_edges.as<int2>(), ctx->x.as<double4>(),
                             m->eperm.as<int>(), m->qspread.as<double>() + 2);
        ctx->launches += (m->nv > 0) + (m->ne > 0);
        m->qorder_ready = true;
    }
    CK(cudaGetLastError());
    return TW_OK;
}

// Runs one resolve on inputs already in ctx->xs / ctx->ys (device, N x 3).
// host_out (nullable): the result is also copied to this host buffer, enqueued
// behind the kernel so that one stream synchronization covers the call
int run_resolve(tw_ctx* ctx, tw_mesh* m, const double* d_xs, const double* d_ys, const tw_resolve_config& cfg,
                double* d_out, tw_resolve_stats* st, double* smd_host, double* path_host, tw_step_trace* trace_host,
                double* host_out) {
    Globals G;
    int retries = 0;
    float dev_ms = 0.f, kern_ms = 0.f;
    const long long launches0 = ctx->launches;
    for (;;) {
        int rc = ensure_buffers(ctx, m, cfg);
        if (rc) return rc;
        Params P = make_params(ctx, m, cfg);
        if (!trace_host) P.trace = nullptr;  // lets the kernel skip work only a trace would show
        P.pw_all = 0;
        CK(cudaMemsetAsync(ctx->globals.p, 0, sizeof(Globals), ctx->stream));
        if (cfg.coloring_mode == TW_COLOR_REFERENCE) {
            // the exact replay runs on one device thread while the grid waits:
            // the barrier watchdog allows it 600 s instead of 20 s
            static const unsigned long long wd = 600000000000ull;
            CK(cudaMemcpyAsync((char*)ctx->globals.p + offsetof(Globals, watchdog_ns), &wd, 8,
                               cudaMemcpyHostToDevice, ctx->stream));
        }
        // color tables return to zero at the end of every step; an attempt
        // aborted for capacity growth may leave counts behind
        CK(cudaMemsetAsync(ctx->ccount.p, 0, (size_t)ctx->colcap * 4, ctx->stream));
        CK(cudaMemsetAsync(ctx->er_color_cnt.p, 0, (size_t)ctx->colcap * 4, ctx->stream));
        CK(cudaEventRecord(ctx->ev0, ctx->stream));
        launch_setup(ctx->stream, m->nv, d_xs, d_ys, m->d_inv_mass.as<double>(), P.x, const_cast<double4*>(P.yk1),
                     P.r, P.dmin, P.voff, P.vcnt, P.imp, &P.g->nonfinite, m->ne, P.edges,
                     const_cast<double*>(P.ly), P.is_er, P.edge_lambda, P.er_color, P.edge_color,
                     cfg.edge_constraints ? 1 : 0, cfg.coloring_mode == TW_COLOR_DEVICE ? 1 : 0);
        ctx->launches += launch_count_last();
        rc = build_bvhs(ctx, m);
        if (rc) return rc;
        CK(cudaEventRecord(ctx->evk, ctx->stream));
        CK(coop_resolve(ctx->stream, P, ctx->nblocks, ctx->minb));
        ctx->launches += 1;
        CK(cudaEventRecord(ctx->ev1, ctx->stream));
        // the result (re-enqueued by a capacity retry) ahead of the globals read-back
        launch_pack(ctx->stream, m->nv, ctx->x.as<double4>(), d_out);
        ctx->launches += launch_count_last();
        if (host_out && m->nv)
            CK(cudaMemcpyAsync(host_out, d_out, (size_t)m->nv * 24, cudaMemcpyDeviceToHost, ctx->stream));
        if (smd_host)
            CK(cudaMemcpyAsync(smd_host, ctx->smd.p, (size_t)cfg.step_limit * 8, cudaMemcpyDeviceToHost, ctx->stream));
        if (trace_host) {
            static_assert(sizeof(Trace) == sizeof(tw_step_trace), "trace layout");
            CK(cudaMemcpyAsync(trace_host, ctx->trace.p, (size_t)cfg.step_limit * sizeof(Trace),
                               cudaMemcpyDeviceToHost, ctx->stream));
        }
        CK(cudaMemcpyAsync(&G, ctx->globals.p, sizeof(Globals), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaEventElapsedTime(&dev_ms, ctx->ev0, ctx->ev1));
        CK(cudaEventElapsedTime(&kern_ms, ctx->evk, ctx->ev1));
        if (G.nonfinite) return fail(ctx, TW_EINVAL, "resolve: non-finite input positions");
        if (G.error & ERR_TIMEOUT) return fail(ctx, TW_ETIMEOUT, "resolve: device watchdog fired");
        if (G.error & ERR_INTERNAL)
            return fail(ctx, TW_ECUDA, "resolve: device invariant violated at tw_phases.cuh:" +
                                           std::to_string(G.internal_line) + " (step " +
                                           std::to_string(G.steps) + ")");
        const int cap = G.error & (ERR_CAP_SLOTS | ERR_CAP_PAIRS | ERR_CAP_ARCH | ERR_CAP_COLORS | ERR_CAP_REFPOOL |
                                   ERR_CAP_STACK | ERR_CAP_CAND | ERR_CAP_PATH);
        if (!cap) break;
        if (++retries > 12) return fail(ctx, TW_ECAPACITY, "resolve: capacity growth did not converge");
        if (G.error & ERR_CAP_STACK) return fail(ctx, TW_ECAPACITY, "resolve: BVH traversal stack overflow");
        if (G.error & ERR_CAP_SLOTS) ctx->K = std::max(ctx->K * 2, ((G.needed_k + 31) / 32) * 32);
        if (G.error & ERR_CAP_PAIRS) grow_ll(ctx->pcap, G.needed_pairs + G.needed_pairs / 4);
        if (G.error & ERR_CAP_CAND) grow_ll(ctx->ccap, (long long)G.ncand + (long long)G.ncand / 4);
        if (G.error & ERR_CAP_ARCH) grow_ll(ctx->arch_cap, ctx->arch_cap * 2);
        if (G.error & ERR_CAP_COLORS) ctx->colcap *= 4;
        if (G.error & ERR_CAP_REFPOOL) ctx->refpool_cap *= 4;
        if (G.error & ERR_CAP_PATH) ctx->path_cap = std::min(cfg.step_limit + 1, ctx->path_cap * 4);
    }
    ctx->last = G;
    ctx->last_path_states = cfg.record_path ? G.steps + 1 : 0;
    ctx->last_nv = m->nv;
    std::memset(st, 0, sizeof *st);
    st->steps = G.steps;
    st->searches = G.searches;
    st->final_residual = G.final_residual;
    st->converged = G.converged;
    st->hit_step_limit = !G.converged;
    st->stagnated = 0;
    st->start_in_contact = G.start_in_contact;
    st->step_law_violated = G.step_law_violated;
    st->num_pairs = (int32_t)G.np;
    st->pairs_evaluated = G.pairs_evaluated;
    st->rows_solved = G.rows_solved;
    st->device_ms = dev_ms;
    st->kernel_ms = kern_ms;
    st->setup_ms = dev_ms - kern_ms;
    st->retries = retries;
    st->kernel_launches = (int32_t)(ctx->launches - launches0);
    if (path_host && cfg.record_path)
        CK(cudaMemcpyAsync(path_host, ctx->path.p, ((size_t)G.steps + 1) * m->nv * 24, cudaMemcpyDeviceToHost,
                           ctx->stream));
    return TW_OK;
}

int check_cfg(tw_ctx* ctx, const tw_resolve_config* cfg) {
    if (!cfg || !config_valid(*cfg)) return fail(ctx, TW_EINVAL, "resolve: invalid configuration");
    if (cfg->solver == TW_SOLVER_AL20 || cfg->solver == TW_SOLVER_AL100)
        return fail(ctx, TW_EUNSUPPORTED, "resolve: the AL baseline solvers are not provided on the device");
    if (cfg->solver != TW_SOLVER_PGS && cfg->solver != TW_SOLVER_JACOBI)
        return fail(ctx, TW_EINVAL, "resolve: unknown solver");
    if (cfg->coloring_mode != TW_COLOR_REFERENCE && cfg->coloring_mode != TW_COLOR_DEVICE)
        return fail(ctx, TW_EINVAL, "resolve: unknown coloring mode");
    if (cfg->family != TW_FAMILY_VOLUME && cfg->family != TW_FAMILY_GAP)
        return fail(ctx, TW_EINVAL, "resolve: unknown constraint family");
    return TW_OK;
}

}  // namespace host
}  // namespace tw

using namespace tw::host;

namespace {
struct Scratch {  // per-call device buffers of the row stage entries
    std::vector<void*> ptrs;
    cudaError_t err = cudaSuccess;
    template <typename T>
    T* up(const T* host, size_t n) {
        void* p = nullptr;
        if (err == cudaSuccess) err = cudaMalloc(&p, std::max<size_t>(16, n * sizeof(T)));
        if (err == cudaSuccess && host && n) err = cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice);
        if (p) ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    template <typename T>
    T* out(size_t n) {
        return up<T>(nullptr, n);
    }
    template <typename T>
    void down(T* host, const T* dev, size_t n) {
        if (err == cudaSuccess && host && n) err = cudaMemcpy(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost);
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFree(p);
    }
};

double4* upload_x4(Scratch& S, int32_t nv, const double* x, const double* inv_mass) {
    std::vector<double4> x4(std::max(1, nv));
    for (int v = 0; v < nv; ++v)
        x4[v] = make_double4(x[3 * v], x[3 * v + 1], x[3 * v + 2], inv_mass ? inv_mass[v] : 1.0);
    return S.up(x4.data(), x4.size());
}
}  // namespace

// ================================================================= C-ABI
extern "C" {

int tw_abi_version(void) { return TW_ABI_VERSION; }

void tw_default_config(tw_resolve_config* c) {
    std::memset(c, 0, sizeof *c);
    c->step_limit = 512;
    c->solver = TW_SOLVER_PGS;
    c->eps = 1e-4;
    c->d_min = 2e-3;
    c->d_max = 4e-3;
    c->delta = 1e-3;
    c->sigma = 1.1;
    c->gamma = 0.9;
    c->sweeps = 1;
    c->family = TW_FAMILY_VOLUME;
    c->under_relax = 0.5;
    c->edge_constraints = 1;
    c->force_fresh_search = 0;
    c->record_path = 0;
    c->coloring_mode = TW_COLOR_DEVICE;
    c->color_seed = 0x5eed;
}

int tw_ctx_create(int device, void* stream, tw_ctx** out) {
    if (!out) return TW_EINVAL;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return TW_ECUDA;
    if (device < 0 || device >= n) return TW_EINVAL;
    tw_ctx* ctx = new tw_ctx();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete ctx;
        return TW_ECUDA;
    }
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (!coop) {
        delete ctx;
        return TW_ECUDA;
    }
    int want = 4;  // measured best on B200 (bow knot): 64 regs, 32 warps/SM
    if (const char* s = std::getenv("TW_BLOCKS_PER_SM")) want = std::min(4, std::max(2, std::atoi(s)));
    ctx->minb = want;
    if (const char* s = std::getenv("TW_PGS_CTAS_PER_SM")) ctx->pgs_per_sm = std::max(1, std::atoi(s));
    if (const char* s = std::getenv("TW_PGS_TAIL")) ctx->pgs_tail_rows = std::max(0LL, std::atoll(s));
    if (const char* s = std::getenv("TW_BVH_REBUILD")) ctx->bvh_rebuild = std::max(1, std::atoi(s));
    // initial partner slots per query (<= 128: lists sorted in registers in the
    // key emission; more: sorted in memory by ph_query_totals)
    if (const char* s = std::getenv("TW_QUERY_SLOTS")) ctx->K = std::max(4, std::atoi(s));
    if (std::getenv("TW_TINY_CAPS")) {  // start every capacity tiny: exercises the grow-and-rerun paths
        ctx->pcap = 256, ctx->ccap = 256, ctx->K = 4, ctx->arch_cap = 16, ctx->refpool_cap = 1024;
        ctx->path_cap = 2;
        ctx->colcap = 8;
    }
    const int per_sm = std::max(1, std::min(resolve_blocks_per_sm(want), want));
    ctx->nblocks = std::min(ctx->sm_count * per_sm, tw::MAX_BLOCKS);
    if (stream) {
        ctx->stream = (cudaStream_t)stream;
    } else {
        // a blocking stream: ordered with the legacy default stream, so callers
        // that enqueue their inputs there (e.g. torch's default stream) never
        // race the context's kernels
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamDefault) != cudaSuccess) {
            delete ctx;
            return TW_ECUDA;
        }
        ctx->own_stream = true;
    }
    cudaEventCreate(&ctx->ev0);
    cudaEventCreate(&ctx->ev1);
    cudaEventCreate(&ctx->evk);
    if (const char* d = std::getenv("TW_DEBUG"); d && d[0] == '1') {
        if (cudaHostAlloc((void**)&ctx->dbg_host, MAX_BLOCKS * sizeof(int), cudaHostAllocMapped) == cudaSuccess) {
            std::memset(ctx->dbg_host, 0xff, MAX_BLOCKS * sizeof(int));
            cudaHostGetDevicePointer((void**)&ctx->dbg_dev, ctx->dbg_host, 0);
        }
    }
    *out = ctx;
    return TW_OK;
}

void tw_ctx_destroy(tw_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    DevMem* all[] = {&ctx->xs, &ctx->ys, &ctx->xo, &ctx->x, &ctx->yk1, &ctx->r, &ctx->imp, &ctx->dmin, &ctx->voff,
                     &ctx->vinc, &ctx->c_slot, &ctx->erank, &ctx->part_v,
                     &ctx->vcnt, &ctx->ly, &ctx->is_er, &ctx->er_edge, &ctx->er_index, &ctx->er_value, &ctx->er_g,
                     &ctx->er_q, &ctx->edge_lambda, &ctx->er_color, &ctx->er_by_color, &ctx->er_color_off,
                     &ctx->er_color_cnt, &ctx->pkey, &ctx->pids, &ctx->pdd, &ctx->pw, &ctx->pflag, &ctx->qcount,
                     &ctx->qslot, &ctx->cand, &ctx->c_key, &ctx->c_ids, &ctx->c_jac, &ctx->c_value, &ctx->c_diag, &ctx->c_q,
                     &ctx->c_lambda, &ctx->c_next, &ctx->c_color, &ctx->c_stamp, &ctx->c_tent, &ctx->c_arch,
                     &ctx->c_lost, &ctx->vmask, &ctx->vbig, &ctx->pk_ids, &ctx->pk_jac, &ctx->pk_q, &ctx->pk_diag, &ctx->pk_lam,
                     &ctx->c_by_color, &ctx->ccount, &ctx->coff, &ctx->arch_key0, &ctx->arch_key1,
                     &ctx->arch_val0, &ctx->arch_val1, &ctx->new_lb, &ctx->new_key, &ctx->new_val, &ctx->refpool,
                     &ctx->part_q, &ctx->part_c, &ctx->part_k, &ctx->globals, &ctx->box,
                     &ctx->bvh_tmp, &ctx->smd, &ctx->trace, &ctx->path, &ctx->s_kinds, &ctx->s_verts, &ctx->s_out,
                     &ctx->s_has};
    for (DevMem* d : all) d->release();
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->evk) cudaEventDestroy(ctx->evk);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* tw_last_error(const tw_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

int64_t tw_ctx_kernel_launches(const tw_ctx* ctx) { return ctx ? ctx->launches : 0; }

int tw_mesh_create(tw_ctx* ctx, int32_t nv, const double* inv_mass, int32_t ne_explicit, const int32_t* edges,
                   int32_t ns, const int32_t* strand_edges, int32_t nt, const int32_t* triangles, tw_mesh** out) {
    if (!ctx || !out || nv < 0 || ne_explicit < 0 || ns < 0 || nt < 0) return fail(ctx, TW_EINVAL, "mesh: bad sizes");
    *out = nullptr;
    CK(cudaSetDevice(ctx->device));
    tw_mesh* m = new tw_mesh();
    m->ctx = ctx;
    m->device = ctx->device;
    m->nv = nv;
    m->nt = nt;
    m->inv_mass.assign(nv, 1.0);
    if (inv_mass) m->inv_mass.assign(inv_mass, inv_mass + nv);
    // MeshState::validate (mesh.cpp:35-55)
    for (int v = 0; v < nv; ++v)
        if (!std::isfinite(m->inv_mass[v]) || m->inv_mass[v] < 0.0) {
            delete m;
            return fail(ctx, TW_EINVAL, "mesh: inv_mass must be finite and >= 0");
        }
    m->edges = finalize_edges(ne_explicit, edges, ns, strand_edges, nt, triangles);
    m->ne = (int)(m->edges.size() / 2);
    for (size_t i = 0; i < m->edges.size(); i += 2) {
        const int a = m->edges[i], b = m->edges[i + 1];
        if (a < 0 || a >= nv || b < 0 || b >= nv || a == b) {
            delete m;
            return fail(ctx, TW_EINVAL, "mesh: bad edge");
        }
    }
    for (int t = 0; t < nt; ++t) {
        const int a = triangles[3 * t], b = triangles[3 * t + 1], c = triangles[3 * t + 2];
        if (a < 0 || a >= nv || b < 0 || b >= nv || c < 0 || c >= nv || a == b || b == c || a == c) {
            delete m;
            return fail(ctx, TW_EINVAL, "mesh: bad triangle");
        }
    }
    // isolated vertices, vertex -> edge CSR (ascending edge index)
    std::vector<uint8_t> touched(nv, 0);
    std::vector<int> voff(nv + 1, 0);
    for (int e = 0; e < m->ne; ++e) {
        touched[m->edges[2 * e]] = touched[m->edges[2 * e + 1]] = 1;
        ++voff[m->edges[2 * e] + 1];
        ++voff[m->edges[2 * e + 1] + 1];
    }
    for (int t = 0; t < 3 * nt; ++t) touched[triangles[t]] = 1;
    for (int v = 0; v < nv; ++v) voff[v + 1] += voff[v];
    std::vector<int> vedge(std::max(1, voff[nv])), fillp(voff.begin(), voff.end() - 1);
    for (int e = 0; e < m->ne; ++e) {
        vedge[fillp[m->edges[2 * e]]++] = e;
        vedge[fillp[m->edges[2 * e + 1]]++] = e;
    }
    std::vector<int> iso;
    for (int v = 0; v < nv; ++v)
        if (!touched[v]) iso.push_back(v);
    m->niso = (int)iso.size();
    std::vector<int4> tris4(std::max(1, nt));
    for (int t = 0; t < nt; ++t) tris4[t] = make_int4(triangles[3 * t], triangles[3 * t + 1], triangles[3 * t + 2], -1);
    cudaStream_t s = ctx->stream;
    auto up = [&](DevMem& d, const void* src, size_t bytes) -> cudaError_t {
        cudaError_t e = d.ensure(bytes);
        if (e != cudaSuccess) return e;
        if (bytes) e = cudaMemcpyAsync(d.p, src, bytes, cudaMemcpyHostToDevice, s);
        return e;
    };
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = up(m->d_inv_mass, m->inv_mass.data(), (size_t)nv * 8);
    if (e == cudaSuccess) e = up(m->d_edges, m->edges.data(), (size_t)m->ne * 8);
    if (e == cudaSuccess) e = up(m->d_tris, tris4.data(), (size_t)nt * 16);
    if (e == cudaSuccess) e = up(m->d_iso, iso.data(), (size_t)m->niso * 4);
    if (e == cudaSuccess) e = up(m->d_vedge_off, voff.data(), (size_t)(nv + 1) * 4);
    if (e == cudaSuccess) e = up(m->d_vedge, vedge.data(), (size_t)voff[nv] * 4);
    // LBVH storage
    const int ncls[3] = {nt, m->ne, m->niso};
    for (int c = 0; c < 3 && e == cudaSuccess; ++c) {
        BvhMem& B = m->bvh[c];
        B.n = ncls[c];
        const size_t n = (size_t)std::max(1, B.n);
        if (e == cudaSuccess) e = B.prim.ensure(n * 4);
        if (e == cudaSuccess) e = B.child.ensure(n * 8);
        if (e == cudaSuccess) e = B.parent.ensure(2 * n * 4);
        if (e == cudaSuccess) e = B.node.ensure(n * 64);  // max(1, n - 1) internal nodes
        if (e == cudaSuccess) e = B.flag.ensure(n * 4);
        if (e == cudaSuccess) e = cudaMemsetAsync(B.flag.p, 0, n * 4, s);
    }
    // broad-phase query order buffers (filled at the mesh's first call)
    if (e == cudaSuccess) e = m->vperm.ensure((size_t)std::max(1, nv) * 4);
    if (e == cudaSuccess) e = m->eperm.ensure((size_t)std::max(1, m->ne) * 4);
    if (e == cudaSuccess) e = m->qspread.ensure(64);
    // device-mode edge-row precoloring (Jones-Plassmann rounds)
    if (e == cudaSuccess) e = m->d_edge_color.ensure((size_t)std::max(1, m->ne) * 4);
    if (e == cudaSuccess && m->ne > 0) {
        DevMem stamp, counter;
        std::vector<int> st(m->ne, 0);
        int participating = 0;
        for (int k = 0; k < m->ne; ++k) {
            const bool both_static = m->inv_mass[m->edges[2 * k]] == 0.0 && m->inv_mass[m->edges[2 * k + 1]] == 0.0;
            st[k] = both_static ? -1 : 0;
            participating += !both_static;
        }
        std::vector<int> col_init(m->ne, -1);
        e = stamp.ensure((size_t)m->ne * 4);
        if (e == cudaSuccess) e = counter.ensure(4);
        if (e == cudaSuccess) e = cudaMemcpyAsync(stamp.p, st.data(), (size_t)m->ne * 4, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(m->d_edge_color.p, col_init.data(), (size_t)m->ne * 4, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(counter.p, 0, 4, s);
        int colored = 0;
        for (int round = 1; e == cudaSuccess && colored < participating; ++round) {
            launch_edge_color_round(s, m->ne, m->d_edges.as<int2>(), m->d_inv_mass.as<double>(),
                                    m->d_vedge_off.as<int>(), m->d_vedge.as<int>(), m->d_edge_color.as<int>(),
                                    stamp.as<int>(), round, counter.as<int>());
            ++ctx->launches;
            e = cudaMemcpyAsync(&colored, counter.p, 4, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (round > m->ne + 2) break;
        }
        std::vector<int> cols(m->ne);
        if (e == cudaSuccess) e = cudaMemcpyAsync(cols.data(), m->d_edge_color.p, (size_t)m->ne * 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        int mx = -1;
        for (int c : cols) mx = std::max(mx, c);
        m->edge_ncolors = mx + 1;
        stamp.release();
        counter.release();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        delete m;
        return cuda_fail(ctx, e, "tw_mesh_create");
    }
    if (ctx->colcap < m->edge_ncolors + 64) ctx->colcap = m->edge_ncolors + 1024;
    *out = m;
    return TW_OK;
}

int32_t tw_mesh_num_edges(const tw_mesh* m) { return m ? m->ne : 0; }

int tw_mesh_edges(const tw_mesh* m, int32_t* out) {
    if (!m || !out) return TW_EINVAL;
    std::memcpy(out, m->edges.data(), m->edges.size() * 4);
    return TW_OK;
}

void tw_mesh_destroy(tw_mesh* m) {
    if (!m) return;
    cudaSetDevice(m->device);
    cudaDeviceSynchronize();
    DevMem* all[] = {&m->d_inv_mass, &m->d_edges, &m->d_tris, &m->d_iso, &m->d_vedge_off, &m->d_vedge, &m->d_edge_color,
                     &m->vperm, &m->eperm, &m->qspread};
    for (DevMem* d : all) d->release();
    for (auto& B : m->bvh) {
        B.prim.release(), B.child.release(), B.parent.release(), B.node.release(), B.flag.release();
    }
    delete m;
}

int tw_resolve(tw_ctx* ctx, tw_mesh* m, const double* x_start, const double* y_target, const tw_resolve_config* cfg,
               double* x_out, tw_resolve_stats* stats, double* step_max_disp, double* path, tw_step_trace* trace) {
    if (!ctx || !m || !x_start || !y_target || !x_out) return fail(ctx, TW_EINVAL, "resolve: null argument");
    int rc = check_cfg(ctx, cfg);
    if (rc) return rc;
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaSetDevice(ctx->device));
    rc = ensure_buffers(ctx, m, *cfg);
    if (rc) return rc;
    const size_t bytes = (size_t)m->nv * 24;
    if (bytes) {
        CK(cudaMemcpyAsync(ctx->xs.p, x_start, bytes, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->ys.p, y_target, bytes, cudaMemcpyHostToDevice, ctx->stream));
    }
    tw_resolve_stats st;
    rc = run_resolve(ctx, m, ctx->xs.as<double>(), ctx->ys.as<double>(), *cfg, ctx->xo.as<double>(), &st,
                     step_max_disp, cfg->record_path ? path : nullptr, trace, x_out);
    if (rc) return rc;
    if (cfg->record_path && path) CK(cudaStreamSynchronize(ctx->stream));
    st.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (stats) *stats = st;
    return TW_OK;
}

int tw_resolve_device(tw_ctx* ctx, tw_mesh* m, const double* d_x, const double* d_y, const tw_resolve_config* cfg,
                      double* d_out, tw_resolve_stats* stats) {
    if (!ctx || !m || !d_x || !d_y || !d_out) return fail(ctx, TW_EINVAL, "resolve: null argument");
    int rc = check_cfg(ctx, cfg);
    if (rc) return rc;
    tw_resolve_config c = *cfg;
    c.record_path = 0;
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaSetDevice(ctx->device));
    tw_resolve_stats st;
    rc = run_resolve(ctx, m, d_x, d_y, c, d_out, &st, nullptr, nullptr, nullptr);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    st.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (stats) *stats = st;
    return TW_OK;
}

// ---------------------------------------------------------------- stages
int tw_ctx_set_grid_share(tw_ctx* ctx, int32_t parts) {
    if (!ctx || parts < 1) return fail(ctx, TW_EINVAL, "set_grid_share: parts must be >= 1");
    const int per_sm = std::max(1, std::min(resolve_blocks_per_sm(ctx->minb), ctx->minb));
    const int full = std::min(ctx->sm_count * per_sm, tw::MAX_BLOCKS);
    ctx->grid_parts = parts;
    ctx->nblocks = std::max(1, full / parts);
    return TW_OK;
}

int tw_last_path(tw_ctx* ctx, int64_t cap_states, double* out, int32_t* nstates) {
    if (!ctx || !nstates || (cap_states > 0 && !out)) return fail(ctx, TW_EINVAL, "last_path: bad argument");
    *nstates = ctx->last_path_states;
    const int64_t n = std::min<int64_t>(cap_states, ctx->last_path_states);
    if (n > 0) {
        CK(cudaSetDevice(ctx->device));
        CK(cudaMemcpyAsync(out, ctx->path.p, (size_t)n * ctx->last_nv * 24, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return TW_OK;
}

int32_t tw_ctx_phase_profile(const tw_ctx* ctx, int32_t* sites, double* ms, int32_t* counts, int32_t cap) {
    if (!ctx) return 0;
    int n = 0;
    for (int i = 0; i < kPhaseSites; ++i) {
        if (!ctx->last.phase_cnt[i]) continue;
        if (n < cap) {
            sites[n] = i;
            ms[n] = ctx->last.phase_ns[i] * 1e-6;
            counts[n] = (int32_t)ctx->last.phase_cnt[i];
        }
        ++n;
    }
    return n;
}

int tw_stage_closest(tw_ctx* ctx, int32_t nv, const double* x, int64_t n, const int32_t* kinds, const int32_t* verts,
                     double* out, int32_t* has) {
    if (!ctx || nv < 0 || n < 0) return fail(ctx, TW_EINVAL, "closest: bad sizes");
    CK(cudaSetDevice(ctx->device));
    std::vector<double4> x4(std::max(1, nv));
    for (int v = 0; v < nv; ++v) x4[v] = make_double4(x[3 * v], x[3 * v + 1], x[3 * v + 2], 0.0);
    CK(ctx->x.ensure((size_t)std::max(1, nv) * 32));
    CK(ctx->s_kinds.ensure((size_t)std::max<int64_t>(1, n) * 8));
    CK(ctx->s_verts.ensure((size_t)std::max<int64_t>(1, n) * 24));
    CK(ctx->s_out.ensure((size_t)std::max<int64_t>(1, n) * 88));
    CK(ctx->s_has.ensure((size_t)std::max<int64_t>(1, n) * 4));
    cudaStream_t s = ctx->stream;
    CK(cudaMemcpyAsync(ctx->x.p, x4.data(), (size_t)nv * 32, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->s_kinds.p, kinds, (size_t)n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->s_verts.p, verts, (size_t)n * 24, cudaMemcpyHostToDevice, s));
    CK(launch_closest(s, nv, ctx->x.as<double4>(), n, ctx->s_kinds.as<int>(), ctx->s_verts.as<int>(),
                      ctx->s_out.as<double>(), ctx->s_has.as<int>()));
    ++ctx->launches;
    CK(cudaMemcpyAsync(out, ctx->s_out.p, (size_t)n * 88, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(has, ctx->s_has.p, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return TW_OK;
}

namespace {
int stage_upload_x(tw_ctx* ctx, tw_mesh* m, const double* x) {
    std::vector<double4> x4(std::max(1, m->nv));
    for (int v = 0; v < m->nv; ++v) x4[v] = make_double4(x[3 * v], x[3 * v + 1], x[3 * v + 2], m->inv_mass[v]);
    CK(cudaMemcpyAsync(ctx->x.p, x4.data(), (size_t)m->nv * 32, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return TW_OK;
}

// pair records in the layout the search writes (ids from the key, VT triangle
// ids from the device triangle table)
int stage_upload_pairs(tw_ctx* ctx, tw_mesh* m, int64_t np, const uint64_t* keys, const double* dist,
                       const double* wa, const double* wb, const double* dir, const uint8_t* flags) {
    // pack the pair records as the search writes them
    std::vector<int4> ids(np);
    std::vector<double4> dd(np), w(np);
    for (int64_t i = 0; i < np; ++i) {
        const uint64_t k = keys[i];
        const int ka = (int)(k >> 62), kb = (int)((k >> 60) & 3), ia = (int)((k >> 30) & 0x3fffffff),
                  ib = (int)(k & 0x3fffffff);
        int va[3] = {-1, -1, -1}, vb[3] = {-1, -1, -1};
        auto ids_of = [&](int kind, int idx, int* v) {
            if (kind == 0) v[0] = idx;
            else if (kind == 1) v[0] = m->edges[2 * idx], v[1] = m->edges[2 * idx + 1];
            else v[0] = v[1] = v[2] = -1;  // triangle ids: filled from the device table below
        };
        ids_of(ka, ia, va);
        ids_of(kb, ib, vb);
        ids[i] = ka == 1 ? make_int4(va[0], va[1], vb[0], vb[1]) : make_int4(va[0], vb[0], vb[1], vb[2]);
        dd[i] = make_double4(dir[3 * i], dir[3 * i + 1], dir[3 * i + 2], dist[i]);
        if (ka == 1) w[i] = make_double4(wa[3 * i], wa[3 * i + 1], wb[3 * i], wb[3 * i + 1]);
        else w[i] = make_double4(wb[3 * i], wb[3 * i + 1], wb[3 * i + 2], 0.0);
    }
    cudaStream_t s = ctx->stream;
    if (np) {
        CK(cudaMemcpyAsync(ctx->pkey.p, keys, np * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(ctx->pids.p, ids.data(), np * 16, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(ctx->pdd.p, dd.data(), np * 32, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(ctx->pw.p, w.data(), np * 32, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(ctx->pflag.p, flags, np, cudaMemcpyHostToDevice, s));
    }
    // triangle ids for VT pairs come from the device triangle table
    std::vector<int4> tris(m->nt);
    if (m->nt) CK(cudaMemcpyAsync(tris.data(), m->d_tris.p, (size_t)m->nt * 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    bool fix = false;
    for (int64_t i = 0; i < np; ++i) {
        const uint64_t k = keys[i];
        if (((k >> 60) & 3) == 2) {
            const int4 t = tris[k & 0x3fffffff];
            ids[i] = make_int4((int)((k >> 30) & 0x3fffffff), t.x, t.y, t.z);
            fix = true;
        }
    }
    if (fix && np) CK(cudaMemcpyAsync(ctx->pids.p, ids.data(), np * 16, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    return TW_OK;
}

int stage_download_pairs(tw_ctx* ctx, int64_t np, uint64_t* keys, double* dist, double* wa, double* wb, double* dir,
                         uint8_t* flags) {
    std::vector<int4> ids(np);
    std::vector<double4> dd(np), w(np);
    cudaStream_t s = ctx->stream;
    if (np) {
        CK(cudaMemcpyAsync(keys, ctx->pkey.p, np * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(dd.data(), ctx->pdd.p, np * 32, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(w.data(), ctx->pw.p, np * 32, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(flags, ctx->pflag.p, np, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < np; ++i) {
        const int ka = (int)(keys[i] >> 62), kb = (int)((keys[i] >> 60) & 3);
        dist[i] = dd[i].w;
        dir[3 * i] = dd[i].x, dir[3 * i + 1] = dd[i].y, dir[3 * i + 2] = dd[i].z;
        double a[3] = {1, 0, 0}, b[3] = {1, 0, 0};
        if (ka == 1) a[0] = w[i].x, a[1] = w[i].y, b[0] = w[i].z, b[1] = w[i].w;
        else if (kb == 2) b[0] = w[i].x, b[1] = w[i].y, b[2] = w[i].z;
        else if (kb == 1) b[0] = w[i].x, b[1] = w[i].y;
        for (int k = 0; k < 3; ++k) wa[3 * i + k] = a[k], wb[3 * i + k] = b[k];
        flags[i] &= (uint8_t)(PF_ACTIVE | PF_ALL_STATIC | PF_DEGENERATE);
    }
    return TW_OK;
}
}  // namespace

int tw_stage_search(tw_ctx* ctx, tw_mesh* m, const double* x, double d_max, int64_t cap, uint64_t* keys, double* dist,
                    double* wa, double* wb, double* dir, uint8_t* flags, int64_t* np) {
    if (!ctx || !m || !x || !np) return fail(ctx, TW_EINVAL, "search: null argument");
    if (!(d_max > 0.0)) return fail(ctx, TW_EINVAL, "proximity_search: d_max must be > 0");
    CK(cudaSetDevice(ctx->device));
    tw_resolve_config cfg;
    tw_default_config(&cfg);
    cfg.d_max = d_max;
    cfg.step_limit = 1;
    int rc = ensure_buffers(ctx, m, cfg);
    if (rc) return rc;
    rc = stage_upload_x(ctx, m, x);
    if (rc) return rc;
    Globals G;
    for (int attempt = 0;; ++attempt) {
        rc = ensure_buffers(ctx, m, cfg);
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
    if (G.np > cap) return fail(ctx, TW_ECAPACITY, "search: output capacity too small");
    return stage_download_pairs(ctx, G.np, keys, dist, wa, wb, dir, flags);
}

int tw_stage_refresh(tw_ctx* ctx, tw_mesh* m, const double* x, double bound, int64_t np, const uint64_t* keys,
                     double* dist, double* wa, double* wb, double* dir, uint8_t* flags, double* vertex_bound) {
    if (!ctx || !m || !x || np < 0) return fail(ctx, TW_EINVAL, "refresh: bad argument");
    CK(cudaSetDevice(ctx->device));
    tw_resolve_config cfg;
    tw_default_config(&cfg);
    cfg.step_limit = 1;
    if (ctx->pcap < np) grow_ll(ctx->pcap, np);
    int rc = ensure_buffers(ctx, m, cfg);
    if (rc) return rc;
    rc = stage_upload_x(ctx, m, x);
    if (rc) return rc;
    rc = stage_upload_pairs(ctx, m, np, keys, dist, wa, wb, dir, flags);
    if (rc) return rc;
    cudaStream_t s = ctx->stream;
    Params P = make_params(ctx, m, cfg);
    CK(cudaMemsetAsync(ctx->globals.p, 0, sizeof(Globals), s));
    CK(cudaMemsetAsync(ctx->dmin.p, 0x7f, (size_t)m->nv * 8, s));
    Globals G;
    std::memset(&G, 0, sizeof G);
    G.np = np;
    CK(cudaMemcpyAsync(ctx->globals.p, &G, sizeof G, cudaMemcpyHostToDevice, s));
    CK(coop_refresh(s, P, ctx->nblocks, bound));
    ++ctx->launches;
    CK(cudaMemcpyAsync(&G, ctx->globals.p, sizeof G, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (G.error) return fail(ctx, TW_ETIMEOUT, "refresh: device error");
    int rc2 = stage_download_pairs(ctx, np, const_cast<uint64_t*>(keys), dist, wa, wb, dir, flags);
    if (rc2) return rc2;
    if (vertex_bound) {
        CK(cudaMemcpyAsync(vertex_bound, ctx->r.p, (size_t)m->nv * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    return TW_OK;
}

int tw_stage_advance(tw_ctx* ctx, int32_t nv, const double* inv_mass, const double* y, const double* D, double gamma,
                     double* x, double* r, double* max_disp) {
    if (!ctx || nv < 0) return fail(ctx, TW_EINVAL, "advance: bad argument");
    CK(cudaSetDevice(ctx->device));
    const size_t n = (size_t)std::max(1, nv);
    CK(ctx->x.ensure(n * 32));
    CK(ctx->yk1.ensure(n * 32));
    CK(ctx->r.ensure(n * 8));
    CK(ctx->imp.ensure(n * 32));
    CK(ctx->dmin.ensure(n * 8));
    CK(ctx->voff.ensure((n + 1) * 4));
    CK(ctx->vcnt.ensure(n * 4));
    CK(ctx->globals.ensure(sizeof(Globals)));
    CK(ctx->part_k.ensure((size_t)ctx->nblocks * 8));
    std::vector<double4> x4(n), y4(n), imp(n, make_double4(0, 0, 0, 0));
    std::vector<double> Db(n);
    for (int v = 0; v < nv; ++v) {
        x4[v] = make_double4(x[3 * v], x[3 * v + 1], x[3 * v + 2], inv_mass[v]);
        y4[v] = make_double4(y[3 * v], y[3 * v + 1], y[3 * v + 2], inv_mass[v]);
        Db[v] = D[v];
    }
    cudaStream_t s = ctx->stream;
    CK(cudaMemcpyAsync(ctx->x.p, x4.data(), n * 32, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->yk1.p, y4.data(), n * 32, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->imp.p, imp.data(), n * 32, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->dmin.p, Db.data(), n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->r.p, r, (size_t)nv * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(ctx->globals.p, 0, sizeof(Globals), s));
    Params P;
    std::memset(&P, 0, sizeof P);
    P.cfg.gamma = gamma;
    P.nv = nv;
    P.x = ctx->x.as<double4>();
    P.yk1 = ctx->yk1.as<double4>();
    P.r = ctx->r.as<double>();
    P.imp = ctx->imp.as<double4>();
    P.dmin = ctx->dmin.as<unsigned long long>();
    P.voff = ctx->voff.as<int>();
    P.vcnt = ctx->vcnt.as<int>();
    P.part_k = ctx->part_k.as<long long>();
    P.g = ctx->globals.as<Globals>();
    CK(launch_advance(s, P, ctx->nblocks));
    ++ctx->launches;
    Globals G;
    CK(cudaMemcpyAsync(&G, ctx->globals.p, sizeof G, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(x4.data(), ctx->x.p, n * 32, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(r, ctx->r.p, (size_t)nv * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int v = 0; v < nv; ++v) x[3 * v] = x4[v].x, x[3 * v + 1] = x4[v].y, x[3 * v + 2] = x4[v].z;
    if (max_disp) {
        unsigned long long b = G.maxdisp_bits;
        double d;
        std::memcpy(&d, &b, 8);
        *max_disp = d;
    }
    return TW_OK;
}

int tw_ccd_certify(tw_ctx* ctx, tw_mesh* m, const double* x0, const double* x1, int32_t* violations,
                   int32_t* certain, int64_t* candidates) {
    if (!ctx || !m || !x0 || !x1 || !violations) return fail(ctx, TW_EINVAL, "ccd_certify: bad argument");
    CK(cudaSetDevice(ctx->device));
    tw_resolve_config cfg;
    tw_default_config(&cfg);
    cfg.step_limit = 1;
    int rc = TW_OK;
    cudaStream_t s = ctx->stream;
    Globals G;
    for (int attempt = 0;; ++attempt) {
        rc = ensure_buffers(ctx, m, cfg);
        if (rc) return rc;
        rc = stage_upload_x(ctx, m, x1);
        if (rc) return rc;
        CK(cudaMemcpyAsync(ctx->yk1.p, ctx->x.p, (size_t)m->nv * 32, cudaMemcpyDeviceToDevice, s));
        rc = stage_upload_x(ctx, m, x0);
        if (rc) return rc;
        Params P = make_params(ctx, m, cfg);
        P.ccd_x1 = ctx->yk1.as<double4>();
        P.niso = 0;  // the certifier has no isolated-vertex classes (VT over every vertex, EE)
        CK(cudaMemsetAsync(ctx->globals.p, 0, sizeof(Globals), s));
        rc = build_bvhs(ctx, m);
        if (rc) return rc;
        CK(coop_ccd(s, P, ctx->nblocks));
        ++ctx->launches;
        CK(cudaMemcpyAsync(&G, ctx->globals.p, sizeof G, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (G.error & ERR_TIMEOUT) return fail(ctx, TW_ETIMEOUT, "ccd_certify: watchdog");
        if (G.error & ERR_CAP_STACK) return fail(ctx, TW_ECAPACITY, "ccd_certify: traversal stack overflow");
        if (!(G.error & ERR_CAP_CAND)) break;
        if (attempt > 10) return fail(ctx, TW_ECAPACITY, "ccd_certify: capacity");
        grow_ll(ctx->ccap, (long long)G.ncand + (long long)G.ncand / 4);
    }
    *violations = G.ccd_violations;
    if (certain) *certain = G.ccd_certain;
    if (candidates) *candidates = (int64_t)G.ncand;
    return TW_OK;
}

int tw_stage_linearize(tw_ctx* ctx, tw_mesh* m, const double* x, int64_t np, const uint64_t* keys,
                       const double* dist, const double* wa, const double* wb, const double* dir,
                       const uint8_t* flags, const double* edge_targets, double delta, double sigma, int32_t family,
                       int32_t edge_constraints, int64_t cap, uint8_t* kind, int32_t* verts, double* value,
                       double* jac, double* diag, uint64_t* pair_key, int32_t* edge_index, int64_t* nrows) {
    if (!ctx || !m || !x || np < 0 || (np && (!keys || !dist || !wa || !wb || !dir || !flags)) || !nrows ||
        (m->ne && edge_constraints && !edge_targets) || !(delta > 0.0) || (family != 0 && family != 1))
        return fail(ctx, TW_EINVAL, "linearize: bad argument");
    CK(cudaSetDevice(ctx->device));
    tw_resolve_config cfg;
    tw_default_config(&cfg);
    cfg.step_limit = 1;
    cfg.delta = delta;
    cfg.sigma = sigma;
    cfg.family = family;
    cfg.edge_constraints = edge_constraints ? 1 : 0;
    if (ctx->pcap < np) grow_ll(ctx->pcap, np);
    int rc = ensure_buffers(ctx, m, cfg);
    if (rc) return rc;
    rc = stage_upload_x(ctx, m, x);
    if (rc) return rc;
    rc = stage_upload_pairs(ctx, m, np, keys, dist, wa, wb, dir, flags);
    if (rc) return rc;
    cudaStream_t s = ctx->stream;
    const int ne = m->ne;
    // frozen edge targets and the edge-row set (constraints.cpp:152-153)
    std::vector<double> ly(std::max(1, ne), 0.0);
    std::vector<uint8_t> is_er(std::max(1, ne), 0);
    for (int e = 0; e < ne && edge_constraints; ++e) {
        ly[e] = edge_targets[e];
        const int i = m->edges[2 * e], j = m->edges[2 * e + 1];
        is_er[e] = (ly[e] > 1e-12 && !(m->inv_mass[i] == 0.0 && m->inv_mass[j] == 0.0)) ? 1 : 0;
    }
    if (ne) {
        CK(cudaMemcpyAsync(ctx->ly.p, ly.data(), (size_t)ne * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(ctx->is_er.p, is_er.data(), (size_t)ne, cudaMemcpyHostToDevice, s));
    }
    CK(cudaMemcpyAsync(ctx->yk1.p, ctx->x.p, (size_t)m->nv * 32, cudaMemcpyDeviceToDevice, s));  // q unused
    CK(cudaMemsetAsync(ctx->vcnt.p, 0, (size_t)std::max(1, m->nv) * 4, s));
    CK(cudaMemsetAsync(ctx->er_color_cnt.p, 0, (size_t)ctx->colcap * 4, s));
    Params P = make_params(ctx, m, cfg);
    P.cfg.coloring_mode = 0;  // no device-mode edge buckets in the prologue
    Globals G;
    std::memset(&G, 0, sizeof G);
    G.np = np;
    CK(cudaMemcpyAsync(ctx->globals.p, &G, sizeof G, cudaMemcpyHostToDevice, s));
    CK(coop_stage_linearize(s, P, ctx->nblocks));
    ++ctx->launches;
    CK(cudaMemcpyAsync(&G, ctx->globals.p, sizeof G, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (G.error) return fail(ctx, TW_ETIMEOUT, "linearize: device error");
    const long long nc = G.nc, ner = G.ner, R = nc + ner;
    *nrows = R;
    if (R > cap) return fail(ctx, TW_ECAPACITY, "linearize: output capacity too small");
    std::vector<uint64_t> ck(nc);
    std::vector<int4> cid(nc);
    std::vector<double> cval(nc), cjac(nc * 12), cdiag(nc), erv(std::max(1, ne));
    std::vector<double4> erg(std::max(1, ne));
    std::vector<int> ere(std::max(1LL, ner));
    if (nc) {
        CK(cudaMemcpyAsync(ck.data(), ctx->c_key.p, nc * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(cid.data(), ctx->c_ids.p, nc * 16, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(cval.data(), ctx->c_value.p, nc * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(cjac.data(), ctx->c_jac.p, nc * 96, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(cdiag.data(), ctx->c_diag.p, nc * 8, cudaMemcpyDeviceToHost, s));
    }
    if (ner) {
        CK(cudaMemcpyAsync(ere.data(), ctx->er_edge.p, ner * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(erv.data(), ctx->er_value.p, (size_t)ne * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(erg.data(), ctx->er_g.p, (size_t)ne * 32, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    static const uint8_t row_kind[3][3] = {{3, 2, 0}, {255, 1, 255}, {255, 255, 255}};  // [ka][kb]: VV VE VT / EE
    for (long long i = 0; i < nc; ++i) {
        kind[i] = row_kind[ck[i] >> 62][(ck[i] >> 60) & 3];
        verts[4 * i] = cid[i].x, verts[4 * i + 1] = cid[i].y, verts[4 * i + 2] = cid[i].z, verts[4 * i + 3] = cid[i].w;
        value[i] = cval[i];
        for (int k = 0; k < 12; ++k) jac[12 * i + k] = cjac[12 * i + k];
        diag[i] = cdiag[i];
        pair_key[i] = ck[i];
        edge_index[i] = -1;
    }
    for (long long k = 0; k < ner; ++k) {
        const long long i = nc + k;
        const int e = ere[k];
        const double4 g = erg[e];
        const bool zero = g.x == 0.0 && g.y == 0.0 && g.z == 0.0;  // edge length <= 1e-12: zero rows
        kind[i] = 4;
        verts[4 * i] = m->edges[2 * e], verts[4 * i + 1] = m->edges[2 * e + 1];
        verts[4 * i + 2] = verts[4 * i + 3] = -1;
        value[i] = erv[e];
        const double j0[3] = {zero ? g.x : -g.x, zero ? g.y : -g.y, zero ? g.z : -g.z};
        const double j1[3] = {g.x, g.y, g.z};
        for (int c = 0; c < 3; ++c) jac[12 * i + c] = j0[c], jac[12 * i + 3 + c] = j1[c];
        for (int c = 6; c < 12; ++c) jac[12 * i + c] = 0.0;
        diag[i] = g.w;
        pair_key[i] = 0;
        edge_index[i] = e;
    }
    return TW_OK;
}

int tw_stage_color(tw_ctx* ctx, tw_mesh* m, int64_t nrows, const uint8_t* kind, const int32_t* verts,
                   const uint64_t* pair_key, const int32_t* edge_index, uint64_t seed, int32_t mode,
                   int32_t edge_constraints, int32_t* color, int32_t* ncolors) {
    if (!ctx || !m || nrows < 0 || (nrows && (!kind || !verts || !edge_index || !color)) || !ncolors ||
        (mode != TW_COLOR_REFERENCE && mode != TW_COLOR_DEVICE))
        return fail(ctx, TW_EINVAL, "color: bad argument");
    long long nc = 0;
    while (nc < nrows && kind[nc] != 4) ++nc;
    for (long long i = nc; i < nrows; ++i)
        if (kind[i] != 4 || edge_index[i] < 0 || edge_index[i] >= m->ne)
            return fail(ctx, TW_EINVAL, "color: contact rows must precede the edge rows");
    CK(cudaSetDevice(ctx->device));
    tw_resolve_config cfg;
    tw_default_config(&cfg);
    cfg.step_limit = 1;
    cfg.coloring_mode = mode;
    cfg.color_seed = seed;
    cfg.edge_constraints = edge_constraints ? 1 : 0;
    if (ctx->pcap < nc) grow_ll(ctx->pcap, nc);
    cudaStream_t s = ctx->stream;
    const int ne = m->ne;
    std::vector<int4> ids(std::max(1LL, nc));
    std::vector<uint64_t> keys(std::max(1LL, nc), 0);
    for (long long i = 0; i < nc; ++i) {
        ids[i] = make_int4(verts[4 * i], verts[4 * i + 1], verts[4 * i + 2], verts[4 * i + 3]);
        if (pair_key) keys[i] = pair_key[i];
    }
    std::vector<uint8_t> is_er(std::max(1, ne), 0);
    for (long long i = nc; i < nrows; ++i) is_er[edge_index[i]] = 1;
    Globals G;
    for (int attempt = 0;; ++attempt) {
        int rc = ensure_buffers(ctx, m, cfg);
        if (rc) return rc;
        if (nc) {
            CK(cudaMemcpyAsync(ctx->c_ids.p, ids.data(), nc * 16, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(ctx->c_key.p, keys.data(), nc * 8, cudaMemcpyHostToDevice, s));
            CK(cudaMemsetAsync(ctx->c_lambda.p, 0, nc * 8, s));
        }
        if (ne) {
            CK(cudaMemcpyAsync(ctx->is_er.p, is_er.data(), (size_t)ne, cudaMemcpyHostToDevice, s));
            CK(cudaMemsetAsync(ctx->edge_lambda.p, 0, (size_t)ne * 8, s));
            CK(cudaMemcpyAsync(ctx->er_color.p, m->d_edge_color.p, (size_t)ne * 4, cudaMemcpyDeviceToDevice, s));
        }
        CK(cudaMemsetAsync(ctx->vcnt.p, 0, (size_t)std::max(1, m->nv) * 4, s));
        CK(cudaMemsetAsync(ctx->ccount.p, 0, (size_t)ctx->colcap * 4, s));
        CK(cudaMemsetAsync(ctx->er_color_cnt.p, 0, (size_t)ctx->colcap * 4, s));
        std::memset(&G, 0, sizeof G);
        G.max_color = -1;  // no contact row colored yet
        if (mode == TW_COLOR_REFERENCE) G.watchdog_ns = 600000000000ull;  // one-thread replay
        CK(cudaMemcpyAsync(ctx->globals.p, &G, sizeof G, cudaMemcpyHostToDevice, s));
        Params P = make_params(ctx, m, cfg);
        CK(coop_stage_color(s, P, ctx->nblocks, nc));
        ++ctx->launches;
        CK(cudaMemcpyAsync(&G, ctx->globals.p, sizeof G, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int capbits = G.error & (ERR_CAP_COLORS | ERR_CAP_REFPOOL);
        if (G.error & ~(ERR_CAP_COLORS | ERR_CAP_REFPOOL)) return fail(ctx, TW_ETIMEOUT, "color: device error");
        if (!capbits) break;
        if (attempt > 8) return fail(ctx, TW_ECAPACITY, "color: capacity growth did not converge");
        if (G.error & ERR_CAP_COLORS) ctx->colcap *= 4;
        if (G.error & ERR_CAP_REFPOOL) ctx->refpool_cap *= 4;
    }
    std::vector<int> cc(std::max(1LL, nc)), ec(std::max(1, ne));
    if (nc) CK(cudaMemcpyAsync(cc.data(), ctx->c_color.p, nc * 4, cudaMemcpyDeviceToHost, s));
    if (ne) CK(cudaMemcpyAsync(ec.data(), ctx->er_color.p, (size_t)ne * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int nco = G.max_color + 1;
    for (long long i = 0; i < nc; ++i) color[i] = cc[i];
    for (long long i = nc; i < nrows; ++i) {
        color[i] = ec[edge_index[i]];
        nco = std::max(nco, color[i] + 1);
    }
    *ncolors = nco;
    return TW_OK;
}

int tw_stage_backward(tw_ctx* ctx, int32_t nv, const double* inv_mass, int64_t nrows, const int32_t* verts,
                      const double* value, const double* jac, const double* diag, const int32_t* color,
                      int32_t ncolors, const double* x, const double* y_target, int32_t solver, int32_t sweeps,
                      double under_relax, double* lambda, double* q_out, double* y_out) {
    if (!y_out) return fail(ctx, TW_EINVAL, "backward: bad argument");
    return tw_stage_lcp(ctx, nv, inv_mass, nrows, verts, value, jac, diag, color, ncolors, x, y_target, solver,
                        sweeps, under_relax, TW_LCP_ASSEMBLE | TW_LCP_SOLVE | TW_LCP_RECOVER, lambda, q_out,
                        nullptr, y_out);
}

int tw_stage_lcp(tw_ctx* ctx, int32_t nv, const double* inv_mass, int64_t nrows, const int32_t* verts,
                 const double* value, const double* jac, const double* diag, const int32_t* color, int32_t ncolors,
                 const double* x, const double* y_target, int32_t solver, int32_t sweeps, double under_relax,
                 int32_t mode, double* lambda, double* q, double* impulse, double* y_out) {
    const bool assemble = mode & TW_LCP_ASSEMBLE, solve = mode & TW_LCP_SOLVE, recover = mode & TW_LCP_RECOVER;
    if (!ctx || nv < 0 || !inv_mass || nrows < 0 || (mode & ~7) || !mode ||
        (nrows && (!verts || !jac || !lambda)) || (nrows && assemble && !value) || (nrows && solve && !diag) ||
        ((assemble || recover) && !y_target) || (assemble && !x) || (recover && !y_out) ||
        (!assemble && (solve || recover) && !impulse) || (!assemble && solve && nrows && !q) || sweeps < 1 ||
        (solve && solver == TW_SOLVER_PGS && nrows && (!color || ncolors < 1)))
        return fail(ctx, TW_EINVAL, "backward: bad argument");
    if (solver != TW_SOLVER_PGS && solver != TW_SOLVER_JACOBI)
        return fail(ctx, TW_EUNSUPPORTED, "backward: only pgs and jacobi run on the device");
    for (int64_t i = 0; i < nrows; ++i) {
        if (solver == TW_SOLVER_PGS && (color[i] < 0 || color[i] >= ncolors))
            return fail(ctx, TW_EINVAL, "backward: color out of range");
        for (int k = 0; k < 4; ++k)
            if (verts[4 * i + k] >= nv) return fail(ctx, TW_EINVAL, "backward: vertex id out of range");
    }
    CK(cudaSetDevice(ctx->device));
    // rows carry their own vertex ids: a vertex-only mesh sizes the buffers
    tw_mesh* m = nullptr;
    int rc = tw_mesh_create(ctx, nv, inv_mass, 0, nullptr, 0, nullptr, 0, nullptr, &m);
    if (rc) return rc;
    struct Guard {
        tw_mesh* m;
        ~Guard() { tw_mesh_destroy(m); }
    } guard{m};
    tw_resolve_config cfg;
    tw_default_config(&cfg);
    cfg.step_limit = 1;
    cfg.solver = solver;
    cfg.sweeps = sweeps;
    cfg.under_relax = under_relax;
    cfg.edge_constraints = 0;
    cfg.coloring_mode = TW_COLOR_REFERENCE;  // colors are given
    if (ctx->pcap < nrows) grow_ll(ctx->pcap, nrows);
    if (ctx->colcap < ncolors + 1) ctx->colcap = ncolors + 1024;
    rc = ensure_buffers(ctx, m, cfg);
    if (rc) return rc;
    cudaStream_t s = ctx->stream;
    const size_t n = (size_t)std::max(1, nv);
    std::vector<double4> x4(n), y4(n), imp4(n);
    for (int v = 0; v < nv; ++v) {
        if (x) x4[v] = make_double4(x[3 * v], x[3 * v + 1], x[3 * v + 2], inv_mass[v]);
        if (y_target) y4[v] = make_double4(y_target[3 * v], y_target[3 * v + 1], y_target[3 * v + 2], inv_mass[v]);
        if (impulse) imp4[v] = make_double4(impulse[3 * v], impulse[3 * v + 1], impulse[3 * v + 2], inv_mass[v]);
    }
    std::vector<int4> ids(std::max<int64_t>(1, nrows));
    for (int64_t i = 0; i < nrows; ++i)
        ids[i] = make_int4(verts[4 * i], verts[4 * i + 1], verts[4 * i + 2], verts[4 * i + 3]);
    CK(cudaMemcpyAsync(ctx->x.p, x4.data(), n * 32, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->yk1.p, y4.data(), n * 32, cudaMemcpyHostToDevice, s));
    if (nrows) {
        CK(cudaMemcpyAsync(ctx->c_ids.p, ids.data(), nrows * 16, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(ctx->c_jac.p, jac, nrows * 96, cudaMemcpyHostToDevice, s));
        if (value) CK(cudaMemcpyAsync(ctx->c_value.p, value, nrows * 8, cudaMemcpyHostToDevice, s));
        if (diag) CK(cudaMemcpyAsync(ctx->c_diag.p, diag, nrows * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(ctx->c_lambda.p, lambda, nrows * 8, cudaMemcpyHostToDevice, s));
        if (!assemble && q) CK(cudaMemcpyAsync(ctx->c_q.p, q, nrows * 8, cudaMemcpyHostToDevice, s));
        if (solve && solver == TW_SOLVER_PGS)
            CK(cudaMemcpyAsync(ctx->c_color.p, color, nrows * 4, cudaMemcpyHostToDevice, s));
    }
    if (!assemble) CK(cudaMemcpyAsync(ctx->imp.p, imp4.data(), n * 32, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(ctx->vcnt.p, 0, n * 4, s));
    CK(cudaMemsetAsync(ctx->ccount.p, 0, (size_t)ctx->colcap * 4, s));
    CK(cudaMemsetAsync(ctx->globals.p, 0, sizeof(Globals), s));
    Params P = make_params(ctx, m, cfg);
    CK(coop_stage_backward(s, P, ctx->nblocks, nrows, solver == TW_SOLVER_PGS ? ncolors : 0, mode));
    ++ctx->launches;
    Globals G;
    CK(cudaMemcpyAsync(&G, ctx->globals.p, sizeof G, cudaMemcpyDeviceToHost, s));
    if (nrows) {
        CK(cudaMemcpyAsync(lambda, ctx->c_lambda.p, nrows * 8, cudaMemcpyDeviceToHost, s));
        if (assemble && q) CK(cudaMemcpyAsync(q, ctx->c_q.p, nrows * 8, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaMemcpyAsync(imp4.data(), ctx->imp.p, n * 32, cudaMemcpyDeviceToHost, s));
    if (recover) CK(cudaMemcpyAsync(x4.data(), ctx->x.p, n * 32, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (G.error) return fail(ctx, TW_ETIMEOUT, "backward: device error");
    if (recover)
        for (int v = 0; v < nv; ++v) y_out[3 * v] = x4[v].x, y_out[3 * v + 1] = x4[v].y, y_out[3 * v + 2] = x4[v].z;
    if (impulse)
        for (int v = 0; v < nv; ++v)
            impulse[3 * v] = imp4[v].x, impulse[3 * v + 1] = imp4[v].y, impulse[3 * v + 2] = imp4[v].z;
    return TW_OK;
}


int tw_stage_build_rows(tw_ctx* ctx, int32_t nv, const double* x, int64_t n, const int32_t* kinds,
                        const int32_t* verts, const double* closest, double delta, int32_t gap, uint8_t* kind,
                        int32_t* nverts, int32_t* row_verts, double* value, double* jac, uint8_t* flavor,
                        double* ref_volume, double* gap_weights, double* denom) {
    if (!ctx || nv < 0 || n < 0 || !x || (n && (!kinds || !verts || !closest || !kind || !nverts || !row_verts ||
                                                 !value || !jac || !flavor || !ref_volume || !gap_weights || !denom)) ||
        !(delta > 0.0))
        return fail(ctx, TW_EINVAL, "build_rows: bad argument");
    for (int64_t i = 0; i < n; ++i) {
        const int ka = kinds[2 * i], kb = kinds[2 * i + 1];
        const bool ok = (ka == 0 && (kb == 0 || kb == 1 || kb == 2)) || (ka == 1 && kb == 1);
        if (!ok) return fail(ctx, TW_EINVAL, "build_rows: unsupported pair kinds");
        for (int k = 0; k < 6; ++k)
            if (verts[6 * i + k] >= nv) return fail(ctx, TW_EINVAL, "build_rows: vertex id out of range");
    }
    CK(cudaSetDevice(ctx->device));
    if (!n) return TW_OK;
    Scratch S;
    const double4* dx = upload_x4(S, nv, x, nullptr);
    const int* dk = S.up(kinds, 2 * (size_t)n);
    const int* dv = S.up(verts, 6 * (size_t)n);
    const double* dc = S.up(closest, 11 * (size_t)n);
    int *okind = S.out<int>(n), *onv = S.out<int>(n), *orv = S.out<int>(4 * n), *ofl = S.out<int>(n);
    double *oval = S.out<double>(n), *ojac = S.out<double>(12 * n), *orefv = S.out<double>(n),
           *ogw = S.out<double>(4 * n), *oden = S.out<double>(n);
    if (S.err) return cuda_fail(ctx, S.err, "build_rows: upload");
    launch_build_rows(ctx->stream, dx, n, dk, dv, dc, delta, gap ? 1 : 0, okind, onv, orv, oval, ojac, ofl, orefv, ogw,
                      oden);
    ++ctx->launches;
    CK(cudaStreamSynchronize(ctx->stream));
    std::vector<int> hk(n), hf(n);
    S.down(hk.data(), okind, n);
    S.down(nverts, onv, n);
    S.down(row_verts, orv, 4 * n);
    S.down(value, oval, n);
    S.down(jac, ojac, 12 * n);
    S.down(hf.data(), ofl, n);
    S.down(ref_volume, orefv, n);
    S.down(gap_weights, ogw, 4 * n);
    S.down(denom, oden, n);
    if (S.err) return cuda_fail(ctx, S.err, "build_rows: download");
    for (int64_t i = 0; i < n; ++i) kind[i] = (uint8_t)hk[i], flavor[i] = (uint8_t)hf[i];
    return TW_OK;
}

int tw_stage_constraint_value(tw_ctx* ctx, int32_t nv, const double* x, int64_t n, const uint8_t* flavor,
                              const int32_t* nverts, const int32_t* row_verts, const double* ref_volume,
                              const double* gap_weights, const double* denom, const double* sigma, double* out) {
    if (!ctx || nv < 0 || n < 0 || !x ||
        (n && (!flavor || !nverts || !row_verts || !ref_volume || !gap_weights || !denom || !sigma || !out)))
        return fail(ctx, TW_EINVAL, "constraint_value: bad argument");
    for (int64_t i = 0; i < n; ++i) {
        if (flavor[i] > 2 || nverts[i] < 1 || nverts[i] > 4) return fail(ctx, TW_EINVAL, "constraint_value: bad row");
        for (int k = 0; k < nverts[i]; ++k)
            if (row_verts[4 * i + k] < 0 || row_verts[4 * i + k] >= nv)
                return fail(ctx, TW_EINVAL, "constraint_value: vertex id out of range");
    }
    CK(cudaSetDevice(ctx->device));
    if (!n) return TW_OK;
    Scratch S;
    std::vector<int> fl(flavor, flavor + n);
    const double4* dx = upload_x4(S, nv, x, nullptr);
    const int* df = S.up(fl.data(), n);
    const int* dn = S.up(nverts, n);
    const int* dv = S.up(row_verts, 4 * (size_t)n);
    const double* drv = S.up(ref_volume, n);
    const double* dg = S.up(gap_weights, 4 * (size_t)n);
    const double* dd = S.up(denom, n);
    const double* ds = S.up(sigma, n);
    double* dout = S.out<double>(n);
    if (S.err) return cuda_fail(ctx, S.err, "constraint_value: upload");
    launch_value_at(ctx->stream, dx, n, df, dn, dv, drv, dg, dd, ds, dout);
    ++ctx->launches;
    CK(cudaStreamSynchronize(ctx->stream));
    S.down(out, dout, n);
    if (S.err) return cuda_fail(ctx, S.err, "constraint_value: download");
    return TW_OK;
}

int tw_stage_fill_diag(tw_ctx* ctx, int32_t nv, const double* inv_mass, int64_t n, const int32_t* nverts,
                       const int32_t* row_verts, const double* jac, double* diag) {
    if (!ctx || nv < 0 || n < 0 || !inv_mass || (n && (!nverts || !row_verts || !jac || !diag)))
        return fail(ctx, TW_EINVAL, "fill_diag: bad argument");
    for (int64_t i = 0; i < n; ++i) {
        if (nverts[i] < 0 || nverts[i] > 4) return fail(ctx, TW_EINVAL, "fill_diag: bad row");
        for (int k = 0; k < nverts[i]; ++k)
            if (row_verts[4 * i + k] < 0 || row_verts[4 * i + k] >= nv)
                return fail(ctx, TW_EINVAL, "fill_diag: vertex id out of range");
    }
    CK(cudaSetDevice(ctx->device));
    if (!n) return TW_OK;
    Scratch S;
    const double* dm = S.up(inv_mass, nv);
    const int* dn = S.up(nverts, n);
    const int* dv = S.up(row_verts, 4 * (size_t)n);
    const double* dj = S.up(jac, 12 * (size_t)n);
    double* dd = S.out<double>(n);
    if (S.err) return cuda_fail(ctx, S.err, "fill_diag: upload");
    launch_fill_diag(ctx->stream, dm, n, dn, dv, dj, dd);
    ++ctx->launches;
    CK(cudaStreamSynchronize(ctx->stream));
    S.down(diag, dd, n);
    if (S.err) return cuda_fail(ctx, S.err, "fill_diag: download");
    return TW_OK;
}

int tw_stage_linearize_ex(tw_ctx* ctx, tw_mesh* m, const double* x, int64_t np, const uint64_t* keys,
                          const double* dist, const double* wa, const double* wb, const double* dir,
                          const uint8_t* flags, const double* edge_targets, double delta, double sigma,
                          int32_t family, int32_t edge_constraints, int64_t cap, uint8_t* kind, int32_t* verts,
                          double* value, double* jac, double* diag, uint64_t* pair_key, int32_t* edge_index,
                          uint8_t* flavor, double* ref_volume, double* gap_weights, double* denom, int64_t* nrows) {
    int rc = tw_stage_linearize(ctx, m, x, np, keys, dist, wa, wb, dir, flags, edge_targets, delta, sigma, family,
                                edge_constraints, cap, kind, verts, value, jac, diag, pair_key, edge_index, nrows);
    if (rc) return rc;
    if (!flavor || !ref_volume || !gap_weights || !denom) return fail(ctx, TW_EINVAL, "linearize_ex: null output");
    const int64_t R = *nrows;
    // contact rows: their re-evaluation data from the device row builder on
    // the same pair records (pair order = key order)
    std::vector<int32_t> kinds, pv;
    std::vector<double> cl;
    std::vector<int64_t> rows;
    for (int64_t i = 0; i < R; ++i) {
        if (kind[i] == 4) continue;
        const uint64_t k = pair_key[i];
        const int64_t p = std::lower_bound(keys, keys + np, k) - keys;
        const int ka = (int)(k >> 62), kb = (int)((k >> 60) & 3);
        const int ia = (int)((k >> 30) & 0x3fffffff), ib = (int)(k & 0x3fffffff);
        int va[3] = {-1, -1, -1}, vb[3] = {-1, -1, -1};
        if (ka == 0) va[0] = ia;
        else va[0] = m->edges[2 * ia], va[1] = m->edges[2 * ia + 1];
        if (kb == 0) vb[0] = ib;
        else if (kb == 1) vb[0] = m->edges[2 * ib], vb[1] = m->edges[2 * ib + 1];
        else vb[0] = verts[4 * i + 1], vb[1] = verts[4 * i + 2], vb[2] = verts[4 * i + 3];  // VT: (a, t0, t1, t2)
        if (kb == 2 && kind[i] != 0) {  // a VT gap row keeps the same vertex order
            vb[0] = verts[4 * i + 1], vb[1] = verts[4 * i + 2], vb[2] = verts[4 * i + 3];
        }
        kinds.insert(kinds.end(), {ka, kb});
        pv.insert(pv.end(), {va[0], va[1], va[2], vb[0], vb[1], vb[2]});
        cl.push_back(dist[p]);
        for (int c = 0; c < 3; ++c) cl.push_back(wa[3 * p + c]);
        for (int c = 0; c < 3; ++c) cl.push_back(wb[3 * p + c]);
        for (int c = 0; c < 3; ++c) cl.push_back(dir[3 * p + c]);
        cl.push_back((flags[p] & PF_DEGENERATE) ? 1.0 : 0.0);
        rows.push_back(i);
    }
    const int64_t nc = (int64_t)rows.size();
    if (nc) {
        std::vector<uint8_t> k2(nc), f2(nc);
        std::vector<int32_t> n2(nc), v2(4 * nc);
        std::vector<double> val2(nc), j2(12 * nc), rv2(nc), g2(4 * nc), d2(nc);
        rc = tw_stage_build_rows(ctx, m->nv, x, nc, kinds.data(), pv.data(), cl.data(), delta, family, k2.data(),
                                 n2.data(), v2.data(), val2.data(), j2.data(), f2.data(), rv2.data(), g2.data(),
                                 d2.data());
        if (rc) return rc;
        for (int64_t r = 0; r < nc; ++r) {
            const int64_t i = rows[r];
            if (val2[r] != value[i] && !(std::isnan(val2[r]) && std::isnan(value[i])))
                return fail(ctx, TW_ECUDA, "linearize_ex: row builder disagrees with the linearization");
            flavor[i] = f2[r];
            ref_volume[i] = rv2[r];
            for (int c = 0; c < 4; ++c) gap_weights[4 * i + c] = g2[4 * r + c];
            denom[i] = d2[r];
        }
    }
    for (int64_t i = 0; i < R; ++i)
        if (kind[i] == 4) {
            flavor[i] = 2;
            ref_volume[i] = 0.0;
            for (int c = 0; c < 4; ++c) gap_weights[4 * i + c] = 0.0;
            denom[i] = edge_targets[edge_index[i]];
        }
    return TW_OK;
}

}  // extern "C"

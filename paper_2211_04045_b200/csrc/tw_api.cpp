// C++ API of the reference (include/twoway/*.hpp) implemented over the C-ABI.
// MeshState helpers restate proj/src/mesh.cpp; resolve()/repair() upload the
// topology once per mesh (cached per thread by topology hash) and run the
// device-resident Alg. 1.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <unordered_map>

#include "tw_c.h"
#include "twoway/resolve.hpp"

namespace twoway {

// ------------------------------------------------------------ MeshState
void MeshState::finalize() {  // mesh.cpp:10-33
    const int n = num_vertices();
    if (velocities.size() != positions.size()) velocities.assign(n, Vec3::Zero());
    if (inv_mass.size() != positions.size()) inv_mass.assign(n, 1.0);
    std::map<std::pair<int, int>, int> seen;
    auto key = [](int a, int b) { return std::make_pair(std::min(a, b), std::max(a, b)); };
    for (const auto& e : edges) seen.emplace(key(e[0], e[1]), 1);
    for (const auto& e : strand_edges)
        if (seen.emplace(key(e[0], e[1]), 1).second) edges.push_back(e);
    for (const auto& t : triangles)
        for (int k = 0; k < 3; ++k) {
            const int a = t[k], b = t[(k + 1) % 3];
            if (seen.emplace(key(a, b), 1).second) edges.push_back({std::min(a, b), std::max(a, b)});
        }
    vertex_triangles.assign(n, {});
    vertex_edges.assign(n, {});
    for (int t = 0; t < static_cast<int>(triangles.size()); ++t)
        for (int k = 0; k < 3; ++k) vertex_triangles[triangles[t][k]].push_back(t);
    for (int e = 0; e < static_cast<int>(edges.size()); ++e)
        for (int k = 0; k < 2; ++k) vertex_edges[edges[e][k]].push_back(e);
}

void MeshState::validate() const {  // mesh.cpp:35-55
    const int n = num_vertices();
    if (velocities.size() != positions.size() || inv_mass.size() != positions.size())
        throw std::invalid_argument("mesh: velocity/mass arrays out of sync with positions");
    for (int v = 0; v < n; ++v) {
        if (!positions[v].allFinite()) throw std::invalid_argument("mesh: non-finite position");
        if (!std::isfinite(inv_mass[v]) || inv_mass[v] < 0.0)
            throw std::invalid_argument("mesh: inv_mass must be finite and >= 0");
    }
    for (const auto& e : edges) {
        if (e[0] < 0 || e[0] >= n || e[1] < 0 || e[1] >= n) throw std::invalid_argument("mesh: edge index out of range");
        if (e[0] == e[1]) throw std::invalid_argument("mesh: degenerate edge");
    }
    for (const auto& t : triangles) {
        for (int k = 0; k < 3; ++k)
            if (t[k] < 0 || t[k] >= n) throw std::invalid_argument("mesh: triangle index out of range");
        if (t[0] == t[1] || t[1] == t[2] || t[0] == t[2]) throw std::invalid_argument("mesh: degenerate triangle");
    }
}

void compute_lumped_masses(MeshState& mesh, double area_density, double line_density) {  // mesh.cpp:57-77
    const int n = mesh.num_vertices();
    std::vector<double> mass(n, 0.0);
    for (const auto& t : mesh.triangles) {
        const Vec3 e1 = mesh.positions[t[1]] - mesh.positions[t[0]];
        const Vec3 e2 = mesh.positions[t[2]] - mesh.positions[t[0]];
        const double m = area_density * 0.5 * e1.cross(e2).norm();
        for (int k = 0; k < 3; ++k) mass[t[k]] += m / 3.0;
    }
    for (const auto& e : mesh.strand_edges) {
        const double m = line_density * (mesh.positions[e[1]] - mesh.positions[e[0]]).norm();
        mass[e[0]] += 0.5 * m;
        mass[e[1]] += 0.5 * m;
    }
    for (int v = 0; v < n; ++v) {
        if (mesh.inv_mass[v] == 0.0) continue;
        mesh.inv_mass[v] = mass[v] > 0.0 ? 1.0 / mass[v] : 1.0;
    }
}

int append_mesh(MeshState& mesh, const MeshState& other) {  // mesh.cpp:79-106
    const int off = mesh.num_vertices();
    mesh.positions.insert(mesh.positions.end(), other.positions.begin(), other.positions.end());
    mesh.velocities.insert(mesh.velocities.end(), other.velocities.begin(), other.velocities.end());
    mesh.inv_mass.insert(mesh.inv_mass.end(), other.inv_mass.begin(), other.inv_mass.end());
    for (const auto& t : other.triangles) mesh.triangles.push_back({t[0] + off, t[1] + off, t[2] + off});
    for (const auto& e : other.strand_edges) mesh.strand_edges.push_back({e[0] + off, e[1] + off});
    for (const auto& e : other.edges) {
        bool from_tri = false;
        for (const auto& t : other.triangles) {
            for (int k = 0; k < 3; ++k) {
                const int a = t[k], b = t[(k + 1) % 3];
                if (std::min(a, b) == std::min(e[0], e[1]) && std::max(a, b) == std::max(e[0], e[1])) from_tri = true;
            }
            if (from_tri) break;
        }
        if (!from_tri) {
            const bool strand =
                std::find(other.strand_edges.begin(), other.strand_edges.end(), e) != other.strand_edges.end();
            if (!strand) mesh.edges.push_back({e[0] + off, e[1] + off});
        }
    }
    mesh.finalize();
    return off;
}

// --------------------------------------------------------- ResolveConfig
void ResolveConfig::validate() const {  // resolve.cpp:12-21
    if (!(d_min > 0.0) || !(d_min <= d_max)) throw std::invalid_argument("resolve: need 0 < d_min <= d_max");
    if (!(delta > 0.0) || !(delta <= d_min)) throw std::invalid_argument("resolve: need 0 < delta <= d_min");
    if (!(gamma > 0.0) || !(gamma < 1.0)) throw std::invalid_argument("resolve: need 0 < gamma < 1");
    if (!(eps > 0.0)) throw std::invalid_argument("resolve: need eps > 0");
    if (step_limit < 1) throw std::invalid_argument("resolve: need step_limit >= 1");
    if (sweeps < 1) throw std::invalid_argument("resolve: need sweeps >= 1");
}

std::string ResolveStats::csv_header() { return "steps,searches,residual,max_disp,ms"; }

std::string ResolveStats::csv_row() const {  // resolve.cpp:23-34
    double md = 0.0;
    for (double d : step_max_disp) md = std::max(md, d);
    char buf[160];
    std::snprintf(buf, sizeof(buf), "%d,%d,%.9g,%.9g,%.3f", steps, searches, final_residual, md, wall_ms);
    return buf;
}

// ----------------------------------------------------------- device path
namespace {

struct CtxDeleter {
    void operator()(tw_ctx* c) const { tw_ctx_destroy(c); }
};
struct MeshDeleter {
    void operator()(tw_mesh* m) const { tw_mesh_destroy(m); }
};

struct ThreadState {
    std::map<int, std::unique_ptr<tw_ctx, CtxDeleter>> ctx;  // per device
    struct Cached {
        uint64_t hash = 0;
        std::unique_ptr<tw_mesh, MeshDeleter> mesh;
    };
    std::map<std::pair<int, const MeshState*>, Cached> meshes;
};

thread_local ThreadState g_state;

uint64_t topology_hash(const MeshState& m) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) {
        h ^= v;
        h *= 1099511628211ull;
    };
    mix(m.positions.size());
    for (const auto& e : m.edges) mix((uint64_t)(uint32_t)e[0] << 32 | (uint32_t)e[1]);
    for (const auto& t : m.triangles) mix(((uint64_t)(uint32_t)t[0] << 40) ^ ((uint64_t)(uint32_t)t[1] << 20) ^ (uint32_t)t[2]);
    for (double im : m.inv_mass) {
        uint64_t b;
        std::memcpy(&b, &im, 8);
        mix(b);
    }
    return h;
}

[[noreturn]] void throw_status(int rc, tw_ctx* ctx) {
    const std::string msg = tw_last_error(ctx);
    if (rc == TW_EINVAL || rc == TW_EUNSUPPORTED) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

tw_ctx* context(int device) {
    auto& slot = g_state.ctx[device];
    if (!slot) {
        tw_ctx* c = nullptr;
        const int rc = tw_ctx_create(device, nullptr, &c);
        if (rc != TW_OK) throw std::runtime_error("twoway: no CUDA device available for the B200 path");
        slot.reset(c);
    }
    return slot.get();
}

tw_mesh* device_mesh(tw_ctx* ctx, int device, const MeshState& mesh) {
    const uint64_t h = topology_hash(mesh);
    auto& c = g_state.meshes[{device, &mesh}];
    if (c.mesh && c.hash == h) return c.mesh.get();
    std::vector<int32_t> edges;
    edges.reserve(mesh.edges.size() * 2);
    for (const auto& e : mesh.edges) edges.push_back(e[0]), edges.push_back(e[1]);
    std::vector<int32_t> tris;
    tris.reserve(mesh.triangles.size() * 3);
    for (const auto& t : mesh.triangles) tris.push_back(t[0]), tris.push_back(t[1]), tris.push_back(t[2]);
    tw_mesh* m = nullptr;
    // the finalized edge list goes in as explicit edges: finalize() is idempotent on it
    const int rc = tw_mesh_create(ctx, mesh.num_vertices(), mesh.inv_mass.data(), (int32_t)mesh.edges.size(),
                                  edges.data(), 0, nullptr, (int32_t)mesh.triangles.size(), tris.data(), &m);
    if (rc != TW_OK) throw_status(rc, ctx);
    c.mesh.reset(m);
    c.hash = h;
    return m;
}

}  // namespace

ResolveResult resolve(PositionsView x_start, PositionsView y_target, const MeshState& mesh, const ResolveConfig& cfg) {
    cfg.validate();
    const size_t n = mesh.positions.size();
    if (x_start.size() != n || y_target.size() != n)
        throw std::invalid_argument("resolve: position arrays do not match mesh");
    if (!all_finite(x_start) || !all_finite(y_target)) throw std::invalid_argument("resolve: non-finite input positions");
    const auto t0 = std::chrono::steady_clock::now();
    tw_ctx* ctx = context(cfg.device);
    tw_mesh* m = device_mesh(ctx, cfg.device, mesh);
    tw_resolve_config c;
    tw_default_config(&c);
    c.step_limit = cfg.step_limit;
    c.solver = static_cast<int32_t>(cfg.solver);
    c.eps = cfg.eps;
    c.d_min = cfg.d_min;
    c.d_max = cfg.d_max;
    c.delta = cfg.delta;
    c.sigma = cfg.sigma;
    c.gamma = cfg.gamma;
    c.sweeps = cfg.sweeps;
    c.family = static_cast<int32_t>(cfg.family);
    c.under_relax = cfg.under_relax;
    c.edge_constraints = cfg.edge_constraints;
    c.force_fresh_search = cfg.force_fresh_search;
    c.record_path = cfg.record_path;
    c.coloring_mode = static_cast<int32_t>(cfg.coloring);
    c.color_seed = cfg.color_seed;
    ResolveResult out;
    out.x.resize(n);
    std::vector<double> smd(cfg.step_limit);
    std::vector<double> path;
    if (cfg.record_path) path.resize(((size_t)cfg.step_limit + 1) * n * 3);
    tw_resolve_stats st;
    static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 layout");
    const int rc = tw_resolve(ctx, m, reinterpret_cast<const double*>(x_start.data()),
                              reinterpret_cast<const double*>(y_target.data()), &c,
                              reinterpret_cast<double*>(out.x.data()), &st, smd.data(),
                              cfg.record_path ? path.data() : nullptr, nullptr);
    if (rc != TW_OK) throw_status(rc, ctx);
    ResolveStats& s = out.stats;
    s.steps = st.steps;
    s.searches = st.searches;
    s.final_residual = st.final_residual;
    s.step_max_disp.assign(smd.begin(), smd.begin() + st.steps);
    s.converged = st.converged;
    s.hit_step_limit = st.hit_step_limit;
    s.stagnated = st.stagnated;
    s.start_in_contact = st.start_in_contact;
    s.step_law_violated = st.step_law_violated;
    s.device_ms = st.device_ms;
    s.pairs_evaluated = st.pairs_evaluated;
    s.num_pairs = st.num_pairs;
    if (cfg.record_path) {
        s.path.resize(st.steps + 1);
        for (int k = 0; k <= st.steps; ++k) {
            s.path[k].resize(n);
            std::memcpy(s.path[k].data(), path.data() + (size_t)k * n * 3, n * 24);
        }
    }
    s.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

ResolveResult repair(PositionsView x_free, PositionsView y_penetrating, const MeshState& mesh, const ResolveConfig& cfg) {
    return resolve(x_free, y_penetrating, mesh, cfg);
}

}  // namespace twoway

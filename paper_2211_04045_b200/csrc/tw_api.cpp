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
#include "twoway/advance.hpp"
#include "twoway/constraints.hpp"
#include "twoway/distance.hpp"
#include "twoway/proximity.hpp"
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

// ------------------------------------------------------------ stage API
// The reference's stage functions (distance/proximity/constraints/advance
// headers) over the stage entries of the C-ABI, on device 0 of this thread's
// context. They serve callers and tests of the reference's stage API.
namespace {

constexpr int kStageDevice = 0;

tw_ctx* stage_ctx() { return context(kStageDevice); }

void check(int rc, tw_ctx* ctx) {
    if (rc != TW_OK) throw_status(rc, ctx);
}

std::vector<double> flat(PositionsView p) {
    std::vector<double> f(p.size() * 3);
    for (size_t i = 0; i < p.size(); ++i) f[3 * i] = p[i].x(), f[3 * i + 1] = p[i].y(), f[3 * i + 2] = p[i].z();
    return f;
}

// closest results of n pairs (kinds 2n, verts 6n) -> out 11n, has n
void closest_batch(PositionsView positions, const std::vector<int32_t>& kinds, const std::vector<int32_t>& verts,
                   std::vector<double>& out, std::vector<int32_t>& has) {
    tw_ctx* ctx = stage_ctx();
    const int64_t n = (int64_t)kinds.size() / 2;
    out.assign(std::max<int64_t>(1, n) * 11, 0.0);
    has.assign(std::max<int64_t>(1, n), 0);
    const std::vector<double> x = flat(positions);
    check(tw_stage_closest(ctx, (int32_t)positions.size(), x.data(), n, kinds.data(), verts.data(), out.data(),
                           has.data()),
          ctx);
}

ClosestResult unpack_closest(const double* o) {
    ClosestResult r;
    r.distance = o[0];
    for (int k = 0; k < 3; ++k) r.weights_a[k] = o[1 + k], r.weights_b[k] = o[4 + k];
    r.direction = Vec3(o[7], o[8], o[9]);
    r.degenerate = o[10] != 0.0;
    return r;
}

std::optional<ClosestResult> closest_of(const Simplex& sa, const Simplex& sb, PositionsView positions) {
    std::vector<int32_t> kinds = {(int32_t)sa.kind, (int32_t)sb.kind}, verts(6, -1);
    for (int k = 0; k < 3; ++k) verts[k] = sa.idx[k], verts[3 + k] = sb.idx[k];
    std::vector<double> out;
    std::vector<int32_t> has;
    closest_batch(positions, kinds, verts, out, has);
    if (has[0] < 0) throw std::invalid_argument("simplex_pair_closest: adjacent pair or unsupported kinds");
    if (has[0] == 0) return std::nullopt;
    return unpack_closest(out.data());
}

Simplex simplex_of(int kind, int index, const MeshState& mesh) {
    if (kind == 0) return Simplex::vertex(index);
    if (kind == 1) return Simplex::edge(mesh.edges[index][0], mesh.edges[index][1]);
    const auto& t = mesh.triangles[index];
    return Simplex::triangle(t[0], t[1], t[2]);
}

}  // namespace

ClosestResult vertex_vertex_closest(const Vec3& p, const Vec3& q) {
    const Vec3 pts[2] = {p, q};
    return *closest_of(Simplex::vertex(0), Simplex::vertex(1), PositionsView(pts, 2));
}

ClosestResult vertex_edge_closest(const Vec3& p, const Vec3& e0, const Vec3& e1) {
    const Vec3 pts[3] = {p, e0, e1};
    return *closest_of(Simplex::vertex(0), Simplex::edge(1, 2), PositionsView(pts, 3));
}

std::optional<ClosestResult> vertex_triangle_closest(const Vec3& p, const Vec3& a, const Vec3& b, const Vec3& c) {
    const Vec3 pts[4] = {p, a, b, c};
    return closest_of(Simplex::vertex(0), Simplex::triangle(1, 2, 3), PositionsView(pts, 4));
}

std::optional<ClosestResult> edge_edge_closest(const Vec3& p1, const Vec3& p2, const Vec3& q1, const Vec3& q2) {
    const Vec3 pts[4] = {p1, p2, q1, q2};
    return closest_of(Simplex::edge(0, 1), Simplex::edge(2, 3), PositionsView(pts, 4));
}

std::optional<ClosestResult> simplex_pair_closest(const Simplex& sa, const Simplex& sb, PositionsView positions) {
    return closest_of(sa, sb, positions);
}

Vec3 weighted_point(const Simplex& s, const std::array<double, 3>& w, PositionsView positions) {  // distance.cpp:28-32
    Vec3 p = Vec3::Zero();
    for (int i = 0; i < s.size(); ++i) p = p + w[i] * positions[s.idx[i]];
    return p;
}

void ProximitySet::rebuild_vertex_index(int num_vertices) {  // proximity.cpp:54-64
    vertex_pairs.assign(num_vertices, {});
    for (int i = 0; i < static_cast<int>(pairs.size()); ++i) {
        const ProximityPair& p = pairs[i];
        for (int k = 0; k < p.a.size(); ++k) vertex_pairs[p.a.idx[k]].push_back(i);
        for (int k = 0; k < p.b.size(); ++k) vertex_pairs[p.b.idx[k]].push_back(i);
    }
}

ProximitySet proximity_search(PositionsView positions, const MeshState& mesh, double d_max) {
    tw_ctx* ctx = stage_ctx();
    tw_mesh* m = device_mesh(ctx, kStageDevice, mesh);
    const std::vector<double> x = flat(positions);
    int64_t cap = std::max<int64_t>(1024, 64 * (int64_t)positions.size()), np = 0;
    std::vector<uint64_t> keys;
    std::vector<double> dist, wa, wb, dir;
    std::vector<uint8_t> flags;
    for (;;) {
        keys.resize(cap), dist.resize(cap), wa.resize(3 * cap), wb.resize(3 * cap), dir.resize(3 * cap);
        flags.resize(cap);
        const int rc = tw_stage_search(ctx, m, x.data(), d_max, cap, keys.data(), dist.data(), wa.data(), wb.data(),
                                       dir.data(), flags.data(), &np);
        if (rc == TW_ECAPACITY && np > cap) {
            cap = np;
            continue;
        }
        check(rc, ctx);
        break;
    }
    ProximitySet set;
    set.bound = d_max;
    set.pairs.resize(np);
    for (int64_t i = 0; i < np; ++i) {
        ProximityPair& p = set.pairs[i];
        const uint64_t k = keys[i];
        const int ka = (int)(k >> 62), kb = (int)((k >> 60) & 3);
        p.index_a = (int)((k >> 30) & 0x3fffffff), p.index_b = (int)(k & 0x3fffffff);
        p.a = simplex_of(ka, p.index_a, mesh), p.b = simplex_of(kb, p.index_b, mesh);
        p.closest.distance = dist[i];
        for (int c = 0; c < 3; ++c) p.closest.weights_a[c] = wa[3 * i + c], p.closest.weights_b[c] = wb[3 * i + c];
        p.closest.direction = Vec3(dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]);
        p.closest.degenerate = (flags[i] & 4) != 0;
        p.active = (flags[i] & 1) != 0;
        p.all_static = (flags[i] & 2) != 0;
    }
    set.rebuild_vertex_index((int)positions.size());
    return set;
}

double shrink_bound(ProximitySet& set, double max_disp) {  // proximity.cpp:185-188
    set.bound -= 2.0 * max_disp;
    return set.bound;
}

void refresh_distances(ProximitySet& set, PositionsView positions) {  // proximity.cpp:190-202
    const size_t n = set.pairs.size();
    std::vector<int32_t> kinds(2 * n), verts(6 * n);
    for (size_t i = 0; i < n; ++i) {
        const ProximityPair& p = set.pairs[i];
        kinds[2 * i] = (int32_t)p.a.kind, kinds[2 * i + 1] = (int32_t)p.b.kind;
        for (int k = 0; k < 3; ++k) verts[6 * i + k] = p.a.idx[k], verts[6 * i + 3 + k] = p.b.idx[k];
    }
    std::vector<double> out;
    std::vector<int32_t> has;
    if (n) closest_batch(positions, kinds, verts, out, has);
    for (size_t i = 0; i < n; ++i) {
        ProximityPair& p = set.pairs[i];
        if (has[i] != 1) {  // nullopt: inactive, the stale result stays
            p.active = false;
            continue;
        }
        const Vec3 prev = p.closest.direction;
        p.closest = unpack_closest(out.data() + 11 * i);
        if (p.closest.degenerate && !prev.isZero()) p.closest.direction = prev;
        p.active = p.closest.distance < set.bound;
    }
}

double per_vertex_bound(const ProximitySet& set, int vertex) {  // proximity.cpp:204-211
    double d = set.bound;
    if (vertex < 0 || vertex >= static_cast<int>(set.vertex_pairs.size())) return d;
    for (int i : set.vertex_pairs[vertex]) {
        const ProximityPair& p = set.pairs[i];
        if (p.active) d = std::min(d, p.closest.distance);
    }
    return d;
}

std::vector<Constraint> linearize_all(const ProximitySet& set, PositionsView positions, const MeshState& mesh,
                                      const std::vector<double>& edge_targets, const AssemblyOptions& opts) {
    tw_ctx* ctx = stage_ctx();
    tw_mesh* m = device_mesh(ctx, kStageDevice, mesh);
    const int64_t np = (int64_t)set.pairs.size();
    std::vector<uint64_t> keys(std::max<int64_t>(1, np));
    std::vector<double> dist(std::max<int64_t>(1, np)), wa(3 * std::max<int64_t>(1, np)), wb(wa.size()), dir(wa.size());
    std::vector<uint8_t> flags(std::max<int64_t>(1, np));
    for (int64_t i = 0; i < np; ++i) {
        const ProximityPair& p = set.pairs[i];
        keys[i] = p.key();
        dist[i] = p.closest.distance;
        for (int c = 0; c < 3; ++c) {
            wa[3 * i + c] = p.closest.weights_a[c], wb[3 * i + c] = p.closest.weights_b[c];
            dir[3 * i + c] = p.closest.direction[c];
        }
        flags[i] = (uint8_t)((p.active ? 1 : 0) | (p.all_static ? 2 : 0) | (p.closest.degenerate ? 4 : 0));
    }
    const std::vector<double> x = flat(positions);
    const int64_t cap = np + (int64_t)mesh.edges.size() + 16;
    std::vector<uint8_t> kind(cap);
    std::vector<int32_t> verts(4 * cap), eidx(cap);
    std::vector<double> value(cap), jac(12 * cap), diag(cap);
    std::vector<uint64_t> pkey(cap);
    int64_t nrows = 0;
    check(tw_stage_linearize(ctx, m, x.data(), np, keys.data(), dist.data(), wa.data(), wb.data(), dir.data(),
                             flags.data(), edge_targets.empty() ? nullptr : edge_targets.data(), opts.delta,
                             opts.sigma, opts.family == ConstraintFamily::Gap ? 1 : 0, opts.edge_constraints ? 1 : 0,
                             cap, kind.data(), verts.data(), value.data(), jac.data(), diag.data(), pkey.data(),
                             eidx.data(), &nrows),
          ctx);
    std::vector<Constraint> rows(nrows);
    for (int64_t i = 0; i < nrows; ++i) {
        Constraint& c = rows[i];
        c.kind = static_cast<ConstraintKind>(kind[i]);
        c.nverts = 0;
        for (int k = 0; k < 4; ++k) {
            c.verts[k] = verts[4 * i + k];
            if (c.verts[k] >= 0) ++c.nverts;
            c.jac[k] = Vec3(jac[12 * i + 3 * k], jac[12 * i + 3 * k + 1], jac[12 * i + 3 * k + 2]);
        }
        c.value = value[i];
        c.diag = diag[i];
        if (c.kind == ConstraintKind::EdgeLength) {
            c.edge_index = eidx[i];
            c.flavor = Constraint::Flavor::LengthRatio;
            c.sigma = opts.sigma;
        } else {
            c.pair_key = pkey[i];
            const auto it = std::lower_bound(set.pairs.begin(), set.pairs.end(), c.pair_key,
                                             [](const ProximityPair& p, uint64_t k) { return p.key() < k; });
            c.pair_index = (int)(it - set.pairs.begin());
        }
    }
    return rows;
}

int color_constraints(std::vector<Constraint>& constraints, std::span<const double> inv_mass, uint64_t seed) {
    // Generic rows (the reference colors every row alike: a shared dynamic
    // vertex conflicts) on a vertex-only device mesh, reference algorithm.
    tw_ctx* ctx = stage_ctx();
    tw_mesh* m = nullptr;
    check(tw_mesh_create(ctx, (int32_t)inv_mass.size(), inv_mass.data(), 0, nullptr, 0, nullptr, 0, nullptr, &m), ctx);
    std::unique_ptr<tw_mesh, MeshDeleter> guard(m);
    const int64_t n = (int64_t)constraints.size();
    std::vector<uint8_t> kind(std::max<int64_t>(1, n), 0);  // all rows as contact rows
    std::vector<int32_t> verts(4 * std::max<int64_t>(1, n)), eidx(std::max<int64_t>(1, n), -1), color(kind.size());
    std::vector<uint64_t> keys(kind.size(), 0);
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 4; ++k) verts[4 * i + k] = k < constraints[i].nverts ? constraints[i].verts[k] : -1;
    int32_t ncolors = 0;
    check(tw_stage_color(ctx, m, n, kind.data(), verts.data(), keys.data(), eidx.data(), seed, TW_COLOR_REFERENCE, 0,
                         color.data(), &ncolors),
          ctx);
    for (int64_t i = 0; i < n; ++i) constraints[i].color = color[i];
    return ncolors;
}

void advance(AdvanceState& state, PositionsView y_target, const ProximitySet& set, double gamma,
             std::span<const double> inv_mass) {
    tw_ctx* ctx = stage_ctx();
    const int nv = (int)state.x.size();
    std::vector<double> D(nv);
    for (int v = 0; v < nv; ++v) D[v] = per_vertex_bound(set, v);
    std::vector<double> x = flat(state.x);
    const std::vector<double> y = flat(y_target);
    double md = 0.0;
    check(tw_stage_advance(ctx, nv, inv_mass.data(), y.data(), D.data(), gamma, x.data(), state.r.data(), &md), ctx);
    for (int v = 0; v < nv; ++v) state.x[v] = Vec3(x[3 * v], x[3 * v + 1], x[3 * v + 2]);
    state.last_max_disp = md;
}

bool termination_reached(const AdvanceState& state, double eps) { return state.max_remainder() < eps; }

}  // namespace twoway

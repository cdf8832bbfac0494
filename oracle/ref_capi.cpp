// ORACLE TEST INFRASTRUCTURE — C-ABI over the REAL reference, compiled from
// /root/reference/proj/src (in place, never copied) against the Eigen-subset
// shim in oracle/ref_shim/ by oracle/Makefile.ref into oracle/_ref/libtwoway_ref.so.
//
// Only tests/ and bench.py's reference / cpu_baseline legs load it, to pin the
// clean-room restatement (oracle/*.c) and to time the reference's own CPU
// resolve. Nothing in paper_2211_04045_b200/ links or loads it.
//
// Struct layouts (or_config, or_stats) are those of oracle/oracle.h.
#include <chrono>
#include <cstring>
#include <stdexcept>

#include "oracle.h"
#include "twoway/dynamics.hpp"
#include "twoway/normal_flow.hpp"
#include "twoway/resolve.hpp"
#include "twoway/testkit/ccd.hpp"
#include "twoway/testkit/fixtures.hpp"

using namespace twoway;

namespace {

thread_local char g_err[512];

int fail(const std::exception& e) {
    std::snprintf(g_err, sizeof(g_err), "%s", e.what());
    return dynamic_cast<const std::invalid_argument*>(&e) ? -1 : -2;
}

Positions to_pos(int nv, const double* x) {
    Positions p(static_cast<size_t>(nv));
    for (int i = 0; i < nv; ++i) p[i] = Vec3(x[3 * i], x[3 * i + 1], x[3 * i + 2]);
    return p;
}

void from_pos(const Positions& p, double* out) {
    for (size_t i = 0; i < p.size(); ++i)
        for (int k = 0; k < 3; ++k) out[3 * i + k] = p[i][k];
}

ResolveConfig to_cfg(const or_config* c) {
    ResolveConfig r;
    r.step_limit = c->step_limit;
    r.solver = static_cast<SolverKind>(c->solver);
    r.eps = c->eps;
    r.d_min = c->d_min;
    r.d_max = c->d_max;
    r.delta = c->delta;
    r.sigma = c->sigma;
    r.gamma = c->gamma;
    r.sweeps = c->sweeps;
    r.family = static_cast<ConstraintFamily>(c->family);
    r.under_relax = c->under_relax;
    r.edge_constraints = c->edge_constraints != 0;
    r.force_fresh_search = c->force_fresh_search != 0;
    r.record_path = c->record_path != 0;
    r.color_seed = c->color_seed;
    return r;
}

struct EnergyParams {  // EnergyModel scalars (dynamics.hpp:12-24)
    double spring_stiffness, bending_stiffness, gravity[3], repulsion_stiffness,
        repulsion_radius, dt;
    int32_t newton_iters;
    double mu, pcg_tol;
    int32_t pcg_max_iters;
};

EnergyModel to_model(const EnergyParams* p) {
    EnergyModel m;
    m.spring_stiffness = p->spring_stiffness;
    m.bending_stiffness = p->bending_stiffness;
    m.gravity = Vec3(p->gravity[0], p->gravity[1], p->gravity[2]);
    m.repulsion_stiffness = p->repulsion_stiffness;
    m.repulsion_radius = p->repulsion_radius;
    m.dt = p->dt;
    m.newton_iters = p->newton_iters;
    m.mu = p->mu;
    m.pcg_tol = p->pcg_tol;
    m.pcg_max_iters = p->pcg_max_iters;
    return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err; }

// MeshState{positions, triangles, strand_edges, inv_mass (NULL -> default)}
// -> finalize() -> validate(), as bindings/module.cpp:32-48 does.
void* ref_mesh_create(int nv, const double* x, int nt, const int* tris, int ns,
                      const int* strands, const double* inv_mass, const double* vel) {
    try {
        auto* m = new MeshState();
        m->positions = to_pos(nv, x);
        for (int t = 0; t < nt; ++t) m->triangles.push_back({tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]});
        for (int e = 0; e < ns; ++e) m->strand_edges.push_back({strands[2 * e], strands[2 * e + 1]});
        if (inv_mass) m->inv_mass.assign(inv_mass, inv_mass + nv);
        m->finalize();
        if (vel) m->velocities = to_pos(nv, vel);
        m->validate();
        return m;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_mesh_destroy(void* m) { delete static_cast<MeshState*>(m); }

// Edge list in MeshState::edges order; returns the count (writes when cap allows).
int ref_mesh_edges(void* mp, int cap, int* out) {
    const auto* m = static_cast<MeshState*>(mp);
    const int ne = static_cast<int>(m->edges.size());
    if (ne <= cap)
        for (int e = 0; e < ne; ++e) out[2 * e] = m->edges[e][0], out[2 * e + 1] = m->edges[e][1];
    return ne;
}

int ref_mesh_positions(void* mp, double* x, double* v, double* inv_mass) {
    const auto* m = static_cast<MeshState*>(mp);
    if (x) from_pos(m->positions, x);
    if (v) from_pos(m->velocities, v);
    if (inv_mass) std::memcpy(inv_mass, m->inv_mass.data(), m->inv_mass.size() * sizeof(double));
    return m->num_vertices();
}

// twoway::resolve (resolve.cpp:36-144). step_max_disp (cap step_limit) and
// path ((steps + 1) * nv * 3, only with record_path) may be NULL.
int ref_resolve(void* mp, const double* x, const double* y, const or_config* cfg, double* x_out,
                or_stats* st, double* step_max_disp, int64_t path_cap, double* path) {
    const auto* m = static_cast<MeshState*>(mp);
    try {
        const int nv = m->num_vertices();
        const Positions xs = to_pos(nv, x), ys = to_pos(nv, y);
        const ResolveResult r = resolve(xs, ys, *m, to_cfg(cfg));
        from_pos(r.x, x_out);
        if (st) {
            st->steps = r.stats.steps;
            st->searches = r.stats.searches;
            st->final_residual = r.stats.final_residual;
            st->wall_ms = r.stats.wall_ms;
            st->converged = r.stats.converged;
            st->hit_step_limit = r.stats.hit_step_limit;
            st->stagnated = r.stats.stagnated;
            st->start_in_contact = r.stats.start_in_contact;
            st->step_law_violated = r.stats.step_law_violated;
            st->status = 0;
        }
        if (step_max_disp)
            for (size_t i = 0; i < r.stats.step_max_disp.size(); ++i) step_max_disp[i] = r.stats.step_max_disp[i];
        if (path) {
            int64_t off = 0;
            for (const Positions& p : r.stats.path) {
                if (off + 3 * nv > path_cap) break;
                from_pos(p, path + off);
                off += 3 * nv;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        if (st) st->status = -1;
        return fail(e);
    }
}

// proximity_search (proximity.cpp:76-183): sorted keys and distances.
// Returns P, or -P when P > cap (nothing written).
int64_t ref_search(void* mp, const double* x, double d_max, int64_t cap, uint64_t* keys,
                   double* dist, uint8_t* flags) {
    const auto* m = static_cast<MeshState*>(mp);
    try {
        const ProximitySet s = proximity_search(to_pos(m->num_vertices(), x), *m, d_max);
        const int64_t P = static_cast<int64_t>(s.pairs.size());
        if (P > cap) return -P;
        for (int64_t i = 0; i < P; ++i) {
            keys[i] = s.pairs[i].key();
            if (dist) dist[i] = s.pairs[i].closest.distance;
            if (flags) flags[i] = (s.pairs[i].active ? 1 : 0) | (s.pairs[i].all_static ? 2 : 0);
        }
        return P;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// proximity_search at x, then linearize_all (constraints.cpp:181-220) with
// edge targets |y_i - y_j|, then color_constraints with `seed`. Per row: kind,
// pair key (contact) or edge index (edge rows), value, diag and color.
// Returns R, or -R when R > cap.
int64_t ref_linearize(void* mp, const double* x, const double* y, double d_max, double delta,
                      double sigma, int family, int edge_constraints, uint64_t seed, int64_t cap,
                      uint8_t* kind, uint64_t* key, int32_t* edge_index, double* value,
                      double* diag, int32_t* color, int32_t* ncolors) {
    const auto* m = static_cast<MeshState*>(mp);
    try {
        const int nv = m->num_vertices();
        const Positions xs = to_pos(nv, x), ys = to_pos(nv, y);
        const ProximitySet s = proximity_search(xs, *m, d_max);
        std::vector<double> targets(m->edges.size());
        for (size_t e = 0; e < m->edges.size(); ++e)
            targets[e] = (ys[m->edges[e][0]] - ys[m->edges[e][1]]).norm();
        AssemblyOptions o;
        o.delta = delta;
        o.sigma = sigma;
        o.family = static_cast<ConstraintFamily>(family);
        o.edge_constraints = edge_constraints != 0;
        std::vector<Constraint> rows = linearize_all(s, xs, *m, targets, o);
        const int nc = color_constraints(rows, m->inv_mass, seed);
        if (ncolors) *ncolors = nc;
        const int64_t R = static_cast<int64_t>(rows.size());
        if (R > cap) return -R;
        for (int64_t i = 0; i < R; ++i) {
            kind[i] = static_cast<uint8_t>(rows[i].kind);
            key[i] = rows[i].pair_key;
            edge_index[i] = rows[i].edge_index;
            value[i] = rows[i].value;
            diag[i] = rows[i].diag;
            color[i] = rows[i].color;
        }
        return R;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- dynamics (dynamics.cpp) ----

// One simulation step (dynamics.cpp:326-349) on a mesh whose positions and
// velocities are the state at t; the rest data is taken from rest_x via
// EnergyModel::prepare. Writes x^{t+1}, v^{t+1}; returns total resolve steps.
int ref_step(void* mp, const double* rest_x, const EnergyParams* ep, const or_config* cfg,
             double* x_out, double* v_out, int32_t* searches) {
    auto* m = static_cast<MeshState*>(mp);
    try {
        EnergyModel model = to_model(ep);
        MeshState rest = *m;
        rest.positions = to_pos(m->num_vertices(), rest_x);
        model.prepare(rest);
        const StepStats st = step(model, *m, to_cfg(cfg));
        from_pos(m->positions, x_out);
        from_pos(m->velocities, v_out);
        if (searches) *searches = st.total_searches();
        return st.total_resolve_steps();
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The target half of step(): search at x, gradient_and_hessian, add_repulsion,
// newton_target (PCG), optional friction_filter (dynamics.cpp:334-339).
// Also returns the gradient (3 nv) when grad != NULL.
int ref_newton_target(void* mp, const double* rest_x, const EnergyParams* ep, double d_max,
                      const double* x, double* y_out, double* grad, int32_t* pcg_iters,
                      int32_t* pcg_converged) {
    auto* m = static_cast<MeshState*>(mp);
    try {
        EnergyModel model = to_model(ep);
        MeshState rest = *m;
        rest.positions = to_pos(m->num_vertices(), rest_x);
        model.prepare(rest);
        const Positions xs = to_pos(m->num_vertices(), x);
        const ProximitySet set = proximity_search(xs, *m, d_max);
        GradientHessian gh = gradient_and_hessian(model, *m, xs);
        add_repulsion(model, set, xs, gh);
        if (grad)
            for (int i = 0; i < 3 * m->num_vertices(); ++i) grad[i] = gh.gradient(i);
        NewtonResult nt = newton_target(model, *m, xs, gh);
        Positions y = std::move(nt.y);
        if (model.mu > 0.0) y = friction_filter(model, *m, xs, y, set);
        from_pos(y, y_out);
        if (pcg_iters) *pcg_iters = nt.pcg_iterations;
        if (pcg_converged) *pcg_converged = nt.pcg_converged;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// friction_filter(model, mesh, x, y_target, proximity_search(x, d_max))
// (dynamics.cpp:272-324), the reference's own function.
int ref_friction_filter(void* mp, const double* rest_x, const EnergyParams* ep, double d_max,
                        const double* x, const double* y_target, double* y_out) {
    auto* m = static_cast<MeshState*>(mp);
    try {
        EnergyModel model = to_model(ep);
        MeshState rest = *m;
        rest.positions = to_pos(m->num_vertices(), rest_x);
        model.prepare(rest);
        const Positions xs = to_pos(m->num_vertices(), x);
        const ProximitySet set = proximity_search(xs, *m, d_max);
        const Positions y = friction_filter(model, *m, xs, to_pos(m->num_vertices(), y_target), set);
        from_pos(y, y_out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

double ref_incremental_energy(void* mp, const double* rest_x, const EnergyParams* ep,
                              const double* x) {
    auto* m = static_cast<MeshState*>(mp);
    EnergyModel model = to_model(ep);
    MeshState rest = *m;
    rest.positions = to_pos(m->num_vertices(), rest_x);
    model.prepare(rest);
    return incremental_energy(model, *m, to_pos(m->num_vertices(), x));
}

// Timed pieces of one simulation frame of the reference (seconds), for the
// bench's reference arm: the Newton target (step()'s search, gradient /
// Hessian, repulsion, PCG; dynamics.cpp:334-337), one proximity_search at the
// start state (the cost of every re-search of resolve) and one non-search
// Alg.-1 iteration at the start state towards the target (linearize_all,
// warm-start-free color_constraints, assemble_lcp, pgs_sweeps, recover_target,
// advance, refresh_distances, shrink_bound: resolve.cpp:84-137), all the
// reference's own functions. out[0..2] = t_target, t_search, t_iteration;
// out[3] = contact rows of that iteration; out[4] = colors.
int ref_frame_sample(void* mp, const double* rest_x, const EnergyParams* ep, const or_config* cfg, double* out) {
    auto* m = static_cast<MeshState*>(mp);
    try {
        using clk = std::chrono::steady_clock;
        auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
        EnergyModel model = to_model(ep);
        MeshState rest = *m;
        rest.positions = to_pos(m->num_vertices(), rest_x);
        model.prepare(rest);
        const ResolveConfig rc = to_cfg(cfg);
        const Positions x = m->positions;
        const auto t0 = clk::now();
        ProximitySet set0 = proximity_search(x, *m, rc.d_max);
        GradientHessian gh = gradient_and_hessian(model, *m, x);
        add_repulsion(model, set0, x, gh);
        NewtonResult nt = newton_target(model, *m, x, gh);
        const auto t1 = clk::now();
        ProximitySet set = proximity_search(x, *m, rc.d_max);
        const auto t2 = clk::now();
        Positions yk1 = nt.y;
        for (int v = 0; v < m->num_vertices(); ++v)
            if (m->inv_mass[v] == 0.0) yk1[v] = x[v];
        std::vector<double> targets(m->edges.size());
        for (size_t e = 0; e < m->edges.size(); ++e) targets[e] = (yk1[m->edges[e][0]] - yk1[m->edges[e][1]]).norm();
        AssemblyOptions opts;
        opts.delta = rc.delta;
        opts.sigma = rc.sigma;
        opts.family = rc.family;
        opts.edge_constraints = rc.edge_constraints;
        AdvanceState st;
        st.reset(x);
        const auto t3 = clk::now();
        std::vector<Constraint> rows = linearize_all(set, st.x, *m, targets, opts);
        const int nc = color_constraints(rows, m->inv_mass, rc.color_seed);
        LcpSystem sys = assemble_lcp(rows, st.x, yk1, m->inv_mass, nc);
        pgs_sweeps(sys, rc.sweeps);
        const Positions y = recover_target(sys, yk1);
        advance(st, y, set, rc.gamma, m->inv_mass);
        const double bound_before = set.bound;
        refresh_distances(set, st.x);
        shrink_bound(set, st.last_max_disp);
        const auto t4 = clk::now();
        (void)bound_before;
        int contacts = 0;
        for (const Constraint& c : rows) contacts += c.kind != ConstraintKind::EdgeLength;
        out[0] = secs(t0, t1);
        out[1] = secs(t1, t2);
        out[2] = secs(t3, t4);
        out[3] = contacts;
        out[4] = nc;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- normal flow (normal_flow.cpp) ----
int ref_normal_flow_target(void* mp, const double* x, double beta, double alpha_smooth,
                           double* y_out) {
    const auto* m = static_cast<MeshState*>(mp);
    try {
        NormalFlowConfig c;
        c.beta = beta;
        c.alpha_smooth = alpha_smooth;
        from_pos(normal_flow_target(*m, to_pos(m->num_vertices(), x), c), y_out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- testkit ----
// ccd_certify on one segment x0 -> x1 (testkit/ccd.cpp:339-498).
int ref_ccd_certify(void* mp, const double* x0, const double* x1, int32_t* certain) {
    const auto* m = static_cast<MeshState*>(mp);
    try {
        const Positions a = to_pos(m->num_vertices(), x0), b = to_pos(m->num_vertices(), x1);
        testkit::PathSegment seg{a, b, m};
        const testkit::CcdReport r = testkit::ccd_certify(seg);
        if (certain) *certain = r.certain_count();
        return static_cast<int>(r.violations.size());
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The reference's fixture battery (testkit/fixtures.cpp:304-314): fixture i of
// scene_fixtures(seed). Returns a mesh handle (positions = x) and writes y
// (cap 3*nv doubles); *nv_out, flags (benign | penetrating << 1).
void* ref_fixture(uint64_t seed, int index, int cap, double* y, int32_t* nv_out, int32_t* flags,
                  char* name, int name_cap) {
    try {
        std::vector<testkit::Fixture> fs = testkit::scene_fixtures(seed);
        if (index < 0 || index >= static_cast<int>(fs.size())) {
            *nv_out = static_cast<int>(fs.size());
            return nullptr;
        }
        testkit::Fixture& f = fs[index];
        auto* m = new MeshState(f.mesh);
        m->positions = f.x;
        *nv_out = m->num_vertices();
        *flags = (f.benign ? 1 : 0) | (f.penetrating ? 2 : 0);
        std::snprintf(name, static_cast<size_t>(name_cap), "%s", f.name.c_str());
        if (3 * m->num_vertices() <= cap) from_pos(f.y, y);
        return m;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

int ref_mesh_topology(void* mp, int32_t* nt, int32_t* tris, int32_t* ns, int32_t* strands) {
    const auto* m = static_cast<MeshState*>(mp);
    if (tris)
        for (size_t t = 0; t < m->triangles.size(); ++t)
            for (int k = 0; k < 3; ++k) tris[3 * t + k] = m->triangles[t][k];
    if (strands)
        for (size_t e = 0; e < m->strand_edges.size(); ++e)
            for (int k = 0; k < 2; ++k) strands[2 * e + k] = m->strand_edges[e][k];
    *nt = static_cast<int32_t>(m->triangles.size());
    *ns = static_cast<int32_t>(m->strand_edges.size());
    return m->num_vertices();
}

}  // extern "C"

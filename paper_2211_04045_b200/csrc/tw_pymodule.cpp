// Python module _twoway mirroring proj/bindings/module.cpp:101-186 (resolve,
// repair, normal_flow_target, certify_segment, vertex_triangle_closest,
// edge_edge_closest) on the B200 path. Inputs
// are numpy (N, 3) float64 / (T, 3) int arrays as in the reference; unknown
// keyword arguments raise ValueError (std::invalid_argument) as there.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>
#include <stdexcept>

#include "tw_c.h"
#include "twoway/resolve.hpp"

namespace py = pybind11;
using namespace twoway;

namespace {

using ArrD = py::array_t<double, py::array::c_style | py::array::forcecast>;
using ArrI = py::array_t<int32_t, py::array::c_style | py::array::forcecast>;

Positions to_positions(const ArrD& a) {
    if (a.ndim() != 2 || a.shape(1) != 3) throw std::invalid_argument("positions must be (N, 3)");
    Positions out(a.shape(0));
    std::memcpy(out.data(), a.data(), out.size() * sizeof(Vec3));
    return out;
}

py::array_t<double> from_positions(PositionsView x) {
    py::array_t<double> out({(py::ssize_t)x.size(), (py::ssize_t)3});
    std::memcpy(out.mutable_data(), x.data(), x.size() * sizeof(Vec3));
    return out;
}

// make_mesh, module.cpp:32-48
MeshState make_mesh(const ArrD& x, const ArrI& triangles, const ArrI& strand_edges, const ArrD& inv_mass) {
    MeshState mesh;
    mesh.positions = to_positions(x);
    if (triangles.size() && (triangles.ndim() != 2 || triangles.shape(1) != 3))
        throw std::invalid_argument("triangles must be (T, 3)");
    if (strand_edges.size() && (strand_edges.ndim() != 2 || strand_edges.shape(1) != 2))
        throw std::invalid_argument("strand_edges must be (S, 2)");
    const int32_t* t = triangles.data();
    for (py::ssize_t i = 0; i < (triangles.size() ? triangles.shape(0) : 0); ++i)
        mesh.triangles.push_back({t[3 * i], t[3 * i + 1], t[3 * i + 2]});
    const int32_t* s = strand_edges.data();
    for (py::ssize_t i = 0; i < (strand_edges.size() ? strand_edges.shape(0) : 0); ++i)
        mesh.strand_edges.push_back({s[2 * i], s[2 * i + 1]});
    if (inv_mass.size() > 0) {
        if (inv_mass.size() != (py::ssize_t)mesh.positions.size())
            throw std::invalid_argument("inv_mass size must match positions");
        mesh.inv_mass.assign(inv_mass.data(), inv_mass.data() + inv_mass.size());
    }
    mesh.finalize();
    mesh.validate();
    return mesh;
}

// config_from_kwargs, module.cpp:50-82 (+ coloring, device)
ResolveConfig config_from_kwargs(const py::kwargs& kw) {
    ResolveConfig cfg;
    for (const auto& item : kw) {
        const std::string key = py::cast<std::string>(item.first);
        if (key == "step_limit") cfg.step_limit = py::cast<int>(item.second);
        else if (key == "eps") cfg.eps = py::cast<double>(item.second);
        else if (key == "d_min") cfg.d_min = py::cast<double>(item.second);
        else if (key == "d_max") cfg.d_max = py::cast<double>(item.second);
        else if (key == "delta") cfg.delta = py::cast<double>(item.second);
        else if (key == "sigma") cfg.sigma = py::cast<double>(item.second);
        else if (key == "gamma") cfg.gamma = py::cast<double>(item.second);
        else if (key == "sweeps") cfg.sweeps = py::cast<int>(item.second);
        else if (key == "edge_constraints") cfg.edge_constraints = py::cast<bool>(item.second);
        else if (key == "record_path") cfg.record_path = py::cast<bool>(item.second);
        else if (key == "color_seed") cfg.color_seed = py::cast<uint64_t>(item.second);
        else if (key == "force_fresh_search") cfg.force_fresh_search = py::cast<bool>(item.second);
        else if (key == "device") cfg.device = py::cast<int>(item.second);
        else if (key == "solver") {
            const std::string s = py::cast<std::string>(item.second);
            if (s == "pgs") cfg.solver = SolverKind::Pgs;
            else if (s == "jacobi") cfg.solver = SolverKind::Jacobi;
            else if (s == "al20") cfg.solver = SolverKind::Al20;
            else if (s == "al100") cfg.solver = SolverKind::Al100;
            else throw std::invalid_argument("unknown solver '" + s + "'");
        } else if (key == "constraint_family") {
            const std::string s = py::cast<std::string>(item.second);
            if (s == "volume") cfg.family = ConstraintFamily::Volume;
            else if (s == "gap") cfg.family = ConstraintFamily::Gap;
            else throw std::invalid_argument("unknown constraint_family '" + s + "'");
        } else if (key == "coloring") {
            const std::string s = py::cast<std::string>(item.second);
            if (s == "reference") cfg.coloring = ColoringMode::Reference;
            else if (s == "device") cfg.coloring = ColoringMode::Device;
            else throw std::invalid_argument("unknown coloring '" + s + "'");
        } else {
            throw std::invalid_argument("unknown config key '" + key + "'");
        }
    }
    return cfg;
}

py::dict stats_to_dict(const ResolveStats& st) {  // module.cpp:84-97 (+ device diagnostics)
    py::dict d;
    d["steps"] = st.steps;
    d["searches"] = st.searches;
    d["final_residual"] = st.final_residual;
    d["converged"] = st.converged;
    d["hit_step_limit"] = st.hit_step_limit;
    d["stagnated"] = st.stagnated;
    d["wall_ms"] = st.wall_ms;
    py::list path;
    for (const auto& p : st.path) path.append(from_positions(p));
    d["path"] = path;
    d["start_in_contact"] = st.start_in_contact;
    d["step_law_violated"] = st.step_law_violated;
    d["step_max_disp"] = st.step_max_disp;
    d["device_ms"] = st.device_ms;
    d["pairs_evaluated"] = st.pairs_evaluated;
    d["num_pairs"] = st.num_pairs;
    return d;
}

py::tuple run(bool rep, const ArrD& x, const ArrD& y, const ArrI& triangles, const ArrI& strand_edges,
              const ArrD& inv_mass, const py::kwargs& kw) {
    MeshState mesh = make_mesh(x, triangles, strand_edges, inv_mass);
    const ResolveConfig cfg = config_from_kwargs(kw);
    const Positions xs = to_positions(x), ys = to_positions(y);
    ResolveResult res;
    {
        py::gil_scoped_release nogil;
        res = rep ? repair(xs, ys, mesh, cfg) : resolve(xs, ys, mesh, cfg);
    }
    return py::make_tuple(from_positions(res.x), stats_to_dict(res.stats));
}

py::dict closest_call(int ka, std::vector<int32_t> va, int kb, std::vector<int32_t> vb, const ArrD& pts) {
    tw_ctx* ctx = nullptr;
    if (tw_ctx_create(0, nullptr, &ctx) != TW_OK) throw std::runtime_error("twoway: no CUDA device");
    int32_t kinds[2] = {ka, kb};
    int32_t verts[6] = {-1, -1, -1, -1, -1, -1};
    for (size_t i = 0; i < va.size(); ++i) verts[i] = va[i];
    for (size_t i = 0; i < vb.size(); ++i) verts[3 + i] = vb[i];
    double out[11];
    int32_t has = 0;
    const int rc = tw_stage_closest(ctx, (int32_t)pts.shape(0), pts.data(), 1, kinds, verts, out, &has);
    tw_ctx_destroy(ctx);
    if (rc != TW_OK) throw std::runtime_error("twoway: closest query failed");
    if (has != 1) throw std::invalid_argument(ka == 0 ? "degenerate triangle" : "degenerate segment");
    py::dict d;
    d["distance"] = out[0];
    if (ka == 0) d["weights"] = py::make_tuple(out[4], out[5], out[6]);
    else d["s"] = out[2], d["t"] = out[5];
    return d;
}

struct OwnedCtx {  // a context for the calls that do not go through twoway::resolve
    tw_ctx* c = nullptr;
    OwnedCtx() {
        if (tw_ctx_create(0, nullptr, &c) != TW_OK) throw std::runtime_error("twoway: no CUDA device");
    }
    ~OwnedCtx() { tw_ctx_destroy(c); }
    void check(int rc) const {
        if (rc == TW_EINVAL || rc == TW_EUNSUPPORTED) throw std::invalid_argument(tw_last_error(c));
        if (rc != TW_OK) throw std::runtime_error(tw_last_error(c));
    }
};

// normal_flow_target binding, module.cpp:134-146
py::array_t<double> normal_flow(const ArrD& x, const ArrI& triangles, double beta, double alpha) {
    MeshState mesh = make_mesh(x, triangles, ArrI(std::vector<py::ssize_t>{0, 2}), ArrD(std::vector<py::ssize_t>{0}));
    std::vector<int32_t> t;
    for (const auto& tr : mesh.triangles) t.insert(t.end(), {tr[0], tr[1], tr[2]});
    py::array_t<double> out({(py::ssize_t)mesh.num_vertices(), (py::ssize_t)3});
    OwnedCtx ctx;
    {
        py::gil_scoped_release nogil;
        ctx.check(tw_normal_flow_target(ctx.c, mesh.num_vertices(), x.data(), (int32_t)mesh.triangles.size(), t.data(),
                                        beta, alpha, out.mutable_data()));
    }
    return out;
}

// certify_segment binding, module.cpp:148-162: the CCD check of the linear
// motion x0 -> x1 runs on the device certifier (tw_ccd_certify)
py::dict certify(const ArrD& x0, const ArrD& x1, const ArrI& triangles, const ArrI& strand_edges) {
    MeshState mesh = make_mesh(x0, triangles, strand_edges, ArrD(std::vector<py::ssize_t>{0}));
    if (x1.ndim() != 2 || x1.shape(0) != x0.shape(0) || x1.shape(1) != 3)
        throw std::invalid_argument("x1 must match x0");
    std::vector<int32_t> e, t;
    for (const auto& ed : mesh.edges) e.insert(e.end(), {ed[0], ed[1]});
    for (const auto& tr : mesh.triangles) t.insert(t.end(), {tr[0], tr[1], tr[2]});
    OwnedCtx ctx;
    int32_t viol = 0, certain = 0;
    {
        py::gil_scoped_release nogil;
        tw_mesh* m = nullptr;
        ctx.check(tw_mesh_create(ctx.c, mesh.num_vertices(), mesh.inv_mass.data(), (int32_t)mesh.edges.size(),
                                 e.data(), 0, nullptr, (int32_t)mesh.triangles.size(), t.data(), &m));
        const int rc = tw_ccd_certify(ctx.c, m, x0.data(), x1.data(), &viol, &certain, nullptr);
        tw_mesh_destroy(m);
        ctx.check(rc);
    }
    py::dict d;
    d["certain"] = certain;
    d["uncertain"] = viol - certain;
    return d;
}

}  // namespace

PYBIND11_MODULE(_twoway, m) {
    m.doc() = "two-way continuous collision handling on B200: resolve/repair a penetrating target onto an "
              "intersection-free state along a certified path";
    const ArrI no_strands(std::vector<py::ssize_t>{0, 2});
    const ArrD no_mass(std::vector<py::ssize_t>{0});
    m.def(
        "resolve",
        [](const ArrD& x, const ArrD& y, const ArrI& t, const ArrI& s, const ArrD& im, const py::kwargs& kw) {
            return run(false, x, y, t, s, im, kw);
        },
        py::arg("x"), py::arg("y"), py::arg("triangles"), py::arg("strand_edges") = no_strands,
        py::arg("inv_mass") = no_mass,
        "Project target y onto an intersection-free state reachable from x (device path).");
    m.def(
        "repair",
        [](const ArrD& x, const ArrD& y, const ArrI& t, const ArrI& s, const ArrD& im, const py::kwargs& kw) {
            return run(true, x, y, t, s, im, kw);
        },
        py::arg("x"), py::arg("y"), py::arg("triangles"), py::arg("strand_edges") = no_strands,
        py::arg("inv_mass") = no_mass, "Intersection-repair entry point (x must be intersection-free).");
    m.def("normal_flow_target", &normal_flow, py::arg("x"), py::arg("triangles"), py::arg("beta") = 5e-4,
          py::arg("alpha") = 0.5,
          "Offset along area-weighted normals plus three cotangent-Jacobi smoothing passes (device).");
    m.def("certify_segment", &certify, py::arg("x0"), py::arg("x1"), py::arg("triangles"),
          py::arg("strand_edges") = no_strands, "CCD check of the linear motion between two states (device certifier).");
    m.def(
        "vertex_triangle_closest",
        [](std::vector<double> p, std::vector<double> a, std::vector<double> b, std::vector<double> c) {
            std::vector<double> pts;
            for (auto* v : {&p, &a, &b, &c}) pts.insert(pts.end(), v->begin(), v->end());
            ArrD arr({(py::ssize_t)4, (py::ssize_t)3}, pts.data());
            return closest_call(0, {0}, 2, {1, 2, 3}, arr);
        },
        py::arg("p"), py::arg("a"), py::arg("b"), py::arg("c"));
    m.def(
        "edge_edge_closest",
        [](std::vector<double> p1, std::vector<double> p2, std::vector<double> q1, std::vector<double> q2) {
            std::vector<double> pts;
            for (auto* v : {&p1, &p2, &q1, &q2}) pts.insert(pts.end(), v->begin(), v->end());
            ArrD arr({(py::ssize_t)4, (py::ssize_t)3}, pts.data());
            return closest_call(1, {0, 1}, 1, {2, 3}, arr);
        },
        py::arg("p1"), py::arg("p2"), py::arg("q1"), py::arg("q2"));
    m.attr("abi_version") = tw_abi_version();
}

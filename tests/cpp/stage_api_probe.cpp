// Exercises the reference's C++ stage API (include/twoway/*.hpp) as a caller
// of the reference would, on a scene read from a binary file; writes every
// result for tests/test_gpu_cpp_api.py to compare with the oracle.
//
//   stage_api_probe in.bin out.bin
// in.bin: int32 nv, nt; double x[nv*3], y[nv*3], inv_mass[nv]; int32 tris[nt*3]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "twoway/advance.hpp"
#include "twoway/constraints.hpp"
#include "twoway/proximity.hpp"
#include "twoway/resolve.hpp"

using namespace twoway;

template <typename T>
static void rd(FILE* f, T* p, size_t n) {
    if (fread(p, sizeof(T), n, f) != n) {
        std::fprintf(stderr, "short read\n");
        std::exit(2);
    }
}
template <typename T>
static void wr(FILE* f, const T* p, size_t n) {
    fwrite(p, sizeof(T), n, f);
}
static void wr_i64(FILE* f, long long v) { wr(f, &v, 1); }

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    FILE* in = std::fopen(argv[1], "rb");
    int32_t nv, nt;
    rd(in, &nv, 1);
    rd(in, &nt, 1);
    std::vector<double> xs(3 * nv), ys(3 * nv), im(nv);
    std::vector<int32_t> tr(3 * nt);
    rd(in, xs.data(), xs.size());
    rd(in, ys.data(), ys.size());
    rd(in, im.data(), im.size());
    rd(in, tr.data(), tr.size());
    std::fclose(in);

    MeshState mesh;
    Positions x(nv), y(nv);
    for (int v = 0; v < nv; ++v) x[v] = Vec3(xs[3 * v], xs[3 * v + 1], xs[3 * v + 2]);
    for (int v = 0; v < nv; ++v) y[v] = Vec3(ys[3 * v], ys[3 * v + 1], ys[3 * v + 2]);
    mesh.positions = x;
    mesh.inv_mass = im;
    for (int t = 0; t < nt; ++t) mesh.triangles.push_back({tr[3 * t], tr[3 * t + 1], tr[3 * t + 2]});
    mesh.finalize();

    FILE* out = std::fopen(argv[2], "wb");
    // proximity_search at y, then refresh at x
    ProximitySet sy = proximity_search(y, mesh, 4e-3);
    wr_i64(out, (long long)sy.pairs.size());
    for (const auto& p : sy.pairs) {
        const uint64_t k = p.key();
        wr(out, &k, 1);
        wr(out, &p.closest.distance, 1);
    }
    ProximitySet sr = sy;
    refresh_distances(sr, x);
    for (const auto& p : sr.pairs) {
        wr(out, &p.closest.distance, 1);
        const int32_t a = p.active ? 1 : 0;
        wr(out, &a, 1);
    }
    // linearize_all at y with targets = edge lengths at x, then the reference coloring
    std::vector<double> targets(mesh.edges.size());
    for (size_t e = 0; e < mesh.edges.size(); ++e) targets[e] = (x[mesh.edges[e][0]] - x[mesh.edges[e][1]]).norm();
    AssemblyOptions opts;
    opts.delta = 1e-3;
    std::vector<Constraint> rows = linearize_all(sy, y, mesh, targets, opts);
    const int ncol = color_constraints(rows, im, 0x5eed);
    wr_i64(out, (long long)rows.size());
    wr_i64(out, ncol);
    for (const auto& c : rows) {
        const int32_t head[4] = {(int32_t)c.kind, c.nverts, c.edge_index, c.color};
        wr(out, head, 4);
        wr(out, c.verts.data(), 4);
        wr(out, &c.value, 1);
        wr(out, &c.diag, 1);
        wr(out, &c.pair_key, 1);
        for (int k = 0; k < 4; ++k) wr(out, c.jac[k].data(), 3);
    }
    // one forward step from x towards y with the pair set at x
    ProximitySet sx = proximity_search(x, mesh, 4e-3);
    AdvanceState st;
    st.reset(x);
    advance(st, y, sx, 0.9, im);
    for (int v = 0; v < nv; ++v) wr(out, st.x[v].data(), 3);
    wr(out, st.r.data(), nv);
    wr(out, &st.last_max_disp, 1);
    // resolve (device coloring: the ResolveConfig default)
    ResolveConfig cfg;
    ResolveResult res = resolve(x, y, mesh, cfg);
    for (int v = 0; v < nv; ++v) wr(out, res.x[v].data(), 3);
    const int32_t steps = res.stats.steps;
    wr(out, &steps, 1);
    std::fclose(out);
    return 0;
}

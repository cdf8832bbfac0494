#pragma once
// Drop-in for proj/include/twoway/constraints.hpp:7-92 (linearized rows, the
// row builders, fill_diag, constraint_value_at and the coloring). Every
// evaluation runs on the device through the C-ABI stage entries
// (tw_stage_linearize_ex / build_rows / constraint_value / fill_diag /
// color); the rows themselves are the reference's host structs.

#include <array>
#include <cstdint>
#include <span>
#include <vector>

#include "twoway/proximity.hpp"

namespace twoway {

enum class ConstraintKind : uint8_t { ContactVT, ContactEE, ContactVE, ContactVV, EdgeLength };

enum class ConstraintFamily : uint8_t { Volume, Gap };

/// One linearized row c + J (y - x) >= 0.
struct Constraint {
    ConstraintKind kind = ConstraintKind::ContactVV;
    int nverts = 0;
    std::array<int, 4> verts{-1, -1, -1, -1};
    double value = 0.0;         // c at the linearization point
    std::array<Vec3, 4> jac{};  // per-vertex Jacobian blocks
    double diag = 0.0;          // regularized J M^-1 J^T entry
    double lambda = 0.0;
    int color = -1;

    int pair_index = -1;  // into ProximitySet::pairs, -1 for edge rows
    uint64_t pair_key = 0;
    int edge_index = -1;  // mesh edge of an EdgeLength row

    // re-evaluation data (constraint_value_at)
    enum class Flavor : uint8_t { VolumeRatio, GapRatio, LengthRatio } flavor = Flavor::GapRatio;
    double ref_volume = 0.0;              // determinant of the reference stencil
    std::array<double, 4> gap_weights{};  // signed closest-point weights (+a, -b)
    double denom = 0.0;                   // delta (contacts) or the target length (edges)
    double sigma = 0.0;                   // EdgeLength only
};

/// Re-evaluates a row at arbitrary positions with its frozen data.
double constraint_value_at(const Constraint& c, PositionsView positions);

/// Eq. (10)/(11) vertex-triangle volume row (gap row when the reference
/// stencil degenerates).
Constraint build_vt_constraint(const ProximityPair& pair, PositionsView positions, double delta);
/// Edge-edge volume row on the four endpoints (gap row for a zero direction or
/// a degenerate reference stencil).
Constraint build_ee_constraint(const ProximityPair& pair, PositionsView positions, double delta);
/// Eq. (12) gap rows.
Constraint build_vv_constraint(const ProximityPair& pair, PositionsView positions, double delta);
Constraint build_ve_constraint(const ProximityPair& pair, PositionsView positions, double delta);
/// Gap row c = dist / delta - 1 for any pair kind.
Constraint build_gap_constraint(const ProximityPair& pair, PositionsView positions, double delta, ConstraintKind kind);
/// Eq. (13) soft unilateral rows, one per edge (zero targets and both-static
/// edges skipped), evaluated at `positions`.
std::vector<Constraint> build_edge_length_constraints(const MeshState& mesh, PositionsView positions,
                                                      const std::vector<double>& target_lengths, double sigma);

struct AssemblyOptions {
    double delta = 1e-3;
    double sigma = 1.1;
    ConstraintFamily family = ConstraintFamily::Volume;
    bool edge_constraints = true;
};

/// Contact rows of the active pairs closer than delta (pair order), then the
/// edge-length rows (edge order), with diag filled from inv_mass.
std::vector<Constraint> linearize_all(const ProximitySet& set, PositionsView positions, const MeshState& mesh,
                                      const std::vector<double>& edge_targets, const AssemblyOptions& opts);

/// diag = max(sum_m inv_mass * |jac_m|^2, 1e-10)
void fill_diag(Constraint& c, std::span<const double> inv_mass);

/// The reference's randomized smallest-last greedy coloring (conflict: a
/// shared vertex with inv_mass > 0); writes Constraint::color, returns the
/// color count.
int color_constraints(std::vector<Constraint>& constraints, std::span<const double> inv_mass, uint64_t seed);

// ------------------------------------------------------------ definitions
namespace detail {

// Row arrays in the C-ABI layout.
struct RowBuffers {
    std::vector<uint8_t> kind, flavor;
    std::vector<int32_t> nverts, verts, edge_index;
    std::vector<double> value, jac, diag, ref_volume, gap_weights, denom;
    std::vector<uint64_t> pair_key;
    explicit RowBuffers(size_t n)
        : kind(n ? n : 1), flavor(n ? n : 1), nverts(n ? n : 1), verts(4 * (n ? n : 1)), edge_index(n ? n : 1),
          value(n ? n : 1), jac(12 * (n ? n : 1)), diag(n ? n : 1), ref_volume(n ? n : 1),
          gap_weights(4 * (n ? n : 1)), denom(n ? n : 1), pair_key(n ? n : 1) {}

    Constraint row(size_t i) const {
        Constraint c;
        c.kind = static_cast<ConstraintKind>(kind[i]);
        c.nverts = 0;
        for (int k = 0; k < 4; ++k) {
            c.verts[k] = verts[4 * i + k];
            if (c.verts[k] >= 0) ++c.nverts;
            c.jac[k] = Vec3(jac[12 * i + 3 * k], jac[12 * i + 3 * k + 1], jac[12 * i + 3 * k + 2]);
            c.gap_weights[k] = gap_weights[4 * i + k];
        }
        c.value = value[i];
        c.diag = diag[i];
        c.flavor = static_cast<Constraint::Flavor>(flavor[i]);
        c.ref_volume = ref_volume[i];
        c.denom = denom[i];
        return c;
    }
};

inline void pack_rows(const std::vector<Constraint>& rows, std::vector<int32_t>& nverts, std::vector<int32_t>& verts,
                      std::vector<double>& jac) {
    const size_t n = rows.size() ? rows.size() : 1;
    nverts.assign(n, 0);
    verts.assign(4 * n, -1);
    jac.assign(12 * n, 0.0);
    for (size_t i = 0; i < rows.size(); ++i) {
        nverts[i] = rows[i].nverts;
        for (int k = 0; k < 4; ++k) {
            verts[4 * i + k] = k < rows[i].nverts ? rows[i].verts[k] : -1;
            for (int c = 0; c < 3; ++c) jac[12 * i + 3 * k + c] = rows[i].jac[k][c];
        }
    }
}

inline Constraint build_row(const ProximityPair& pair, PositionsView x, double delta, int gap,
                            ConstraintKind gap_kind) {
    tw_ctx* ctx = context(kStageDevice);
    const int32_t kinds[2] = {static_cast<int32_t>(pair.a.kind), static_cast<int32_t>(pair.b.kind)};
    int32_t verts[6];
    for (int k = 0; k < 3; ++k) verts[k] = pair.a.idx[k], verts[3 + k] = pair.b.idx[k];
    double closest[11];
    closest[0] = pair.closest.distance;
    for (int k = 0; k < 3; ++k) closest[1 + k] = pair.closest.weights_a[k], closest[4 + k] = pair.closest.weights_b[k];
    for (int k = 0; k < 3; ++k) closest[7 + k] = pair.closest.direction[k];
    closest[10] = pair.closest.degenerate ? 1.0 : 0.0;
    const std::vector<double> xf = flatten(x);
    RowBuffers b(1);
    check(tw_stage_build_rows(ctx, static_cast<int32_t>(x.size()), xf.data(), 1, kinds, verts, closest, delta, gap,
                              b.kind.data(), b.nverts.data(), b.verts.data(), b.value.data(), b.jac.data(),
                              b.flavor.data(), b.ref_volume.data(), b.gap_weights.data(), b.denom.data()),
          ctx);
    b.diag[0] = 0.0;
    Constraint c = b.row(0);
    if (gap) c.kind = gap_kind;
    return c;
}

}  // namespace detail

inline double constraint_value_at(const Constraint& c, PositionsView positions) {
    tw_ctx* ctx = detail::context(detail::kStageDevice);
    const std::vector<double> xf = detail::flatten(positions);
    const uint8_t flavor = static_cast<uint8_t>(c.flavor);
    const int32_t nverts = c.nverts;
    int32_t verts[4];
    for (int k = 0; k < 4; ++k) verts[k] = k < c.nverts ? c.verts[k] : -1;
    double out = 0.0;
    detail::check(tw_stage_constraint_value(ctx, static_cast<int32_t>(positions.size()), xf.data(), 1, &flavor,
                                            &nverts, verts, &c.ref_volume, c.gap_weights.data(), &c.denom, &c.sigma,
                                            &out),
                  ctx);
    return out;
}

inline Constraint build_vt_constraint(const ProximityPair& pair, PositionsView positions, double delta) {
    return detail::build_row(pair, positions, delta, 0, ConstraintKind::ContactVT);
}
inline Constraint build_ee_constraint(const ProximityPair& pair, PositionsView positions, double delta) {
    return detail::build_row(pair, positions, delta, 0, ConstraintKind::ContactEE);
}
inline Constraint build_vv_constraint(const ProximityPair& pair, PositionsView positions, double delta) {
    return detail::build_row(pair, positions, delta, 1, ConstraintKind::ContactVV);
}
inline Constraint build_ve_constraint(const ProximityPair& pair, PositionsView positions, double delta) {
    return detail::build_row(pair, positions, delta, 1, ConstraintKind::ContactVE);
}
inline Constraint build_gap_constraint(const ProximityPair& pair, PositionsView positions, double delta,
                                       ConstraintKind kind) {
    return detail::build_row(pair, positions, delta, 1, kind);
}

inline std::vector<Constraint> linearize_all(const ProximitySet& set, PositionsView positions, const MeshState& mesh,
                                             const std::vector<double>& edge_targets, const AssemblyOptions& opts) {
    tw_ctx* ctx = detail::context(detail::kStageDevice);
    tw_mesh* m = detail::device_mesh(ctx, detail::kStageDevice, mesh);
    const size_t np = set.pairs.size(), n1 = np ? np : 1;
    std::vector<uint64_t> keys(n1);
    std::vector<double> dist(n1), wa(3 * n1), wb(3 * n1), dir(3 * n1);
    std::vector<uint8_t> flags(n1);
    for (size_t i = 0; i < np; ++i) {
        const ProximityPair& p = set.pairs[i];
        keys[i] = p.key();
        dist[i] = p.closest.distance;
        for (int c = 0; c < 3; ++c) {
            wa[3 * i + c] = p.closest.weights_a[c], wb[3 * i + c] = p.closest.weights_b[c];
            dir[3 * i + c] = p.closest.direction[c];
        }
        flags[i] = static_cast<uint8_t>((p.active ? 1 : 0) | (p.all_static ? 2 : 0) | (p.closest.degenerate ? 4 : 0));
    }
    const std::vector<double> xf = detail::flatten(positions);
    const int64_t cap = static_cast<int64_t>(np + mesh.edges.size() + 16);
    detail::RowBuffers b(static_cast<size_t>(cap));
    int64_t nrows = 0;
    detail::check(tw_stage_linearize_ex(ctx, m, xf.data(), static_cast<int64_t>(np), keys.data(), dist.data(),
                                        wa.data(), wb.data(), dir.data(), flags.data(),
                                        edge_targets.empty() ? nullptr : edge_targets.data(), opts.delta, opts.sigma,
                                        opts.family == ConstraintFamily::Gap ? 1 : 0, opts.edge_constraints ? 1 : 0,
                                        cap, b.kind.data(), b.verts.data(), b.value.data(), b.jac.data(),
                                        b.diag.data(), b.pair_key.data(), b.edge_index.data(), b.flavor.data(),
                                        b.ref_volume.data(), b.gap_weights.data(), b.denom.data(), &nrows),
                  ctx);
    std::vector<Constraint> rows(static_cast<size_t>(nrows));
    for (int64_t i = 0; i < nrows; ++i) {
        Constraint& c = rows[i] = b.row(static_cast<size_t>(i));
        if (c.kind == ConstraintKind::EdgeLength) {
            c.edge_index = b.edge_index[i];
            c.sigma = opts.sigma;
        } else {
            c.pair_key = b.pair_key[i];
            const auto it = std::lower_bound(set.pairs.begin(), set.pairs.end(), c.pair_key,
                                             [](const ProximityPair& p, uint64_t k) { return p.key() < k; });
            c.pair_index = static_cast<int>(it - set.pairs.begin());
        }
    }
    return rows;
}

inline std::vector<Constraint> build_edge_length_constraints(const MeshState& mesh, PositionsView positions,
                                                             const std::vector<double>& target_lengths,
                                                             double sigma) {
    AssemblyOptions o;
    o.sigma = sigma;
    std::vector<Constraint> rows = linearize_all(ProximitySet{}, positions, mesh, target_lengths, o);
    for (Constraint& c : rows) c.diag = 0.0;  // the builder leaves diag to fill_diag
    return rows;
}

inline void fill_diag(Constraint& c, std::span<const double> inv_mass) {
    tw_ctx* ctx = detail::context(detail::kStageDevice);
    std::vector<int32_t> nv, verts;
    std::vector<double> jac;
    detail::pack_rows({c}, nv, verts, jac);
    detail::check(tw_stage_fill_diag(ctx, static_cast<int32_t>(inv_mass.size()), inv_mass.data(), 1, nv.data(),
                                     verts.data(), jac.data(), &c.diag),
                  ctx);
}

inline int color_constraints(std::vector<Constraint>& constraints, std::span<const double> inv_mass, uint64_t seed) {
    // Every row is colored alike (a shared dynamic vertex conflicts), on a
    // vertex-only device mesh with the reference algorithm.
    tw_ctx* ctx = detail::context(detail::kStageDevice);
    detail::MeshPtr m = detail::vertex_mesh(ctx, inv_mass);
    const size_t n = constraints.size(), n1 = n ? n : 1;
    std::vector<uint8_t> kind(n1, 0);
    std::vector<int32_t> nv, verts, eidx(n1, -1), color(n1);
    std::vector<double> jac;
    std::vector<uint64_t> keys(n1, 0);
    detail::pack_rows(constraints, nv, verts, jac);
    int32_t ncolors = 0;
    detail::check(tw_stage_color(ctx, m.get(), static_cast<int64_t>(n), kind.data(), verts.data(), keys.data(),
                                 eidx.data(), seed, TW_COLOR_REFERENCE, 0, color.data(), &ncolors),
                  ctx);
    for (size_t i = 0; i < n; ++i) constraints[i].color = color[i];
    return ncolors;
}

}  // namespace twoway

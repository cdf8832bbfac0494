#pragma once
// Drop-in for proj/include/twoway/constraints.hpp:7-92 (linearized rows and
// their coloring). linearize_all runs on the device (tw_stage_linearize),
// color_constraints replays the reference coloring on the device
// (tw_stage_color, reference mode).

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

    // Re-evaluation data of the reference (constraint_value_at); the device
    // linearization does not return it: flavor/ref_volume/gap_weights/denom
    // stay at their defaults here.
    enum class Flavor : uint8_t { VolumeRatio, GapRatio, LengthRatio } flavor = Flavor::GapRatio;
    double ref_volume = 0.0;
    std::array<double, 4> gap_weights{};
    double denom = 0.0;
    double sigma = 0.0;
};

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

/// The reference's randomized smallest-last greedy coloring (conflict: a
/// shared vertex with inv_mass > 0); writes Constraint::color, returns the
/// color count.
int color_constraints(std::vector<Constraint>& constraints, std::span<const double> inv_mass, uint64_t seed);

}  // namespace twoway

#pragma once
// Drop-in for proj/include/twoway/lcp.hpp:12-53 (the backward step). The
// system stays the reference's host struct; assemble_lcp, the PGS / Jacobi
// sweeps and recover_target run on the device (tw_stage_lcp with the
// ASSEMBLE / SOLVE / RECOVER stages), with the reference's row order for the
// warm start, colors ascending then rows ascending for PGS, and the ordered
// impulse application of the Jacobi variant (bit-exact with lcp.cpp).

#include <span>
#include <stdexcept>
#include <vector>

#include "twoway/constraints.hpp"

namespace twoway {

/// Matrix-free view of lambda >= 0 perp q + J M^-1 J^T lambda >= 0 with
/// q_i = c_i + [J (y_target - x)]_i; `impulse` caches M^-1 J^T lambda.
struct LcpSystem {
    std::vector<Constraint>* constraints = nullptr;
    std::span<const double> inv_mass;
    std::vector<double> target_gap;  // q
    Positions impulse;               // M^-1 J^T lambda, one 3-vector per vertex
    int num_colors = 0;

    /// (J M^-1 J^T lambda)_row read off the impulse cache
    double coupling(int row) const {
        const Constraint& c = (*constraints)[row];
        double s = 0.0;
        for (int m = 0; m < c.nverts; ++m) s += c.jac[m].dot(impulse[c.verts[m]]);
        return s;
    }
    /// impulse += M^-1 J_row^T dlambda
    void add_impulse(int row, double dlambda) {
        const Constraint& c = (*constraints)[row];
        for (int m = 0; m < c.nverts; ++m) {
            const int v = c.verts[m];
            impulse[v] += inv_mass[v] * dlambda * c.jac[m];
        }
    }
};

/// Builds q and folds the warm-start multipliers stored on the rows into the
/// impulse cache.
LcpSystem assemble_lcp(std::vector<Constraint>& constraints, PositionsView x, PositionsView y_target,
                       std::span<const double> inv_mass, int num_colors);
/// Multi-color projected Gauss-Seidel (colors ascending; rows of one color
/// share no dynamic vertex).
void pgs_sweeps(LcpSystem& sys, int n_iters);
/// Simultaneous (Jacobi) variant with under-relaxation.
void projected_jacobi_sweeps(LcpSystem& sys, int n_iters, double under_relax);
/// The AL gradient-descent baseline (lcp.cpp:61-129) is a paper comparison
/// baseline that is not provided on the device: throws std::invalid_argument
/// (the C-ABI's TW_EUNSUPPORTED).
void al_gradient_descent(LcpSystem& sys, int n_inner);
/// y = y_target + impulse for dynamic vertices; static ones keep y_target.
Positions recover_target(const LcpSystem& sys, PositionsView y_target);

// ------------------------------------------------------------ definitions
namespace detail {

inline void lcp_stage(LcpSystem& sys, int mode, PositionsView x, PositionsView y, int solver, int iters,
                      double under_relax, Positions* y_out) {
    tw_ctx* ctx = context(kStageDevice);
    std::vector<Constraint>& rows = *sys.constraints;
    const int32_t nv = static_cast<int32_t>(sys.inv_mass.size());
    const size_t n = rows.size(), n1 = n ? n : 1;
    std::vector<int32_t> nverts, verts, color(n1, 0);
    std::vector<double> jac, value(n1), diag(n1), lambda(n1);
    pack_rows(rows, nverts, verts, jac);
    for (size_t i = 0; i < n; ++i) {
        value[i] = rows[i].value, diag[i] = rows[i].diag, lambda[i] = rows[i].lambda;
        color[i] = rows[i].color;
    }
    if (sys.target_gap.size() < n) sys.target_gap.resize(n);
    if (sys.impulse.size() != sys.inv_mass.size()) sys.impulse.assign(sys.inv_mass.size(), Vec3::Zero());
    std::vector<double> imp = flatten(sys.impulse);
    std::vector<double> xf = x.empty() ? std::vector<double>() : flatten(x);
    std::vector<double> yf = y.empty() ? std::vector<double>() : flatten(y);
    std::vector<double> yo(y_out ? 3 * static_cast<size_t>(nv) : 0);
    detail::check(tw_stage_lcp(ctx, nv, sys.inv_mass.data(), static_cast<int64_t>(n), verts.data(), value.data(),
                               jac.data(), diag.data(), color.data(), sys.num_colors > 0 ? sys.num_colors : 1,
                               xf.empty() ? nullptr : xf.data(), yf.empty() ? nullptr : yf.data(), solver,
                               iters, under_relax, mode, lambda.data(), sys.target_gap.data(), imp.data(),
                               y_out ? yo.data() : nullptr),
                  ctx);
    for (size_t i = 0; i < n; ++i) rows[i].lambda = lambda[i];
    sys.impulse = unflatten(imp.data(), sys.inv_mass.size());
    if (y_out) *y_out = unflatten(yo.data(), static_cast<size_t>(nv));
}

}  // namespace detail

inline LcpSystem assemble_lcp(std::vector<Constraint>& constraints, PositionsView x, PositionsView y_target,
                              std::span<const double> inv_mass, int num_colors) {
    LcpSystem sys;
    sys.constraints = &constraints;
    sys.inv_mass = inv_mass;
    sys.num_colors = num_colors;
    sys.target_gap.assign(constraints.size(), 0.0);
    sys.impulse.assign(inv_mass.size(), Vec3::Zero());
    detail::lcp_stage(sys, TW_LCP_ASSEMBLE, x, y_target, TW_SOLVER_PGS, 1, 0.5, nullptr);
    return sys;
}

inline void pgs_sweeps(LcpSystem& sys, int n_iters) {
    if (n_iters < 1 || sys.constraints->empty()) return;
    for (const Constraint& c : *sys.constraints)
        if (c.color < 0 || c.color >= sys.num_colors) throw std::invalid_argument("pgs_sweeps: row color out of range");
    detail::lcp_stage(sys, TW_LCP_SOLVE, {}, {}, TW_SOLVER_PGS, n_iters, 0.5, nullptr);
}

inline void projected_jacobi_sweeps(LcpSystem& sys, int n_iters, double under_relax) {
    if (n_iters < 1 || sys.constraints->empty()) return;
    detail::lcp_stage(sys, TW_LCP_SOLVE, {}, {}, TW_SOLVER_JACOBI, n_iters, under_relax, nullptr);
}

inline void al_gradient_descent(LcpSystem&, int) {
    throw std::invalid_argument("al_gradient_descent: the AL baseline solvers are not provided on the device");
}

inline Positions recover_target(const LcpSystem& sys, PositionsView y_target) {
    LcpSystem copy = sys;
    std::vector<Constraint> none;
    copy.constraints = &none;
    Positions y;
    detail::lcp_stage(copy, TW_LCP_RECOVER, {}, y_target, TW_SOLVER_PGS, 1, 0.5, &y);
    return y;
}

}  // namespace twoway

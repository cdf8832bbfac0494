/*
 * ORACLE — test infrastructure only.
 * Restatement of proj/src/lcp.cpp (assemble_lcp, pgs_sweeps,
 * projected_jacobi_sweeps, recover_target; LcpSystem::coupling/add_impulse in
 * proj/include/twoway/lcp.hpp:19-31) and proj/src/advance.cpp.
 */
#include <stdlib.h>
#include <string.h>

#include "or_internal.h"

static double coupling(const or_lcp* s, int64_t row) { /* lcp.hpp:19-24 */
    const or_row* c = &s->rows[row];
    double acc = 0.0;
    for (int m = 0; m < c->nverts; ++m) acc += v3_dot(c->jac[m], v3_load(s->impulse + 3 * (size_t)c->verts[m]));
    return acc;
}

static void add_impulse(or_lcp* s, int64_t row, double dlambda) { /* lcp.hpp:25-31 */
    const or_row* c = &s->rows[row];
    for (int m = 0; m < c->nverts; ++m) {
        const int v = c->verts[m];
        double* imp = s->impulse + 3 * (size_t)v;
        const v3 add = v3_scale(s->inv_mass[v] * dlambda, c->jac[m]);
        imp[0] = imp[0] + add.x;
        imp[1] = imp[1] + add.y;
        imp[2] = imp[2] + add.z;
    }
}

/* assemble_lcp, lcp.cpp:8-25 */
void or_lcp_assemble(or_lcp* s, or_row* rows, int64_t n, const double* x, const double* y,
                     const double* inv_mass, int nv, int ncolors) {
    s->rows = rows;
    s->n = n;
    s->inv_mass = inv_mass;
    s->nv = nv;
    s->ncolors = ncolors;
    s->impulse = (double*)or_xcalloc((size_t)nv * 3 + 1, sizeof(double));
    s->q = (double*)or_xmalloc(((size_t)n + 1) * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        const or_row* c = &rows[i];
        double q = c->value;
        for (int m = 0; m < c->nverts; ++m) {
            const int v = c->verts[m];
            q += v3_dot(c->jac[m], v3_sub(v3_load(y + 3 * (size_t)v), v3_load(x + 3 * (size_t)v)));
        }
        s->q[i] = q;
        if (c->lambda != 0.0) add_impulse(s, i, c->lambda); /* warm start */
    }
}

/* pgs_sweeps, lcp.cpp:27-42 */
void or_lcp_pgs(or_lcp* s, int iters) {
    for (int it = 0; it < iters; ++it)
        for (int color = 0; color < s->ncolors; ++color)
            for (int64_t i = 0; i < s->n; ++i) {
                or_row* c = &s->rows[i];
                if (c->color != color) continue;
                const double w = s->q[i] + coupling(s, i);
                const double lam = or_max(0.0, c->lambda - w / c->diag);
                const double d = lam - c->lambda;
                if (d != 0.0) add_impulse(s, i, d);
                c->lambda = lam;
            }
}

/* projected_jacobi_sweeps, lcp.cpp:44-59 */
void or_lcp_jacobi(or_lcp* s, int iters, double under_relax) {
    double* next = (double*)or_xmalloc(((size_t)s->n + 1) * sizeof(double));
    for (int it = 0; it < iters; ++it) {
        for (int64_t i = 0; i < s->n; ++i) {
            const or_row* c = &s->rows[i];
            const double w = s->q[i] + coupling(s, i);
            next[i] = or_max(0.0, c->lambda - under_relax * w / c->diag);
        }
        for (int64_t i = 0; i < s->n; ++i) {
            const double d = next[i] - s->rows[i].lambda;
            if (d != 0.0) add_impulse(s, i, d);
            s->rows[i].lambda = next[i];
        }
    }
    free(next);
}

/* recover_target, lcp.cpp:131-136 */
void or_lcp_recover(const or_lcp* s, const double* y_target, double* y_out) {
    for (int v = 0; v < s->nv; ++v)
        for (int k = 0; k < 3; ++k) {
            const size_t i = 3 * (size_t)v + k;
            y_out[i] = s->inv_mass[v] > 0.0 ? y_target[i] + s->impulse[i] : y_target[i];
        }
}

void or_lcp_free(or_lcp* s) {
    free(s->impulse);
    free(s->q);
    s->impulse = s->q = NULL;
}

int or_backward(int nv, const double* inv_mass, int64_t nrows, const int32_t* nverts,
                const int32_t* verts, const double* value, const double* jac, const double* diag,
                const int32_t* color, int ncolors, const double* x, const double* y_target,
                int solver, int sweeps, double under_relax, double* lambda, double* q_out,
                double* impulse_out, double* y_out) {
    if (solver != OR_SOLVER_PGS && solver != OR_SOLVER_JACOBI) return -2;
    or_row* rows = (or_row*)or_xcalloc((size_t)nrows + 1, sizeof(or_row));
    for (int64_t i = 0; i < nrows; ++i) {
        or_row* c = &rows[i];
        c->nverts = nverts[i];
        for (int m = 0; m < 4; ++m) {
            c->verts[m] = verts[4 * i + m];
            c->jac[m] = v3_load(jac + 12 * i + 3 * m);
        }
        c->value = value[i];
        c->diag = diag[i];
        c->color = color ? color[i] : 0;
        c->lambda = lambda[i];
    }
    or_lcp s;
    or_lcp_assemble(&s, rows, nrows, x, y_target, inv_mass, nv, ncolors);
    if (q_out) memcpy(q_out, s.q, (size_t)nrows * sizeof(double));
    if (solver == OR_SOLVER_PGS) or_lcp_pgs(&s, sweeps);
    else or_lcp_jacobi(&s, sweeps, under_relax);
    if (y_out) or_lcp_recover(&s, y_target, y_out);
    if (impulse_out) memcpy(impulse_out, s.impulse, (size_t)nv * 3 * sizeof(double));
    for (int64_t i = 0; i < nrows; ++i) lambda[i] = rows[i].lambda;
    or_lcp_free(&s);
    free(rows);
    return 0;
}

/* advance, advance.cpp:8-39 (D = per_vertex_bound for every vertex) */
double or_advance(int nv, const double* inv_mass, const double* y, const double* D, double gamma,
                  double* x, double* r) {
    double max_disp = 0.0;
    for (int i = 0; i < nv; ++i) {
        if (inv_mass[i] == 0.0) {
            r[i] = 0.0;
            continue;
        }
        const v3 xi = v3_load(x + 3 * (size_t)i);
        const v3 d = v3_sub(v3_load(y + 3 * (size_t)i), xi);
        const double dn = v3_norm(d);
        if (dn == 0.0) {
            r[i] = 0.0;
            continue;
        }
        const double limit = 0.5 * gamma * D[i];
        double alpha = or_min(limit / dn, 1.0);
        v3 disp = v3_scale(alpha, d);
        if (alpha < 1.0) {
            const double dnorm = v3_norm(disp);
            if (dnorm > limit) { /* last-ulp rounding guard */
                const double s = (limit / dnorm) * (1.0 - 1e-14);
                disp = v3_make(disp.x * s, disp.y * s, disp.z * s);
                alpha *= s;
            }
        }
        v3_store(x + 3 * (size_t)i, v3_add(xi, disp));
        r[i] *= (1.0 - alpha);
        max_disp = or_max(max_disp, v3_norm(disp));
    }
    return max_disp;
}

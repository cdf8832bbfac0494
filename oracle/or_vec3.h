/*
 * ORACLE — test infrastructure only (never linked into the product path).
 *
 * FP64 3-vector helpers with the evaluation order of Eigen's fixed-size
 * Vector3d that the reference relies on (reference: proj/include/twoway/
 * types.hpp:10-14; association pinned in SURVEY.md Appendix A):
 *   dot         = (a0*b0 + a1*b1) + a2*b2
 *   squaredNorm = (x*x + y*y) + z*z,   norm = sqrt(squaredNorm)
 *   cross       = (a1*b2 - a2*b1, a2*b0 - a0*b2, a0*b1 - a1*b0)
 *   s*v / v/s   = per component multiply / divide (no reciprocal)
 *   normalized  = v / sqrt(sqn) if sqn > 0 else v
 *   isZero      = all |c| <= 1e-12 (Eigen dummy precision for double)
 * Must be compiled with -ffp-contract=off (no FMA contraction).
 */
#ifndef OR_VEC3_H
#define OR_VEC3_H

#include <math.h>

typedef struct {
    double x, y, z;
} v3;

static inline v3 v3_make(double x, double y, double z) {
    v3 r = {x, y, z};
    return r;
}
static inline v3 v3_zero(void) { return v3_make(0.0, 0.0, 0.0); }
static inline v3 v3_load(const double* p) { return v3_make(p[0], p[1], p[2]); }
static inline void v3_store(double* p, v3 a) {
    p[0] = a.x;
    p[1] = a.y;
    p[2] = a.z;
}
static inline v3 v3_add(v3 a, v3 b) { return v3_make(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline v3 v3_sub(v3 a, v3 b) { return v3_make(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline v3 v3_neg(v3 a) { return v3_make(-a.x, -a.y, -a.z); }
/* s * v */
static inline v3 v3_scale(double s, v3 a) { return v3_make(s * a.x, s * a.y, s * a.z); }
/* v / s */
static inline v3 v3_div(v3 a, double s) { return v3_make(a.x / s, a.y / s, a.z / s); }
static inline double v3_dot(v3 a, v3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
static inline double v3_sqn(v3 a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
static inline double v3_norm(v3 a) { return sqrt(v3_sqn(a)); }
static inline v3 v3_cross(v3 a, v3 b) {
    return v3_make(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline v3 v3_normalized(v3 a) {
    const double z = v3_sqn(a);
    return z > 0.0 ? v3_div(a, sqrt(z)) : a;
}
static inline int v3_is_zero(v3 a) {
    return fabs(a.x) <= 1e-12 && fabs(a.y) <= 1e-12 && fabs(a.z) <= 1e-12;
}
/* std::clamp(v, lo, hi) */
static inline double or_clamp(double v, double lo, double hi) {
    return v < lo ? lo : (hi < v ? hi : v);
}
/* std::min(a, b) / std::max(a, b) */
static inline double or_min(double a, double b) { return b < a ? b : a; }
static inline double or_max(double a, double b) { return a < b ? b : a; }

#endif

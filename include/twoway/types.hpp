#pragma once
// Drop-in for proj/include/twoway/types.hpp:10-22. The reference aliases
// Eigen::Vector3d; Eigen is not a dependency here, so Vec3 is a 24-byte FP64
// vector with the Eigen members the reference's callers use and the same
// evaluation order (dot = (a0 b0 + a1 b1) + a2 b2, norm = sqrt(squaredNorm)).
// Define TWOWAY_USE_EIGEN to alias Eigen::Vector3d instead.

#include <cmath>
#include <cstdint>
#include <span>
#include <vector>

#ifdef TWOWAY_USE_EIGEN
#include <Eigen/Dense>
#endif

namespace twoway {

#ifdef TWOWAY_USE_EIGEN
using Vec3 = Eigen::Vector3d;
#else
class Vec3 {
public:
    constexpr Vec3() : v_{0.0, 0.0, 0.0} {}
    constexpr Vec3(double x, double y, double z) : v_{x, y, z} {}

    static constexpr Vec3 Zero() { return {0.0, 0.0, 0.0}; }
    static constexpr Vec3 UnitX() { return {1.0, 0.0, 0.0}; }
    static constexpr Vec3 UnitY() { return {0.0, 1.0, 0.0}; }
    static constexpr Vec3 UnitZ() { return {0.0, 0.0, 1.0}; }

    double& x() { return v_[0]; }
    double& y() { return v_[1]; }
    double& z() { return v_[2]; }
    double x() const { return v_[0]; }
    double y() const { return v_[1]; }
    double z() const { return v_[2]; }
    double& operator[](int i) { return v_[i]; }
    double operator[](int i) const { return v_[i]; }
    double& operator()(int i) { return v_[i]; }
    double operator()(int i) const { return v_[i]; }
    double* data() { return v_; }
    const double* data() const { return v_; }

    Vec3 operator+(const Vec3& o) const { return {v_[0] + o.v_[0], v_[1] + o.v_[1], v_[2] + o.v_[2]}; }
    Vec3 operator-(const Vec3& o) const { return {v_[0] - o.v_[0], v_[1] - o.v_[1], v_[2] - o.v_[2]}; }
    Vec3 operator-() const { return {-v_[0], -v_[1], -v_[2]}; }
    Vec3 operator*(double s) const { return {v_[0] * s, v_[1] * s, v_[2] * s}; }
    Vec3 operator/(double s) const { return {v_[0] / s, v_[1] / s, v_[2] / s}; }
    Vec3& operator+=(const Vec3& o) { return *this = *this + o; }
    Vec3& operator-=(const Vec3& o) { return *this = *this - o; }
    Vec3& operator*=(double s) { return *this = *this * s; }
    Vec3& operator/=(double s) { return *this = *this / s; }
    bool operator==(const Vec3& o) const { return v_[0] == o.v_[0] && v_[1] == o.v_[1] && v_[2] == o.v_[2]; }

    double dot(const Vec3& o) const { return (v_[0] * o.v_[0] + v_[1] * o.v_[1]) + v_[2] * o.v_[2]; }
    Vec3 cross(const Vec3& o) const {
        return {v_[1] * o.v_[2] - v_[2] * o.v_[1], v_[2] * o.v_[0] - v_[0] * o.v_[2],
                v_[0] * o.v_[1] - v_[1] * o.v_[0]};
    }
    double squaredNorm() const { return dot(*this); }
    double norm() const { return std::sqrt(squaredNorm()); }
    Vec3 normalized() const {
        const double z = squaredNorm();
        return z > 0.0 ? *this / std::sqrt(z) : *this;
    }
    void normalize() { *this = normalized(); }
    Vec3 cwiseMin(const Vec3& o) const {
        return {o.v_[0] < v_[0] ? o.v_[0] : v_[0], o.v_[1] < v_[1] ? o.v_[1] : v_[1],
                o.v_[2] < v_[2] ? o.v_[2] : v_[2]};
    }
    Vec3 cwiseMax(const Vec3& o) const {
        return {v_[0] < o.v_[0] ? o.v_[0] : v_[0], v_[1] < o.v_[1] ? o.v_[1] : v_[1],
                v_[2] < o.v_[2] ? o.v_[2] : v_[2]};
    }
    double maxCoeff() const {
        double m = v_[0];
        if (m < v_[1]) m = v_[1];
        if (m < v_[2]) m = v_[2];
        return m;
    }
    bool allFinite() const { return std::isfinite(v_[0]) && std::isfinite(v_[1]) && std::isfinite(v_[2]); }
    bool isZero(double prec = 1e-12) const {
        return std::abs(v_[0]) <= prec && std::abs(v_[1]) <= prec && std::abs(v_[2]) <= prec;
    }

private:
    double v_[3];
};

inline Vec3 operator*(double s, const Vec3& v) { return {s * v.x(), s * v.y(), s * v.z()}; }
static_assert(sizeof(Vec3) == 24, "Vec3 must have the byte layout of Eigen::Vector3d");
#endif

using Positions = std::vector<Vec3>;
using PositionsView = std::span<const Vec3>;

inline bool is_finite(const Vec3& v) { return v.allFinite(); }

inline bool all_finite(PositionsView xs) {
    for (const Vec3& x : xs)
        if (!x.allFinite()) return false;
    return true;
}

}  // namespace twoway

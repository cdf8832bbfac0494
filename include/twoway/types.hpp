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
using Mat3 = Eigen::Matrix3d;
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

/// 3x3 FP64 matrix (the reference's Mat3 = Eigen::Matrix3d, types.hpp:11),
/// column-major like Eigen, with the members the reference's dynamics code
/// uses: Zero/Identity, (r, c), + - and scalar products, transpose, M * v
/// (row sums (m0 v0 + m1 v1) + m2 v2) and the outer product outer(u, v).
class Mat3 {
public:
    constexpr Mat3() : m_{0, 0, 0, 0, 0, 0, 0, 0, 0} {}
    static constexpr Mat3 Zero() { return Mat3(); }
    static constexpr Mat3 Identity() {
        Mat3 m;
        m.m_[0] = m.m_[4] = m.m_[8] = 1.0;
        return m;
    }
    static Mat3 outer(const Vec3& u, const Vec3& v) {
        Mat3 m;
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) m(r, c) = u[r] * v[c];
        return m;
    }
    double& operator()(int r, int c) { return m_[r + 3 * c]; }
    double operator()(int r, int c) const { return m_[r + 3 * c]; }
    double* data() { return m_; }
    const double* data() const { return m_; }

    Mat3 operator+(const Mat3& o) const { return zip(o, [](double a, double b) { return a + b; }); }
    Mat3 operator-(const Mat3& o) const { return zip(o, [](double a, double b) { return a - b; }); }
    Mat3 operator-() const { return zip(*this, [](double a, double) { return -a; }); }
    Mat3 operator*(double s) const { return zip(*this, [s](double a, double) { return a * s; }); }
    Mat3 operator/(double s) const { return zip(*this, [s](double a, double) { return a / s; }); }
    Mat3& operator+=(const Mat3& o) { return *this = *this + o; }
    Mat3& operator-=(const Mat3& o) { return *this = *this - o; }
    Mat3& operator*=(double s) { return *this = *this * s; }
    bool operator==(const Mat3& o) const {
        for (int i = 0; i < 9; ++i)
            if (m_[i] != o.m_[i]) return false;
        return true;
    }
    Vec3 operator*(const Vec3& v) const {
        Vec3 out;
        for (int r = 0; r < 3; ++r) out[r] = ((*this)(r, 0) * v[0] + (*this)(r, 1) * v[1]) + (*this)(r, 2) * v[2];
        return out;
    }
    Mat3 operator*(const Mat3& o) const {
        Mat3 out;
        for (int c = 0; c < 3; ++c) {
            Vec3 col = *this * Vec3(o(0, c), o(1, c), o(2, c));
            for (int r = 0; r < 3; ++r) out(r, c) = col[r];
        }
        return out;
    }
    Mat3 transpose() const {
        Mat3 t;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) t(c, r) = (*this)(r, c);
        return t;
    }
    Vec3 col(int c) const { return {(*this)(0, c), (*this)(1, c), (*this)(2, c)}; }
    Vec3 row(int r) const { return {(*this)(r, 0), (*this)(r, 1), (*this)(r, 2)}; }
    double trace() const { return ((*this)(0, 0) + (*this)(1, 1)) + (*this)(2, 2); }

private:
    template <typename F>
    Mat3 zip(const Mat3& o, F f) const {
        Mat3 out;
        for (int i = 0; i < 9; ++i) out.m_[i] = f(m_[i], o.m_[i]);
        return out;
    }
    double m_[9];
};

inline Mat3 operator*(double s, const Mat3& m) { return m * s; }
static_assert(sizeof(Mat3) == 72, "Mat3 must have the byte layout of Eigen::Matrix3d");
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

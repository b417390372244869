// Small fixed-size linear algebra for the host side (load-time geometry,
// init poses, squeeze). Replaces the Eigen value types the reference uses in
// its public headers (reference: proj/include/grasp/geometry.hpp:12-44).
// Mat3 is column-major like Eigen::Matrix3d so state layouts line up
// (rotation block = 9 column-major entries, proj/include/grasp/hand.hpp:56-61).
#pragma once

#include <cmath>
#include <stdexcept>
#include <vector>

namespace grasp {

struct Vec3 {
  double x = 0, y = 0, z = 0;
  Vec3() = default;
  constexpr Vec3(double a, double b, double c) : x(a), y(b), z(c) {}
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  static Vec3 Zero() { return {0, 0, 0}; }
  static Vec3 UnitX() { return {1, 0, 0}; }
  static Vec3 UnitY() { return {0, 1, 0}; }
  static Vec3 UnitZ() { return {0, 0, 1}; }
  static Vec3 Constant(double v) { return {v, v, v}; }
};

inline Vec3 operator+(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline Vec3 operator-(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline Vec3 operator-(const Vec3& a) { return {-a.x, -a.y, -a.z}; }
inline Vec3 operator*(double s, const Vec3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline Vec3 operator*(const Vec3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline Vec3 operator/(const Vec3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline Vec3& operator+=(Vec3& a, const Vec3& b) { a.x += b.x; a.y += b.y; a.z += b.z; return a; }
inline Vec3& operator-=(Vec3& a, const Vec3& b) { a.x -= b.x; a.y -= b.y; a.z -= b.z; return a; }
inline Vec3& operator*=(Vec3& a, double s) { a.x *= s; a.y *= s; a.z *= s; return a; }
inline Vec3& operator/=(Vec3& a, double s) { a.x /= s; a.y /= s; a.z /= s; return a; }
inline bool operator==(const Vec3& a, const Vec3& b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
inline bool operator!=(const Vec3& a, const Vec3& b) { return !(a == b); }

// Left-to-right association. Eigen's own association depends on its packet
// path, so agreement with the reference is at rounding level, not bitwise.
inline double dot(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline double squared_norm(const Vec3& a) { return dot(a, a); }
inline double norm(const Vec3& a) { return std::sqrt(squared_norm(a)); }
inline Vec3 cross(const Vec3& a, const Vec3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline Vec3 normalized(const Vec3& a) {
  const double n2 = squared_norm(a);
  if (n2 > 0) return a / std::sqrt(n2);
  return a;
}
inline Vec3 cwise_min(const Vec3& a, const Vec3& b) {
  return {b.x < a.x ? b.x : a.x, b.y < a.y ? b.y : a.y, b.z < a.z ? b.z : a.z};
}
inline Vec3 cwise_max(const Vec3& a, const Vec3& b) {
  return {a.x < b.x ? b.x : a.x, a.y < b.y ? b.y : a.y, a.z < b.z ? b.z : a.z};
}

struct Mat3 {
  double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};  // column-major
  double& operator()(int r, int c) { return m[c * 3 + r]; }
  double operator()(int r, int c) const { return m[c * 3 + r]; }
  Vec3 col(int c) const { return {m[c * 3], m[c * 3 + 1], m[c * 3 + 2]}; }
  Vec3 row(int r) const { return {m[r], m[3 + r], m[6 + r]}; }
  void set_col(int c, const Vec3& v) { m[c * 3] = v.x; m[c * 3 + 1] = v.y; m[c * 3 + 2] = v.z; }
  static Mat3 Identity() { return {}; }
  static Mat3 Zero() { Mat3 z; for (double& v : z.m) v = 0; return z; }
  Mat3 transpose() const {
    Mat3 t;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) t(r, c) = (*this)(c, r);
    return t;
  }
  double determinant() const {
    const Mat3& a = *this;
    return a(0, 0) * (a(1, 1) * a(2, 2) - a(2, 1) * a(1, 2)) -
           a(1, 0) * (a(0, 1) * a(2, 2) - a(2, 1) * a(0, 2)) +
           a(2, 0) * (a(0, 1) * a(1, 2) - a(1, 1) * a(0, 2));
  }
};

inline Vec3 operator*(const Mat3& a, const Vec3& v) {
  Vec3 r;
  r.x = a(0, 0) * v.x + a(0, 1) * v.y + a(0, 2) * v.z;
  r.y = a(1, 0) * v.x + a(1, 1) * v.y + a(1, 2) * v.z;
  r.z = a(2, 0) * v.x + a(2, 1) * v.y + a(2, 2) * v.z;
  return r;
}
inline Mat3 operator*(const Mat3& a, const Mat3& b) {
  Mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = a(i, 0) * b(0, j) + a(i, 1) * b(1, j) + a(i, 2) * b(2, j);
  return r;
}
inline Mat3 operator*(double s, const Mat3& a) { Mat3 r; for (int i = 0; i < 9; ++i) r.m[i] = s * a.m[i]; return r; }
inline Mat3 operator+(const Mat3& a, const Mat3& b) { Mat3 r; for (int i = 0; i < 9; ++i) r.m[i] = a.m[i] + b.m[i]; return r; }
inline Mat3 operator-(const Mat3& a, const Mat3& b) { Mat3 r; for (int i = 0; i < 9; ++i) r.m[i] = a.m[i] - b.m[i]; return r; }
inline Mat3 outer(const Vec3& a, const Vec3& b) {
  Mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = a[i] * b[j];
  return r;
}

inline Mat3 skew(const Vec3& v) {
  Mat3 m = Mat3::Zero();
  m(0, 1) = -v.z;
  m(0, 2) = v.y;
  m(1, 0) = v.z;
  m(1, 2) = -v.x;
  m(2, 0) = -v.y;
  m(2, 1) = v.x;
  return m;
}

/// Dynamic dense matrix, column-major like Eigen::MatrixXd (Jacobians are
/// 3 x (12 + dof), reference hand.hpp:111-121).
struct MatrixXd {
  int n_rows = 0, n_cols = 0;
  std::vector<double> data;
  MatrixXd() = default;
  MatrixXd(int r, int c) : n_rows(r), n_cols(c), data(static_cast<size_t>(r) * c, 0.0) {}
  static MatrixXd Zero(int r, int c) { return MatrixXd(r, c); }
  int rows() const { return n_rows; }
  int cols() const { return n_cols; }
  double& operator()(int r, int c) { return data[static_cast<size_t>(c) * n_rows + r]; }
  double operator()(int r, int c) const { return data[static_cast<size_t>(c) * n_rows + r]; }
  Vec3 col3(int c) const { return {(*this)(0, c), (*this)(1, c), (*this)(2, c)}; }
};

/// Rigid transform p' = R p + t (reference: proj/include/grasp/geometry.hpp:17-28).
struct RigidTransform {
  Mat3 R = Mat3::Identity();
  Vec3 t = Vec3::Zero();
  Vec3 apply(const Vec3& p) const { return R * p + t; }
  Vec3 rotate(const Vec3& v) const { return R * v; }
  RigidTransform inverse() const { Mat3 rt = R.transpose(); return {rt, -(rt * t)}; }
  RigidTransform operator*(const RigidTransform& o) const { return {R * o.R, R * o.t + t}; }
  static RigidTransform identity() { return {}; }
};

/// Eigen::AngleAxisd(angle, axis).toRotationMatrix() with Eigen's expression
/// order (Eigen/src/Geometry/AngleAxis.h); used by FK and init poses.
inline Mat3 angle_axis_matrix(double angle, const Vec3& axis) {
  Mat3 res;
  const Vec3 sin_axis = std::sin(angle) * axis;
  const double c = std::cos(angle);
  const Vec3 cos1_axis = (1.0 - c) * axis;
  double tmp = cos1_axis.x * axis.y;
  res(0, 1) = tmp - sin_axis.z;
  res(1, 0) = tmp + sin_axis.z;
  tmp = cos1_axis.x * axis.z;
  res(0, 2) = tmp + sin_axis.y;
  res(2, 0) = tmp - sin_axis.y;
  tmp = cos1_axis.y * axis.z;
  res(1, 2) = tmp - sin_axis.x;
  res(2, 1) = tmp + sin_axis.x;
  res(0, 0) = cos1_axis.x * axis.x + c;
  res(1, 1) = cos1_axis.y * axis.y + c;
  res(2, 2) = cos1_axis.z * axis.z + c;
  return res;
}

}  // namespace grasp

// ORACLE (test infrastructure only; never linked into the product).
// Small dense types for the fp64 CPU restatement of the reference hot path.
// The reference uses Eigen (proj/CMakeLists.txt:11), which is absent here;
// these restate just the operations the hot path needs.
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <limits>
#include <vector>

namespace oracle {

struct V3 {
  double v[3] = {0, 0, 0};
  V3() = default;
  V3(double a, double b, double c) { v[0] = a; v[1] = b; v[2] = c; }
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
  double x() const { return v[0]; }
  double y() const { return v[1]; }
  double z() const { return v[2]; }
  static V3 unit(int k) { V3 r; r.v[k] = 1.0; return r; }
};
inline V3 operator+(const V3& a, const V3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
inline V3 operator-(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline V3 operator-(const V3& a) { return {-a[0], -a[1], -a[2]}; }
inline V3 operator*(double s, const V3& a) { return {s * a[0], s * a[1], s * a[2]}; }
inline V3 operator*(const V3& a, double s) { return {a[0] * s, a[1] * s, a[2] * s}; }
inline V3 operator/(const V3& a, double s) { return {a[0] / s, a[1] / s, a[2] / s}; }
inline V3& operator+=(V3& a, const V3& b) { for (int i = 0; i < 3; ++i) a[i] += b[i]; return a; }
inline V3& operator-=(V3& a, const V3& b) { for (int i = 0; i < 3; ++i) a[i] -= b[i]; return a; }
inline double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double sqnorm(const V3& a) { return dot(a, a); }
inline double norm(const V3& a) { return std::sqrt(sqnorm(a)); }
inline V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
inline V3 normalized(const V3& a) {
  const double n2 = sqnorm(a);
  return n2 > 0 ? a / std::sqrt(n2) : a;
}
inline bool finite3(const V3& a) { return std::isfinite(a[0]) && std::isfinite(a[1]) && std::isfinite(a[2]); }

// Row-major 3x3 for readability; state layout conversion is explicit.
struct M3 {
  double a[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  double& operator()(int r, int c) { return a[r][c]; }
  double operator()(int r, int c) const { return a[r][c]; }
  static M3 zero() { M3 m; for (auto& r : m.a) for (double& v : r) v = 0; return m; }
  static M3 identity() { return M3(); }
  V3 col(int c) const { return {a[0][c], a[1][c], a[2][c]}; }
  V3 row(int r) const { return {a[r][0], a[r][1], a[r][2]}; }
  void set_col(int c, const V3& v) { for (int r = 0; r < 3; ++r) a[r][c] = v[r]; }
  M3 t() const { M3 m; for (int r = 0; r < 3; ++r) for (int c = 0; c < 3; ++c) m.a[r][c] = a[c][r]; return m; }
  double det() const {
    return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) - a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
           a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
  }
  double trace() const { return a[0][0] + a[1][1] + a[2][2]; }
};
inline M3 operator*(const M3& x, const M3& y) {
  M3 r = M3::zero();
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[i][j] = x.a[i][0] * y.a[0][j] + x.a[i][1] * y.a[1][j] + x.a[i][2] * y.a[2][j];
  return r;
}
inline V3 operator*(const M3& x, const V3& v) {
  return {x.a[0][0] * v[0] + x.a[0][1] * v[1] + x.a[0][2] * v[2], x.a[1][0] * v[0] + x.a[1][1] * v[1] + x.a[1][2] * v[2],
          x.a[2][0] * v[0] + x.a[2][1] * v[1] + x.a[2][2] * v[2]};
}
inline M3 operator+(const M3& x, const M3& y) { M3 r; for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.a[i][j] = x.a[i][j] + y.a[i][j]; return r; }
inline M3 operator-(const M3& x, const M3& y) { M3 r; for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.a[i][j] = x.a[i][j] - y.a[i][j]; return r; }
inline M3 operator*(double s, const M3& x) { M3 r; for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.a[i][j] = s * x.a[i][j]; return r; }
inline M3 skew(const V3& v) {
  M3 m = M3::zero();
  m.a[0][1] = -v[2]; m.a[0][2] = v[1];
  m.a[1][0] = v[2];  m.a[1][2] = -v[0];
  m.a[2][0] = -v[1]; m.a[2][1] = v[0];
  return m;
}
inline M3 outer(const V3& x, const V3& y) { M3 r; for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.a[i][j] = x[i] * y[j]; return r; }

// Eigen::AngleAxisd::toRotationMatrix expression order.
inline M3 angle_axis(double angle, const V3& axis) {
  M3 res;
  const V3 s = std::sin(angle) * axis;
  const double c = std::cos(angle);
  const V3 k = (1.0 - c) * axis;
  double tmp = k[0] * axis[1];
  res.a[0][1] = tmp - s[2];
  res.a[1][0] = tmp + s[2];
  tmp = k[0] * axis[2];
  res.a[0][2] = tmp + s[1];
  res.a[2][0] = tmp - s[1];
  tmp = k[1] * axis[2];
  res.a[1][2] = tmp - s[0];
  res.a[2][1] = tmp + s[0];
  res.a[0][0] = k[0] * axis[0] + c;
  res.a[1][1] = k[1] * axis[1] + c;
  res.a[2][2] = k[2] * axis[2] + c;
  return res;
}

struct Rigid {
  M3 R;
  V3 t;
  V3 apply(const V3& p) const { return R * p + t; }
  Rigid operator*(const Rigid& o) const { return {R * o.R, R * o.t + t}; }
};

// Dynamic dense matrix, column-major.
struct MatX {
  int rows = 0, cols = 0;
  std::vector<double> d;
  MatX() = default;
  MatX(int r, int c, double v = 0.0) : rows(r), cols(c), d(static_cast<size_t>(r) * c, v) {}
  double& operator()(int r, int c) { return d[static_cast<size_t>(c) * rows + r]; }
  double operator()(int r, int c) const { return d[static_cast<size_t>(c) * rows + r]; }
  bool empty() const { return d.empty(); }
};

using VecX = std::vector<double>;

}  // namespace oracle

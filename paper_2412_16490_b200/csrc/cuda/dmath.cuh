// Device-side fp64 3-vector / 3x3 helpers (sm_100a). Matrices are row-major
// double[9] in registers: m[r*3+c].
#pragma once

#include <cuda_runtime.h>
#include <math.h>

#if defined(__CUDA_ARCH__)
#define GDEV_LDG(p) __ldg(p)
#else
#define GDEV_LDG(p) (*(p))
#endif
#define GDEV_FN __host__ __device__ __forceinline__
#define GDEV_INL __host__ __device__ inline

#include "crmath.cuh"

namespace gdev {

struct D3 {
  double x, y, z;
};

// p ? a : b as one selp.f64. nvcc 12.9's optimiser miscompiles the
// unrolled select chains of the pivoting swaps in fullpiv_solve_t (a swap
// was applied with the pivot already in place; reproduced in isolation on
// sm_100a at every ptxas level), so those selects are opaque to it.
GDEV_FN double psel(bool p, double a, double b) {
#if defined(__CUDA_ARCH__)
  double r;
  asm("{ .reg .pred q; setp.ne.u32 q, %1, 0; selp.f64 %0, %2, %3, q; }" : "=d"(r) : "r"((unsigned)p), "d"(a), "d"(b));
  return r;
#else
  return p ? a : b;
#endif
}

GDEV_FN D3 mk(double x, double y, double z) { return D3{x, y, z}; }
GDEV_FN D3 operator+(D3 a, D3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
GDEV_FN D3 operator-(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
GDEV_FN D3 operator-(D3 a) { return {-a.x, -a.y, -a.z}; }
GDEV_FN D3 operator*(double s, D3 a) { return {s * a.x, s * a.y, s * a.z}; }
GDEV_FN D3 operator*(D3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
GDEV_FN D3 operator/(D3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
GDEV_FN D3& operator+=(D3& a, D3 b) { a.x += b.x; a.y += b.y; a.z += b.z; return a; }
GDEV_FN D3& operator-=(D3& a, D3 b) { a.x -= b.x; a.y -= b.y; a.z -= b.z; return a; }
GDEV_FN double dot(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
GDEV_FN double sqn(D3 a) { return dot(a, a); }
GDEV_FN double nrm(D3 a) { return sqrt(sqn(a)); }
GDEV_FN D3 cross(D3 a, D3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
GDEV_FN D3 normalized(D3 a) {
  const double n2 = sqn(a);
  return n2 > 0 ? a / sqrt(n2) : a;
}
GDEV_FN bool finite3(D3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }
GDEV_FN double comp(D3 a, int k) { return k == 0 ? a.x : (k == 1 ? a.y : a.z); }
GDEV_FN D3 unit(int k) { return {k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0}; }

GDEV_FN D3 ld3(const double* p) { return {p[0], p[1], p[2]}; }
GDEV_FN void st3(double* p, D3 v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; }
GDEV_FN D3 ldg3(const double* __restrict__ p) { return {GDEV_LDG(p), GDEV_LDG(p + 1), GDEV_LDG(p + 2)}; }

// Contact frame p, n, d, e (contact.cpp:9-21); n is the inward normal.
GDEV_FN void build_frame(D3 p, D3 n, double* f) {
  const D3 seed = fabs(n.x) > 0.99 ? mk(0, 1, 0) : mk(1, 0, 0);
  const D3 d = normalized(cross(n, seed));
  const D3 e = cross(n, d);
  st3(f, p);
  st3(f + 3, n);
  st3(f + 6, d);
  st3(f + 9, e);
}

// Row-major 3x3.
struct M33 {
  double m[9];
};
GDEV_FN M33 eye() { return {{1, 0, 0, 0, 1, 0, 0, 0, 1}}; }
GDEV_FN D3 mul(const M33& a, D3 v) {
  return {a.m[0] * v.x + a.m[1] * v.y + a.m[2] * v.z, a.m[3] * v.x + a.m[4] * v.y + a.m[5] * v.z,
          a.m[6] * v.x + a.m[7] * v.y + a.m[8] * v.z};
}
GDEV_FN D3 mulT(const M33& a, D3 v) {  // a^T v
  return {a.m[0] * v.x + a.m[3] * v.y + a.m[6] * v.z, a.m[1] * v.x + a.m[4] * v.y + a.m[7] * v.z,
          a.m[2] * v.x + a.m[5] * v.y + a.m[8] * v.z};
}
GDEV_FN M33 mul(const M33& a, const M33& b) {
  M33 r;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r.m[i * 3 + j] = a.m[i * 3] * b.m[j] + a.m[i * 3 + 1] * b.m[3 + j] + a.m[i * 3 + 2] * b.m[6 + j];
  return r;
}
GDEV_FN M33 transpose(const M33& a) {
  return {{a.m[0], a.m[3], a.m[6], a.m[1], a.m[4], a.m[7], a.m[2], a.m[5], a.m[8]}};
}
GDEV_FN double det(const M33& a) {
  return a.m[0] * (a.m[4] * a.m[8] - a.m[5] * a.m[7]) - a.m[1] * (a.m[3] * a.m[8] - a.m[5] * a.m[6]) +
         a.m[2] * (a.m[3] * a.m[7] - a.m[4] * a.m[6]);
}
GDEV_FN D3 col(const M33& a, int c) { return {a.m[c], a.m[3 + c], a.m[6 + c]}; }
GDEV_FN D3 row(const M33& a, int r) { return {a.m[3 * r], a.m[3 * r + 1], a.m[3 * r + 2]}; }
GDEV_FN void set_col(M33& a, int c, D3 v) { a.m[c] = v.x; a.m[3 + c] = v.y; a.m[6 + c] = v.z; }

// Eigen::AngleAxisd::toRotationMatrix expression order (hand.cpp:144).
// AngleAxis(angle, axis).toRotationMatrix() from a precomputed sin/cos.
GDEV_FN M33 angle_axis_sc(double s, double c, D3 axis) {
  const D3 sa = s * axis;
  const D3 ka = (1.0 - c) * axis;
  M33 r;
  double tmp = ka.x * axis.y;
  r.m[1] = tmp - sa.z;
  r.m[3] = tmp + sa.z;
  tmp = ka.x * axis.z;
  r.m[2] = tmp + sa.y;
  r.m[6] = tmp - sa.y;
  tmp = ka.y * axis.z;
  r.m[5] = tmp - sa.x;
  r.m[7] = tmp + sa.x;
  r.m[0] = ka.x * axis.x + c;
  r.m[4] = ka.y * axis.y + c;
  r.m[8] = ka.z * axis.z + c;
  return r;
}

GDEV_FN M33 angle_axis(double angle, D3 axis) {
  double s, c;
#if defined(__CUDA_ARCH__)
  cr_sincos(angle, &s, &c);  // correctly rounded: matches glibc except near midpoints (crmath.cuh)
#else
  s = ::sin(angle);
  c = ::cos(angle);
#endif
  return angle_axis_sc(s, c, axis);
}

// Nearest proper rotation to a raw 3x3 block (hand.cpp:45-73): polar factor
// from a one-sided Jacobi SVD with the determinant fix on the smallest
// singular direction; column Gram-Schmidt fallback when s2 < 1e-9 s0.
GDEV_INL M33 project_rotation(const M33& raw, bool* fallback) {
  double c[3][3];  // c[col][row]
  double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int i = 0; i < 3; ++i) c[j][i] = raw.m[i * 3 + j];
  for (int sweep = 0; sweep < 20; ++sweep) {
    bool changed = false;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0;
      const int q = pq == 0 ? 1 : 2;
      double al = 0, be = 0, ga = 0;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        al += c[p][i] * c[p][i];
        be += c[q][i] * c[q][i];
        ga += c[p][i] * c[q][i];
      }
      if (ga != 0.0 && fabs(ga) > 1e-15 * sqrt(al * be)) {
        changed = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double xp = c[p][i], xq = c[q][i];
          c[p][i] = cs * xp - sn * xq;
          c[q][i] = sn * xp + cs * xq;
          const double vp = v[p][i], vq = v[q][i];
          v[p][i] = cs * vp - sn * vq;
          v[q][i] = sn * vp + cs * vq;
        }
      }
    }
    if (!changed) break;
  }
  double s[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) s[j] = sqrt(c[j][0] * c[j][0] + c[j][1] * c[j][1] + c[j][2] * c[j][2]);
  // Descending order of singular values (stable for ties).
  int o0 = 0, o1 = 1, o2 = 2;
  if (s[o1] > s[o0]) { int t = o0; o0 = o1; o1 = t; }
  if (s[o2] > s[o1]) { int t = o1; o1 = o2; o2 = t; }
  if (s[o1] > s[o0]) { int t = o0; o0 = o1; o1 = t; }
  const double s0 = s[o0], s2 = s[o2];
  M33 R;
  if (!(s0 > 0) || s2 < 1e-9 * s0) {
    *fallback = true;
    D3 c0 = col(raw, 0);
    if (nrm(c0) < 1e-12) c0 = mk(1, 0, 0);
    c0 = normalized(c0);
    D3 c1 = col(raw, 1) - c0 * dot(c0, col(raw, 1));
    if (nrm(c1) < 1e-12) {
      c1 = mk(0, 1, 0) - c0 * c0.y;
      if (nrm(c1) < 1e-12) c1 = mk(0, 0, 1) - c0 * c0.z;
    }
    c1 = normalized(c1);
    set_col(R, 0, c0);
    set_col(R, 1, c1);
    set_col(R, 2, cross(c0, c1));
    return R;
  }
  *fallback = false;
  // U columns (normalized working columns), V columns, in descending order.
  const int ord[3] = {o0, o1, o2};
  M33 U, V;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int j = ord[k];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      U.m[i * 3 + k] = c[j][i] / s[j];
      V.m[i * 3 + k] = v[j][i];
    }
  }
  const M33 Vt = transpose(V);
  const double sign = det(mul(U, Vt)) < 0 ? -1.0 : 1.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) U.m[i * 3 + 2] *= sign;
  return mul(U, Vt);
}

// make_pose_state tail (hand.cpp:81-93): a_inv = ((tr S) I - S)^-1, S = sym(R^T raw).
GDEV_INL bool pose_a_inv(const M33& R, const M33& raw, M33& a_inv) {
  const M33 sf = mul(transpose(R), raw);
  M33 s;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) s.m[i * 3 + j] = 0.5 * (sf.m[i * 3 + j] + sf.m[j * 3 + i]);
  const double tr = s.m[0] + s.m[4] + s.m[8];
  M33 a;
#pragma unroll
  for (int i = 0; i < 9; ++i) a.m[i] = -s.m[i];
  a.m[0] += tr;
  a.m[4] += tr;
  a.m[8] += tr;
  const double d = det(a);
  if (fabs(d) < 1e-12) return false;
  a_inv.m[0] = (a.m[4] * a.m[8] - a.m[5] * a.m[7]) / d;
  a_inv.m[1] = (a.m[2] * a.m[7] - a.m[1] * a.m[8]) / d;
  a_inv.m[2] = (a.m[1] * a.m[5] - a.m[2] * a.m[4]) / d;
  a_inv.m[3] = (a.m[5] * a.m[6] - a.m[3] * a.m[8]) / d;
  a_inv.m[4] = (a.m[0] * a.m[8] - a.m[2] * a.m[6]) / d;
  a_inv.m[5] = (a.m[2] * a.m[3] - a.m[0] * a.m[5]) / d;
  a_inv.m[6] = (a.m[3] * a.m[7] - a.m[4] * a.m[6]) / d;
  a_inv.m[7] = (a.m[1] * a.m[6] - a.m[0] * a.m[7]) / d;
  a_inv.m[8] = (a.m[0] * a.m[4] - a.m[1] * a.m[3]) / d;
  return true;
}

}  // namespace gdev

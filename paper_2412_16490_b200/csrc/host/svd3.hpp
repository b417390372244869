// 3x3 polar/SVD helper for the host pose utilities: one-sided (Hestenes)
// Jacobi SVD, singular values sorted descending. The reference uses
// Eigen::JacobiSVD (proj/src/hand.cpp:47); the polar factor it feeds is
// unique for the inputs that reach it, so any accurate SVD agrees to rounding.
#pragma once

#include "grasp/la.hpp"

#include <algorithm>
#include <cmath>

namespace grasp {

struct Svd3 {
  Mat3 U, V;
  Vec3 s;  // descending
};

inline Svd3 svd3(const Mat3& a) {
  double c[3][3];  // c[col][row] working columns
  double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};  // v[col][row]
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) c[j][i] = a(i, j);
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (int i = 0; i < 3; ++i) {
          alpha += c[p][i] * c[p][i];
          beta += c[q][i] * c[q][i];
          gamma += c[p][i] * c[q][i];
        }
        if (gamma == 0.0 || std::abs(gamma) <= 1e-15 * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (int i = 0; i < 3; ++i) {
          const double xp = c[p][i], xq = c[q][i];
          c[p][i] = cs * xp - sn * xq;
          c[q][i] = sn * xp + cs * xq;
          const double vp = v[p][i], vq = v[q][i];
          v[p][i] = cs * vp - sn * vq;
          v[q][i] = sn * vp + cs * vq;
        }
      }
    if (!rotated) break;
  }
  double sv[3];
  for (int j = 0; j < 3; ++j) sv[j] = std::sqrt(c[j][0] * c[j][0] + c[j][1] * c[j][1] + c[j][2] * c[j][2]);
  int order[3] = {0, 1, 2};
  std::sort(order, order + 3, [&](int x, int y) { return sv[x] > sv[y]; });
  Svd3 out;
  for (int k = 0; k < 3; ++k) {
    const int j = order[k];
    out.s[k] = sv[j];
    for (int i = 0; i < 3; ++i) {
      out.V(i, k) = v[j][i];
      out.U(i, k) = sv[j] > 0 ? c[j][i] / sv[j] : 0.0;
    }
  }
  // Complete U where singular values vanished (only reachable on fallback inputs).
  if (!(out.s[2] > 0)) {
    const Vec3 u0 = out.U.col(0), u1 = out.U.col(1);
    out.U.set_col(2, normalized(cross(u0, u1)));
  }
  return out;
}

}  // namespace grasp

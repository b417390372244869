// Host-side exactness checks of device math shared with the GPU kernels
// (compiled as host code from the same headers; run by tests/test_device_math_host.py):
//  * closed forms for the 1- and 2-point KKT solves == FullPivLU, bit for bit;
//  * FullPivLU on a zero-padded system == the unpadded one;
//  * correctly rounded sin/cos agrees with glibc on >= 99.5% of arguments.
#include "../../paper_2412_16490_b200/csrc/cuda/gjk.cuh"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

using namespace gdev;

int main() {
  std::mt19937_64 rng(5);
  std::uniform_real_distribution<double> U(-1, 1);
  long bad1 = 0, bad2 = 0, fast2 = 0, badpad = 0;
  for (long t = 0; t < 400000; ++t) {
    D3 p0 = mk(U(rng), U(rng), U(rng)), p1 = mk(U(rng), U(rng), U(rng));
    const double sc = std::ldexp(1.0, -(int)(rng() % 12));
    p0 = sc * p0;
    p1 = sc * p1;
    if (t % 7 == 0) p1 = p0;
    if (t % 11 == 0) p1 = p0 + 1e-9 * mk(1, 0, 0);
    if (t % 13 == 0) p0 = mk(p0.x, p0.y, 0.0), p1 = mk(p1.x, p1.y, 0.0);
    if (t % 17 == 0) p0 = mk(0, 0, 0);
    const double a = dot(p0, p0), b = dot(p0, p1), c = dot(p1, p1);
    {  // 1-point
      double m[2][2] = {{a, 1}, {1, 0}}, rhs[2] = {0, 1}, s[2];
      fullpiv_solve_t<2>(m, rhs, s);
      if (std::fabs(a) < 1.0 && !(s[0] == 1.0 && s[1] == -a)) ++bad1;
    }
    {  // 2-point
      double m[3][3] = {{a, b, 1}, {b, c, 1}, {1, 1, 0}}, rhs[3] = {0, 0, 1}, s1[3], s2[3];
      fullpiv_solve_t<3>(m, rhs, s1);
      if (kkt2_fast(a, b, c, s2)) {
        ++fast2;
        if (std::memcmp(s1, s2, sizeof s1)) ++bad2;
      }
      // zero-padded into 5x5
      double mp[5][5] = {}, rp[5] = {}, sp[5];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) mp[i][j] = (i < 2 && j < 2) ? (i == j ? (i ? c : a) : b) : ((i == 2) != (j == 2) ? 1.0 : 0.0);
      rp[2] = 1.0;
      fullpiv_solve_t<5>(mp, rp, sp, 3);
      if (std::memcmp(s1, sp, sizeof s1) || sp[3] != 0.0 || sp[4] != 0.0) ++badpad;
    }
  }
  // 3- and 4-point KKT systems: fixed-pivot fast path == generic FullPivLU
  long bad34 = 0;
  for (long t = 0; t < 300000; ++t) {
    const int K = 3 + (int)(t & 1);
    D3 P[4];
    const double sc = std::ldexp(1.0, -(int)(rng() % 10));
    for (int i = 0; i < 4; ++i) P[i] = sc * mk(U(rng), U(rng), U(rng));
    if (t % 5 == 0) P[2] = P[0] + 0.5 * (P[1] - P[0]);  // collinear
    if (t % 7 == 0) P[3] = P[0] + 0.3 * (P[1] - P[0]) + 0.2 * (P[2] - P[0]);  // coplanar
    if (t % 9 == 0) P[1] = P[0];
    if (t % 11 == 0) for (int i = 0; i < 4; ++i) P[i] = mk(P[i].x, P[i].y, 0.0);
    double g[4][4];
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) g[i][j] = dot(P[i], P[j]);
    if (K == 3) {
      double m1[4][4], m2[4][4], r[4] = {0, 0, 0, 1}, s1[4], s2[4];
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) m1[i][j] = (i < 3 && j < 3) ? g[i][j] : ((i == 3) != (j == 3) ? 1.0 : 0.0);
      std::memcpy(m2, m1, sizeof m1);
      fullpiv_solve_t<4>(m1, r, s1);
      fullpiv_solve_t<4, true>(m2, r, s2);
      if (std::memcmp(s1, s2, sizeof s1)) ++bad34;
    } else {
      double m1[5][5], m2[5][5], r[5] = {0, 0, 0, 0, 1}, s1[5], s2[5];
      for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) m1[i][j] = (i < 4 && j < 4) ? g[i][j] : ((i == 4) != (j == 4) ? 1.0 : 0.0);
      std::memcpy(m2, m1, sizeof m1);
      fullpiv_solve_t<5>(m1, r, s1);
      fullpiv_solve_t<5, true>(m2, r, s2);
      if (std::memcmp(s1, s2, sizeof s1)) ++bad34;
    }
  }
  std::printf("bad34 %ld\n", bad34);
  if (bad34) return 1;
  long cr_bad = 0, n_cr = 2000000;
  std::uniform_real_distribution<double> A(-4.0, 4.0);
  for (long i = 0; i < n_cr; ++i) {
    const double x = A(rng);
    double s, co;
    cr_sincos(x, &s, &co);
    cr_bad += (s != std::sin(x)) + (co != std::cos(x));
  }
  std::printf("bad1 %ld fast2 %ld bad2 %ld badpad %ld cr_mismatch %ld of %ld\n", bad1, fast2, bad2, badpad, cr_bad,
              2 * n_cr);
  const bool ok = bad1 == 0 && bad2 == 0 && badpad == 0 && fast2 > 300000 && cr_bad < 0.005 * 2 * n_cr;
  return ok ? 0 : 1;
}

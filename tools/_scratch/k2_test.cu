#include "../../paper_2412_16490_b200/csrc/cuda/gjk.cuh"
#include <cstdio>
#include <random>
#include <cstring>
using namespace gdev;
int main() {
  std::mt19937_64 rng(5); std::uniform_real_distribution<double> U(-1, 1);
  long bad = 0, fast = 0, n = 3000000;
  for (long t = 0; t < n; ++t) {
    D3 p0 = mk(U(rng), U(rng), U(rng)), p1 = mk(U(rng), U(rng), U(rng));
    double sc = std::ldexp(1.0, -(int)(rng() % 12));
    p0 = sc * p0; p1 = sc * p1;
    if (t % 7 == 0) p1 = p0;                      // duplicate point
    if (t % 11 == 0) p1 = p0 + 1e-9 * mk(1, 0, 0); // near duplicate
    if (t % 13 == 0) p1 = mk(p0.x, p0.y, 0.0), p0 = mk(p0.x, p0.y, 0.0); // zeros
    if (t % 17 == 0) p0 = mk(0, 0, 0);
    double a = dot(p0, p0), b = dot(p0, p1), c = dot(p1, p1);
    double m[3][3] = {{a, b, 1}, {b, c, 1}, {1, 1, 0}}, rhs[3] = {0, 0, 1}, s1[3], s2[3];
    fullpiv_solve_t<3>(m, rhs, s1);
    if (kkt2_fast(a, b, c, s2)) {
      ++fast;
      if (memcmp(s1, s2, sizeof s1)) { if (bad < 5) printf("t %ld a %.17g b %.17g c %.17g lu %.17g %.17g %.17g fast %.17g %.17g %.17g\n", t, a, b, c, s1[0], s1[1], s1[2], s2[0], s2[1], s2[2]); ++bad; }
    }
  }
  printf("n %ld fast %ld bad %ld\n", n, fast, bad);
}

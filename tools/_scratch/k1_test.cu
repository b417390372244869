#include "../../paper_2412_16490_b200/csrc/cuda/gjk.cuh"
#include <cstdio>
#include <random>
using namespace gdev;
int main() {
  std::mt19937_64 rng(3); std::uniform_real_distribution<double> U(-0.9, 0.9);
  long bad = 0;
  for (int t = 0; t < 1000000; ++t) {
    double g = U(rng) * U(rng); if (t % 3 == 0) g = std::fabs(g);
    double m[2][2] = {{g, 1}, {1, 0}}, rhs[2] = {0, 1}, sol[2];
    fullpiv_solve_t<2>(m, rhs, sol);
    if (sol[0] != 1.0 || sol[1] != -g) { if (bad < 3) printf("g %.17g sol %.17g %.17g\n", g, sol[0], sol[1]); ++bad; }
  }
  printf("bad %ld\n", bad);
}

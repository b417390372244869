#include "../../paper_2412_16490_b200/csrc/cuda/dmath.cuh"
#include <cstdio>
#include <random>
#include <cmath>
int main() {
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(-4.0, 4.0);
  long bad_s = 0, bad_c = 0, n = 20000000;
  for (long i = 0; i < n; ++i) {
    double x = U(rng);
    if (i % 4 == 1) x = std::ldexp(x, -(int)(rng() % 40));
    if (i % 4 == 2) x = (double)(rng() % 5) * 1.5707963267948966 + std::ldexp(U(rng), -(int)(rng() % 30));
    double s, c;
    gdev::cr_sincos(x, &s, &c);
    if (s != std::sin(x)) { if (bad_s < 5) printf("sin x=%.17g cr=%.17g glibc=%.17g\n", x, s, std::sin(x)); ++bad_s; }
    if (c != std::cos(x)) { if (bad_c < 5) printf("cos x=%.17g cr=%.17g glibc=%.17g\n", x, c, std::cos(x)); ++bad_c; }
  }
  printf("n %ld sin mismatches %ld cos mismatches %ld\n", n, bad_s, bad_c);
}

#include "../../paper_2412_16490_b200/csrc/cuda/gjk.cuh"
#include <cstdio>
#include <random>
#include <cstring>
using namespace gdev;
namespace gdev {
#include "old_lu.inc"
}
template <int S> int run(std::mt19937_64& rng) {
  std::uniform_real_distribution<double> U(-1, 1);
  int bad = 0;
  for (int t = 0; t < 200000; ++t) {
    double m[S][S], m2[S][S], rhs[S], a[S], b[S];
    int mode = t % 4;
    for (int i = 0; i < S; ++i) for (int j = 0; j < S; ++j) m[i][j] = U(rng);
    if (mode == 1) for (int j = 0; j < S; ++j) m[S-1][j] = m[0][j];        // singular
    if (mode == 2) for (int j = 0; j < S; ++j) m[j][S-1] = 0;            // zero column
    if (mode == 3) { for (int i = 0; i < S; ++i) { m[i][S-1] = 1; m[S-1][i] = 1; } m[S-1][S-1] = 0; for (int i=0;i<S-1;++i) rhs[i]=0; }
    for (int i = 0; i < S; ++i) rhs[i] = (mode == 3) ? (i == S-1) : U(rng);
    memcpy(m2, m, sizeof m);
    old_solve_t<S>(m, rhs, a);
    fullpiv_solve_t<S>(m2, rhs, b);
    if (memcmp(a, b, sizeof a)) { if (bad < 3) { printf("S=%d mode %d mismatch:", S, mode); for (int i=0;i<S;++i) printf(" %g/%g", a[i], b[i]); printf("\n"); } ++bad; }
  }
  return bad;
}
int main() { std::mt19937_64 r(1); int b = run<2>(r) + run<3>(r) + run<4>(r) + run<5>(r); printf("bad %d\n", b); }

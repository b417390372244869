#include "../../paper_2412_16490_b200/csrc/cuda/gjk.cuh"
#include <cstdio>
using namespace gdev;
namespace gdev {
#include "old_lu.inc"
}
__host__ __device__ void go() {
  double m[3][3] = {{0.1, 0.9, 0.3}, {0.5, 0.2, -0.7}, {0.4, 0.6, 0.8}}, m2[3][3], rhs[3] = {1, 2, 3}, a[3], b[3];
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) m2[i][j] = m[i][j];
  old_solve_t<3>(m, rhs, a);
  fullpiv_solve_t<3>(m2, rhs, b);
  printf("old %.17g %.17g %.17g\nnew %.17g %.17g %.17g\n", a[0], a[1], a[2], b[0], b[1], b[2]);
}
__global__ void k() { go(); }
int main() { printf("host\n"); go(); printf("dev\n"); k<<<1,1>>>(); cudaDeviceSynchronize(); }

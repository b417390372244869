#include "../../paper_2412_16490_b200/csrc/cuda/dmath.cuh"
#include <cstdio>
#include <random>
#include <vector>
#include <cmath>
__global__ void k(const double* x, double* s1, double* c1, double* s2, double* c2, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
  sincos(x[i], s1 + i, c1 + i);
  gdev::cr_sincos(x[i], s2 + i, c2 + i);
}
int main() {
  const int n = 4000000; std::mt19937_64 rng(2); std::uniform_real_distribution<double> U(-3.2, 3.2);
  std::vector<double> x(n), s1(n), c1(n), s2(n), c2(n);
  for (auto& v : x) v = U(rng);
  double *dx, *a, *b, *c, *d; cudaMalloc(&dx, n*8); cudaMalloc(&a, n*8); cudaMalloc(&b, n*8); cudaMalloc(&c, n*8); cudaMalloc(&d, n*8);
  cudaMemcpy(dx, x.data(), n*8, cudaMemcpyHostToDevice);
  k<<<(n+255)/256, 256>>>(dx, a, b, c, d, n);
  cudaMemcpy(s1.data(), a, n*8, cudaMemcpyDeviceToHost); cudaMemcpy(c1.data(), b, n*8, cudaMemcpyDeviceToHost);
  cudaMemcpy(s2.data(), c, n*8, cudaMemcpyDeviceToHost); cudaMemcpy(c2.data(), d, n*8, cudaMemcpyDeviceToHost);
  long m1 = 0, m2 = 0, m3 = 0;
  for (int i = 0; i < n; ++i) {
    double gs = std::sin(x[i]), gc = std::cos(x[i]); double hs, hc; gdev::cr_sincos(x[i], &hs, &hc);
    m1 += (s1[i] != gs) + (c1[i] != gc); m2 += (s2[i] != gs) + (c2[i] != gc); m3 += (s2[i] != hs) + (c2[i] != hc);
  }
  printf("calls %d: cuda sincos vs glibc %ld, device cr vs glibc %ld, device cr vs host cr %ld\n", 2*n, m1, m2, m3);
}

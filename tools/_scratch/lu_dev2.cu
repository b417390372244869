#include "../../paper_2412_16490_b200/csrc/cuda/gjk.cuh"
#include <cstdio>
#include <random>
#include <vector>
using namespace gdev;
namespace gdev {
#include "old_lu.inc"
}
template <int S> __global__ void k(const double* M, const double* R, double* A, double* B, int n) {
  int t = blockIdx.x * blockDim.x + threadIdx.x; if (t >= n) return;
  double m[S][S], m2[S][S], rhs[S], a[S], b[S];
  for (int i = 0; i < S; ++i) { rhs[i] = R[t*S+i]; for (int j = 0; j < S; ++j) m[i][j] = m2[i][j] = M[(t*S+i)*S+j]; }
  old_solve_t<S>(m, rhs, a); fullpiv_solve_t<S>(m2, rhs, b);
  for (int i = 0; i < S; ++i) { A[t*S+i] = a[i]; B[t*S+i] = b[i]; }
}
template <int S> void run() {
  const int n = 100000; std::mt19937_64 rng(S); std::uniform_real_distribution<double> U(-1, 1);
  std::vector<double> M(n*S*S), R(n*S), A(n*S), B(n*S), H(n*S);
  for (int t = 0; t < n; ++t) { int mode = t % 2;
    for (int i = 0; i < S; ++i) for (int j = 0; j < S; ++j) M[(t*S+i)*S+j] = U(rng);
    for (int i = 0; i < S; ++i) R[t*S+i] = U(rng);
    if (mode) { for (int i = 0; i < S; ++i) { M[(t*S+i)*S+S-1] = 1; M[(t*S+S-1)*S+i] = 1; R[t*S+i] = i == S-1; } M[(t*S+S-1)*S+S-1] = 0; } }
  double *dM, *dR, *dA, *dB; cudaMalloc(&dM, M.size()*8); cudaMalloc(&dR, R.size()*8); cudaMalloc(&dA, A.size()*8); cudaMalloc(&dB, B.size()*8);
  cudaMemcpy(dM, M.data(), M.size()*8, cudaMemcpyHostToDevice); cudaMemcpy(dR, R.data(), R.size()*8, cudaMemcpyHostToDevice);
  k<S><<<(n+127)/128, 128>>>(dM, dR, dA, dB, n);
  cudaMemcpy(A.data(), dA, A.size()*8, cudaMemcpyDeviceToHost); cudaMemcpy(B.data(), dB, B.size()*8, cudaMemcpyDeviceToHost);
  for (int t = 0; t < n; ++t) { double m[S][S], rhs[S], h[S]; for (int i = 0; i < S; ++i) { rhs[i] = R[t*S+i]; for (int j = 0; j < S; ++j) m[i][j] = M[(t*S+i)*S+j]; } old_solve_t<S>(m, rhs, h); for (int i = 0; i < S; ++i) H[t*S+i] = h[i]; }
  int ba = 0, bb = 0; for (size_t i = 0; i < A.size(); ++i) { ba += A[i] != H[i]; bb += B[i] != H[i];
    if (B[i] != H[i] && bb <= 2) { size_t t = i / S; printf("t=%zu comp %zu: dev-new %.17g host %.17g dev-old %.17g\n", t, i % S, B[i], H[i], A[i]);
      for (int r = 0; r < S; ++r) { for (int c = 0; c < S; ++c) printf(" %.17g", M[(t*S+r)*S+c]); printf(" | %.17g\n", R[t*S+r]); } } }
  printf("S=%d dev-old vs host mismatches %d, dev-new vs host %d (%s)\n", S, ba, bb, cudaGetErrorString(cudaGetLastError()));
}
int main() { run<2>(); run<3>(); run<4>(); run<5>(); }

#include "../../paper_2412_16490_b200/csrc/cuda/gjk.cuh"
#include <cstdio>
using namespace gdev;
namespace gdev {
template <int S>
GDEV_FN void dbg_solve_t(double (&m)[S][S], const double (&rhs)[S], double (&sol)[S]) {
  int rowt[S], colt[S];
  int nonzero = S;
  double maxpivot = 0.0;
  bool stopped = false;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    rowt[k] = k;
    colt[k] = k;
    if (stopped) continue;
    double biggest = -1.0;
    int br = k, bc = k;
#pragma unroll
    for (int c = k; c < S; ++c)
#pragma unroll
      for (int r = k; r < S; ++r) {
        const double v = fabs(m[r][c]);
        if (v > biggest) {
          biggest = v;
          br = r;
          bc = c;
        }
      }
    if (biggest == 0.0) {
      nonzero = k;
      stopped = true;
      continue;
    }
    printf("k=%d br=%d bc=%d biggest=%.17g\n", k, br, bc, biggest);
    maxpivot = fmax(maxpivot, biggest);
    rowt[k] = br;
    colt[k] = bc;
    // Row and column swaps as select chains: the pivot position differs
    // from lane to lane, and branches here would serialise the warp.
#pragma unroll
    for (int c = 0; c < S; ++c) {
      const double old = m[k][c];
      double pick = old;
#pragma unroll
      for (int r = k + 1; r < S; ++r) pick = (br == r) ? m[r][c] : pick;
#pragma unroll
      for (int r = k + 1; r < S; ++r) m[r][c] = (br == r) ? old : m[r][c];
      m[k][c] = pick;
    }
#pragma unroll
    for (int r = 0; r < S; ++r) {
      const double old = m[r][k];
      double pick = old;
#pragma unroll
      for (int c = k + 1; c < S; ++c) pick = (bc == c) ? m[r][c] : pick;
#pragma unroll
      for (int c = k + 1; c < S; ++c) m[r][c] = (bc == c) ? old : m[r][c];
      m[r][k] = pick;
    }
    for (int r = 0; r < S; ++r) printf("  after swap row %d: %.17g %.17g %.17g\n", r, m[r][0], m[r][1], m[r][2]);
    if (k < S - 1) {
      const double piv = m[k][k];
#pragma unroll
      for (int r = k + 1; r < S; ++r) m[r][k] /= piv;
#pragma unroll
      for (int c = k + 1; c < S; ++c) {
        const double mkc = m[k][c];
#pragma unroll
        for (int r = k + 1; r < S; ++r) m[r][c] -= m[r][k] * mkc;
      }
    }
  }
  const double thresh = maxpivot * (S * 2.220446049250313e-16);
  int rank = 0;
#pragma unroll
  for (int i = 0; i < S; ++i) rank += (i < nonzero && fabs(m[i][i]) > thresh) ? 1 : 0;
  if (rank == 0) {
#pragma unroll
    for (int i = 0; i < S; ++i) sol[i] = 0.0;
    return;
  }
  double c[S];
#pragma unroll
  for (int i = 0; i < S; ++i) c[i] = rhs[i];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const double old = c[k];
    double pick = old;
#pragma unroll
    for (int r = k + 1; r < S; ++r) pick = (rowt[k] == r) ? c[r] : pick;
#pragma unroll
    for (int r = k + 1; r < S; ++r) c[r] = (rowt[k] == r) ? old : c[r];
    c[k] = pick;
  }
  // Substitutions with the reference's zero skips as selects (same
  // operations on the taken path, no lane-dependent branches).
#pragma unroll
  for (int i = 0; i < S; ++i) {
    const bool nz = c[i] != 0.0;
#pragma unroll
    for (int r = i + 1; r < S; ++r) c[r] = nz ? c[r] - c[i] * m[r][i] : c[r];
  }
#pragma unroll
  for (int i = S - 1; i >= 0; --i) {
    const bool act = i < rank && c[i] != 0.0;
    const double ci = c[i] / (act ? m[i][i] : 1.0);
    c[i] = act ? ci : c[i];
#pragma unroll
    for (int r = 0; r < i; ++r) c[r] = act ? c[r] - ci * m[r][i] : c[r];
  }
  int perm[S];
#pragma unroll
  for (int i = 0; i < S; ++i) perm[i] = i;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int old = perm[k];
    int pick = old;
#pragma unroll
    for (int r = k + 1; r < S; ++r) pick = (colt[k] == r) ? perm[r] : pick;
#pragma unroll
    for (int r = k + 1; r < S; ++r) perm[r] = (colt[k] == r) ? old : perm[r];
    perm[k] = pick;
  }
#pragma unroll
  for (int j = 0; j < S; ++j) sol[j] = 0.0;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    const double v = i < rank ? c[i] : 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j) sol[j] = (perm[i] == j) ? v : sol[j];
  }
}
template <int S>
GDEV_FN void odbg_solve_t(double (&m)[S][S], const double (&rhs)[S], double (&sol)[S]) {
  int rowt[S], colt[S];
  int nonzero = S;
  double maxpivot = 0.0;
  bool stopped = false;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    rowt[k] = k;
    colt[k] = k;
    if (stopped) continue;
    double biggest = -1.0;
    int br = k, bc = k;
#pragma unroll
    for (int c = k; c < S; ++c)
#pragma unroll
      for (int r = k; r < S; ++r) {
        const double v = fabs(m[r][c]);
        if (v > biggest) {
          biggest = v;
          br = r;
          bc = c;
        }
      }
    if (biggest == 0.0) {
      nonzero = k;
      stopped = true;
      continue;
    }
    printf("k=%d br=%d bc=%d biggest=%.17g\n", k, br, bc, biggest);
    maxpivot = fmax(maxpivot, biggest);
    rowt[k] = br;
    colt[k] = bc;
#pragma unroll
    for (int r = k + 1; r < S; ++r)
      if (r == br)
#pragma unroll
        for (int c = 0; c < S; ++c) {
          const double t = m[k][c];
          m[k][c] = m[r][c];
          m[r][c] = t;
        }
#pragma unroll
    for (int c = k + 1; c < S; ++c)
      if (c == bc)
#pragma unroll
        for (int r = 0; r < S; ++r) {
          const double t = m[r][k];
          m[r][k] = m[r][c];
          m[r][c] = t;
        }
    for (int r = 0; r < S; ++r) printf("  after swap row %d: %.17g %.17g %.17g\n", r, m[r][0], m[r][1], m[r][2]);
    if (k < S - 1) {
      const double piv = m[k][k];
#pragma unroll
      for (int r = k + 1; r < S; ++r) m[r][k] /= piv;
#pragma unroll
      for (int c = k + 1; c < S; ++c) {
        const double mkc = m[k][c];
#pragma unroll
        for (int r = k + 1; r < S; ++r) m[r][c] -= m[r][k] * mkc;
      }
    }
  }
  const double thresh = maxpivot * (S * 2.220446049250313e-16);
  int rank = 0;
#pragma unroll
  for (int i = 0; i < S; ++i) rank += (i < nonzero && fabs(m[i][i]) > thresh) ? 1 : 0;
  if (rank == 0) {
#pragma unroll
    for (int i = 0; i < S; ++i) sol[i] = 0.0;
    return;
  }
  double c[S];
#pragma unroll
  for (int i = 0; i < S; ++i) c[i] = rhs[i];
#pragma unroll
  for (int k = 0; k < S; ++k)
#pragma unroll
    for (int r = k + 1; r < S; ++r)
      if (r == rowt[k]) {
        const double t = c[k];
        c[k] = c[r];
        c[r] = t;
      }
#pragma unroll
  for (int i = 0; i < S; ++i)
    if (c[i] != 0.0)
#pragma unroll
      for (int r = i + 1; r < S; ++r) c[r] -= c[i] * m[r][i];
#pragma unroll
  for (int i = S - 1; i >= 0; --i)
    if (i < rank && c[i] != 0.0) {
      c[i] /= m[i][i];
#pragma unroll
      for (int r = 0; r < i; ++r) c[r] -= c[i] * m[r][i];
    }
  int perm[S];
#pragma unroll
  for (int i = 0; i < S; ++i) perm[i] = i;
#pragma unroll
  for (int k = 0; k < S; ++k)
#pragma unroll
    for (int r = k + 1; r < S; ++r)
      if (r == colt[k]) {
        const int t = perm[k];
        perm[k] = perm[r];
        perm[r] = t;
      }
#pragma unroll
  for (int i = 0; i < S; ++i) {
    const double v = i < rank ? c[i] : 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j)
      if (perm[i] == j) sol[j] = v;
  }
}

}
__global__ void k(const double* M, const double* R) {
  double m[3][3], m2[3][3], rhs[3], a[3], b[3];
  for (int i = 0; i < 3; ++i) { rhs[i] = R[i]; for (int j = 0; j < 3; ++j) m[i][j] = m2[i][j] = M[i*3+j]; }
  printf("OLD\n"); odbg_solve_t<3>(m, rhs, a);
  printf("NEW\n"); dbg_solve_t<3>(m2, rhs, b);
  printf("old %.17g %.17g %.17g\nnew %.17g %.17g %.17g\n", a[0], a[1], a[2], b[0], b[1], b[2]);
}
int main() {
  double M[9] = {0.56651354581996727, 0.97764572163279695, -0.33470568961427127, 0.72734123884778756, -0.80450475511964836, 0.82277867425154305, -0.089859057079953786, -0.79881247174485059, -0.18252776157156536};
  double R[3] = {0.0056711498452954867, -0.080426327843320267, -0.13618048224131574};
  double *dM, *dR; cudaMalloc(&dM, 72); cudaMalloc(&dR, 24); cudaMemcpy(dM, M, 72, cudaMemcpyHostToDevice); cudaMemcpy(dR, R, 24, cudaMemcpyHostToDevice);
  k<<<1,1>>>(dM, dR); cudaDeviceSynchronize();
}

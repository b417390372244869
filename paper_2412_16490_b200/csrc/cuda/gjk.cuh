// Device GJK / EPA signed distance between a posed hand-link hull and an
// object part (reference proj/src/geometry.cpp:17-324, 399-412, 500-525).
// One thread owns one pair; warps are laid out so their 32 threads share the
// same (link, part) and differ in grasp, so vertex loads in the support scans
// are warp-uniform (broadcast) loads. The EPA polytope lives in a fixed
// per-thread buffer; dead faces are compacted in order, which keeps the
// reference's face iteration order (and thus its tie-breaks) unchanged.
#pragma once

#include "dmath.cuh"
#include "model.cuh"

namespace gdev {

constexpr double kTouchTol = 1e-10;   // geometry.cpp:12
constexpr double kGjkRelTol = 1e-14;  // geometry.cpp:13
constexpr int kGjkMaxIters = 128;     // geometry.cpp:14
constexpr int kEpaMaxIters = 512;     // geometry.cpp:15

// Pair status bits written next to each result.
constexpr int kPairEpa = 1;
constexpr int kPairOverflow = 2;
constexpr int kPairDegenerate = 4;
constexpr int kPairCulled = 8;  // provably separated, GJK skipped (d stored as +inf)

struct Hull {
  const double* __restrict__ verts;  // nv*3
  int nv;
  bool posed;  // false: identity pose (object frame)
  M33 R;       // row-major
  D3 t;
  const int* cm_off = nullptr;             // support map of this hull (kSupportCells + 1 offsets), or none
  const unsigned short* cm_idx = nullptr;  // candidate lists (model.cuh)
};

// A Minkowski-difference point w = a - b with its support vertices as a key
// (ia | ib << 16). The points a and b themselves are rebuilt from the key
// (hull_point, the same operations support() used), so simplices, EPA
// polytopes and EPA job records carry 4 bytes instead of 48 per point.
struct SP {
  D3 w;
  unsigned key;
};

GDEV_FN D3 support(const Hull& h, D3 dir, int& arg_out) {
  const D3 dl = h.posed ? mulT(h.R, dir) : dir;
  double best = -INFINITY;
  int arg = 0;
  const double* __restrict__ V = h.verts;
  const int cell = h.cm_off ? support_cell(dl.x, dl.y, dl.z) : -1;
  if (cell >= 0) {
    // Candidates of the direction's cell, ascending: every vertex that can be
    // the computed maximum is listed, so the first maximum is the full scan's.
    const int k1 = GDEV_LDG(h.cm_off + cell + 1);
    for (int k = GDEV_LDG(h.cm_off + cell); k < k1; ++k) {
      const int i = GDEV_LDG(h.cm_idx + k);
      const double s = dl.x * GDEV_LDG(V + 3 * i) + dl.y * GDEV_LDG(V + 3 * i + 1) + dl.z * GDEV_LDG(V + 3 * i + 2);
      if (s > best) {
        best = s;
        arg = i;
      }
    }
    const D3 v = ldg3(h.verts + 3 * arg);
    arg_out = arg;
    return h.posed ? mul(h.R, v) + h.t : v;
  }
  int i = 0;
  // Four independent dot products per step for ILP; the compares stay in
  // index order, so the first maximum still wins (geometry.cpp:404-409).
  for (; i + 4 <= h.nv; i += 4) {
    const double s0 = dl.x * GDEV_LDG(V + 3 * i) + dl.y * GDEV_LDG(V + 3 * i + 1) + dl.z * GDEV_LDG(V + 3 * i + 2);
    const double s1 = dl.x * GDEV_LDG(V + 3 * i + 3) + dl.y * GDEV_LDG(V + 3 * i + 4) + dl.z * GDEV_LDG(V + 3 * i + 5);
    const double s2 = dl.x * GDEV_LDG(V + 3 * i + 6) + dl.y * GDEV_LDG(V + 3 * i + 7) + dl.z * GDEV_LDG(V + 3 * i + 8);
    const double s3 = dl.x * GDEV_LDG(V + 3 * i + 9) + dl.y * GDEV_LDG(V + 3 * i + 10) + dl.z * GDEV_LDG(V + 3 * i + 11);
    if (s0 > best) { best = s0; arg = i; }
    if (s1 > best) { best = s1; arg = i + 1; }
    if (s2 > best) { best = s2; arg = i + 2; }
    if (s3 > best) { best = s3; arg = i + 3; }
  }
  for (; i < h.nv; ++i) {
    const double s = dl.x * GDEV_LDG(V + 3 * i) + dl.y * GDEV_LDG(V + 3 * i + 1) + dl.z * GDEV_LDG(V + 3 * i + 2);
    if (s > best) {
      best = s;
      arg = i;
    }
  }
  const D3 v = ldg3(h.verts + 3 * arg);
  arg_out = arg;
  return h.posed ? mul(h.R, v) + h.t : v;
}

// Vertex i of a hull in the world frame, exactly as support() returns it.
GDEV_FN D3 hull_point(const Hull& h, int i) {
  const D3 v = ldg3(h.verts + 3 * i);
  return h.posed ? mul(h.R, v) + h.t : v;
}
GDEV_FN D3 sp_a(const Hull& A, const SP& p) { return hull_point(A, (int)(p.key & 0xffffu)); }
GDEV_FN D3 sp_b(const Hull& B, const SP& p) { return hull_point(B, (int)(p.key >> 16)); }

GDEV_FN SP support_pair(const Hull& A, const Hull& B, D3 dir) {
  SP s;
  int ia, ib;
  const D3 a = support(A, dir, ia);
  const D3 b = support(B, -dir, ib);
  s.w = a - b;
  s.key = (unsigned)ia | ((unsigned)ib << 16);
  return s;
}

// Exact cycle detection for GJK (Brent). The loop state at the top of an
// iteration is the ordered simplex, and every simplex point is a function
// of its support-vertex pair, so the state is fully described by the keys
// of its points. Once the state at iteration i equals the one at i - p, the
// run is periodic, and the state at the iteration cap (geometry.cpp:111,
// 136-149) is the current one after jumping a multiple of p: the output is
// unchanged, bit for bit, and the cycling iterations are not executed.
// (Pairs of hulls with >= 65535 vertices run without detection.)
struct GjkCycle {
  unsigned long long s0, s1;
  int power, lam;
  bool on;
};

GDEV_FN void cycle_init(GjkCycle& c, int nva, int nvb) {
  c.s0 = c.s1 = ~0ull;
  c.power = 1;
  c.lam = 0;
  c.on = nva < 65535 && nvb < 65535;
}

// Returns the number of iterations to jump (0 when no cycle was closed).
GDEV_FN int cycle_step(GjkCycle& c, const SP (&simp)[4], int ns, int iter) {
  if (!c.on) return 0;
  unsigned k[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) k[i] = i < ns ? simp[i].key : ~0u;
  const unsigned long long a = (unsigned long long)k[0] | ((unsigned long long)k[1] << 32);
  const unsigned long long b = (unsigned long long)k[2] | ((unsigned long long)k[3] << 32);
  if (a == c.s0 && b == c.s1) {
    c.on = false;
    return ((kGjkMaxIters - iter) / c.lam) * c.lam;
  }
  if (c.lam == c.power) {
    c.s0 = a;
    c.s1 = b;
    c.power <<= 1;
    c.lam = 0;
  }
  ++c.lam;
  return 0;
}

// Eigen::FullPivLU::solve restated for a compile-time size S (complete
// pivoting on the largest |entry|, first in column-major order on ties;
// rank = #{|u_ii| > max_pivot * S * eps}; unit-lower then upper substitution
// on the rank block; free unknowns 0). Every index is compile-time or a
// predicated select, so the matrix stays in registers.
//
// Zero padding is exact: a system of size s_real < S embedded in the top-left
// corner with zeros elsewhere gets the same pivots (padded entries are 0 and
// never beat a nonzero one; the column-major scan keeps the real entries'
// order), the same eliminations (padded entries stay +0), stops at the same
// step, and the rank threshold uses s_real. So one body of size S serves all
// smaller systems (instruction-cache footprint).
//
// KKT = true: m is a subset KKT matrix [[G, 1], [1^T, 0]]. When every |G_r0|
// < 1 and every other |G_rc| <= 1, the first pivot is the 1 at (S-1, 0) (the
// first entry of largest magnitude in column-major order); after that
// elimination the step-1 block's last column is exactly 1, so when its other
// columns are all below 1 in magnitude the second pivot is the 1 at
// (1, S-1). On that path the two searches and the select-chain swaps are
// replaced by the known fixed swaps; every arithmetic operation is the same.
template <int S, bool KKT = false>
GDEV_FN void fullpiv_solve_t(double (&m)[S][S], const double (&rhs)[S], double (&sol)[S], int s_real = S) {
  int rowt[S], colt[S];
  int nonzero = S;
  double maxpivot = 0.0;
  bool stopped = false;
  bool fast = false;
  if constexpr (KKT) {
    fast = true;
#pragma unroll
    for (int r = 0; r < S - 1; ++r) {
      fast = fast && fabs(m[r][0]) < 1.0;
#pragma unroll
      for (int c = 1; c < S - 1; ++c) fast = fast && fabs(m[r][c]) <= 1.0;
    }
  }
#pragma unroll
  for (int k = 0; k < S; ++k) {
    rowt[k] = k;
    colt[k] = k;
    if (stopped) continue;
    if constexpr (KKT) {
      if (k == 1 && fast) {
#pragma unroll
        for (int r = 1; r < S; ++r)
#pragma unroll
          for (int c = 1; c < S - 1; ++c) fast = fast && fabs(m[r][c]) < 1.0;
      }
      if (k < 2 && fast) {
        maxpivot = fmax(maxpivot, 1.0);
        if (k == 0) {
          rowt[0] = S - 1;
#pragma unroll
          for (int c = 0; c < S; ++c) {
            const double t = m[0][c];
            m[0][c] = m[S - 1][c];
            m[S - 1][c] = t;
          }
        } else {
          colt[1] = S - 1;
#pragma unroll
          for (int r = 0; r < S; ++r) {
            const double t = m[r][1];
            m[r][1] = m[r][S - 1];
            m[r][S - 1] = t;
          }
        }
        // The pivot is exactly 1 (the KKT ones; see above), and x / 1 = x
        // exactly, so the column scaling is the identity and is skipped. At
        // k = 0 the pivot row is the ones row (1, ..., 1, 0): m[r][0] * 1 is
        // exact, and the last column (all 1) minus m[r][0] * 0 stays 1, so
        // only the subtractions remain.
        if (k == 0) {
#pragma unroll
          for (int c = 1; c < S - 1; ++c)
#pragma unroll
            for (int r = 1; r < S; ++r) m[r][c] -= m[r][0];
        } else {
#pragma unroll
          for (int c = k + 1; c < S; ++c) {
            const double mkc = m[k][c];
#pragma unroll
            for (int r = k + 1; r < S; ++r) m[r][c] -= m[r][k] * mkc;
          }
        }
        continue;
      }
    }
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
      for (int r = k + 1; r < S; ++r) pick = psel(br == r, m[r][c], pick);
#pragma unroll
      for (int r = k + 1; r < S; ++r) m[r][c] = psel(br == r, old, m[r][c]);
      m[k][c] = pick;
    }
#pragma unroll
    for (int r = 0; r < S; ++r) {
      const double old = m[r][k];
      double pick = old;
#pragma unroll
      for (int c = k + 1; c < S; ++c) pick = psel(bc == c, m[r][c], pick);
#pragma unroll
      for (int c = k + 1; c < S; ++c) m[r][c] = psel(bc == c, old, m[r][c]);
      m[r][k] = pick;
    }
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
  const double thresh = maxpivot * (s_real * 2.220446049250313e-16);
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
  bool permute = true;
  if constexpr (KKT) {
    // rhs = e_{S-1} and the fast path's row transpositions are (0, S-1), none,
    // then swaps among rows >= 2 (zeros): the permuted rhs is e_0 exactly
    if (fast) {
#pragma unroll
      for (int i = 0; i < S; ++i) c[i] = i == 0 ? 1.0 : 0.0;
      permute = false;
    }
  }
  if (permute) {
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
    // u_00 = u_11 = 1 exactly on the KKT fast path (columns 0 and 1 are never
    // swapped again), so those divisions are identities
    double ci = c[i];
    if (!(KKT && i < 2 && fast)) ci = c[i] / (act ? m[i][i] : 1.0);
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
  bool general = true;
  if constexpr (KKT && S > 2) {
    // fast path: column transpositions (none, (1, S-1), then among >= 2), so
    // perm[0] = 0 and perm[1] = S - 1, and rank >= 2 (two unit pivots); the
    // rest of perm permutes 1 .. S-2
    if (fast) {
      general = false;
      sol[0] = c[0];
      sol[S - 1] = c[1];
#pragma unroll
      for (int i = 2; i < S; ++i) {
        const double v = i < rank ? c[i] : 0.0;
#pragma unroll
        for (int j = 1; j < S - 1; ++j) sol[j] = (perm[i] == j) ? v : sol[j];
      }
    }
  }
  if (general) {
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const double v = i < rank ? c[i] : 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) sol[j] = (perm[i] == j) ? v : sol[j];
    }
  }
}

// FullPivLU on the 2-point KKT system [[a, b, 1], [b, c, 1], [1, 1, 0]],
// rhs e_2, along its pivot path when |a|, |b| < 1 and |c| <= 1 (first pivot:
// the 1 at (2, 0), the first entry of largest magnitude in column-major
// order) and |c - b|, |b - a| < 1 (second: the 1 at (1, 2), columns 1 and 2
// swapped): the same operations on the same operands as fullpiv_solve_t,
// so the result is bit-identical; returns false off that path.
GDEV_FN bool kkt2_fast(double a, double b, double c, double (&sol)[3]) {
  if (!(fabs(a) < 1.0 && fabs(b) < 1.0 && fabs(c) <= 1.0)) return false;
  const double cb = c - b * 1.0, ba = b - a * 1.0;
  if (!(fabs(cb) < 1.0 && fabs(ba) < 1.0)) return false;
  const double e = ba - 1.0 * cb;
  const double maxpivot = e != 0.0 ? fmax(1.0, fabs(e)) : 1.0;
  const double thresh = maxpivot * (3 * 2.220446049250313e-16);
  const bool rank3 = e != 0.0 && fabs(e) > thresh;
  // forward substitution (unit lower) on the permuted rhs (1, 0, 0)
  double c0 = 1.0, c1 = 0.0 - 1.0 * b, c2 = 0.0 - 1.0 * a;
  if (c1 != 0.0) c2 = c2 - c1 * 1.0;
  // back substitution on the rank block
  if (rank3 && c2 != 0.0) {
    c2 = c2 / e;
    c1 = c1 - c2 * cb;
    c0 = c0 - c2 * 1.0;
  }
  if (c1 != 0.0) {
    c1 = c1 / 1.0;
    c0 = c0 - c1 * 0.0;
  }
  if (c0 != 0.0) c0 = c0 / 1.0;
  // column permutation (0, 2, 1)
  sol[0] = c0;
  sol[2] = c1;
  sol[1] = rank3 ? c2 : 0.0;
  return true;
}

struct Simplex {
  double dist2;
  D3 v;
  int keep[4];
  double wts[4];
  int nkeep;
  bool contains;
};

// One subset of closest_on_simplex (geometry.cpp:61-93): solve the
// (K+1)x(K+1) affine least-norm KKT system for the gathered points P[0..K)
// (original simplex indices id[0..K)) and apply the acceptance and tie rules
// against the running best. Gram entries are dot(P_i, P_j), bit-identical
// to the reference's gram(idx_i, idx_j) (products commute exactly, sums in
// the same order, no contraction in this TU). (A single zero-padded size-5
// body for every K cuts the kernel's code by a fifth but costs more than
// the instruction-cache stalls it removes; measured.)
template <int K>
GDEV_FN void simplex_subset(const D3 (&P)[4], const int (&id)[4], Simplex& best) {
  double m[K + 1][K + 1];
  double rhs[K + 1];
#pragma unroll
  for (int i = 0; i < K; ++i) {
#pragma unroll
    for (int j = i; j < K; ++j) {
      m[i][j] = dot(P[i], P[j]);
      m[j][i] = m[i][j];
    }
    m[i][K] = 1.0;
    m[K][i] = 1.0;
    rhs[i] = 0.0;
  }
  m[K][K] = 0.0;
  rhs[K] = 1.0;
  double sol[K + 1];
  if constexpr (K == 1) {
    // [[g, 1], [1, 0]] with |g| < 1: FullPivLU pivots on the (1, 0) one,
    // and its solve gives exactly (1, -g) (every step is exact).
    if (fabs(m[0][0]) < 1.0) {
      sol[0] = 1.0;
      sol[1] = -m[0][0];
    } else {
      fullpiv_solve_t<K + 1>(m, rhs, sol);
    }
  } else if constexpr (K == 2) {
    if (!kkt2_fast(m[0][0], m[0][1], m[1][1], sol)) fullpiv_solve_t<K + 1>(m, rhs, sol);
  } else {
    fullpiv_solve_t<K + 1, true>(m, rhs, sol);
  }
  bool ok = true;
#pragma unroll
  for (int i = 0; i <= K; ++i) ok = ok && isfinite(sol[i]);
#pragma unroll
  for (int i = 0; i < K; ++i) ok = ok && !(sol[i] < -1e-12);
  if (!ok) return;
  D3 v = mk(0, 0, 0);
#pragma unroll
  for (int i = 0; i < K; ++i) v += sol[i] * P[i];
  const double d2 = sqn(v);
  if (d2 < best.dist2 - 1e-300 || (K < best.nkeep && d2 <= best.dist2 * (1.0 + 1e-12))) {
    best.dist2 = d2;
    best.v = v;
    best.nkeep = K;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      best.keep[i] = i < K ? id[i] : 0;
      best.wts[i] = i < K ? sol[i < K ? i : 0] : 0.0;
    }
    best.contains = K == 4;
  }
}

// Gathers the points of subset `mask` (ascending index order) into P/id.
GDEV_FN int gather_subset(const SP* simp, int mask, D3 (&P)[4], int (&id)[4]) {
  int k = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool bit = (mask >> i) & 1;
#pragma unroll
    for (int s = 0; s <= i; ++s) {
      const bool put = bit && k == s;
      P[s].x = psel(put, simp[i].w.x, P[s].x);
      P[s].y = psel(put, simp[i].w.y, P[s].y);
      P[s].z = psel(put, simp[i].w.z, P[s].z);
      id[s] = put ? i : id[s];
    }
    k += bit ? 1 : 0;
  }
  return k;
}

// Closest point of conv(simp[0..n)) to the origin by subset enumeration in
// mask order 1..2^n-1 (geometry.cpp:58-95). The mask loop is a runtime loop
// over one solver body per subset size: every lane sees the same size at
// the same mask, so lanes stay converged, and the code stays small enough
// for the instruction cache (a fully unrolled enumeration is ~18k SASS
// instructions and stalled on instruction fetch).
GDEV_FN Simplex closest_on_simplex(const SP* simp, int n) {
  Simplex best;
  best.dist2 = INFINITY;
  best.v = mk(0, 0, 0);
  best.nkeep = 0;
  best.contains = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    best.keep[i] = 0;
    best.wts[i] = 0.0;
  }
  const int last = (1 << n) - 1;
#pragma unroll 1
  for (int mask = 1; mask <= last; ++mask) {
    D3 P[4];
    int id[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      P[i] = mk(0, 0, 0);
      id[i] = 0;
    }
    const int K = gather_subset(simp, mask, P, id);
    switch (K) {
      case 1: simplex_subset<1>(P, id, best); break;
      case 2: simplex_subset<2>(P, id, best); break;
      case 3: simplex_subset<3>(P, id, best); break;
      default: simplex_subset<4>(P, id, best); break;
    }
  }
  return best;
}


struct PairResult {
  double d;
  D3 pa, pb, n;
  int flags;
  unsigned n_support, gjk_iters, epa_iters, gjk_skipped;  // op counters
};

struct EpaFace {
  int v0, v1, v2;
  D3 n;
  double d;
};

GDEV_FN bool lex_less(D3 a, D3 b) {
  if (a.x != b.x) return a.x < b.x;
  if (a.y != b.y) return a.y < b.y;
  return a.z < b.z;
}

// EPA polytope storage. The common case fits a small per-thread buffer;
// pairs that outgrow it are redone with the large buffer (global memory),
// which covers the reference's 512-iteration cap (geometry.cpp:15).
template <int V, int F, int HZ>
struct EpaScratchT {
  static constexpr int kV = V, kF = F, kH = HZ;
  SP verts[V];
  EpaFace faces[F];
  int hk[HZ];  // horizon edges (u << 16) | v, in kill order
};
using EpaScratch = EpaScratchT<64, 128, 96>;
using EpaScratchBig = EpaScratchT<kEpaMaxIters + 8, 4 * kEpaMaxIters, 4 * kEpaMaxIters>;

GDEV_INL EpaFace epa_make_face(const SP* verts, D3 interior, int i0, int i1, int i2) {
  EpaFace f;
  f.v0 = i0;
  f.v1 = i1;
  f.v2 = i2;
  const D3 c = cross(verts[i1].w - verts[i0].w, verts[i2].w - verts[i0].w);
  const double len = nrm(c);
  f.n = len > 0 ? c / len : mk(0, 0, 1);
  f.d = dot(f.n, verts[i0].w);
  if (dot(f.n, interior) > f.d) {
    const int t = f.v1;
    f.v1 = f.v2;
    f.v2 = t;
    f.n = -f.n;
    f.d = -f.d;
  }
  return f;
}

// geometry.cpp:168-205 + 227-324.
struct EpaDebug {
  int iters, nv, nf, v[3];
  double n[3], d, tri_w[9], tri_a[9], wts[3];
  int keep[3], nkeep;
};

template <class Scratch>
GDEV_FN bool epa(const SP (&simp)[4], int ns, const Hull& A, const Hull& B, double scale, Scratch& s,
                 PairResult& out, EpaDebug* dbg = nullptr) {
  constexpr int kEpaMaxVerts = Scratch::kV, kEpaMaxFaces = Scratch::kF, kEpaMaxHorizon = Scratch::kH;
  // pad_to_tetrahedron
  const double tol = 1e-12 * scale;
  D3 dirs[10];
  int nd = 0;
  if (ns == 2) {
    const D3 d = normalized(simp[1].w - simp[0].w);
    const D3 t = fabs(d.x) < 0.9 ? mk(1, 0, 0) : mk(0, 1, 0);
    const D3 e1 = normalized(cross(d, t));
    const D3 e2 = cross(d, e1);
    dirs[nd++] = e1;
    dirs[nd++] = -e1;
    dirs[nd++] = e2;
    dirs[nd++] = -e2;
  }
  if (ns == 3) {
    const D3 n = normalized(cross(simp[1].w - simp[0].w, simp[2].w - simp[0].w));
    dirs[nd++] = n;
    dirs[nd++] = -n;
  }
  dirs[nd++] = mk(1, 0, 0);
  dirs[nd++] = mk(-1, 0, 0);
  dirs[nd++] = mk(0, 1, 0);
  dirs[nd++] = mk(0, -1, 0);
  dirs[nd++] = mk(0, 0, 1);
  dirs[nd++] = mk(0, 0, -1);
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < ns) s.verts[i] = simp[i];
  int nv = ns;
  for (int k = 0; k < nd && nv < 4; ++k) {
    const SP cand = support_pair(A, B, dirs[k]);
    ++out.n_support;
    bool indep;
    if (nv == 0) {
      indep = true;
    } else if (nv == 1) {
      indep = nrm(cand.w - s.verts[0].w) > tol;
    } else if (nv == 2) {
      const D3 d = normalized(s.verts[1].w - s.verts[0].w);
      const D3 r = cand.w - s.verts[0].w;
      indep = nrm(r - d * dot(d, r)) > tol;
    } else {
      const D3 n = normalized(cross(s.verts[1].w - s.verts[0].w, s.verts[2].w - s.verts[0].w));
      indep = fabs(dot(n, cand.w - s.verts[0].w)) > tol;
    }
    if (indep) s.verts[nv++] = cand;
  }
  if (nv != 4) {
    out.flags |= kPairDegenerate;
    return false;
  }
  const D3 interior = (s.verts[0].w + s.verts[1].w + s.verts[2].w + s.verts[3].w) / 4.0;
  int nf = 0;
  s.faces[nf++] = epa_make_face(s.verts, interior, 0, 1, 2);
  s.faces[nf++] = epa_make_face(s.verts, interior, 0, 2, 3);
  s.faces[nf++] = epa_make_face(s.verts, interior, 0, 3, 1);
  s.faces[nf++] = epa_make_face(s.verts, interior, 1, 3, 2);

  const double grow_tol = 1e-10 * scale;
  EpaFace best_copy = s.faces[0];
  // Closest face (geometry.cpp:255-262), scanned in face-array order. The
  // scan of the next iteration runs incrementally as the kill loop compacts
  // the kept faces and the horizon loop appends the new ones: the same
  // comparisons in the same order, one pass over the faces fewer.
  int best = -1;
  double best_d = INFINITY;
  auto consider = [&](int i) {
    const double di = s.faces[i].d;
    if (di < best_d - 1e-12 * scale ||
        (di < best_d + 1e-12 * scale && best >= 0 && lex_less(-s.faces[i].n, -s.faces[best].n))) {
      best_d = fmin(best_d, di);
      best = i;
    }
  };
  for (int i = 0; i < nf; ++i) consider(i);
  for (int iter = 0; iter < kEpaMaxIters; ++iter) {
    if (best < 0) {
      out.flags |= kPairDegenerate;
      return false;
    }
    best_copy = s.faces[best];
    const SP w = support_pair(A, B, best_copy.n);
    ++out.n_support;
    ++out.epa_iters;
    if (dot(best_copy.n, w.w) - best_copy.d <= grow_tol) break;
    if (nv >= kEpaMaxVerts) {
      out.flags |= kPairOverflow;
      break;
    }
    const int wi = nv;
    s.verts[nv++] = w;
    // Kill visible faces in order, collecting their directed edges.
    int nh = 0;
    int kept = 0;
    bool overflow = false;
    best = -1;
    best_d = INFINITY;
    for (int i = 0; i < nf; ++i) {
      const EpaFace f = s.faces[i];
      if (dot(f.n, w.w) - f.d > 1e-12 * scale) {
        if (nh + 3 > kEpaMaxHorizon) {
          overflow = true;
        } else {
          s.hk[nh++] = (f.v0 << 16) | f.v1;
          s.hk[nh++] = (f.v1 << 16) | f.v2;
          s.hk[nh++] = (f.v2 << 16) | f.v0;
        }
      } else {
        s.faces[kept] = f;
        consider(kept++);
      }
    }
    nf = kept;
    if (overflow) {
      out.flags |= kPairOverflow;
      break;
    }
    int n_boundary = 0;
    for (int e = 0; e < nh; ++e) {
      const int ke = s.hk[e], rev = ((ke & 0xffff) << 16) | (ke >> 16);
      bool paired = false;
      for (int o = 0; o < nh; ++o)
        if (s.hk[o] == rev) paired = true;
      if (!paired) {
        if (nf >= kEpaMaxFaces) {
          overflow = true;
          break;
        }
        s.faces[nf] = epa_make_face(s.verts, interior, ke >> 16, ke & 0xffff, wi);
        consider(nf++);
        ++n_boundary;
      }
    }
    if (overflow) {
      out.flags |= kPairOverflow;
      break;
    }
    if (n_boundary == 0) break;
  }
  out.d = -fmax(best_copy.d, 0.0);
  out.n = -best_copy.n;
  const SP tri[3] = {s.verts[best_copy.v0], s.verts[best_copy.v1], s.verts[best_copy.v2]};
  const Simplex sx = closest_on_simplex(tri, 3);
  D3 wa = mk(0, 0, 0), wb = mk(0, 0, 0);
  double wsum = 0.0;
  for (int i = 0; i < sx.nkeep; ++i) {
    const SP& p = tri[sx.keep[i]];
    wa += sx.wts[i] * sp_a(A, p);
    wb += sx.wts[i] * sp_b(B, p);
    wsum += sx.wts[i];
  }
  if (wsum > 0.5) {
    out.pa = wa;
    out.pb = wb;
  } else {
    out.pa = sp_a(A, tri[0]);
    out.pb = sp_b(B, tri[0]);
  }
  out.flags |= kPairEpa;
  if (dbg) {
    dbg->nv = nv;
    dbg->nf = nf;
    dbg->v[0] = best_copy.v0; dbg->v[1] = best_copy.v1; dbg->v[2] = best_copy.v2;
    st3(dbg->n, best_copy.n);
    dbg->d = best_copy.d;
    for (int i = 0; i < 3; ++i) { st3(dbg->tri_w + 3 * i, tri[i].w); st3(dbg->tri_a + 3 * i, sp_a(A, tri[i])); }
    dbg->nkeep = sx.nkeep;
    for (int i = 0; i < sx.nkeep; ++i) { dbg->keep[i] = sx.keep[i]; dbg->wts[i] = sx.wts[i]; }
  }
  return true;
}

// GJK part of signed_distance (geometry.cpp:105-164, 500-516). Returns true
// on overlap, leaving the terminal simplex (the EPA seed) in simp/ns;
// otherwise `out` holds the separated result.
GDEV_FN bool gjk_phase(const Hull& A, const Hull& B, double scale, PairResult& out, SP (&simp)[4], int& ns) {
  out.flags = 0;
  out.n_support = 1;
  out.gjk_iters = 0;
  out.epa_iters = 0;
  out.gjk_skipped = 0;
  // The simplex is only ever indexed by compile-time constants (unrolled
  // loops with predicates) so it stays in registers. One support_pair and
  // one closest_on_simplex call site (instruction-cache footprint): the
  // loop enters at the seed support (direction +x, geometry.cpp:107-108),
  // and the iteration cap (geometry.cpp:151-163: the estimate on the
  // unreduced simplex, i.e. its support subset, no contact test) leaves
  // through the common separated exit.
  ns = 0;
  GjkCycle cyc;
  cycle_init(cyc, A.nv, B.nv);
  bool overlap = false;
  Simplex sx;
  D3 dir = mk(1, 0, 0);
  for (int iter = -1;;) {
    const SP w = support_pair(A, B, dir);
    if (iter < 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) simp[i] = w;
    } else {
      ++out.n_support;
      ++out.gjk_iters;
      const double gap = sx.dist2 - dot(sx.v, w.w);
      bool repeat = false;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < ns && nrm(simp[i].w - w.w) < 1e-14 * scale) repeat = true;
      if (gap <= kGjkRelTol * sx.dist2 + 1e-300 || repeat || ns == 4) break;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i == ns) simp[i] = w;
    }
    ++ns;
    ++iter;
    const int jump = cycle_step(cyc, simp, ns, iter);
    iter += jump;
    out.gjk_skipped += jump;
    sx = closest_on_simplex(simp, ns);
    SP red[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int src = sx.keep[i];
      red[i] = simp[0];
      if (src == 1) red[i] = simp[1];
      if (src == 2) red[i] = simp[2];
      if (src == 3) red[i] = simp[3];
    }
    ns = sx.nkeep;
#pragma unroll
    for (int i = 0; i < 4; ++i) simp[i] = red[i];
    if (iter == kGjkMaxIters) break;
    if (sx.contains || sqrt(sx.dist2) < kTouchTol * scale) {
      overlap = true;
      break;
    }
    dir = -sx.v;
  }
  if (!overlap) {
    D3 wa = mk(0, 0, 0), wb = mk(0, 0, 0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i < ns) {
        wa += sx.wts[i] * sp_a(A, simp[i]);
        wb += sx.wts[i] * sp_b(B, simp[i]);
      }
    }
    const double d = sqrt(sx.dist2);
    out.d = d;
    out.pa = wa;
    out.pb = wb;
    out.n = d > 1e-14 ? (wa - wb) / d : mk(0, 0, 1);
    return false;
  }
  return true;
}

// signed_distance(a, pose_a, b, identity) (geometry.cpp:500-525).
template <class Scratch>
GDEV_INL PairResult signed_distance(const Hull& A, const Hull& B, double scale, Scratch& scratch,
                                    EpaDebug* dbg = nullptr) {
  PairResult out;
  SP simp[4];
  int ns;
  if (gjk_phase(A, B, scale, out, simp, ns)) epa(simp, ns, A, B, scale, scratch, out, dbg);
  return out;
}

}  // namespace gdev

// Lower-level QP kernel (separate translation unit, compiled with FMA
// contraction; the geometry/kinematics kernels in kernels.cuh are compiled
// without it so their discrete decisions match the fp64 oracle bit for bit).
//
// One warp = one grasp's batch of 6 closure-direction QPs (energy.cpp:60-92,
// qpsolve.cpp:45-120, 193-235). Lane (j, c) = (direction j, contact c) owns
// the K edge weights of contact c in column j, their identity rows and the
// cap row c; the total-weight row is replicated in the M lanes of a column.
// K = P + sigma I + rho A'A is B + U U^T with B block-diagonal (closed-form
// inverse) and U = [sqrt2 W^T | sqrt(rho) 1] of rank 7, so
//   K^-1 r = B^-1 r - Z (G^T r),  G = B^-1 U,  Z = G (I + U^T G)^-1,
// i.e. each ADMM sweep is a handful of K-long dot products per lane plus
// 8 fixed-order column reductions. Templated on (K, M) so every per-lane
// array is register-resident; (0, 0) is the generic runtime-size fallback.
#pragma once

#include "dmath.cuh"
#include "model.cuh"

namespace gdev {

#ifndef GDEV_FULL_MASK
#define GDEV_FULL_MASK
constexpr unsigned kFull = 0xffffffffu;
#endif

// Pairwise sum of N register values (short dependency chains: the sweep is
// bound by fp64 latency at ~4 warps per scheduler, not by the fp64 pipe).
template <int N>
__device__ __forceinline__ double tree_sum(const double* v) {
  if constexpr (N == 1) {
    return v[0];
  } else {
    return tree_sum<N / 2>(v) + tree_sum<N - N / 2>(v + N / 2);
  }
}

// max(v, 0) by clearing negative values' bits (ALU pipe, not the fp64 pipe).
__device__ __forceinline__ double relu_bits(double v) {
  const long long b = __double_as_longlong(v);
  return __longlong_as_double(b & ~(b >> 63));
}

// Fixed-order sum over lanes base..base+cnt-1 (identical on all lanes): all
// shuffles first, then a pairwise tree when the count is known.
template <int CNT>
__device__ __forceinline__ double qp_group_sum(double v, int base, int cnt) {
  if constexpr (CNT == 4 || CNT == 5) {
    // shift-down partial sums: the group's head lane (base) ends with the
    // whole sum reading only lanes base..base+CNT-1, then broadcasts it
    // (CNT = 5: 4 shuffles and 3 adds instead of 5 and 4)
    const double s1 = v + __shfl_down_sync(kFull, v, 1);
    double s = s1 + __shfl_down_sync(kFull, s1, 2);
    if constexpr (CNT == 5) s += __shfl_down_sync(kFull, v, 4);
    return __shfl_sync(kFull, s, base);
  } else if constexpr (CNT > 0) {
    double t[CNT];
#pragma unroll
    for (int b = 0; b < CNT; ++b) t[b] = __shfl_sync(kFull, v, base + b);
    return tree_sum<CNT>(t);
  } else {
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < kMaxTips; ++b)
      if (b < cnt) s += __shfl_sync(kFull, v, base + b);
    return s;
  }
}
template <int CNT>
__device__ __forceinline__ double qp_group_max(double v, int base, int cnt) {
  double s = 0.0;
  const int n = CNT > 0 ? CNT : cnt;
#pragma unroll
  for (int b = 0; b < (CNT > 0 ? CNT : kMaxTips); ++b)
    if (b < n) s = fmax(s, __shfl_sync(kFull, v, base + b));
  return s;
}

// Per-contact blocks are padded to an odd number of doubles so that the
// m contacts a warp reads at once (lanes of one contact broadcast) fall in
// distinct shared-memory bank pairs.
constexpr int kQpWStride = kMaxEdges | 1;        // W: [6][m][ws] with ws = k | 1
constexpr int kQpGStride = (7 * kMaxEdges) | 1;  // G, Z: [m][gs] with gs = 7k | 1, rows of 7
struct QpSmem {
  double frame[kMaxTips * 12];
  double W[6 * kMaxTips * kQpWStride];  // W(r, c, e) = W[r * m * ws + c * ws + e]
  double Gm[kMaxTips * kQpGStride];     // B^-1 U: G(c, e, p) = Gm[c * gs + e * 7 + p]
  double C[49];                         // I + U^T G
  double Cinv[49];
};

// mode 0: coarse (frames from the tip point queries, warm start from the
// per-grasp scratch, envelope-gradient forces written when with_grad).
// mode 1: final record (frames from st.frames, cold start).
// mode 2: standalone batch (frames from st.frames, warm if qp_ready).
#ifndef GDEV_QP_MIN_BLOCKS
#define GDEV_QP_MIN_BLOCKS 3  // 168 registers, no spills (measured best since the scaled-dual sweep; 4 and 5 spill)
#endif
#ifndef GDEV_QP_WARPS
#define GDEV_QP_WARPS 4  // grasps (warps) per block; 1 and 2 measured slower (qp 440 / 434 vs 432 ms)
#endif
template <int KT, int MT>
#ifndef GDEV_QP_RESIDENT_WARPS
#define GDEV_QP_RESIDENT_WARPS (GDEV_QP_MIN_BLOCKS * 4)
#endif
__global__ void __launch_bounds__(32 * GDEV_QP_WARPS, GDEV_QP_RESIDENT_WARPS / GDEV_QP_WARPS)
    k_qp_t(DevHand H, DevParams P, DevState st, int m_rt, int mode, int with_grad) {
  __shared__ QpSmem smem_all[GDEV_QP_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * GDEV_QP_WARPS + warp;
  if (g >= st.G) return;
  if (st.failed[g]) return;
  QpSmem& s = smem_all[warp];
  constexpr int KMAX = KT > 0 ? KT : kMaxEdges;
  const int k = KT > 0 ? KT : P.k;
  const int m = MT > 0 ? MT : m_rt;
  const int n = m * k, M = m + 1 + n;
  const int ws = k | 1, wn = m * ws, gs = (7 * k) | 1;

  // Frames.
  if (lane < m) {
    if (mode == 0) {
      const double* q = st.qres + ((size_t)g * st.NQ + H.tip_proxy[lane]) * 8;
      build_frame(ld3(q + 1), -ld3(q + 4), s.frame + 12 * lane);
    } else {
      const double* f = st.frames + ((size_t)g * m + lane) * 12;
      for (int i = 0; i < 12; ++i) s.frame[12 * lane + i] = f[i];
    }
  }
  __syncwarp();
  const double a_diag = P.sigma + P.rho;
  const double betap = P.rho / (a_diag + k * P.rho);
  const double sqrt2 = 1.4142135623730951, sqrt_rho = sqrt(P.rho);
  // Wrench basis block c (contact.cpp:47-53) and G = B^-1 U rows.
  if (lane < m) {
    const int c = lane;
    const D3 p = ld3(s.frame + 12 * c), nn = ld3(s.frame + 12 * c + 3);
    const D3 d = ld3(s.frame + 12 * c + 6), e = ld3(s.frame + 12 * c + 9);
    for (int j = 0; j < k; ++j) {
      const D3 edge = nn + P.mu * (P.cos_t[j] * d + P.sin_t[j] * e);
      const D3 tq = cross(p, edge);
      const int col = c * ws + j;
      s.W[0 * wn + col] = edge.x;
      s.W[1 * wn + col] = edge.y;
      s.W[2 * wn + col] = edge.z;
      s.W[3 * wn + col] = tq.x;
      s.W[4 * wn + col] = tq.y;
      s.W[5 * wn + col] = tq.z;
    }
    for (int q = 0; q < 7; ++q) {
      double bs = 0.0;
      for (int j = 0; j < k; ++j) bs += q < 6 ? sqrt2 * s.W[q * wn + c * ws + j] : sqrt_rho;
      for (int j = 0; j < k; ++j) {
        const double u = q < 6 ? sqrt2 * s.W[q * wn + c * ws + j] : sqrt_rho;
        s.Gm[c * gs + j * 7 + q] = (u - betap * bs) / a_diag;
      }
    }
  }
  __syncwarp();
  // Capacitance C = I + U^T G (symmetric, 28 unique entries).
  if (lane < 28) {
    int p = 0, q = lane;
    while (q >= 7 - p) {
      q -= 7 - p;
      ++p;
    }
    q += p;
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
      const int ci = i / k, ei = i - ci * k;
      const double u = p < 6 ? sqrt2 * s.W[p * wn + ci * ws + ei] : sqrt_rho;
      acc += u * s.Gm[ci * gs + ei * 7 + q];
    }
    const double v = acc + (p == q ? 1.0 : 0.0);
    s.C[p * 7 + q] = v;
    s.C[q * 7 + p] = v;
  }
  __syncwarp();
  // C^-1 (7x7): every lane factors C (Cholesky) redundantly; lane q < 7
  // solves for column q.
  {
    double L[7][7];
#pragma unroll
    for (int j = 0; j < 7; ++j) {
      double dsum = s.C[j * 7 + j];
#pragma unroll
      for (int q = 0; q < j; ++q) dsum -= L[j][q] * L[j][q];
      const double ljj = sqrt(dsum);
      L[j][j] = ljj;
#pragma unroll
      for (int i = j + 1; i < 7; ++i) {
        double v = s.C[i * 7 + j];
#pragma unroll
        for (int q = 0; q < j; ++q) v -= L[i][q] * L[j][q];
        L[i][j] = v / ljj;
      }
    }
    __syncwarp();
    if (lane < 7) {
      double y[7];
#pragma unroll
      for (int r = 0; r < 7; ++r) {
        double v = r == lane ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < r; ++q) v -= L[r][q] * y[q];
        y[r] = v / L[r][r];
      }
#pragma unroll
      for (int r = 6; r >= 0; --r) {
        double v = y[r];
#pragma unroll
        for (int q = r + 1; q < 7; ++q) v -= L[q][r] * y[q];
        y[r] = v / L[r][r];
      }
#pragma unroll
      for (int r = 0; r < 7; ++r) s.Cinv[r * 7 + lane] = y[r];
    }
  }
  __syncwarp();

  const bool active = lane < 6 * m;
  const int j = active ? lane / m : 0;
  const int c = active ? lane % m : 0;
  const int base = j * m;
  const int axis = j >> 1;
  const double tsign = ((j & 1) ? -1.0 : 1.0) * P.target_sign;
  const double rho = P.rho, sigma = P.sigma, alpha = P.alpha, mu = P.mu;
  const double inv_a = 1.0 / a_diag;
  const double inv_rho = 1.0 / rho;
  // This lane's contact frame (contact.cpp:47-53): edge_e = n + mu (cos_e d +
  // sin_e e), torque_e = p x edge_e. Every product with W or W^T is formed
  // from it: W v = (f, p x f) with f = n S0 + mu (d S1 + e S2), S0 = sum v_e,
  // S1 = sum cos_e v_e, S2 = sum sin_e v_e; (W^T u)_e = edge_e . (u_f + u_t x p).
  const D3 fp = ld3(s.frame + 12 * c);
  // The sweep uses the frame only as sqrt2 n, sqrt2 mu d, sqrt2 mu e (the U
  // rows); the residual check reloads the unscaled frame from shared memory.
  const D3 sn = sqrt2 * ld3(s.frame + 12 * c + 3);
  const D3 sdv = (sqrt2 * mu) * ld3(s.frame + 12 * c + 6), sev = (sqrt2 * mu) * ld3(s.frame + 12 * c + 9);
  double ccos = 0.0, csin = 0.0;
#pragma unroll
  for (int e = 0; e < KMAX; ++e)
    if (e < k) ccos += P.cos_t[e], csin += P.sin_t[e];
  auto w_times = [&](const double (&v)[KMAX], D3& f, D3& t, double& s0) {
    const D3 fn = ld3(s.frame + 12 * c + 3), fd = ld3(s.frame + 12 * c + 6), fe = ld3(s.frame + 12 * c + 9);
    double s1 = 0.0, s2 = 0.0;
    s0 = 0.0;
#pragma unroll
    for (int e = 0; e < KMAX; ++e) {
      if (e < k) {
        s0 += v[e];
        s1 += P.cos_t[e] * v[e];
        s2 += P.sin_t[e] * v[e];
      }
    }
    f = s0 * fn + mu * (s1 * fd + s2 * fe);
    t = cross(fp, f);
  };

  // Scaled duals u = y / rho (ADMM scaled form): the projection step costs
  // two adds per row; y = rho u is formed only for the residual check and
  // the snapshot. nq = -q.
  double x[KMAX], zid[KMAX], uid[KMAX], nq[KMAX];
  double zc, uc, ztot, utot;
  const bool warm = (mode == 0 || mode == 2) && st.qp_ready[g];
  const double* wx = st.warm_x + (size_t)g * n * 6;
  const double* wy = st.warm_y + (size_t)g * M * 6;
#pragma unroll
  for (int e = 0; e < KMAX; ++e) {
    if (e < k) {
      const int i = c * k + e;
      x[e] = warm ? wx[j * n + i] : 0.0;
      uid[e] = warm ? wy[j * M + m + 1 + i] * inv_rho : 0.0;
      nq[e] = (2.0 * P.beta) * (tsign * s.W[axis * wn + c * ws + e]);
    } else {
      x[e] = uid[e] = nq[e] = 0.0;
    }
    zid[e] = x[e];
  }
  uc = warm ? wy[j * M + c] * inv_rho : 0.0;
  utot = warm ? wy[j * M + m] * inv_rho : 0.0;
  {
    const double bs = tree_sum<KMAX>(x);
    zc = bs;
    ztot = qp_group_sum<MT>(bs, base, m);
  }
  const double gamma = P.gamma_total;
  const double oma = 1.0 - alpha, a_inv_a = alpha * inv_a;
  bool frozen = !active;
  double* ox = st.warm_x + (size_t)g * n * 6;
  double* oy = st.warm_y + (size_t)g * M * 6;
  double* oz = st.out_z + (size_t)g * M * 6;

  // After a projection z = max(v, 0) and u = min(v, 0) for v = zbar + u, so
  // z - u = |v| and (1 - alpha) z + u = (v >= 0 ? 1 - alpha : 1) v: from the
  // second sweep on, the per-edge state is (x, v) and the edge update is four
  // fp64 operations. The first sweep starts from the warm (z, u), which need
  // not be complementary, and is peeled (kFirst).
  double vz[KMAX];
  // countdown to the next check sweep (iter % check_interval == 0) without
  // an integer division per sweep
  const int interval = P.check_interval > 0 ? P.check_interval : 1;
  int to_check = interval;
  auto sweep = [&]<bool kFirst>(int iter) -> bool {
    // rhs = A'(rho z - y) + sigma x - q = rq + vct (vct: the cap and total
    // rows, common to the lane's edges) ; r' = B^-1 rhs
    const double vct = rho * ((zc - uc) + (ztot - utot));
    double rq[KMAX];
#pragma unroll
    for (int e = 0; e < KMAX; ++e)
      rq[e] = e < k ? rho * (kFirst ? zid[e] - uid[e] : fabs(vz[e])) + (sigma * x[e] + nq[e]) : 0.0;
    const double bsum = tree_sum<KMAX>(rq) + k * vct;
    const double bb = betap * bsum;
    double tv[7];
    {
      // two interleaved accumulators per sum (padded rq entries are zero)
      double s1a = 0.0, s1b = 0.0, s2a = 0.0, s2b = 0.0;
#pragma unroll
      for (int e = 0; e < KMAX; e += 2) {
        s1a += P.cos_t[e] * rq[e];
        s2a += P.sin_t[e] * rq[e];
        if (e + 1 < KMAX) {
          s1b += P.cos_t[e + 1] * rq[e + 1];
          s2b += P.sin_t[e + 1] * rq[e + 1];
        }
      }
      const double s1r = (s1a + s1b) + ccos * vct, s2r = (s2a + s2b) + csin * vct;
      const double s0 = (bsum - k * bb) * inv_a;
      const double s1 = (s1r - ccos * bb) * inv_a, s2 = (s2r - csin * bb) * inv_a;
      const D3 f2 = s0 * sn + (s1 * sdv + s2 * sev);  // sqrt2 f
      const D3 t2 = cross(fp, f2);                       // sqrt2 t
      const double tl[7] = {f2.x, f2.y, f2.z, t2.x, t2.y, t2.z, sqrt_rho * s0};
#pragma unroll
      for (int p = 0; p < 7; ++p) tv[p] = qp_group_sum<MT>(tl[p], base, m);
    }
    // s = C^-1 t ; G s = B^-1 U s ; xt = r' - G s. With the contact count
    // known at compile time the 7 rows of C^-1 t are split over the m lanes
    // of the column (lane c takes rows c, c + m, ...) and shared by shuffles.
    double sv[7];
    if constexpr (MT > 0) {
      constexpr int RPL = (7 + MT - 1) / MT;  // rows per lane
      double mine[RPL];
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = c + i * MT;
        double a0 = 0.0, a1 = 0.0;
        if (r < 7) {
#pragma unroll
          for (int p = 0; p < 7; p += 2) {
            a0 += s.Cinv[r * 7 + p] * tv[p];
            if (p + 1 < 7) a1 += s.Cinv[r * 7 + p + 1] * tv[p + 1];
          }
        }
        mine[i] = a0 + a1;
      }
#pragma unroll
      for (int r = 0; r < 7; ++r) sv[r] = __shfl_sync(kFull, mine[r / MT], base + r % MT);
    } else {
#pragma unroll
      for (int r = 0; r < 7; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int p = 0; p < 7; ++p) acc += s.Cinv[r * 7 + p] * tv[p];
        sv[r] = acc;
      }
    }
    const D3 wv = mk(sv[0], sv[1], sv[2]) + cross(mk(sv[3], sv[4], sv[5]), fp);
    // (U s)_e = ua + ub cos_e + ue sin_e, so (G s)_e = (U s - betap sum U s)_e / a
    // is ga + gb cos_e + gc sin_e.
    const double ua = dot(sn, wv) + sqrt_rho * sv[6], ub = dot(sdv, wv), ue = dot(sev, wv);
    const double us_sum = k * ua + ccos * ub + csin * ue;
    const double ga = (ua - betap * us_sum) * inv_a, gb = ub * inv_a, gc = ue * inv_a;
    const double h0 = bb * inv_a + ga;
    // alpha xt_e = alpha (inv_a (rq_e + vct) - h0 - gb cos_e - gc sin_e)
    const double hh = alpha * (inv_a * vct - h0), agb = alpha * gb, agc = alpha * gc;
    double axt[KMAX];
#pragma unroll
    for (int e = 0; e < KMAX; ++e)
      axt[e] = e < k ? ((a_inv_a * rq[e] + hh) - agb * P.cos_t[e]) - agc * P.sin_t[e] : 0.0;
    // (a closed form from the sums already formed saves the tree but rounds
    // differently; the end-to-end comparison with the oracle drifted past
    // its 1e-5 tolerance on the short trident schedule, so the tree stays)
    const double aztc = tree_sum<KMAX>(axt);
    const double aztt = qp_group_sum<MT>(aztc, base, m);
    // Relaxed updates and projection (z = Pi(zbar + u), u += zbar - z).
#pragma unroll
    for (int e = 0; e < KMAX; ++e) {
      if (e < k) {
        x[e] = oma * x[e] + axt[e];
        if constexpr (kFirst) {
          vz[e] = (oma * zid[e] + axt[e]) + uid[e];
        } else {
          const double fac = __double2hiint(vz[e]) >= 0 ? oma : 1.0;  // sign bit: ALU, not fp64
          vz[e] = fac * vz[e] + axt[e];
        }
      } else {
        vz[e] = 0.0;
      }
    }
    {
      const double v = (oma * zc + aztc) + uc;
      const double zn = fmin(relu_bits(v), 1.0);
      uc = v - zn;
      zc = zn;
    }
    {
      const double v = (oma * ztot + aztt) + utot;
      const double zn = fmax(v, gamma);
      utot = v - zn;
      ztot = zn;
    }
    const bool check_now = --to_check == 0;
    if (check_now) to_check = interval;
    if (check_now || iter == P.max_iters) {
      double axc = 0.0;
#pragma unroll
      for (int e = 0; e < KMAX; ++e)
        if (e < k) axc += x[e];
      const double axt = qp_group_sum<MT>(axc, base, m);
      double rp_ = fmax(fabs(axc - zc), fabs(axt - ztot));
#pragma unroll
      for (int e = 0; e < KMAX; ++e)
        if (e < k) rp_ = fmax(rp_, fabs(x[e] - relu_bits(vz[e])));
      rp_ = qp_group_max<MT>(rp_, base, m);
      // The dual residual only matters for a live column whose primal residual
      // passed: skipped (warp-uniformly) when there is none (ok is false then).
      double rd = INFINITY;
      if (__any_sync(kFull, !frozen && rp_ <= P.eps_primal)) {
      // W x over the column, then (W^T W x)_e = edge_e . (wf + wt x p)
      D3 wf, wt;
      double sx_;
      w_times(x, wf, wt, sx_);
      wf = mk(qp_group_sum<MT>(wf.x, base, m), qp_group_sum<MT>(wf.y, base, m), qp_group_sum<MT>(wf.z, base, m));
      wt = mk(qp_group_sum<MT>(wt.x, base, m), qp_group_sum<MT>(wt.y, base, m), qp_group_sum<MT>(wt.z, base, m));
      const D3 u = wf + cross(wt, fp);
      const D3 fn = ld3(s.frame + 12 * c + 3), fd = ld3(s.frame + 12 * c + 6), fe = ld3(s.frame + 12 * c + 9);
      const double nu = dot(fn, u), du = dot(fd, u), eu = dot(fe, u);
      rd = 0.0;
#pragma unroll
      for (int e = 0; e < KMAX; ++e) {
        if (e < k) {
          const double px = nu + mu * (P.cos_t[e] * du + P.sin_t[e] * eu);
          const double dual = (2.0 * px + rho * ((uc + utot) + (vz[e] - relu_bits(vz[e])))) - nq[e];
          rd = fmax(rd, fabs(dual));
        }
      }
      rd = qp_group_max<MT>(rd, base, m);
      }
      if (!frozen) {
        const bool ok = rp_ <= P.eps_primal && rd <= P.eps_dual;
        if (ok || iter == P.max_iters) {
          frozen = true;
#pragma unroll
          for (int e = 0; e < KMAX; ++e) {
            if (e < k) {
              const int i = c * k + e;
              ox[j * n + i] = x[e];
              oy[j * M + m + 1 + i] = rho * (vz[e] - relu_bits(vz[e]));
              oz[j * M + m + 1 + i] = relu_bits(vz[e]);
            }
          }
          oy[j * M + c] = rho * uc;
          oz[j * M + c] = zc;
          if (c == 0) {
            oy[j * M + m] = rho * utot;
            oz[j * M + m] = ztot;
            st.qp_iters[(size_t)g * 6 + j] = iter;
            st.qp_conv[(size_t)g * 6 + j] = ok ? 1 : 0;
          }
        }
      }
      if (__all_sync(kFull, frozen)) return true;
    }
    return false;
  };
  int sweeps = 0;
  if (P.max_iters >= 1) {
    sweeps = 1;
    bool stop = sweep.template operator()<true>(1);
    for (int iter = 2; iter <= P.max_iters && !stop; ++iter) {
      sweeps = iter;
      stop = sweep.template operator()<false>(iter);
    }
  }
  if (lane == 0) {
    st.qp_ready[g] = 1;
    if (st.ops) {
      atomicAdd(st.ops + kOpQpColumnSweeps, 6ull * sweeps);
      atomicAdd(st.ops + kOpQpSolves, 1ull);
    }
  }

  // Energy report from the snapshot (energy.cpp:78-90), read back from the
  // warm-start copy this lane wrote when its column froze.
  double xs[KMAX];
#pragma unroll
  for (int e = 0; e < KMAX; ++e) xs[e] = (active && e < k) ? ox[j * n + c * k + e] : 0.0;
  double res[6];
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < KMAX; ++e)
      if (e < k) acc += s.W[r * wn + c * ws + e] * xs[e];
    const double wl = qp_group_sum<MT>(acc, base, m);
    res[r] = P.beta * (r == axis ? tsign : 0.0) - wl;
  }
  double pd = 0.0;
#pragma unroll
  for (int r = 0; r < 6; ++r) pd += res[r] * res[r];
  if (active && c == 0) st.qp_perdir[(size_t)g * 6 + j] = pd;
  double total = 0.0;
  for (int jj = 0; jj < 6; ++jj) total += __shfl_sync(kFull, pd, jj * m);
  if (lane == 0) st.qp_energy[g] = total;
  if (!with_grad) return;

  // Envelope gradient (energy.cpp:94-145) reduced to one force per tip.
  const D3 p = ld3(s.frame + 12 * c), nn = ld3(s.frame + 12 * c + 3);
  const D3 dd = ld3(s.frame + 12 * c + 6), ee = ld3(s.frame + 12 * c + 9);
  const D3 seed = fabs(nn.x) > 0.99 ? mk(0, 1, 0) : mk(1, 0, 0);
  const double cnorm = nrm(cross(nn, seed));
  const D3 rf = mk(res[0], res[1], res[2]), rt = mk(res[3], res[4], res[5]);
  double sum = 0.0, sum_cos = 0.0, sum_sin = 0.0;
  D3 fsum = mk(0, 0, 0);
#pragma unroll
  for (int e = 0; e < KMAX; ++e) {
    if (e < k) {
      sum += xs[e];
      sum_cos += xs[e] * P.cos_t[e];
      sum_sin += xs[e] * P.sin_t[e];
      fsum += xs[e] * (nn + P.mu * (P.cos_t[e] * dd + P.sin_t[e] * ee));
    }
  }
  const D3 gv = rf + cross(rt, p);
  // md = -(I - d d^T)[seed]x / cnorm  ->  md^T g = seed x ((I - d d^T) g) / cnorm
  const D3 proj = gv - dd * dot(dd, gv);
  const D3 mdTg = cross(seed, proj) / cnorm;
  // me = [n]x md - [d]x  ->  me^T g = md^T (g x n) + d x g
  const D3 gxn = cross(gv, nn);
  const D3 proj2 = gxn - dd * dot(dd, gxn);
  const D3 meTg = cross(seed, proj2) / cnorm + cross(dd, gv);
  const D3 an = sum * gv + (P.mu * sum_cos) * mdTg + (P.mu * sum_sin) * meTg;
  const D3 ap = cross(fsum, rt);
  // Sum over the 6 directions of contact c, fixed order.
  D3 AN = mk(0, 0, 0), AP = mk(0, 0, 0);
  for (int jj = 0; jj < 6; ++jj) {
    const int src = jj * m + c;
    AN.x += __shfl_sync(kFull, an.x, src);
    AN.y += __shfl_sync(kFull, an.y, src);
    AN.z += __shfl_sync(kFull, an.z, src);
    AP.x += __shfl_sync(kFull, ap.x, src);
    AP.y += __shfl_sync(kFull, ap.y, src);
    AP.z += __shfl_sync(kFull, ap.z, src);
  }
  if (active && j == 0) {
    const double* qb = st.qres + (size_t)g * st.NQ * 8;
    const double h2 = 2.0 * P.fd_step;
    double vals_p[3], vals_n[3];  // (dp^T AP)_k = dp.col(k) . AP
    for (int kk = 0; kk < 3; ++kk) {
      const double* qp = qb + (size_t)(H.S + c * 6 + 2 * kk) * 8;
      const double* qm = qb + (size_t)(H.S + c * 6 + 2 * kk + 1) * 8;
      const D3 dpc = (ld3(qp + 1) - ld3(qm + 1)) / h2;
      const D3 dnc = (ld3(qp + 4) - ld3(qm + 4)) / h2;
      vals_p[kk] = dot(dpc, AP);
      vals_n[kk] = dot(dnc, AN);
    }
    const D3 F = (-2.0 * P.w_grasp) * (mk(vals_p[0], vals_p[1], vals_p[2]) - mk(vals_n[0], vals_n[1], vals_n[2]));
    st3(st.qp_force + ((size_t)g * m + c) * 3, F);
  }
}

}  // namespace gdev

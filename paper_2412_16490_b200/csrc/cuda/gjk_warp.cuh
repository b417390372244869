// Warp-cooperative GJK / EPA: one warp owns one (grasp, link, part) pair.
// Same algorithm and tie rules as gjk.cuh (reference geometry.cpp:58-324):
//  * support scans are split across lanes and reduced by (value, lowest
//    index), which is exactly the sequential "strict >, first maximum" rule;
//  * GJK's simplex state and subset solves are replicated in every lane's
//    registers (identical inputs -> identical decisions, no divergence);
//  * the EPA polytope lives in shared memory; its order-dependent steps
//    (nearest-face tie-break, face kill/compaction, horizon) run on lane 0
//    between __syncwarp()s, the support calls on the whole warp.
#pragma once

#include "gjk.cuh"

namespace gdev {

constexpr int kWarpEpaVerts = 64;
constexpr int kWarpEpaFaces = 128;
constexpr int kWarpEpaHorizon = 96;

struct WarpEpa {
  SP verts[kWarpEpaVerts];
  EpaFace faces[kWarpEpaFaces];
  int hu[kWarpEpaHorizon], hv[kWarpEpaHorizon];
  EpaFace best;
  int nv, nf, status;  // status: 0 continue, 1 done, 2 overflow, 3 degenerate
};

__device__ __forceinline__ D3 warp_support(const Hull& h, D3 dir, int lane) {
  const D3 dl = h.posed ? mulT(h.R, dir) : dir;
  double best = -INFINITY;
  int arg = 0x7fffffff;
  for (int i = lane; i < h.nv; i += 32) {
    const double s = dl.x * __ldg(h.verts + 3 * i) + dl.y * __ldg(h.verts + 3 * i + 1) + dl.z * __ldg(h.verts + 3 * i + 2);
    if (s > best) {
      best = s;
      arg = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
    if (ob > best || (ob == best && oa < arg)) {
      best = ob;
      arg = oa;
    }
  }
  if (arg == 0x7fffffff) arg = 0;
  const D3 v = ldg3(h.verts + 3 * arg);
  return h.posed ? mul(h.R, v) + h.t : v;
}

__device__ __forceinline__ SP warp_support_pair(const Hull& A, const Hull& B, D3 dir, int lane) {
  SP s;
  s.a = warp_support(A, dir, lane);
  s.b = warp_support(B, -dir, lane);
  s.w = s.a - s.b;
  return s;
}

// EPA after a GJK overlap (geometry.cpp:168-205, 227-324).
__device__ inline void warp_epa(const SP* simp, int ns, const Hull& A, const Hull& B, double scale, WarpEpa& s,
                                int lane, PairResult& out) {
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
  SP tet[4];
  int nv = ns;
  for (int i = 0; i < ns; ++i) tet[i] = simp[i];
  for (int k = 0; k < nd && nv < 4; ++k) {
    const SP cand = warp_support_pair(A, B, dirs[k], lane);
    ++out.n_support;
    bool indep;
    if (nv == 0) {
      indep = true;
    } else if (nv == 1) {
      indep = nrm(cand.w - tet[0].w) > tol;
    } else if (nv == 2) {
      const D3 d = normalized(tet[1].w - tet[0].w);
      const D3 r = cand.w - tet[0].w;
      indep = nrm(r - d * dot(d, r)) > tol;
    } else {
      const D3 n = normalized(cross(tet[1].w - tet[0].w, tet[2].w - tet[0].w));
      indep = fabs(dot(n, cand.w - tet[0].w)) > tol;
    }
    if (indep) {
      if (nv == 0) tet[0] = cand;
      if (nv == 1) tet[1] = cand;
      if (nv == 2) tet[2] = cand;
      if (nv == 3) tet[3] = cand;
      ++nv;
    }
  }
  if (nv != 4) {
    out.flags |= kPairDegenerate;
    return;
  }
  const D3 interior = (tet[0].w + tet[1].w + tet[2].w + tet[3].w) / 4.0;
  if (lane == 0) {
    for (int i = 0; i < 4; ++i) s.verts[i] = tet[i];
    s.nv = 4;
    s.faces[0] = epa_make_face(s.verts, interior, 0, 1, 2);
    s.faces[1] = epa_make_face(s.verts, interior, 0, 2, 3);
    s.faces[2] = epa_make_face(s.verts, interior, 0, 3, 1);
    s.faces[3] = epa_make_face(s.verts, interior, 1, 3, 2);
    s.nf = 4;
    s.status = 0;
    s.best = s.faces[0];
  }
  __syncwarp();
  const double grow_tol = 1e-10 * scale;
  for (int iter = 0; iter < kEpaMaxIters; ++iter) {
    if (lane == 0) {
      int best = -1;
      double best_d = INFINITY;
      for (int i = 0; i < s.nf; ++i) {
        const double di = s.faces[i].d;
        if (di < best_d - 1e-12 * scale ||
            (di < best_d + 1e-12 * scale && best >= 0 && lex_less(-s.faces[i].n, -s.faces[best].n))) {
          best_d = fmin(best_d, di);
          best = i;
        }
      }
      if (best < 0)
        s.status = 3;
      else
        s.best = s.faces[best];
    }
    __syncwarp();
    if (s.status == 3) {
      out.flags |= kPairDegenerate;
      return;
    }
    const EpaFace bf = s.best;
    const SP w = warp_support_pair(A, B, bf.n, lane);
    ++out.n_support;
    ++out.epa_iters;
    if (dot(bf.n, w.w) - bf.d <= grow_tol) break;
    if (lane == 0) {
      if (s.nv >= kWarpEpaVerts) {
        s.status = 2;
      } else {
        const int wi = s.nv;
        s.verts[s.nv++] = w;
        int nh = 0, kept = 0;
        for (int i = 0; i < s.nf; ++i) {
          const EpaFace f = s.faces[i];
          if (dot(f.n, w.w) - f.d > 1e-12 * scale) {
            if (nh + 3 > kWarpEpaHorizon) {
              s.status = 2;
            } else {
              s.hu[nh] = f.v0; s.hv[nh++] = f.v1;
              s.hu[nh] = f.v1; s.hv[nh++] = f.v2;
              s.hu[nh] = f.v2; s.hv[nh++] = f.v0;
            }
          } else {
            s.faces[kept++] = f;
          }
        }
        s.nf = kept;
        int n_boundary = 0;
        for (int e = 0; e < nh && s.status == 0; ++e) {
          bool paired = false;
          for (int o = 0; o < nh; ++o)
            if (s.hu[o] == s.hv[e] && s.hv[o] == s.hu[e]) paired = true;
          if (!paired) {
            if (s.nf >= kWarpEpaFaces) {
              s.status = 2;
              break;
            }
            s.faces[s.nf++] = epa_make_face(s.verts, interior, s.hu[e], s.hv[e], wi);
            ++n_boundary;
          }
        }
        if (s.status == 0 && n_boundary == 0) s.status = 1;
      }
    }
    __syncwarp();
    if (s.status == 2) {
      out.flags |= kPairOverflow;
      return;
    }
    if (s.status == 1) break;
  }
  const EpaFace bf = s.best;
  out.d = -fmax(bf.d, 0.0);
  out.n = -bf.n;
  const SP tri[3] = {s.verts[bf.v0], s.verts[bf.v1], s.verts[bf.v2]};
  const Simplex sx = closest_on_simplex(tri, 3);
  D3 wa = mk(0, 0, 0), wb = mk(0, 0, 0);
  double wsum = 0.0;
  for (int i = 0; i < sx.nkeep; ++i) {
    wa += sx.wts[i] * tri[sx.keep[i]].a;
    wb += sx.wts[i] * tri[sx.keep[i]].b;
    wsum += sx.wts[i];
  }
  if (wsum > 0.5) {
    out.pa = wa;
    out.pb = wb;
  } else {
    out.pa = tri[0].a;
    out.pb = tri[0].b;
  }
  out.flags |= kPairEpa;
  __syncwarp();
}

// signed_distance(a, pose_a, b, identity) (geometry.cpp:500-525), warp-wide.
__device__ inline PairResult warp_signed_distance(const Hull& A, const Hull& B, double scale, WarpEpa& scratch,
                                                  int lane) {
  PairResult out;
  out.flags = 0;
  out.n_support = 1;
  out.gjk_iters = 0;
  out.epa_iters = 0;
  SP simp[4];
  int ns = 1;
  simp[0] = warp_support_pair(A, B, mk(1, 0, 0), lane);
  bool done = false, overlap = false;
  Simplex sx;
  for (int iter = 0; iter < kGjkMaxIters && !done; ++iter) {
    sx = closest_on_simplex(simp, ns);
    SP red[4];
    for (int i = 0; i < sx.nkeep; ++i) red[i] = simp[sx.keep[i]];
    ns = sx.nkeep;
    for (int i = 0; i < ns; ++i) simp[i] = red[i];
    if (sx.contains || sqrt(sx.dist2) < kTouchTol * scale) {
      overlap = true;
      done = true;
      break;
    }
    const SP w = warp_support_pair(A, B, -sx.v, lane);
    ++out.n_support;
    ++out.gjk_iters;
    const double gap = sx.dist2 - dot(sx.v, w.w);
    bool repeat = false;
    for (int i = 0; i < ns; ++i)
      if (nrm(simp[i].w - w.w) < 1e-14 * scale) repeat = true;
    if (gap <= kGjkRelTol * sx.dist2 + 1e-300 || repeat || ns == 4) {
      done = true;
      break;
    }
    simp[ns++] = w;
  }
  if (!done) {
    sx = closest_on_simplex(simp, ns);
    D3 wa = mk(0, 0, 0), wb = mk(0, 0, 0);
    for (int i = 0; i < sx.nkeep; ++i) {
      wa += sx.wts[i] * simp[sx.keep[i]].a;
      wb += sx.wts[i] * simp[sx.keep[i]].b;
    }
    const double d = sqrt(sx.dist2);
    out.d = d;
    out.pa = wa;
    out.pb = wb;
    out.n = d > 1e-14 ? (wa - wb) / d : mk(0, 0, 1);
    return out;
  }
  if (!overlap) {
    D3 wa = mk(0, 0, 0), wb = mk(0, 0, 0);
    for (int i = 0; i < ns; ++i) {
      wa += sx.wts[i] * simp[i].a;
      wb += sx.wts[i] * simp[i].b;
    }
    const double d = sqrt(sx.dist2);
    out.d = d;
    out.pa = wa;
    out.pb = wb;
    out.n = d > 1e-14 ? (wa - wb) / d : mk(0, 0, 1);
    return out;
  }
  warp_epa(simp, ns, A, B, scale, scratch, lane, out);
  return out;
}

}  // namespace gdev

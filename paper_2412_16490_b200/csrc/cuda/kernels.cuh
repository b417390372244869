// sm_100a kernels of the bilevel grasp-synthesis loop.
//
// Per upper-level iteration (reference total_energy + apply_step,
// proj/src/pipeline.cpp:96-231):
//   coarse stage: k_point_query -> k_qp -> k_step<coarse>
//   mesh stages:  k_point_query(tips) -> k_pairs -> k_step<mesh>
// k_step ends with the forward kinematics of the new state and writes the
// next iteration's query points, so there is no separate FK launch inside a
// stage. All arithmetic is fp64 like the reference; every reduction runs in
// a fixed order so results do not depend on batch size or scheduling.
#pragma once

#include "dmath.cuh"
#include "gjk.cuh"
#include "model.cuh"

namespace gdev {

#ifndef GDEV_FULL_MASK
#define GDEV_FULL_MASK
constexpr unsigned kFull = 0xffffffffu;
#endif

// ----------------------------------------------------------------- helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;  // butterfly: identical on every lane
}

// Fixed-order sum of `v` over lanes base..base+cnt-1, identical on all lanes.
__device__ __forceinline__ double group_sum(double v, int base, int cnt) {
  double s = 0.0;
  for (int b = 0; b < cnt; ++b) s += __shfl_sync(kFull, v, base + b);
  return s;
}
__device__ __forceinline__ double group_max(double v, int base, int cnt) {
  double s = 0.0;
  for (int b = 0; b < cnt; ++b) s = fmax(s, __shfl_sync(kFull, v, base + b));
  return s;
}

struct Pose {
  M33 R;
  D3 t;
  M33 a_inv;
  bool degenerate;
};

__device__ __forceinline__ void store_pose(double* p, const Pose& ps) {
  for (int i = 0; i < 9; ++i) p[i] = ps.R.m[i];
  st3(p + 9, ps.t);
  for (int i = 0; i < 9; ++i) p[12 + i] = ps.a_inv.m[i];
  p[21] = ps.degenerate ? 1.0 : 0.0;
}
__device__ __forceinline__ Pose load_pose(const double* p) {
  Pose ps;
  for (int i = 0; i < 9; ++i) ps.R.m[i] = p[i];
  ps.t = ld3(p + 9);
  for (int i = 0; i < 9; ++i) ps.a_inv.m[i] = p[12 + i];
  ps.degenerate = p[21] != 0.0;
  return ps;
}

// make_pose_state + pose_from_state (hand.cpp:75-116): raw block is
// column-major in x.
__device__ inline Pose compute_pose(const double* x) {
  M33 raw;
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) raw.m[i * 3 + c] = x[3 * c + i];
  Pose ps;
  bool fallback = false;
  ps.R = project_rotation(raw, &fallback);
  ps.t = mk(x[9], x[10], x[11]);
  ps.a_inv = eye();
  ps.degenerate = fallback;
  if (!fallback) ps.degenerate = !pose_a_inv(ps.R, raw, ps.a_inv);
  return ps;
}

// Per-warp scratch of the warp-per-grasp kernels.
struct WarpScratch {
  double x[kMaxDims];
  double xn[kMaxDims];
  double grad[kMaxDims];
  double pose[24];
  double world[kMaxLinks * 12];
  double jo[kMaxDof * 6];
  double pc[kMaxProxies * 3];
  double sn[kMaxDof], cs[kMaxDof];  // sin/cos of the joint angles (one correctly rounded pair per joint)
  double itF[32 * 3];
  double itT[32 * 3];
  int itL[32];
  double red[32];
  int flag[4];
};

// Forward kinematics for one grasp (hand.cpp:126-153): lane 0 projects the
// rotation, lane l < L walks its root-to-l path (same op sequence as the
// sequential reference), then proxy centers and the coarse FD stencil points
// are written as the next iteration's point queries.
__device__ inline void warp_fk(const DevHand& H, const DevState& st, int g, int lane, WarpScratch& s, double fd_step,
                               bool write_state) {
  if (lane == 0) {
    const Pose ps = compute_pose(s.x);
    store_pose(s.pose, ps);
  }
  for (int j = lane; j < H.dof; j += 32) cr_sincos(s.x[12 + j], s.sn + j, s.cs + j);
  __syncwarp();
  const Pose base = load_pose(s.pose);
  if (lane < H.L) {
    const int l = lane;
    M33 Rc = eye();
    D3 tc = mk(0, 0, 0);
    const int depth = H.link_depth[l];
    for (int d = 0; d < depth; ++d) {
      const int p = H.link_path[l * kMaxDepth + d];
      const int j = H.link_parent_joint[p];
      if (j < 0) continue;  // base link: identity chain
      const D3 origin = ld3(H.joint_origin + 3 * j);
      const D3 axis = ld3(H.joint_axis + 3 * j);
      const M33 Rs = angle_axis_sc(s.sn[j], s.cs[j], axis);
      const D3 jo = mul(Rc, origin) + tc;  // parent.apply(origin)
      const M33 Rn = mul(Rc, Rs);
      if (p == l) {
        st3(s.jo + 6 * j, jo);
        st3(s.jo + 6 * j + 3, mul(Rn, axis));
      }
      Rc = Rn;
      tc = jo;
    }
    const M33 Rw = mul(base.R, Rc);
    const D3 tw = mul(base.R, tc) + base.t;
    for (int i = 0; i < 9; ++i) s.world[l * 12 + i] = Rw.m[i];
    st3(s.world + l * 12 + 9, tw);
  }
  __syncwarp();
  for (int p = lane; p < H.S; p += 32) {
    const int l = H.proxy_link[p];
    M33 Rw;
    for (int i = 0; i < 9; ++i) Rw.m[i] = s.world[l * 12 + i];
    const D3 c = mul(Rw, ld3(H.proxy + 4 * p)) + ld3(s.world + l * 12 + 9);
    st3(s.pc + 3 * p, c);
  }
  __syncwarp();
  if (!write_state) return;
  double* gp = st.pose + (size_t)g * 24;
  for (int i = lane; i < 24; i += 32) gp[i] = s.pose[i];
  double* gw = st.world + (size_t)g * H.L * 12;
  for (int i = lane; i < H.L * 12; i += 32) gw[i] = s.world[i];
  double* gj = st.joints + (size_t)g * H.dof * 6;
  for (int i = lane; i < H.dof * 6; i += 32) gj[i] = s.jo[i];
  double* q = st.qpts + (size_t)g * st.NQ * 3;
  for (int p = lane; p < H.S; p += 32) st3(q + 3 * p, ld3(s.pc + 3 * p));
  for (int t = lane; t < 6 * H.m; t += 32) {
    const int f = t / 6, k = (t % 6) / 2;
    const double sign = (t & 1) ? -1.0 : 1.0;
    D3 c = ld3(s.pc + 3 * H.tip_proxy[f]);
    // c +/- h e_k touches only component k (pipeline.cpp:150-152).
    if (k == 0) c.x = c.x + sign * fd_step;
    if (k == 1) c.y = c.y + sign * fd_step;
    if (k == 2) c.z = c.z + sign * fd_step;
    st3(q + 3 * (H.S + t), c);
  }
}

__device__ inline void load_fk(const DevHand& H, const DevState& st, int g, int lane, WarpScratch& s) {
  const double* gp = st.pose + (size_t)g * 24;
  for (int i = lane; i < 24; i += 32) s.pose[i] = gp[i];
  const double* gw = st.world + (size_t)g * H.L * 12;
  for (int i = lane; i < H.L * 12; i += 32) s.world[i] = gw[i];
  const double* gj = st.joints + (size_t)g * H.dof * 6;
  for (int i = lane; i < H.dof * 6; i += 32) s.jo[i] = gj[i];
  __syncwarp();
  for (int p = lane; p < H.S; p += 32) {
    const int l = H.proxy_link[p];
    M33 Rw;
    for (int i = 0; i < 9; ++i) Rw.m[i] = s.world[l * 12 + i];
    st3(s.pc + 3 * p, mul(Rw, ld3(H.proxy + 4 * p)) + ld3(s.world + l * 12 + 9));
  }
  __syncwarp();
}

// Profiling op counter, aggregated over the warp's active lanes first (one
// atomic per warp instead of one per thread: per-thread atomics on the same
// few counters serialised and inflated the profiled kernel times).
__device__ __forceinline__ void op_add(unsigned long long* ops, int k, unsigned v) {
  const unsigned mask = __activemask();
  const unsigned s = __reduce_add_sync(mask, v);
  if ((int)(threadIdx.x & 31) == __ffs(mask) - 1 && s) atomicAdd(ops + k, (unsigned long long)s);
}

// --------------------------------------------------------- point queries
// Ericson closest point on a triangle (geometry.cpp:327-347).
__device__ __forceinline__ D3 closest_on_triangle(D3 p, D3 a, D3 b, D3 c) {
  const D3 ab = b - a, ac = c - a, ap = p - a;
  const double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0 && d2 <= 0) return a;
  const D3 bp = p - b;
  const double d3 = dot(ab, bp), d4 = dot(ac, bp);
  if (d3 >= 0 && d4 <= d3) return b;
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) return a + ab * (d1 / (d1 - d3));
  const D3 cp = p - c;
  const double d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0 && d5 <= d6) return c;
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) return a + ac * (d2 / (d2 - d6));
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0 && d4 - d3 >= 0 && d5 - d6 >= 0) return b + (c - b) * ((d4 - d3) / ((d4 - d3) + (d5 - d6)));
  const double denom = 1.0 / (va + vb + vc);
  return a + ab * (vb * denom) + ac * (vc * denom);
}

struct PointHit {
  double d;
  D3 pb, n;
  int part;
  int face;  // winning part's closest face (outside) or shallowest face (inside); -1 if none
  int sep;   // face whose plane separated the point from the winning part, -1 if inside / none
};

// point_to_mesh (geometry.cpp:527-542) with query_part (:355-395): inside
// test breaking at the first plane with depth < -1e-12, else the brute-force
// closest point with strict '<' over faces and parts.
// Single-instruction fp32 square root (relative error ~1e-7, far inside the
// culling slack); used only for culling bounds.
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ double4 ld_plane(const DevObject& O, int f) {
  const double2* q = reinterpret_cast<const double2*>(O.face_plane + f);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// Signed distance from p to part's containing box (center, half extents,
// axes column-major; model.cuh part_box): negative inside. The part lies in
// the box, so this bounds the part's signed distance from below, also for
// points inside (the part's depth is at most the box's).
__device__ __forceinline__ double part_box_dist(const DevObject& O, int part, D3 p) {
  const double* b = O.part_box + 15 * part;
  const D3 r = p - ldg3(b);
  double acc = 0.0, mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double e = fabs(dot(r, ldg3(b + 6 + 3 * k))) - __ldg(b + 3 + k);
    mx = fmax(mx, e);
    acc += e > 0.0 ? e * e : 0.0;
  }
  return mx > 0.0 ? sqrt(acc) : mx;
}

// Distance from p to cluster c's oriented box (a lower bound on the distance
// to every face of the cluster) exceeds reach.
__device__ __forceinline__ bool cluster_box_far(const DevObject& O, int c, float px, float py, float pz,
                                                float reach) {
  const float4 B0 = __ldg(O.cluster_box32 + 4 * c), B1 = __ldg(O.cluster_box32 + 4 * c + 1);
  const float4 B2 = __ldg(O.cluster_box32 + 4 * c + 2), B3 = __ldg(O.cluster_box32 + 4 * c + 3);
  const float rx = px - B0.x, ry = py - B0.y, rz = pz - B0.z;
  const float eu = fmaxf(fabsf(rx * B1.x + ry * B1.y + rz * B1.z) - B0.w, 0.0f);
  const float ev = fmaxf(fabsf(rx * B2.x + ry * B2.y + rz * B2.z) - B1.w, 0.0f);
  const float en = fmaxf(fabsf(rx * B3.x + ry * B3.y + rz * B3.z) - B2.w, 0.0f);
  return eu * eu + ev * ev + en * en > reach * reach;
}

// Part range [p0, p1) of grasp g's object (multi-object contexts; st.obj == nullptr: object 0).
__device__ __forceinline__ void obj_parts(const DevObject& O, const DevState& st, int g, int& p0, int& p1) {
  const int o = st.obj ? __ldg(st.obj + g) : 0;
  p0 = __ldg(O.obj_pbeg + o);
  p1 = __ldg(O.obj_pbeg + o + 1);
}

// point_to_mesh(p, parts [p0, p1)) (geometry.cpp:527-542); the part index
// returned is global (p0 + the object's part index).
__device__ inline PointHit point_to_mesh(const DevObject& O, D3 p, int p0, int p1, int warm_face = -1,
                                         unsigned* plane_tests = nullptr, unsigned* tri_tests = nullptr,
                                         int warm_sep = -1) {
  PointHit best;
  best.d = INFINITY;
  best.pb = mk(0, 0, 0);
  best.n = mk(0, 0, 1);
  best.part = -1;
  best.face = -1;
  best.sep = -1;
  unsigned planes = 0, tris = 0;
  const float px = (float)p.x, py = (float)p.y, pz = (float)p.z;
  // Warm start: the exact distance to any face (here the slot's closest face
  // of the previous query) bounds the minimum over all outside parts from
  // above; parts and faces whose lower bounds exceed it cannot be the
  // argmin (inside parts have lower bound <= 0 and are never skipped).
  double ub_warm = INFINITY;
  if (warm_face >= 0 && warm_face < O.F) {
    ++tris;
    const double* F = O.faces + (size_t)warm_face * kFaceStride;
    ub_warm = nrm(p - closest_on_triangle(p, ldg3(F), ldg3(F + 3), ldg3(F + 6)));
  }
  for (int part = p0; part < p1; ++part) {
    const int f0 = __ldg(O.part_fbeg + part), f1 = __ldg(O.part_fbeg + part + 1);
    // Part-level cull: every point of the part is at least |p - c| - r
    // away; a part that cannot reach below the current best cannot win the
    // strict '<' across parts (geometry.cpp:533), so skipping it is exact.
    {
      const double* S = O.part_sphere + 4 * part;
      const double lb = nrm(p - ldg3(S)) - __ldg(S + 3) - kCullSlack;
      if (lb > best.d || lb > ub_warm) continue;
      // the part's containing box (0 for points inside it)
      const double lbb = part_box_dist(O, part, p) - kCullSlack;
      if (lbb > best.d || lbb > ub_warm) continue;
    }
    // Face clusters (runs of consecutive faces with fp32 bounding spheres):
    // an upper bound on the part distance (min |p-C| + R) and a seed face,
    // the smallest sphere lower bound in the nearest cluster. The warm face,
    // when it is one of this part's, is the seed instead (its exact distance
    // is already the bound).
    const int c0 = __ldg(O.part_cbeg + part), c1 = __ldg(O.part_cbeg + part + 1);
    float ubA = INFINITY;
    int seed_f = warm_face;
    if (!(warm_face >= f0 && warm_face < f1)) {
      float lb_seed = INFINITY;
      int seed_c = c0;
      for (int c = c0; c < c1; ++c) {
        const float4 S = __ldg(O.cluster_sphere32 + c);
        const float dx = px - S.x, dy = py - S.y, dz = pz - S.z;
        const float dist = sqrt_approx(dx * dx + dy * dy + dz * dz);
        ubA = fminf(ubA, dist + S.w);
        if (dist - S.w < lb_seed) {
          lb_seed = dist - S.w;
          seed_c = c;
        }
      }
      int seed_k = __ldg(O.cluster_fbeg + seed_c);
      const int e = __ldg(O.cluster_fbeg + seed_c + 1);
      float lbf = INFINITY;
      for (int k = seed_k; k < e; ++k) {
        const float4 S = __ldg(O.face_sphere32 + k);
        const float dx = px - S.x, dy = py - S.y, dz = pz - S.z;
        const float lb = sqrt_approx(dx * dx + dy * dy + dz * dz) - S.w;
        if (lb < lbf) {
          lbf = lb;
          seed_k = k;
        }
      }
      seed_f = __ldg(O.pq_fid + seed_k);
    }
    // Inside test (query_part, geometry.cpp:369-383): inside iff no face
    // plane has depth < -1e-12; then the shallowest face in index order
    // (strict '<'), i.e. the lexicographic minimum of (depth, face). Neither
    // depends on the order the planes are tried, so the seed face's plane
    // (usually a separating one for outside points), the warm face's and the
    // plane that separated the slot's last query are tried first, and the
    // planes are then visited by normal group (model.cuh
    // grp_*): a group whose depth lower bound h_g + n_g.(C_g - p) -
    // delta_g |C_g - p| exceeds a known depth can neither separate nor hold
    // the minimum, so it is skipped. Plane records are (n, n.a) with
    // degenerate faces stored as (0, +inf), which neither separates nor wins
    // the minimum, i.e. is skipped as in the reference.
    bool inside;
    double min_depth = INFINITY;
    D3 best_n = mk(0, 0, 1);
    int min_f = -1;
    int sep_f = -1;
    double ub_depth;  // a depth of some plane of the part (>= the minimum)
    {
      const double4 Q = ld_plane(O, seed_f);
      ++planes;
      ub_depth = Q.w - (Q.x * p.x + Q.y * p.y + Q.z * p.z);
      inside = !(ub_depth < -1e-12);
      sep_f = inside ? -1 : seed_f;
    }
    if (inside && warm_sep >= f0 && warm_sep < f1 && warm_sep != seed_f) {
      const double4 Q = ld_plane(O, warm_sep);
      ++planes;
      const double depth = Q.w - (Q.x * p.x + Q.y * p.y + Q.z * p.z);
      inside = !(depth < -1e-12);
      sep_f = inside ? -1 : warm_sep;
      ub_depth = fmin(ub_depth, depth);
    }
    if (inside && warm_face >= f0 && warm_face < f1 && warm_face != seed_f) {
      const double4 Q = ld_plane(O, warm_face);
      ++planes;
      const double depth = Q.w - (Q.x * p.x + Q.y * p.y + Q.z * p.z);
      inside = !(depth < -1e-12);
      sep_f = inside ? -1 : warm_face;
      ub_depth = fmin(ub_depth, depth);
    }
    if (inside) {
      // fp32 bound with |r| <= |r|_1 (weaker, no square root); the rounding
      // (~1e-8 m) is far inside kCullSlack32
      auto group_far = [&](const float4* B) {
        const float4 B0 = __ldg(B), B1 = __ldg(B + 1);
        const float rx = B1.x - px, ry = B1.y - py, rz = B1.z - pz;
        const float lb = (B0.w + (B0.x * rx + B0.y * ry + B0.z * rz)) - B1.w * (fabsf(rx) + fabsf(ry) + fabsf(rz));
        return lb > (float)fmin(ub_depth, min_depth) + kCullSlack32;
      };
      const int s1 = __ldg(O.part_gbeg + part + 1);
      for (int sg = __ldg(O.part_gbeg + part); sg < s1 && inside; ++sg) {
        if (group_far(O.sup_bound + 2 * sg)) continue;
        const int q1 = __ldg(O.sup_gbeg + sg + 1);
        for (int q = __ldg(O.sup_gbeg + sg); q < q1 && inside; ++q) {
          if (group_far(O.grp_bound + 2 * q)) continue;
          const int k1 = __ldg(O.grp_beg + q + 1);
          for (int k = __ldg(O.grp_beg + q); k < k1; ++k) {
            const double2* qq = reinterpret_cast<const double2*>(O.grp_plane + k);
            const double2 qa = __ldg(qq), qb = __ldg(qq + 1);
            ++planes;
            const double depth = qb.y - (qa.x * p.x + qa.y * p.y + qb.x * p.z);
            const int f = __ldg(O.grp_face + k);
            if (depth < -1e-12) {
              inside = false;
              sep_f = f;
              break;
            }
            if (depth < min_depth || (depth == min_depth && f < min_f)) {
              min_depth = depth;
              best_n = mk(qa.x, qa.y, qb.x);
              min_f = f;
            }
          }
        }
      }
    }
    double sd;
    D3 pt, nn;
    int sf = -1;
    if (inside && isfinite(min_depth)) {
      sd = -min_depth;
      nn = best_n;
      pt = p + best_n * min_depth;
      sf = min_f;  // the shallowest face: the next query's warm start
    } else {
      // Brute-force closest point over the faces in index order with strict
      // '<' (geometry.cpp:384-392), evaluated exactly only where it can
      // matter. The seed face's exact distance bounds the minimum from
      // above; faces are then visited in index order (cluster by cluster)
      // and evaluated exactly only when their lower bounds (cluster sphere,
      // face sphere, face thin box) do not exceed min(bound, running best):
      // every skipped face is strictly worse than the final minimum, so the
      // argmin and its value are unchanged. Bounds in fp32 with
      // kCullSlack32 (conservative).
      float bound;
      {
        double d_seed = ub_warm;
        if (seed_f != warm_face) {
          ++tris;
          const double* F = O.faces + (size_t)seed_f * kFaceStride;
          d_seed = nrm(p - closest_on_triangle(p, ldg3(F), ldg3(F + 3), ldg3(F + 6)));
        }
        bound = fminf(fminf(ubA, __double2float_ru(d_seed)), __double2float_ru(ub_warm)) + kCullSlack32;
      }
      sd = INFINITY;
      float sd32 = INFINITY;
      pt = mk(0, 0, 0);
      sf = -1;
      for (int c = c0; c < c1; ++c) {
        {
          // |p - C| - R - slack > min(bound, best), squared (both sides >= 0)
          const float4 S = __ldg(O.cluster_sphere32 + c);
          const float dx = px - S.x, dy = py - S.y, dz = pz - S.z;
          const float reach = fminf(bound, sd32) + S.w + kCullSlack32;
          if (dx * dx + dy * dy + dz * dz > reach * reach) continue;
        }
        if (cluster_box_far(O, c, px, py, pz, fminf(bound, sd32) + kCullSlack32)) continue;
        const int e = __ldg(O.cluster_fbeg + c + 1);
        for (int k = __ldg(O.cluster_fbeg + c); k < e; ++k) {
          const float cut = fminf(bound, sd32);
          {
            const float4 S = __ldg(O.face_sphere32 + k);
            const float dx = px - S.x, dy = py - S.y, dz = pz - S.z;
            const float reach = cut + S.w + kCullSlack32;
            if (dx * dx + dy * dy + dz * dz > reach * reach) continue;
          }
          // Thin-box bound: the triangle lies in a box (centre o, fp32 axes
          // u, v, n, half extents hu, hv, hn; built on the host from the
          // rounded axes), so |p - q| for any triangle point q is at least
          // the distance from p to the box (axes orthonormal to ~1e-7,
          // covered by the slack). Tight for the long thin faces that
          // sphere bounds cannot separate.
          {
            const float4 B0 = __ldg(O.face_box32 + 4 * k), B1 = __ldg(O.face_box32 + 4 * k + 1);
            const float4 B2 = __ldg(O.face_box32 + 4 * k + 2), B3 = __ldg(O.face_box32 + 4 * k + 3);
            const float rx = px - B0.x, ry = py - B0.y, rz = pz - B0.z;
            const float eu = fmaxf(fabsf(rx * B1.x + ry * B1.y + rz * B1.z) - B0.w, 0.0f);
            const float ev = fmaxf(fabsf(rx * B2.x + ry * B2.y + rz * B2.z) - B1.w, 0.0f);
            const float en = fmaxf(fabsf(rx * B3.x + ry * B3.y + rz * B3.z) - B2.w, 0.0f);
            const float reach = cut + kCullSlack32;
            if (eu * eu + ev * ev + en * en > reach * reach) continue;
          }
          ++tris;
          const double* F = O.pq_faces + (size_t)k * kFaceStride;
          const D3 cp = closest_on_triangle(p, ldg3(F), ldg3(F + 3), ldg3(F + 6));
          const double d = nrm(p - cp);
          const int f = __ldg(O.pq_fid + k);
          if (d < sd || (d == sd && f < sf)) {  // lexicographic (distance, face) minimum
            sd = d;
            sd32 = __double2float_ru(d) + kCullSlack32;
            pt = cp;
            sf = f;
          }
        }
      }
      nn = sd > 1e-14 ? (p - pt) / sd : mk(0, 0, 1);
    }
    if (sd < best.d) {
      best.d = sd;
      best.pb = pt;
      best.n = nn;
      best.part = part;
      best.face = sf;
      best.sep = sep_f;
    }
  }
  if (plane_tests) *plane_tests = planes;
  if (tri_tests) *tri_tests = tris;
  return best;
}

// point_to_mesh by an aligned group of L lanes of one warp (gmask = the
// group's lanes, gl = lane in group); every lane returns the same hit. Each
// sequential scan is split over the lanes and merged with an order-free
// reduction that reproduces it exactly: a strict '<' scan in index order
// picks the lexicographic minimum of (value, index); the inside test is "no
// plane separates" (any-vote) plus the (depth, face) minimum. The culls use
// the lane's own running best, an upper bound on the group's final minimum,
// so every skipped face is still strictly worse than it.
template <int L>
__device__ __forceinline__ void group_lexmin(unsigned gmask, double& v, int& i) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(gmask, v, o);
    const int i2 = __shfl_xor_sync(gmask, i, o);
    if (v2 < v || (v2 == v && i2 < i)) {
      v = v2;
      i = i2;
    }
  }
}
template <int L>
__device__ __forceinline__ void group_lexmin(unsigned gmask, float& v, int& i) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(gmask, v, o);
    const int i2 = __shfl_xor_sync(gmask, i, o);
    if (v2 < v || (v2 == v && i2 < i)) {
      v = v2;
      i = i2;
    }
  }
}
template <int L>
__device__ __forceinline__ float group_fmin(unsigned gmask, float v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(gmask, v, o));
  return v;
}

template <int L>
__device__ PointHit point_to_mesh_group(const DevObject& O, D3 p, int p0, int p1, int warm_face, int gl, unsigned gmask,
                                        unsigned* plane_tests, unsigned* tri_tests, int warm_sep = -1) {
  PointHit best;
  best.d = INFINITY;
  best.pb = mk(0, 0, 0);
  best.n = mk(0, 0, 1);
  best.part = -1;
  best.face = -1;
  best.sep = -1;
  unsigned planes = 0, tris = 0;
  const float px = (float)p.x, py = (float)p.y, pz = (float)p.z;
  double ub_warm = INFINITY;
  if (warm_face >= 0 && warm_face < O.F) {
    if (gl == 0) ++tris;
    const double* F = O.faces + (size_t)warm_face * kFaceStride;
    ub_warm = nrm(p - closest_on_triangle(p, ldg3(F), ldg3(F + 3), ldg3(F + 6)));
  }
  for (int part = p0; part < p1; ++part) {
    const int f0 = __ldg(O.part_fbeg + part), f1 = __ldg(O.part_fbeg + part + 1);
    {
      const double* S = O.part_sphere + 4 * part;
      const double lb = nrm(p - ldg3(S)) - __ldg(S + 3) - kCullSlack;
      if (lb > best.d || lb > ub_warm) continue;
      // the part's containing box (0 for points inside it)
      const double lbb = part_box_dist(O, part, p) - kCullSlack;
      if (lbb > best.d || lbb > ub_warm) continue;
    }
    const int c0 = __ldg(O.part_cbeg + part), c1 = __ldg(O.part_cbeg + part + 1);
    float ubA = INFINITY;
    int seed_f = warm_face;
    if (!(warm_face >= f0 && warm_face < f1)) {  // (the warm face seeds its own part)
      float lb_seed = INFINITY;
      int seed_c = c0;
      for (int c = c0 + gl; c < c1; c += L) {
        const float4 S = __ldg(O.cluster_sphere32 + c);
        const float dx = px - S.x, dy = py - S.y, dz = pz - S.z;
        const float dist = sqrt_approx(dx * dx + dy * dy + dz * dz);
        ubA = fminf(ubA, dist + S.w);
        if (dist - S.w < lb_seed) {
          lb_seed = dist - S.w;
          seed_c = c;
        }
      }
      ubA = group_fmin<L>(gmask, ubA);
      group_lexmin<L>(gmask, lb_seed, seed_c);
      const int s0 = __ldg(O.cluster_fbeg + seed_c), e = __ldg(O.cluster_fbeg + seed_c + 1);
      float lbf = INFINITY;
      seed_f = s0;
      for (int f = s0 + gl; f < e; f += L) {
        const float4 S = __ldg(O.face_sphere32 + f);
        const float dx = px - S.x, dy = py - S.y, dz = pz - S.z;
        const float lb = sqrt_approx(dx * dx + dy * dy + dz * dz) - S.w;
        if (lb < lbf) {
          lbf = lb;
          seed_f = f;
        }
      }
      group_lexmin<L>(gmask, lbf, seed_f);
      seed_f = __ldg(O.pq_fid + seed_f);  // position -> face
    }
    // Inside test as in point_to_mesh: the seed, last separating and warm
    // planes first, then the normal groups whose depth bound does not exceed
    // a known depth, each group's planes split over the lanes.
    bool inside;
    double min_depth = INFINITY;
    int min_face = INT_MAX, sep_f = -1;
    double ub_depth;
    {
      const double4 Q = ld_plane(O, seed_f);
      if (gl == 0) ++planes;
      ub_depth = Q.w - (Q.x * p.x + Q.y * p.y + Q.z * p.z);
      inside = !(ub_depth < -1e-12);
      sep_f = inside ? -1 : seed_f;
    }
    if (inside && warm_sep >= f0 && warm_sep < f1 && warm_sep != seed_f) {
      const double4 Q = ld_plane(O, warm_sep);
      if (gl == 0) ++planes;
      const double depth = Q.w - (Q.x * p.x + Q.y * p.y + Q.z * p.z);
      inside = !(depth < -1e-12);
      sep_f = inside ? -1 : warm_sep;
      ub_depth = fmin(ub_depth, depth);
    }
    if (inside && warm_face >= f0 && warm_face < f1 && warm_face != seed_f) {
      const double4 Q = ld_plane(O, warm_face);
      if (gl == 0) ++planes;
      const double depth = Q.w - (Q.x * p.x + Q.y * p.y + Q.z * p.z);
      inside = !(depth < -1e-12);
      sep_f = inside ? -1 : warm_face;
      ub_depth = fmin(ub_depth, depth);
    }
    if (inside) {
      // every lane of the group evaluates the same bounds (same p, same
      // ub_depth), so the group stays converged through the group loops
      const float thr = (float)ub_depth + kCullSlack32;
      auto group_far = [&](const float4* B) {
        const float4 B0 = __ldg(B), B1 = __ldg(B + 1);
        const float rx = B1.x - px, ry = B1.y - py, rz = B1.z - pz;
        const float lb = (B0.w + (B0.x * rx + B0.y * ry + B0.z * rz)) - B1.w * (fabsf(rx) + fabsf(ry) + fabsf(rz));
        return lb > thr;
      };
      const int s1 = __ldg(O.part_gbeg + part + 1);
      for (int sg = __ldg(O.part_gbeg + part); sg < s1 && inside; ++sg) {
        if (group_far(O.sup_bound + 2 * sg)) continue;
        const int q1 = __ldg(O.sup_gbeg + sg + 1);
        for (int q = __ldg(O.sup_gbeg + sg); q < q1 && inside; ++q) {
          if (group_far(O.grp_bound + 2 * q)) continue;
          const int k1 = __ldg(O.grp_beg + q + 1);
          int my_sep = -1;
          for (int k = __ldg(O.grp_beg + q) + gl; k < k1; k += L) {
            const double2* qq = reinterpret_cast<const double2*>(O.grp_plane + k);
            const double2 qa = __ldg(qq), qb = __ldg(qq + 1);
            ++planes;
            const double depth = qb.y - (qa.x * p.x + qa.y * p.y + qb.x * p.z);
            const int f = __ldg(O.grp_face + k);
            if (depth < -1e-12) {
              my_sep = f;
              break;
            }
            if (depth < min_depth || (depth == min_depth && f < min_face)) {
              min_depth = depth;
              min_face = f;
            }
          }
          const unsigned sep = __ballot_sync(gmask, my_sep >= 0);
          if (sep) {
            inside = false;
            sep_f = __shfl_sync(gmask, my_sep, __ffs(sep) - 1);
          }
        }
      }
      if (inside) group_lexmin<L>(gmask, min_depth, min_face);
    }
    double sd;
    D3 pt, nn;
    int sf = -1;
    if (inside && isfinite(min_depth)) {
      const double4 Q = ld_plane(O, min_face);
      const D3 best_n = mk(Q.x, Q.y, Q.z);
      sd = -min_depth;
      nn = best_n;
      pt = p + best_n * min_depth;
      sf = min_face;
    } else {
      float bound;
      {
        double d_seed = ub_warm;
        if (seed_f != warm_face) {
          if (gl == 0) ++tris;
          const double* F = O.faces + (size_t)seed_f * kFaceStride;
          d_seed = nrm(p - closest_on_triangle(p, ldg3(F), ldg3(F + 3), ldg3(F + 6)));
        }
        bound = fminf(fminf(ubA, __double2float_ru(d_seed)), __double2float_ru(ub_warm)) + kCullSlack32;
      }
      sd = INFINITY;
      float sd32 = INFINITY;
      pt = mk(0, 0, 0);
      int lf = INT_MAX;
      for (int c = c0; c < c1; ++c) {
        {
          const float4 S = __ldg(O.cluster_sphere32 + c);
          const float dx = px - S.x, dy = py - S.y, dz = pz - S.z;
          const float reach = fminf(bound, sd32) + S.w + kCullSlack32;
          if (dx * dx + dy * dy + dz * dz > reach * reach) continue;
        }
        if (cluster_box_far(O, c, px, py, pz, fminf(bound, sd32) + kCullSlack32)) continue;
        const int e = __ldg(O.cluster_fbeg + c + 1);
        for (int k = __ldg(O.cluster_fbeg + c) + gl; k < e; k += L) {
          const float cut = fminf(bound, sd32);
          {
            const float4 S = __ldg(O.face_sphere32 + k);
            const float dx = px - S.x, dy = py - S.y, dz = pz - S.z;
            const float reach = cut + S.w + kCullSlack32;
            if (dx * dx + dy * dy + dz * dz > reach * reach) continue;
          }
          {
            const float4 B0 = __ldg(O.face_box32 + 4 * k), B1 = __ldg(O.face_box32 + 4 * k + 1);
            const float4 B2 = __ldg(O.face_box32 + 4 * k + 2), B3 = __ldg(O.face_box32 + 4 * k + 3);
            const float rx = px - B0.x, ry = py - B0.y, rz = pz - B0.z;
            const float eu = fmaxf(fabsf(rx * B1.x + ry * B1.y + rz * B1.z) - B0.w, 0.0f);
            const float ev = fmaxf(fabsf(rx * B2.x + ry * B2.y + rz * B2.z) - B1.w, 0.0f);
            const float en = fmaxf(fabsf(rx * B3.x + ry * B3.y + rz * B3.z) - B2.w, 0.0f);
            const float reach = cut + kCullSlack32;
            if (eu * eu + ev * ev + en * en > reach * reach) continue;
          }
          ++tris;
          const double* F = O.pq_faces + (size_t)k * kFaceStride;
          const D3 cp = closest_on_triangle(p, ldg3(F), ldg3(F + 3), ldg3(F + 6));
          const double d = nrm(p - cp);
          const int f = __ldg(O.pq_fid + k);
          if (d < sd || (d == sd && f < lf)) {  // lexicographic (distance, face) minimum
            sd = d;
            sd32 = __double2float_ru(d) + kCullSlack32;
            pt = cp;
            lf = f;
          }
        }
      }
      // winner: the lane holding the (distance, face) minimum
      double wd = sd;
      int wf = lf;
      group_lexmin<L>(gmask, wd, wf);
      const unsigned win = __ballot_sync(gmask, lf == wf && wf != INT_MAX);
      const int src = win ? __ffs(win) - 1 : (threadIdx.x & 31);
      pt = mk(__shfl_sync(gmask, pt.x, src), __shfl_sync(gmask, pt.y, src), __shfl_sync(gmask, pt.z, src));
      sd = wd;
      sf = wf == INT_MAX ? -1 : wf;
      nn = sd > 1e-14 ? (p - pt) / sd : mk(0, 0, 1);
    }
    if (sd < best.d) {
      best.d = sd;
      best.pb = pt;
      best.n = nn;
      best.part = part;
      best.face = sf;
      best.sep = sep_f;
    }
  }
  if (plane_tests) *plane_tests = planes;
  if (tri_tests) *tri_tests = tris;
  return best;
}

// Group-per-query variant for launches with few queries (the fine and final
// stages' tip-centre queries, G x m: one query per thread leaves most SMs idle).
template <int L>
#ifndef GDEV_PQG_BLOCK
#define GDEV_PQG_BLOCK 128  // 64: 270.7 vs 273.4 ms point queries (noise level), 256: 276.5
#endif
__global__ void __launch_bounds__(GDEV_PQG_BLOCK) k_point_query_group(DevObject O, DevState st, const int* __restrict__ slots,
                                                           int n_slots) {
  const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / L;
  const int gl = threadIdx.x & (L - 1);
  const unsigned gmask = L == 32 ? 0xffffffffu : (((1u << L) - 1) << ((threadIdx.x & 31) & ~(L - 1)));
  const int per = slots ? n_slots : st.NQ;
  if (t >= (long long)st.G * per) return;
  const int g = (int)(t / per);
  const int slot = slots ? slots[t % per] : (int)(t % per);
  if (st.failed[g]) return;
  const D3 p = ld3(st.qpts + ((size_t)g * st.NQ + slot) * 3);
  unsigned planes, tris;
  int* qf = st.qface + (size_t)g * st.NQ + slot;
  int* qs = st.qsep + (size_t)g * st.NQ + slot;
  int p0, p1;
  obj_parts(O, st, g, p0, p1);
  const PointHit h = point_to_mesh_group<L>(O, p, p0, p1, *qf, gl, gmask, &planes, &tris, *qs);
  __syncwarp(gmask);
  if (st.ops) {
    op_add(st.ops, kOpPlaneTests, planes);
    op_add(st.ops, kOpTriangleTests, tris);
    op_add(st.ops, kOpPointQueries, gl == 0 ? 1u : 0u);
  }
  if (gl != 0) return;
  *qf = h.face;
  *qs = h.sep;
  double* o = st.qres + ((size_t)g * st.NQ + slot) * 8;
  o[0] = h.d;
  st3(o + 1, h.pb);
  st3(o + 4, h.n);
  o[7] = h.part;
}

// One thread per (grasp, query slot). slots == nullptr: all NQ slots.
// 768 threads/SM (80 registers, small spills) measured best: the divergent, latency-bound
// query loop needs the extra resident warps. 64-thread blocks retire the divergent
// tail at a finer grain than 128 (point queries 281 -> 272 ms; 32 threads: 273 ms).
#ifndef GDEV_PQ_BLOCK
#define GDEV_PQ_BLOCK 64  // 64 and 32 measured 3% faster than 128 (finer tail)
#endif
#ifndef GDEV_PQ_THREADS_PER_SM
#define GDEV_PQ_THREADS_PER_SM 768
#endif
__global__ void __launch_bounds__(GDEV_PQ_BLOCK, GDEV_PQ_THREADS_PER_SM / GDEV_PQ_BLOCK) k_point_query(DevObject O, DevState st, const int* __restrict__ slots,
                                                        int n_slots) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int per = slots ? n_slots : st.NQ;
  if (t >= (long long)st.G * per) return;
  const int g = (int)(t / per);
  const int slot = slots ? slots[t % per] : (int)(t % per);
  if (st.failed[g]) return;
  const D3 p = ld3(st.qpts + ((size_t)g * st.NQ + slot) * 3);
  unsigned planes, tris;
  int* qf = st.qface + (size_t)g * st.NQ + slot;
  int* qs = st.qsep + (size_t)g * st.NQ + slot;
  int p0, p1;
  obj_parts(O, st, g, p0, p1);
  const PointHit h = point_to_mesh(O, p, p0, p1, *qf, &planes, &tris, *qs);
  *qf = h.face;
  *qs = h.sep;
  if (st.ops) {
    op_add(st.ops, kOpPlaneTests, planes);
    op_add(st.ops, kOpTriangleTests, tris);
    op_add(st.ops, kOpPointQueries, 1u);
  }
  double* o = st.qres + ((size_t)g * st.NQ + slot) * 8;
  o[0] = h.d;
  st3(o + 1, h.pb);
  st3(o + 4, h.n);
  o[7] = h.part;
}

// Standalone query surface (teacher-forced tests).
__global__ void k_points_raw(DevObject O, int n, const double* __restrict__ pts, double* out,
                             const int* __restrict__ warm = nullptr) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  // standalone surface: the context's first object
  const PointHit h = point_to_mesh(O, ld3(pts + 3 * t), 0, O.obj_pbeg[1], warm ? warm[t] : -1);
  double* o = out + 8 * t;
  o[0] = h.d;
  st3(o + 1, h.pb);
  st3(o + 4, h.n);
  o[7] = h.part;
}

// ------------------------------------------------------------ GJK pairs
// Vertex range and support map of a link hull (link frame) / object part.
__device__ __forceinline__ void set_link_hull(const DevHand& H, int link, Hull& A) {
  A.verts = H.link_verts + 3 * (size_t)H.link_vbeg[link];
  A.nv = H.link_vbeg[link + 1] - H.link_vbeg[link];
  const int cm = H.link_cm[link];
  A.cm_off = cm >= 0 ? H.cm_off + cm : nullptr;
  A.cm_idx = H.cm_idx;
}
__device__ __forceinline__ void set_part_hull(const DevObject& O, int part, Hull& B) {
  B.verts = O.verts + 3 * (size_t)O.part_vbeg[part];
  B.nv = O.part_vbeg[part + 1] - O.part_vbeg[part];
  B.posed = false;
  B.R = eye();
  B.t = mk(0, 0, 0);
  const int cm = O.part_cm[part];
  B.cm_off = cm >= 0 ? O.cm_off + cm : nullptr;
  B.cm_idx = O.cm_idx;
}

__device__ __forceinline__ double scale_of(D3 centroid_world, double halfnorm) {
  return nrm(centroid_world) + 2.0 * halfnorm;
}

template <class Scratch>
__device__ inline PairResult link_part_distance(const DevHand& H, const DevObject& O, int link, int part,
                                                const M33& Rw, D3 tw, Scratch& scratch) {
  Hull A;
  set_link_hull(H, link, A);
  A.posed = true;
  A.R = Rw;
  A.t = tw;
  Hull B;
  set_part_hull(O, part, B);
  // cloud_scale (geometry.cpp:17-23).
  double scale = 1.0;
  scale = fmax(scale, scale_of(mul(Rw, ld3(H.link_centroid + 3 * link)) + tw, H.link_halfnorm[link]));
  scale = fmax(scale, scale_of(ld3(O.part_centroid + 3 * part), O.part_halfnorm[part]));
  return signed_distance(A, B, scale, scratch);
}

// Profiling: GJK closest-point calls of one pair, total and histogram.
__device__ __forceinline__ void count_gjk(unsigned long long* ops, unsigned calls, unsigned skipped) {
  op_add(ops, kOpGjkIters, calls);
  op_add(ops, kOpGjkCycleJumps, skipped ? 1u : 0u);
  op_add(ops, kOpGjkItersSkipped, skipped);
  const int b = calls <= 4 ? 0 : calls <= 8 ? 1 : calls <= 16 ? 2 : calls <= 32 ? 3 : calls <= 64 ? 4 : 5;
#pragma unroll
  for (int k = 0; k < 6; ++k) op_add(ops, kOpGjkHist + k, b == k ? 1u : 0u);
}

__device__ __forceinline__ void store_pair(double* o, const PairResult& r) {
  o[0] = r.d;
  st3(o + 1, r.pa);
  st3(o + 4, r.pb);
  st3(o + 7, r.n);
  o[10] = r.flags;
}

// OBB-vs-sphere lower bound against an object part (geometry.cpp:544-557).
__device__ __forceinline__ double obb_sphere(const double* obb, D3 center, double radius) {
  const D3 oc = ld3(obb);
  const D3 half = ld3(obb + 3);
  // rotation column-major: columns are axes; q = rot^T (c - oc)
  const D3 rel = center - oc;
  const D3 q = mk(obb[6] * rel.x + obb[7] * rel.y + obb[8] * rel.z, obb[9] * rel.x + obb[10] * rel.y + obb[11] * rel.z,
                  obb[12] * rel.x + obb[13] * rel.y + obb[14] * rel.z);
  const D3 ex = mk(fabs(q.x) - half.x, fabs(q.y) - half.y, fabs(q.z) - half.z);
  double dist;
  if (ex.x <= 0 && ex.y <= 0 && ex.z <= 0)
    dist = fmax(ex.x, fmax(ex.y, ex.z));
  else
    dist = nrm(mk(fmax(ex.x, 0.0), fmax(ex.y, 0.0), fmax(ex.z, 0.0)));
  return dist - radius;
}

// True when the signed distance of (link, part) must be computed. By default
// every pair is: the reference runs GJK on every pair (pipeline.cpp:176-188)
// and its GJK reports a spurious overlap for some provably separated pairs
// (a coplanar 4-point simplex whose rank-deficient KKT solve wins the
// subset enumeration by an ulp, so contains = true; about 1 in 6e4 late-stage
// pairs, gaps up to mm measured), which then enters the penetration hinge.
// Reproducing those needs the GJK. With the opt-in cull (GRASP_CULL=1) a
// pair is skipped (+inf) unless it is in a fingertip's witness keep-set (the
// OBB test select_witness applies, pipeline.cpp:332-334) or it may
// penetrate by the link-sphere vs part-OBB and link-box vs part-box (SAT)
// lower bounds: exact for the true geometry, not for those spurious overlaps.
// Separating-axis test between the link box (posed by Rw, tw) and the part
// box (object frame), 15 axes (Gottschalk's OBB test). true only if the
// projections on some axis are disjoint with a gap > margin, which proves
// the hulls inside are separated (d > 0). |R| is padded by 1e-12, and the
// unnormalised cross axes only make the margin test stricter.
__device__ __forceinline__ bool boxes_separated(const double* la, const M33& Rw, D3 tw, const double* pb,
                                                double margin) {
  D3 A[3], B[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    A[i] = mul(Rw, ld3(la + 6 + 3 * i));
    B[i] = ld3(pb + 6 + 3 * i);
  }
  const double ah[3] = {la[3], la[4], la[5]}, bh[3] = {pb[3], pb[4], pb[5]};
  const D3 T = ld3(pb) - (mul(Rw, ld3(la)) + tw);
  double R[3][3], AR[3][3], t[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    t[i] = dot(T, A[i]);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      R[i][j] = dot(A[i], B[j]);
      AR[i][j] = fabs(R[i][j]) + 1e-12;
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (fabs(t[i]) > ah[i] + bh[0] * AR[i][0] + bh[1] * AR[i][1] + bh[2] * AR[i][2] + margin) return true;
#pragma unroll
  for (int j = 0; j < 3; ++j)
    if (fabs(t[0] * R[0][j] + t[1] * R[1][j] + t[2] * R[2][j]) >
        ah[0] * AR[0][j] + ah[1] * AR[1][j] + ah[2] * AR[2][j] + bh[j] + margin)
      return true;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int j1 = (j + 1) % 3, j2 = (j + 2) % 3;
      const double ra = ah[i1] * AR[i2][j] + ah[i2] * AR[i1][j];
      const double rb = bh[j1] * AR[i][j2] + bh[j2] * AR[i][j1];
      if (fabs(t[i2] * R[i1][j] - t[i1] * R[i2][j]) > ra + rb + margin) return true;
    }
  }
  return false;
}

__device__ __forceinline__ bool pair_needed(const DevHand& H, const DevObject& O, const DevState& st, int g,
                                            int link, int part, const M33& Rw, D3 tw) {
  if (!H.cull) return true;
  const int f = H.link_tip[link];
  if (f >= 0) {
    const int tp = H.tip_proxy[f];
    const D3 center = mul(Rw, ld3(H.proxy + 4 * tp)) + tw;
    const double reference = st.qres[((size_t)g * st.NQ + tp) * 8] - H.proxy[4 * tp + 3];
    // Superset of select_witness's keep test (reference + 1e-9 there): the
    // tip centre here comes from st.world, the step kernel's from its own FK
    // copy, so a wider margin keeps every pair it may read exact.
    if (obb_sphere(O.part_obb + 15 * part, center, H.tip_envelope[f]) < reference + 1e-6) return true;
  }
  const double* bs = H.link_bsphere + 4 * link;
  const D3 c = mul(Rw, ld3(bs)) + tw;
  if (obb_sphere(O.part_obb + 15 * part, c, bs[3]) > kCullSlack) return false;
  return !(H.link_box && boxes_separated(H.link_box + 15 * link, Rw, tw, O.part_box + 15 * part, kCullSlack));
}


// Compacted pair evaluation. The list is segmented by (link, part) so that a
// GJK warp works on one hull pair: its vertex loads are warp-uniform
// (broadcast) and its support loops have one trip count.
//
// Pass 1a: one thread per (grasp, link, part) launch index t (lp-major) runs
// the cull test; culled slots get their (+inf) result directly, the others
// set need[t] and are counted into their segment (one atomic per segment
// present in the warp).
__device__ __forceinline__ int warp_segment_add(int* counters, int seg, bool active) {
  // Adds 1 per active lane to counters[seg] with one atomic per distinct seg;
  // returns this lane's position (old value + rank among active lanes of seg).
  const unsigned act = __ballot_sync(kFull, active);
  const unsigned peers = __match_any_sync(kFull, seg) & act;
  const int lane = threadIdx.x & 31;
  int base = 0;
  const int leader = peers ? __ffs(peers) - 1 : lane;
  if (active && lane == leader) base = atomicAdd(counters + seg, __popc(peers));
  base = __shfl_sync(kFull, base, leader);
  return base + __popc(peers & ((1u << lane) - 1));
}

// List segments: 0 = the early pairs (the slot's last EPA took more than
// st.early_pred iterations: GJK + EPA in one thread by k_pairs_early,
// concurrently with k_pairs_list), then (link-part, GJK-length bucket).
constexpr int kPairEarly = 254;  // (pair_need stores 1 + bucket in a byte)
__device__ __forceinline__ int pair_segment(int lp, int b) { return b == kPairEarly ? 0 : 1 + lp * kPairBuckets + b; }

__global__ void __launch_bounds__(128) k_pairs_cull(DevHand H, DevObject O, DevState st,
                                                    const int* __restrict__ links, int n_links) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = (long long)st.G * n_links * O.Pmax;
  bool need = false;
  int lp = 0, b = 0;
  if (t < n) {
    const int g = (int)(t % st.G);
    lp = (int)(t / st.G);
    const int link = links ? links[lp / O.Pmax] : lp / O.Pmax;
    const int part = lp % O.Pmax;  // the grasp's object's part index
    if (!st.failed[g]) {
      int p0, p1;
      obj_parts(O, st, g, p0, p1);
      const double* w = st.world + ((size_t)g * H.L + link) * 12;
      M33 Rw;
      for (int i = 0; i < 9; ++i) Rw.m[i] = w[i];
      // slots past the object's parts (multi-object contexts) hold +inf and are never read as pairs
      need = part < p1 - p0 && pair_needed(H, O, st, g, link, p0 + part, Rw, ld3(w + 9));
      if (!need) {
        double* o = st.pairs + ((size_t)g * st.NP + link * O.Pmax + part) * 12;
        o[0] = INFINITY;
        o[10] = kPairCulled;
      } else {
        const size_t slot = (size_t)g * st.NP + link * O.Pmax + part;
        b = st.epa_hist[slot] > st.early_pred ? kPairEarly : pair_bucket(st.pair_hist[slot]);
      }
    }
    st.pair_need[t] = need ? (unsigned char)(1 + b) : 0;
  }
  warp_segment_add(st.seg_count, pair_segment(lp, b), need);
}

// Pass 1b: exclusive scan of the segment counts (one block); seg_count turns
// into the fill cursor of pass 1c, *pair_count into the list length.
__global__ void __launch_bounds__(1024) k_pairs_scan(DevState st, int n_seg) {
  __shared__ int part_sum[1024];
  const int tid = threadIdx.x;
  const int per = (n_seg + 1023) / 1024;
  const int b = tid * per, e = min(n_seg, b + per);
  int s = 0;
  for (int i = b; i < e; ++i) s += st.seg_count[i];
  part_sum[tid] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int v = tid >= off ? part_sum[tid - off] : 0;
    __syncthreads();
    part_sum[tid] += v;
    __syncthreads();
  }
  int run = part_sum[tid] - s;
  for (int i = b; i < e; ++i) {
    const int c = st.seg_count[i];
    st.seg_offset[i] = run;
    st.seg_count[i] = run;
    run += c;
  }
  if (tid == 1023) *st.pair_count = part_sum[1023];
}

// Pass 1c: scatter the needed slots into their segments.
__global__ void __launch_bounds__(128) k_pairs_scatter(DevState st, const int* __restrict__ links, int n_links,
                                                       int P) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = (long long)st.G * n_links * P;
  const int code = t < n ? st.pair_need[t] : 0;
  const bool need = code != 0;
  const int lp = t < n ? (int)(t / st.G) : 0;
  const int pos = warp_segment_add(st.seg_count, pair_segment(lp, need ? code - 1 : 0), need);
  if (need) {
    const int g = (int)(t % st.G);
    const int link = links ? links[lp / P] : lp / P;
    st.pair_list[pos] = (int)((size_t)g * st.NP + link * P + lp % P);
  }
}

// Spatially bucketed all-slot point queries. A slot's query of the last
// iteration tells where its point is now: near the cluster of its last
// closest face, or inside a part. Listing the queries by that bucket puts
// queries with the same path through point_to_mesh (same parts culled, same
// clusters scanned, same inside test) into the same warps. Which thread runs
// a query does not change its result, so the order is free.
// Query class: 0 = what the QP reads (tip proxies and their FD stencils),
// 1 = the other proxies (read by the step kernel only), listed after class 0
// so the two can run as separate launches (class 1 next to the QP).
__device__ __forceinline__ int pq_class(const DevHand& H, const DevState& st, size_t t) {
  const int slot = (int)(t % st.NQ);
  if (slot >= H.S) return 0;
  for (int f = 0; f < H.m; ++f)
    if (__ldg(H.tip_proxy + f) == slot) return 0;
  return 1;
}

__device__ __forceinline__ int pq_bucket(const DevObject& O, const DevState& st, size_t t) {
  const int f = st.qface[t];
  const double d = st.qres[t * 8];
  // inside queries (last result negative) apart from outside ones: they take
  // the plane-group path, the others the face scan
  if (f >= 0 && f < O.F) return __ldg(O.face_cluster + f) + (d < 0.0 ? O.NC : 0);
  const double pd = st.qres[t * 8 + 7];
  if (d < 0.0 && pd >= 0.0 && pd < O.P) return 2 * O.NC + (int)pd;
  return 2 * O.NC + O.P;
}

__global__ void __launch_bounds__(128) k_pq_count(DevHand H, DevObject O, DevState st) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = (long long)st.G * st.NQ;
  bool active = false;
  int key = 0;
  if (t < n) {
    active = !st.failed[t / st.NQ];
    if (active) key = pq_bucket(O, st, (size_t)t) + pq_class(H, st, (size_t)t) * (2 * O.NC + O.P + 1);
    st.pq_key[t] = active ? key : -1;
  }
  warp_segment_add(st.pq_count, key, active);
}

// Exclusive scan of n counts in place (one block); *total = their sum.
// split_out (optional): the exclusive prefix at index split_at (0 <= split_at <= n).
__global__ void __launch_bounds__(1024) k_exclusive_scan(int* counts, int n, int* total, int split_at = -1,
                                                         int* split_out = nullptr) {
  __shared__ int part_sum[1024];
  const int tid = threadIdx.x;
  const int per = (n + 1023) / 1024;
  const int b = tid * per, e = min(n, b + per);
  int s = 0;
  for (int i = b; i < e; ++i) s += counts[i];
  part_sum[tid] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int v = tid >= off ? part_sum[tid - off] : 0;
    __syncthreads();
    part_sum[tid] += v;
    __syncthreads();
  }
  int run = part_sum[tid] - s;
  for (int i = b; i < e; ++i) {
    const int c = counts[i];
    if (split_out && i == split_at) *split_out = run;
    counts[i] = run;
    run += c;
  }
  if (tid == 1023) {
    *total = part_sum[1023];
    if (split_out && split_at == n) *split_out = part_sum[1023];
  }
}

__global__ void __launch_bounds__(128) k_pq_scatter(DevState st) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = (long long)st.G * st.NQ;
  const int key = t < n ? st.pq_key[t] : -1;
  const bool active = key >= 0;
  const int pos = warp_segment_add(st.pq_count, active ? key : 0, active);
  if (active) st.pq_list[pos] = (int)t;
}

// k_point_query over the bucketed list.
// Entries [*begin, *end) of the bucketed list (begin == nullptr: 0).
__global__ void __launch_bounds__(GDEV_PQ_BLOCK, GDEV_PQ_THREADS_PER_SM / GDEV_PQ_BLOCK) k_point_query_list(
    DevObject O, DevState st, const int* begin, const int* end) {
  const int i = (begin ? *begin : 0) + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *end) return;
  const int t = st.pq_list[i];
  const int g = t / st.NQ;
  if (st.failed[g]) return;  // (the list may predate the grasp's failure)
  const D3 p = ld3(st.qpts + (size_t)t * 3);
  unsigned planes, tris;
  int* qf = st.qface + t;
  int* qs = st.qsep + t;
  int p0, p1;
  obj_parts(O, st, g, p0, p1);
  const PointHit h = point_to_mesh(O, p, p0, p1, *qf, &planes, &tris, *qs);
  *qf = h.face;
  *qs = h.sep;
  if (st.ops) {
    op_add(st.ops, kOpPlaneTests, planes);
    op_add(st.ops, kOpTriangleTests, tris);
    op_add(st.ops, kOpPointQueries, 1u);
  }
  double* o = st.qres + (size_t)t * 8;
  o[0] = h.d;
  st3(o + 1, h.pb);
  st3(o + 4, h.n);
  o[7] = h.part;
}

// Hulls and cloud_scale (geometry.cpp:17-23) of a pair slot.
__device__ __forceinline__ void slot_hulls(const DevHand& H, const DevObject& O, const DevState& st, int slot, Hull& A,
                                           Hull& B, double& scale) {
  const int g = slot / st.NP, lp = slot % st.NP;
  int p0, p1;
  obj_parts(O, st, g, p0, p1);
  const int link = lp / O.Pmax, part = p0 + lp % O.Pmax;
  const double* w = st.world + ((size_t)g * H.L + link) * 12;
  set_link_hull(H, link, A);
  A.posed = true;
  for (int k = 0; k < 9; ++k) A.R.m[k] = w[k];
  A.t = ld3(w + 9);
  set_part_hull(O, part, B);
  scale = 1.0;
  scale = fmax(scale, scale_of(mul(A.R, ld3(H.link_centroid + 3 * link)) + A.t, H.link_halfnorm[link]));
  scale = fmax(scale, scale_of(ld3(O.part_centroid + 3 * part), O.part_halfnorm[part]));
}

__device__ __forceinline__ void queue_overflow(const DevState& st, int slot) {
  const int o = atomicAdd(st.ovf_count, 1);
  if (o < st.ovf_cap)
    st.ovf_list[o] = slot;
  else
    atomicAdd(st.err + 1, 1);
}

// Pass 2: GJK, one thread per listed pair (dense warps, register simplex,
// no EPA buffer). Overlapping pairs pass their terminal simplex to k_pairs_epa.
#ifndef GDEV_PAIRS_BLOCK
#define GDEV_PAIRS_BLOCK 128
#endif
#ifndef GDEV_PAIRS_MIN_BLOCKS
#define GDEV_PAIRS_MIN_BLOCKS 3  // 168 registers: 376 vs 382 ms at 2 blocks (232 registers) since SP keys; before them 2 > 3 > 4 > 5 > 6
#endif
// Jobs whose slot needed more than kEpaLongPred EPA iterations last time go
// to a second region (launched first, packed into their own warps): a
// thread-per-job warp otherwise runs as long as its longest lane.
#ifndef GDEV_EPA_LONG_PRED
#define GDEV_EPA_LONG_PRED 6
#endif
constexpr int kEpaLongPred = GDEV_EPA_LONG_PRED;
__device__ __forceinline__ void write_epa_job(const DevState& st, int slot, const SP (&simp)[4], int ns) {
  const bool long_job = st.epa_hist[slot] > kEpaLongPred;
  const int job = atomicAdd(long_job ? st.epa_long_count : st.epa_count, 1);
  if (job >= st.epa_cap) {
    if (st.ops) atomicAdd(st.ops + kOpEpaOverflow, 1ull);
    queue_overflow(st, slot);
    return;
  }
  double* jb = st.epa_jobs + ((size_t)job + (long_job ? st.epa_cap : 0)) * kEpaJobStride;
  jb[0] = slot;
  jb[1] = ns;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    st3(jb + 2 + 4 * k, simp[k].w);
    jb[5 + 4 * k] = simp[k].key;
  }
}

// Pass 2 (default): GJK, one thread per listed pair from start to end.
__global__ void __launch_bounds__(GDEV_PAIRS_BLOCK, GDEV_PAIRS_MIN_BLOCKS) k_pairs_list(DevHand H, DevObject O, DevState st) {
  const int i = st.seg_offset[1] + blockIdx.x * blockDim.x + threadIdx.x;  // after the early pairs
  if (i >= *st.pair_count) return;
  const int slot = st.pair_list[i];
  Hull A, B;
  double scale;
  slot_hulls(H, O, st, slot, A, B, scale);
  PairResult r;
  SP simp[4];
  int ns;
  const bool overlap = gjk_phase(A, B, scale, r, simp, ns);
  st.pair_hist[slot] = (unsigned char)min(255u, r.gjk_iters + 1);
  if (st.ops) {
    op_add(st.ops, kOpSupportVerts, r.n_support * (A.nv + B.nv));
    count_gjk(st.ops, r.gjk_iters + 1, r.gjk_skipped);
    op_add(st.ops, kOpPairsNeeded, 1u);
  }
  if (!overlap) {
    store_pair(st.pairs + (size_t)slot * 12, r);
    return;
  }
  write_epa_job(st, slot, simp, ns);
}

// Pass 3: EPA for the overlapping pairs (geometry.cpp:168-205, 227-324), one
// thread per job, polytope in local memory.
#ifndef GDEV_EPA_MIN_BLOCKS
#define GDEV_EPA_MIN_BLOCKS 1
#endif
__device__ __forceinline__ void epa_job(const DevHand& H, const DevObject& O, const DevState& st, int job);

// (grid-stride over the jobs: the grid is sized for the usual job count)
__global__ void __launch_bounds__(32, GDEV_EPA_MIN_BLOCKS) k_pairs_epa(DevHand H, DevObject O, DevState st) {
  const int n_long = min(*st.epa_long_count, st.epa_cap);
  const int n_all = n_long + min(*st.epa_count, st.epa_cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_all; i += gridDim.x * blockDim.x)
    epa_job(H, O, st, i < n_long ? st.epa_cap + i : i - n_long);  // predicted-long jobs first
}

__device__ __forceinline__ void epa_job(const DevHand& H, const DevObject& O, const DevState& st, int job) {
  const double* jb = st.epa_jobs + (size_t)job * kEpaJobStride;
  const int slot = (int)jb[0], ns = (int)jb[1];
  SP simp[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    simp[k].w = ld3(jb + 2 + 4 * k);
    simp[k].key = (unsigned)jb[5 + 4 * k];
  }
  Hull A, B;
  double scale;
  slot_hulls(H, O, st, slot, A, B, scale);
  PairResult r;
  r.flags = 0;
  r.n_support = 0;
  r.gjk_iters = 0;
  r.epa_iters = 0;
  EpaScratch scratch;
  epa(simp, ns, A, B, scale, scratch, r);
  if (st.ops) {
    atomicAdd(st.ops + kOpSupportVerts, (unsigned long long)r.n_support * (A.nv + B.nv));
    atomicAdd(st.ops + kOpEpaIters, (unsigned long long)r.epa_iters);
    atomicMax(st.ops + kOpEpaMaxIters, (unsigned long long)r.epa_iters);
    if (r.epa_iters > 8) atomicAdd(st.ops + kOpEpaLongJobs, 1ull);
    if (r.flags & kPairOverflow) atomicAdd(st.ops + kOpEpaOverflow, 1ull);
  }
  st.epa_hist[slot] = (unsigned char)min(255, r.epa_iters);
  if (r.flags & kPairDegenerate) atomicAdd(st.err + 0, 1);
  if (r.flags & kPairOverflow) {
    queue_overflow(st, slot);
    return;
  }
  store_pair(st.pairs + (size_t)slot * 12, r);
}


// The early pairs (list segment 0): GJK and, on overlap, EPA in one thread,
// launched on a second stream next to k_pairs_list so that the long EPA runs
// overlap the GJK pass instead of forming k_pairs_epa's tail. Same functions,
// same results as the two-pass path.
__device__ __forceinline__ void pair_early(const DevHand& H, const DevObject& O, const DevState& st, int slot) {
  Hull A, B;
  double scale;
  slot_hulls(H, O, st, slot, A, B, scale);
  PairResult r;
  SP simp[4];
  int ns;
  const bool overlap = gjk_phase(A, B, scale, r, simp, ns);
  st.pair_hist[slot] = (unsigned char)min(255u, r.gjk_iters + 1);
  if (st.ops) {
    op_add(st.ops, kOpSupportVerts, r.n_support * (A.nv + B.nv));
    count_gjk(st.ops, r.gjk_iters + 1, r.gjk_skipped);
    op_add(st.ops, kOpPairsNeeded, 1u);
  }
  if (overlap) {
    r.n_support = 0;
    EpaScratch scratch;
    epa(simp, ns, A, B, scale, scratch, r);
    if (st.ops) {
      op_add(st.ops, kOpSupportVerts, r.n_support * (A.nv + B.nv));
      op_add(st.ops, kOpEpaIters, r.epa_iters);
      atomicMax(st.ops + kOpEpaMaxIters, (unsigned long long)r.epa_iters);
      op_add(st.ops, kOpEpaLongJobs, r.epa_iters > 8 ? 1u : 0u);
      op_add(st.ops, kOpEpaOverflow, (r.flags & kPairOverflow) ? 1u : 0u);
    }
    if (r.flags & kPairDegenerate) atomicAdd(st.err + 0, 1);
    if (r.flags & kPairOverflow) {
      st.epa_hist[slot] = (unsigned char)min(255, r.epa_iters);
      queue_overflow(st, slot);
      return;
    }
  }
  st.epa_hist[slot] = (unsigned char)min(255, overlap ? r.epa_iters : 0);
  store_pair(st.pairs + (size_t)slot * 12, r);
}

__global__ void __launch_bounds__(32) k_pairs_early(DevHand H, DevObject O, DevState st) {
  const int n_early = st.seg_offset[1];
  // (grid-stride: the grid is sized for the usual count, not the worst case)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_early; i += gridDim.x * blockDim.x)
    pair_early(H, O, st, st.pair_list[i]);
}

// Redoes the queued pairs with the large global-memory EPA buffer.
__global__ void __launch_bounds__(128) k_pairs_big(DevHand H, DevObject O, DevState st) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int count = min(*st.ovf_count, st.ovf_cap);
  if (tid >= st.big_slots) return;
  EpaScratchBig& scratch = static_cast<EpaScratchBig*>(st.big_scratch)[tid];
  for (int i = tid; i < count; i += st.big_slots) {
    const int slot = st.ovf_list[i];
    const int g = slot / st.NP, lp = slot % st.NP;
    int p0, p1;
    obj_parts(O, st, g, p0, p1);
    const int link = lp / O.Pmax, part = p0 + lp % O.Pmax;
    const double* w = st.world + ((size_t)g * H.L + link) * 12;
    M33 Rw;
    for (int k = 0; k < 9; ++k) Rw.m[k] = w[k];
    const PairResult r = link_part_distance(H, O, link, part, Rw, ld3(w + 9), scratch);
    store_pair(st.pairs + (size_t)slot * 12, r);
    if (r.flags & kPairDegenerate) atomicAdd(st.err + 0, 1);
    if (r.flags & kPairOverflow) atomicAdd(st.err + 1, 1);
  }
}

// Standalone pair surface (teacher-forced tests): poses[n*12] column-major R
// + t; grid-stride over n with one large EPA buffer per thread.
__global__ void k_pairs_raw(DevHand H, DevObject O, int n, const int* __restrict__ links, const int* __restrict__ parts,
                            const double* __restrict__ poses, double* out, EpaScratchBig* big,
                            unsigned long long* ops) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int t = tid; t < n; t += gridDim.x * blockDim.x) {
    M33 Rw;
    for (int c = 0; c < 3; ++c)
      for (int i = 0; i < 3; ++i) Rw.m[i * 3 + c] = poses[12 * t + 3 * c + i];
    const PairResult r = link_part_distance(H, O, links[t], parts[t], Rw, ld3(poses + 12 * t + 9), big[tid]);
    store_pair(out + 11 * t, r);
    out[11 * t + 10] = r.flags;
    if (ops) count_gjk(ops, r.gjk_iters + 1, r.gjk_skipped);
  }
}

// ------------------------------------------------------------- evaluation
// Grasp evaluation (eval.cpp:51-89) on the state in st.x / st.world.
// Self-penetration pairs: signed_distance(link a posed, link b posed)
// (eval.cpp:63-72; geometry.cpp:500-525 with both poses), one thread per
// (grasp, collision pair); d written to out[g * ncp + i]. Pairs whose EPA
// polytope outgrows the small per-thread scratch are queued (st.ovf_list) and
// redone by k_eval_self_pairs_big with the reference's full 512-iteration
// capacity, like k_pairs_big for object pairs.
template <class Scratch>
__device__ PairResult self_pair_distance(const DevHand& H, const DevState& st, long long t, Scratch& scratch) {
  const int g = (int)(t / H.ncp), i = (int)(t % H.ncp);
  const int la = H.cp_a[i], lb = H.cp_b[i];
  Hull A, B;
  M33 Ra, Rb;
  const double* wa = st.world + ((size_t)g * H.L + la) * 12;
  const double* wb = st.world + ((size_t)g * H.L + lb) * 12;
  for (int k = 0; k < 9; ++k) Ra.m[k] = wa[k], Rb.m[k] = wb[k];
  const D3 ta = ld3(wa + 9), tb = ld3(wb + 9);
  set_link_hull(H, la, A);
  A.posed = true;
  A.R = Ra;
  A.t = ta;
  set_link_hull(H, lb, B);
  B.posed = true;
  B.R = Rb;
  B.t = tb;
  // cloud_scale (geometry.cpp:17-23)
  double scale = 1.0;
  scale = fmax(scale, scale_of(mul(Ra, ld3(H.link_centroid + 3 * la)) + ta, H.link_halfnorm[la]));
  scale = fmax(scale, scale_of(mul(Rb, ld3(H.link_centroid + 3 * lb)) + tb, H.link_halfnorm[lb]));
  return signed_distance(A, B, scale, scratch);
}

__global__ void __launch_bounds__(128) k_eval_self_pairs(DevHand H, DevState st, double* out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)st.G * H.ncp) return;
  EpaScratch scratch;
  const PairResult r = self_pair_distance(H, st, t, scratch);
  if (r.flags & kPairOverflow) {
    const int k = atomicAdd(st.ovf_count, 1);
    if (k < st.ovf_cap) st.ovf_list[k] = (int)t;
    else atomicAdd(st.err + 1, 1);
    return;
  }
  if (r.flags & kPairDegenerate) atomicAdd(st.err + 0, 1);
  out[t] = r.d;
}

__global__ void __launch_bounds__(128) k_eval_self_pairs_big(DevHand H, DevState st, double* out) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int count = min(*st.ovf_count, st.ovf_cap);
  if (tid >= st.big_slots) return;
  EpaScratchBig& scratch = static_cast<EpaScratchBig*>(st.big_scratch)[tid];
  for (int i = tid; i < count; i += st.big_slots) {
    const long long t = st.ovf_list[i];
    const PairResult r = self_pair_distance(H, st, t, scratch);
    if (r.flags & kPairDegenerate) atomicAdd(st.err + 0, 1);
    if (r.flags & kPairOverflow) atomicAdd(st.err + 1, 1);
    out[t] = r.d;
  }
}

// Per grasp: penetration depth over every (link, part) pair record and
// self-penetration depth over the collision pairs, in mm (max(0, -d)).
__global__ void k_eval_depths(DevHand H, DevObject O, DevState st, const double* __restrict__ self_d, double* pd,
                              double* spd) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= st.G) return;
  double depth = 0.0;
  const int np = H.L * O.Pmax;  // slots past the object's parts hold +inf
  for (int i = 0; i < np; ++i) depth = fmax(depth, -st.pairs[((size_t)g * st.NP + i) * 12]);
  pd[g] = 1000.0 * depth;
  depth = 0.0;
  for (int i = 0; i < H.ncp; ++i) depth = fmax(depth, -self_d[(size_t)g * H.ncp + i]);
  spd[g] = 1000.0 * depth;
}

// ------------------------------------------------------ gradient assembly
// A force f (world) at world point p on link l contributes J(l,p)^T f to
// the state gradient (hand.cpp:155-169). With v = R^T (p - t) and
// f' = R^T f this is: rotation block J_tan^T (v x f'), translation f, joint j
// (ancestor of l) a_j . ((v - o_j) x f'). Forces are therefore accumulated
// per link as F_l = sum f', T_l = sum v x f' and expanded once per iteration.
struct LinkAcc {
  D3 F, T;
};

// Adds one chunk of up to 32 items (item lane t owns itL/itF/itT[t]) to the
// per-link accumulator held by lane == link. Fixed item order; only the lanes
// holding an item (itL >= 0, each lane wrote its own slot) are visited.
__device__ __forceinline__ void flush_items(WarpScratch& s, int lane, LinkAcc& acc, bool any) {
  __syncwarp();
  if (any) {
    for (unsigned m = __ballot_sync(kFull, s.itL[lane] >= 0); m; m &= m - 1) {
      const int i = __ffs(m) - 1;
      if (s.itL[i] == lane) {
        acc.F += ld3(s.itF + 3 * i);
        acc.T += ld3(s.itT + 3 * i);
      }
    }
  }
  __syncwarp();
}

// Adds a chunk of per-lane energy terms to lane 0's running total in lane
// order (the reference's sequential sum). Zero terms are skipped: the total
// starts at +0 and x + 0 == x for every x other than -0, which a sum from +0
// never reaches, so the result is bitwise the full sequential sum.
__device__ __forceinline__ void add_terms(WarpScratch& s, int lane, double term, double& total) {
  const unsigned nz = __ballot_sync(kFull, term != 0.0);
  s.red[lane] = term;
  __syncwarp();
  if (lane == 0)
    for (unsigned m = nz; m; m &= m - 1) total += s.red[__ffs(m) - 1];
}

__device__ __forceinline__ void put_item(WarpScratch& s, int lane, int link, D3 pw, D3 fw) {
  const M33 R = {{s.pose[0], s.pose[1], s.pose[2], s.pose[3], s.pose[4], s.pose[5], s.pose[6], s.pose[7], s.pose[8]}};
  const D3 v = mulT(R, pw - ld3(s.pose + 9));
  const D3 f = mulT(R, fw);
  s.itL[lane] = link;
  st3(s.itF + 3 * lane, f);
  st3(s.itT + 3 * lane, cross(v, f));
}

// Expands per-link accumulators into the state gradient s.grad (adds to the
// limit gradient already there).
__device__ inline void expand_gradient(const DevHand& H, WarpScratch& s, int lane, const LinkAcc& acc) {
  // Totals and per-joint subtree sums, fixed link order. Links whose
  // accumulator is all zeros are skipped: the sums start at +0 and adding an
  // exact zero changes no value other than -0, which they never reach.
  D3 Ftot = mk(0, 0, 0), Ttot = mk(0, 0, 0), Fsub = mk(0, 0, 0), Tsub = mk(0, 0, 0);
  const unsigned sub = lane < H.dof ? H.joint_subtree[lane] : 0u;
  const bool nz = lane < H.L && (acc.F.x != 0.0 || acc.F.y != 0.0 || acc.F.z != 0.0 || acc.T.x != 0.0 ||
                                 acc.T.y != 0.0 || acc.T.z != 0.0);
  for (unsigned m = __ballot_sync(kFull, nz); m; m &= m - 1) {
    const int l = __ffs(m) - 1;
    const D3 F = mk(__shfl_sync(kFull, acc.F.x, l), __shfl_sync(kFull, acc.F.y, l), __shfl_sync(kFull, acc.F.z, l));
    const D3 T = mk(__shfl_sync(kFull, acc.T.x, l), __shfl_sync(kFull, acc.T.y, l), __shfl_sync(kFull, acc.T.z, l));
    Ftot += F;
    Ttot += T;
    if (sub & (1u << l)) {
      Fsub += F;
      Tsub += T;
    }
  }
  if (lane < H.dof) {
    const D3 o = ld3(s.jo + 6 * lane), a = ld3(s.jo + 6 * lane + 3);
    s.grad[12 + lane] += dot(a, Tsub - cross(o, Fsub));
  }
  if (lane < 9) {
    // grad_raw[3l+i] = (e_l x r_i) . (a_inv^T T), zero when degenerate.
    const bool degenerate = s.pose[21] != 0.0;
    const int l = lane / 3, i = lane % 3;
    const M33 ai = {{s.pose[12], s.pose[13], s.pose[14], s.pose[15], s.pose[16], s.pose[17], s.pose[18], s.pose[19],
                     s.pose[20]}};
    const D3 w = mulT(ai, Ttot);
    const D3 ri = mk(s.pose[3 * i], s.pose[3 * i + 1], s.pose[3 * i + 2]);
    s.grad[lane] += degenerate ? 0.0 : dot(cross(unit(l), ri), w);
  } else if (lane < 12) {
    const M33 R = {{s.pose[0], s.pose[1], s.pose[2], s.pose[3], s.pose[4], s.pose[5], s.pose[6], s.pose[7], s.pose[8]}};
    s.grad[lane] += comp(mul(R, Ftot), lane - 9);
  }
  __syncwarp();
}

// Joint-limit and sphere self-penetration terms (hand.cpp:207-245); items
// for self pairs are pushed in pair order.
__device__ inline void limit_and_self(const DevHand& H, const DevParams& P, WarpScratch& s, int lane, LinkAcc& acc,
                                      bool with_grad, double& e_lim, double& e_self) {
  double el = 0.0;
  for (int j = lane; j < H.dof; j += 32) {
    const double qj = s.x[12 + j];
    const double over = fmax(qj - H.joint_upper[j], 0.0);
    const double under = fmax(H.joint_lower[j] - qj, 0.0);
    el += over * over + under * under;
    s.grad[12 + j] = with_grad ? P.w_limit * (2.0 * over - 2.0 * under) : 0.0;
  }
  for (int i = lane; i < 12; i += 32) s.grad[i] = 0.0;
  e_lim = warp_sum(el);
  double es = 0.0;
  for (int base = 0; base < H.nsp; base += 32) {
    const int t = base + lane;
    bool active = false;
    D3 ca, cb, dir;
    double overlap = 0.0;
    int la = -1, lb = -1;
    if (t < H.nsp) {
      const int pa = H.sp_a[t], pb = H.sp_b[t];
      ca = ld3(s.pc + 3 * pa);
      cb = ld3(s.pc + 3 * pb);
      const double dist = nrm(ca - cb);
      overlap = H.proxy[4 * pa + 3] + H.proxy[4 * pb + 3] - dist;
      if (overlap > 0) {
        es += overlap * overlap;
        if (dist > 1e-12) {
          active = true;
          dir = (ca - cb) / dist;
          la = H.proxy_link[pa];
          lb = H.proxy_link[pb];
        }
      }
    }
    if (!with_grad) continue;
    const bool any = __any_sync(kFull, active);
    if (!any) continue;
    // item a
    s.itL[lane] = -1;
    if (active) put_item(s, lane, la, ca, (-2.0 * P.w_self * overlap) * dir);
    flush_items(s, lane, acc, true);
    s.itL[lane] = -1;
    if (active) put_item(s, lane, lb, cb, (2.0 * P.w_self * overlap) * dir);
    flush_items(s, lane, acc, true);
  }
  e_self = warp_sum(es);
}

// apply_step (pipeline.cpp:214-231) on lane 0 + divergence/failure checks
// (pipeline.cpp:264-277). Returns the failure code (0 ok).
__device__ inline int step_lane0(const DevHand& H, const StageArgs& A, WarpScratch& s, double energy) {
  const int D = H.D;
  bool finite = isfinite(energy);
  for (int i = 0; i < D; ++i) finite = finite && isfinite(s.grad[i]);
  if (!finite) return 1;
  for (int i = 0; i < D; ++i) s.xn[i] = s.x[i];
  auto move = [&](int start, int len, double step) {
    double n2 = 0.0;
    for (int i = 0; i < len; ++i) n2 += s.grad[start + i] * s.grad[start + i];
    const double scale = step * A.decay / fmax(1.0, sqrt(n2));
    for (int i = 0; i < len; ++i) s.xn[start + i] -= scale * s.grad[start + i];
  };
  move(0, 9, A.step_rot);
  move(9, 3, A.step_trans);
  if (H.dof > 0) {
    move(12, H.dof, A.step_joints);
    for (int j = 0; j < H.dof; ++j) s.xn[12 + j] = fmin(fmax(s.xn[12 + j], H.joint_lower[j]), H.joint_upper[j]);
  }
  bool xf = true;
  for (int i = 0; i < D; ++i) xf = xf && isfinite(s.xn[i]);
  const double tn = sqrt(s.xn[9] * s.xn[9] + s.xn[10] * s.xn[10] + s.xn[11] * s.xn[11]);
  if (!xf || tn > 1e3) return 2;
  for (int i = 0; i < D; ++i) s.x[i] = s.xn[i];
  return 0;
}

// Common tail of both step kernels: finite check, step, state write, FK.
__device__ inline void finish_iteration(const DevHand& H, const DevParams& P, const StageArgs& A, const DevState& st,
                                        int g, int lane, WarpScratch& s, double total) {
  if (lane == 0) {
    st.energy[g] = total;
    if (A.mode == 0 && A.it == 0) st.stage_energy[(size_t)g * 6 + 2 * A.stage] = total;
    if (A.mode == 1) st.stage_energy[(size_t)g * 6 + 2 * A.stage + 1] = total;
  }
  if (A.mode == 2) {
    for (int i = lane; i < H.D; i += 32) st.grad[(size_t)g * H.D + i] = s.grad[i];
    return;
  }
  if (A.mode != 0) return;
  if (lane == 0) {
    const int code = step_lane0(H, A, s, total);
    s.flag[0] = code;
    if (code) st.failed[g] = code;
  }
  __syncwarp();
  const int code = s.flag[0];
  double* gx = st.x + (size_t)g * H.D;
  for (int i = lane; i < H.D; i += 32) {
    st.grad[(size_t)g * H.D + i] = s.grad[i];
    gx[i] = s.x[i];
  }
  if (code) return;
  __syncwarp();
  warp_fk(H, st, g, lane, s, P.fd_step, true);
}

// Sphere-proxy (coarse) stage iteration: total_energy (pipeline.cpp:114-174)
// with the QP part from k_qp, then the step and FK.
__global__ void __launch_bounds__(64) k_step_coarse(DevHand H, DevParams P, StageArgs A, DevState st) {
  __shared__ WarpScratch smem_all[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * 2 + warp;
  if (g >= st.G || st.failed[g]) return;
  WarpScratch& s = smem_all[warp];
  for (int i = lane; i < H.D; i += 32) s.x[i] = st.x[(size_t)g * H.D + i];
  load_fk(H, st, g, lane, s);
  const bool with_grad = A.mode != 1;
  LinkAcc acc{mk(0, 0, 0), mk(0, 0, 0)};
  double e_lim, e_self;
  limit_and_self(H, P, s, lane, acc, with_grad, e_lim, e_self);

  const double* qres = st.qres + (size_t)g * st.NQ * 8;
  // Energy accumulated on lane 0 in the reference's order (pipeline.cpp:104-171).
  double total = P.w_limit * e_lim;
  total += P.w_self * e_self;
  // Hinge over every proxy (pipeline.cpp:116-129), items in proxy order.
  for (int base = 0; base < H.S; base += 32) {
    const int p = base + lane;
    double term = 0.0;
    bool active = false;
    if (p < H.S) {
      const double sd = qres[(size_t)p * 8] - H.proxy[4 * p + 3];
      if (sd < 0.0) {
        term = P.w_pen * sd * sd;
        active = true;
        s.itL[lane] = -1;
        if (with_grad) put_item(s, lane, H.proxy_link[p], ld3(s.pc + 3 * p), (P.w_pen * 2.0 * sd) * ld3(qres + p * 8 + 4));
      } else {
        s.itL[lane] = -1;
      }
    } else {
      s.itL[lane] = -1;
    }
    // Energy in reference order: sequential over proxies.
    add_terms(s, lane, term, total);
    if (with_grad) flush_items(s, lane, acc, __any_sync(kFull, active));
    __syncwarp();
  }
  // Tip distance terms (pipeline.cpp:133-163) and the QP force at the tip.
  {
    const int f = lane;
    double term = 0.0;
    s.itL[lane] = -1;
    if (f < H.m) {
      const int tp = H.tip_proxy[f];
      const double* q0 = qres + (size_t)tp * 8;
      const double r = q0[0] - H.proxy[4 * tp + 3] - A.offset;
      term = P.w_distance * r * r;
      if (with_grad) {
        const D3 n0 = ld3(q0 + 4);
        double dpn[3];
        const double h2 = 2.0 * P.fd_step;
        for (int kk = 0; kk < 3; ++kk) {
          const double* qp = qres + (size_t)(H.S + f * 6 + 2 * kk) * 8;
          const double* qm = qres + (size_t)(H.S + f * 6 + 2 * kk + 1) * 8;
          dpn[kk] = dot((ld3(qp + 1) - ld3(qm + 1)) / h2, n0);  // (dp^T n)_k
        }
        // dd = n^T (I - dp) -> force 2 w r (n - dp^T n)
        const D3 fw = (P.w_distance * 2.0 * r) * (n0 - mk(dpn[0], dpn[1], dpn[2]));
        put_item(s, lane, H.tip_link[f], ld3(s.pc + 3 * tp), fw);
      }
    }
    s.red[lane] = term;
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < H.m; ++i) total += s.red[i];
    if (with_grad) flush_items(s, lane, acc, true);
    s.itL[lane] = -1;
    if (with_grad && f < H.m)
      put_item(s, lane, H.tip_link[f], ld3(s.pc + 3 * H.tip_proxy[f]), ld3(st.qp_force + ((size_t)g * H.m + f) * 3));
    if (with_grad) flush_items(s, lane, acc, true);
  }
  if (lane == 0) total += P.w_grasp * st.qp_energy[g];
  total = __shfl_sync(kFull, total, 0);
  if (with_grad) expand_gradient(H, s, lane, acc);
  finish_iteration(H, P, A, st, g, lane, s, total);
}

struct Witness {
  D3 c_w, p_w, n;
  double d;
};

// fine_contact_query for tip f (pipeline.cpp:320-353) from the tip-center
// point query and the (tip link, part) pair results of this iteration.
__device__ inline Witness select_witness(const DevHand& H, const DevObject& O, const DevState& st, int g, int f,
                                         D3 center) {
  const int tp = H.tip_proxy[f];
  const double reference = st.qres[((size_t)g * st.NQ + tp) * 8] - H.proxy[4 * tp + 3];
  const double env = H.tip_envelope[f];
  const int link = H.tip_link[f];
  Witness w;
  w.d = INFINITY;
  w.c_w = w.p_w = mk(0, 0, 0);
  w.n = mk(0, 0, 1);
  int p0, p1;
  obj_parts(O, st, g, p0, p1);
  for (int p = 0; p < p1 - p0; ++p) {
    if (!(obb_sphere(O.part_obb + 15 * (p0 + p), center, env) < reference + 1e-9)) continue;
    const double* r = st.pairs + ((size_t)g * st.NP + link * O.Pmax + p) * 12;
    if (r[0] < w.d) {
      w.d = r[0];
      w.c_w = ld3(r + 1);
      w.p_w = ld3(r + 4);
      w.n = ld3(r + 7);
    }
  }
  return w;
}

// Mesh stages (pipeline.cpp:175-208): hinge over every (link part, object
// part), witness distance, detached-witness surrogate; then step and FK.
__global__ void __launch_bounds__(64) k_step_mesh(DevHand H, DevObject O, DevParams P, StageArgs A, DevState st) {
  __shared__ WarpScratch smem_all[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * 2 + warp;
  if (g >= st.G || st.failed[g]) return;
  WarpScratch& s = smem_all[warp];
  for (int i = lane; i < H.D; i += 32) s.x[i] = st.x[(size_t)g * H.D + i];
  load_fk(H, st, g, lane, s);
  const bool with_grad = A.mode != 1;
  LinkAcc acc{mk(0, 0, 0), mk(0, 0, 0)};
  double e_lim, e_self;
  limit_and_self(H, P, s, lane, acc, with_grad, e_lim, e_self);

  const int npairs = H.L * O.Pmax;  // slots past the object's parts hold +inf (no hinge)
  const double* pr = st.pairs + (size_t)g * st.NP * 12;
  double total = P.w_limit * e_lim;
  total += P.w_self * e_self;
  for (int base = 0; base < npairs; base += 32) {
    const int t = base + lane;
    double term = 0.0;
    bool active = false;
    s.itL[lane] = -1;
    if (t < npairs) {
      const double d = pr[(size_t)t * 12];
      if (d < 0.0) {
        term = P.w_pen * d * d;
        active = true;
        if (with_grad) put_item(s, lane, t / O.Pmax, ld3(pr + (size_t)t * 12 + 1), (P.w_pen * 2.0 * d) * ld3(pr + (size_t)t * 12 + 7));
      }
    }
    add_terms(s, lane, term, total);
    if (with_grad) flush_items(s, lane, acc, __any_sync(kFull, active));
    __syncwarp();
  }
  // Witness distance and surrogate terms.
  double sur = 0.0;
  {
    const int f = lane;
    double term = 0.0, sq = 0.0;
    Witness w;
    s.itL[lane] = -1;
    if (f < H.m) {
      w = select_witness(H, O, st, g, f, ld3(s.pc + 3 * H.tip_proxy[f]));
      const double r = w.d - A.offset;
      term = P.w_distance * r * r;
      if (with_grad) put_item(s, lane, H.tip_link[f], w.c_w, (P.w_distance * 2.0 * r) * w.n);
      const D3 diff = w.c_w - ld3(st.anchors + ((size_t)g * H.m + f) * 3);
      sq = sqn(diff);
      w.p_w = diff;  // reuse as the surrogate direction
    }
    s.red[lane] = term;
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < H.m; ++i) total += s.red[i];
    __syncwarp();
    s.red[lane] = sq;
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < H.m; ++i) sur += s.red[i];
    if (with_grad) flush_items(s, lane, acc, true);
    s.itL[lane] = -1;
    if (with_grad && f < H.m) put_item(s, lane, H.tip_link[f], w.c_w, (2.0 * P.w_grasp) * w.p_w);
    if (with_grad) flush_items(s, lane, acc, true);
  }
  if (lane == 0) total += P.w_grasp * sur;
  total = __shfl_sync(kFull, total, 0);
  if (with_grad) expand_gradient(H, s, lane, acc);
  finish_iteration(H, P, A, st, g, lane, s, total);
}

// FK from st.x for every live grasp (stage starts, teacher-forced calls).
__global__ void __launch_bounds__(64) k_fk(DevHand H, DevParams P, DevState st) {
  __shared__ WarpScratch smem_all[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * 2 + warp;
  if (g >= st.G || st.failed[g]) return;
  WarpScratch& s = smem_all[warp];
  for (int i = lane; i < H.D; i += 32) s.x[i] = st.x[(size_t)g * H.D + i];
  __syncwarp();
  warp_fk(H, st, g, lane, s, P.fd_step, true);
}

// After the coarse stage: anchors = nearest surface points of the tip
// centers at the final state (pipeline.cpp:69-78, 284-289).
__global__ void k_anchors(DevHand H, DevState st, int skip_fine) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= st.G || st.failed[g]) return;
  for (int f = 0; f < H.m; ++f) {
    const double* q = st.qres + ((size_t)g * st.NQ + H.tip_proxy[f]) * 8;
    st3(st.anchors + ((size_t)g * H.m + f) * 3, ld3(q + 1));
  }
  if (skip_fine) {
    for (int i = 0; i < H.D; ++i) st.x_p[(size_t)g * H.D + i] = st.x[(size_t)g * H.D + i];
    st.have_pregrasp[g] = 1;
  }
}

__global__ void k_set_pregrasp(DevHand H, DevState st) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= st.G || st.failed[g]) return;
  for (int i = 0; i < H.D; ++i) st.x_p[(size_t)g * H.D + i] = st.x[(size_t)g * H.D + i];
  st.have_pregrasp[g] = 1;
}

// Final record: witnesses at x -> contact frames (p_w, -n) for the cold QP
// (pipeline.cpp:302-311); also exposes the raw witnesses.
__global__ void k_final_frames(DevHand H, DevObject O, DevState st, double* witness_out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= st.G * H.m) return;
  const int g = t / H.m, f = t % H.m;
  if (st.failed[g]) return;
  const int l = H.tip_link[f];
  const double* w = st.world + ((size_t)g * H.L + l) * 12;
  M33 Rw;
  for (int i = 0; i < 9; ++i) Rw.m[i] = w[i];
  const D3 center = mul(Rw, ld3(H.proxy + 4 * H.tip_proxy[f])) + ld3(w + 9);
  const Witness wt = select_witness(H, O, st, g, f, center);
  build_frame(wt.p_w, -wt.n, st.frames + ((size_t)g * H.m + f) * 12);
  if (witness_out) {
    double* o = witness_out + ((size_t)g * H.m + f) * 11;
    st3(o, wt.c_w);
    st3(o + 3, wt.p_w);
    st3(o + 6, wt.n);
    o[9] = wt.d;
    o[10] = l;
  }
}

// Failed grasps report NaN energy and no QP fields (pipeline.cpp:312-314):
// the record buffers of failed rows are overwritten on the device, so host
// and device outputs of grasp_synthesize carry the same values.
__global__ void k_mask_failed(DevHand H, DevState st, int n_edges) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= st.G || !st.failed[g]) return;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  const int n = H.m * n_edges;
  st.qp_energy[g] = nan;
  for (int j = 0; j < 6; ++j) {
    st.qp_perdir[(size_t)g * 6 + j] = nan;
    st.qp_conv[(size_t)g * 6 + j] = 0;
  }
  for (int i = 0; i < n * 6; ++i) st.warm_x[(size_t)g * n * 6 + i] = nan;
  for (int i = 0; i < H.m * 12; ++i) st.frames[(size_t)g * H.m * 12 + i] = nan;
}

// Fingertip-centre query points from given world link transforms (the
// FkResult overload of fine_contact_query, pipeline.cpp:326-330).
__global__ void k_tip_points(DevHand H, DevState st) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= st.G * H.m) return;
  const int g = t / H.m, f = t % H.m;
  const double* w = st.world + ((size_t)g * H.L + H.tip_link[f]) * 12;
  M33 Rw;
  for (int i = 0; i < 9; ++i) Rw.m[i] = w[i];
  const D3 c = mul(Rw, ld3(H.proxy + 4 * H.tip_proxy[f])) + ld3(w + 9);
  st3(st.qpts + ((size_t)g * st.NQ + H.tip_proxy[f]) * 3, c);
}

// x_p fallback and squeeze (pipeline.cpp:296-300, 426-434).
__global__ void k_squeeze(DevHand H, DevState st, double* x_s) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= st.G) return;
  const int D = H.D;
  const double* x = st.x + (size_t)g * D;
  double* xp = st.x_p + (size_t)g * D;
  if (!st.have_pregrasp[g])
    for (int i = 0; i < D; ++i) xp[i] = x[i];
  double* xs = x_s + (size_t)g * D;
  if (st.failed[g]) {
    for (int i = 0; i < D; ++i) xs[i] = x[i];
    return;
  }
  M33 rg, rp;
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) {
      rg.m[i * 3 + c] = x[3 * c + i];
      rp.m[i * 3 + c] = xp[3 * c + i];
    }
  bool fb;
  const M33 Rg = project_rotation(rg, &fb);
  const M33 Rp = project_rotation(rp, &fb);
  const M33 R = mul(Rg, mul(transpose(Rp), Rg));
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) xs[3 * c + i] = R.m[i * 3 + c];
  for (int i = 9; i < 12; ++i) xs[i] = 2.0 * x[i] - xp[i];
  for (int j = 0; j < H.dof; ++j)
    xs[12 + j] = fmin(fmax(2.0 * x[12 + j] - xp[12 + j], H.joint_lower[j]), H.joint_upper[j]);
}

}  // namespace gdev

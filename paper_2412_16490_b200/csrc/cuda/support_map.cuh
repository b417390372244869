// Host construction of the GJK support maps (model.cuh: kSupportMapN,
// support_cell). Shared by engine.cu (upload) and the host exactness test
// tests/cpp/support_map_exact.cu.
#pragma once

#include "model.cuh"

#include <algorithm>
#include <cmath>
#include <vector>

namespace gdev {

// Support map of one hull (model.cuh): for every cube-map cell, the ascending
// list of vertices that can be the computed argmax of d . v for a direction d
// in the cell. Vertex i is left out only when the cell's maximiser j at the
// cell axis a beats it by a margin no rounding can close: for unit d in the
// cell's cone (half-angle th around a, dilated), d . (v_j - v_i) >=
// a . w - 2 sin(th / 2) |w|, and the device's fp64 dot products d . v carry
// at most gamma_3 |d| |v| < 4u |d| R error each (R = max |v|), so excluding
// only when that lower bound exceeds 8u R (+ 16u |w| for this host
// arithmetic) never drops a computed maximum. Appends the cell offsets
// (absolute into idx) to off and returns the map's base in off.
inline int build_support_map(const double* v, int nv, std::vector<int>& off, std::vector<unsigned short>& idx) {
  const int N = kSupportMapN;
  const double u = std::ldexp(1.0, -53);
  double R = 0.0;
  for (int i = 0; i < nv; ++i) R = std::max(R, std::sqrt(v[3 * i] * v[3 * i] + v[3 * i + 1] * v[3 * i + 1] + v[3 * i + 2] * v[3 * i + 2]));
  const int base = static_cast<int>(off.size());
  auto unit_dir = [](int face, double pu, double pv, double d[3]) {
    const int a = face / 2;
    const int b = a == 0 ? 1 : 0, c = a == 2 ? 1 : 2;
    d[a] = (face % 2 == 0) ? 1.0 : -1.0;
    d[b] = pu;
    d[c] = pv;
    const double n = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int k = 0; k < 3; ++k) d[k] /= n;
  };
  for (int face = 0; face < 6; ++face)
    for (int iv = 0; iv < N; ++iv)
      for (int iu = 0; iu < N; ++iu) {
        const double u0 = -1.0 + 2.0 * iu / N, u1 = -1.0 + 2.0 * (iu + 1) / N;
        const double v0 = -1.0 + 2.0 * iv / N, v1 = -1.0 + 2.0 * (iv + 1) / N;
        double a[3], cd[3];
        unit_dir(face, 0.5 * (u0 + u1), 0.5 * (v0 + v1), a);
        double th = 0.0;
        const double cu[2] = {u0, u1}, cv[2] = {v0, v1};
        for (double pu : cu)
          for (double pv : cv) {
            unit_dir(face, pu, pv, cd);
            const double c = std::min(1.0, std::max(-1.0, a[0] * cd[0] + a[1] * cd[1] + a[2] * cd[2]));
            th = std::max(th, std::acos(c));
          }
        th += 1e-6;  // covers directions the device bins across a cell boundary by rounding
        const double s2 = 2.0 * std::sin(0.5 * th);
        int j = 0;
        double tj = -INFINITY;
        for (int i = 0; i < nv; ++i) {
          const double t = a[0] * v[3 * i] + a[1] * v[3 * i + 1] + a[2] * v[3 * i + 2];
          if (t > tj) tj = t, j = i;
        }
        off.push_back(static_cast<int>(idx.size()));
        for (int i = 0; i < nv; ++i) {
          const double w[3] = {v[3 * j] - v[3 * i], v[3 * j + 1] - v[3 * i + 1], v[3 * j + 2] - v[3 * i + 2]};
          const double wn = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
          const double lower = a[0] * w[0] + a[1] * w[1] + a[2] * w[2] - s2 * wn;
          if (!(lower > 8.0 * u * R + 16.0 * u * wn)) idx.push_back(static_cast<unsigned short>(i));
        }
      }
  off.push_back(static_cast<int>(idx.size()));
  return base;
}

// Support maps for the hulls [begin[k], begin[k+1]) of a packed vertex array
// with at least kSupportMapMinVerts vertices; base[k] = -1 for the others.
inline void build_support_maps(const double* verts, const int* begin, int count, std::vector<int>& base,
                        std::vector<int>& off, std::vector<unsigned short>& idx) {
  base.assign(count, -1);
  for (int k = 0; k < count; ++k) {
    const int nv = begin[k + 1] - begin[k];
    if (nv >= kSupportMapMinVerts && nv <= 65535)
      base[k] = build_support_map(verts + 3 * static_cast<size_t>(begin[k]), nv, off, idx);
  }
  if (off.empty()) off.push_back(0);
  if (idx.empty()) idx.push_back(0);
}

}  // namespace gdev

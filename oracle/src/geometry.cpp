// ORACLE (test infrastructure only). Restates /root/reference/proj/src/geometry.cpp
// query functions in plain fp64: closest_on_triangle/query_part/point_to_mesh
// (:326-395, :527-542), support/GJK/EPA (:17-324, :399-412, :477-525) with an
// explicit restatement of Eigen::FullPivLU for the simplex solve (:76), and
// the OBB broad phase (:544-572).
#include "oracle_impl.hpp"

#include <cmath>
#include <limits>

namespace oracle {

namespace {
thread_local Stats* g_stats = nullptr;
}
Stats* stats_sink() { return g_stats; }
void set_stats_sink(Stats* s) { g_stats = s; }
void Stats::add(const Stats& o) {
  point_queries += o.point_queries; inside_faces += o.inside_faces; outside_faces += o.outside_faces;
  gjk_calls += o.gjk_calls; gjk_iters += o.gjk_iters; gjk_support_verts += o.gjk_support_verts;
  epa_calls += o.epa_calls; epa_iters += o.epa_iters; epa_face_scans += o.epa_face_scans;
  qp_solves += o.qp_solves; qp_sweeps += o.qp_sweeps; qp_column_sweeps += o.qp_column_sweeps;
  jacobians += o.jacobians; self_pairs += o.self_pairs; obb_tests += o.obb_tests;
}

namespace {

constexpr double kTouchTol = 1e-10;   // geometry.cpp:12
constexpr double kGjkRelTol = 1e-14;  // geometry.cpp:13
constexpr int kGjkMaxIters = 128;     // geometry.cpp:14
constexpr int kEpaMaxIters = 512;     // geometry.cpp:15
constexpr double kInf = std::numeric_limits<double>::infinity();

// Ericson closest point on a triangle (geometry.cpp:327-347).
V3 closest_on_triangle(const V3& p, const V3& a, const V3& b, const V3& c) {
  const V3 ab = b - a, ac = c - a, ap = p - a;
  const double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0 && d2 <= 0) return a;
  const V3 bp = p - b;
  const double d3 = dot(ab, bp), d4 = dot(ac, bp);
  if (d3 >= 0 && d4 <= d3) return b;
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) return a + ab * (d1 / (d1 - d3));
  const V3 cp = p - c;
  const double d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0 && d5 <= d6) return c;
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) return a + ac * (d2 / (d2 - d6));
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0 && d4 - d3 >= 0 && d5 - d6 >= 0) return b + (c - b) * ((d4 - d3) / ((d4 - d3) + (d5 - d6)));
  const double denom = 1.0 / (va + vb + vc);
  return a + ab * (vb * denom) + ac * (vc * denom);
}

struct PartHit {
  double sdist = kInf;
  V3 point;
  V3 normal = V3(0, 0, 1);
};

// geometry.cpp:355-395: inside test (break at first depth < -1e-12), else
// brute-force closest point over every face with strict '<'.
PartHit query_part(const V3& p, const Part& part) {
  Stats* st = g_stats;
  PartHit q;
  bool inside = true;
  double min_depth = kInf;
  V3 best_n(0, 0, 1);
  long long scanned = 0;
  for (const auto& t : part.faces) {
    ++scanned;
    const V3& a = part.verts[t[0]];
    V3 n = cross(part.verts[t[1]] - a, part.verts[t[2]] - a);
    const double len = norm(n);
    if (len < 1e-30) continue;
    n = n / len;
    const double depth = dot(n, a) - dot(n, p);
    if (depth < -1e-12) {
      inside = false;
      break;
    }
    if (depth < min_depth) {
      min_depth = depth;
      best_n = n;
    }
  }
  if (st) st->inside_faces += scanned;
  if (inside && std::isfinite(min_depth)) {
    q.sdist = -min_depth;
    q.normal = best_n;
    q.point = p + best_n * min_depth;
    return q;
  }
  for (const auto& t : part.faces) {
    const V3 c = closest_on_triangle(p, part.verts[t[0]], part.verts[t[1]], part.verts[t[2]]);
    const double d = norm(p - c);
    if (d < q.sdist) {
      q.sdist = d;
      q.point = c;
    }
  }
  if (st) st->outside_faces += static_cast<long long>(part.faces.size());
  q.normal = q.sdist > 1e-14 ? (p - q.point) / q.sdist : V3(0, 0, 1);
  return q;
}

// ---------------------------------------------------------------- GJK/EPA
struct SupportPoint {
  V3 w, a, b;
};

V3 support_point(const Part& part, const Rigid& pose, const V3& dir) {
  const V3 dl = pose.R.t() * dir;
  double best = -kInf;
  int arg = 0;
  for (int i = 0; i < static_cast<int>(part.verts.size()); ++i) {
    const double s = dot(dl, part.verts[i]);
    if (s > best) {
      best = s;
      arg = i;
    }
  }
  if (g_stats) g_stats->gjk_support_verts += static_cast<long long>(part.verts.size());
  return pose.apply(part.verts[arg]);
}

struct Support {
  const Part* pa;
  const Part* pb;
  Rigid ta, tb;
  SupportPoint operator()(const V3& dir) const {
    SupportPoint s;
    s.a = support_point(*pa, ta, dir);
    s.b = support_point(*pb, tb, -dir);
    s.w = s.a - s.b;
    return s;
  }
};

double cloud_scale(const Part& a, const Rigid& pa, const Part& b, const Rigid& pb) {
  double s = 1.0;
  s = std::max(s, norm(pa.apply(a.centroid)) + 2.0 * norm(a.obb_half));
  s = std::max(s, norm(pb.apply(b.centroid)) + 2.0 * norm(b.obb_half));
  return s;
}

// Eigen::FullPivLU(M).solve(rhs) restated: complete pivoting on the largest
// |entry| (first in column-major order on ties), rank from the threshold
// |u_ii| > max_pivot * n * eps, unit-lower then upper substitution on the
// rank-sized block, non-pivot unknowns set to zero.
void fullpiv_solve(int n, double* m /* n*n column-major */, const double* rhs, double* sol) {
  auto at = [&](int r, int c) -> double& { return m[c * n + r]; };
  int rowt[5], colt[5];
  int nonzero = n;
  double maxpivot = 0.0;
  for (int k = 0; k < n; ++k) {
    double biggest = -1.0;
    int br = k, bc = k;
    for (int c = k; c < n; ++c)
      for (int r = k; r < n; ++r) {
        const double v = std::abs(at(r, c));
        if (v > biggest) {
          biggest = v;
          br = r;
          bc = c;
        }
      }
    if (biggest == 0.0) {
      nonzero = k;
      for (int i = k; i < n; ++i) rowt[i] = colt[i] = i;
      break;
    }
    if (biggest > maxpivot) maxpivot = biggest;
    rowt[k] = br;
    colt[k] = bc;
    if (br != k)
      for (int c = 0; c < n; ++c) std::swap(at(k, c), at(br, c));
    if (bc != k)
      for (int r = 0; r < n; ++r) std::swap(at(r, k), at(r, bc));
    if (k < n - 1) {
      const double piv = at(k, k);
      for (int r = k + 1; r < n; ++r) at(r, k) /= piv;
      for (int c = k + 1; c < n; ++c)
        for (int r = k + 1; r < n; ++r) at(r, c) -= at(r, k) * at(k, c);
    }
  }
  const double thresh = maxpivot * (n * std::numeric_limits<double>::epsilon());
  int rank = 0;
  for (int i = 0; i < nonzero; ++i) rank += std::abs(at(i, i)) > thresh;
  if (rank == 0) {
    for (int i = 0; i < n; ++i) sol[i] = 0.0;
    return;
  }
  double c[5];
  for (int i = 0; i < n; ++i) c[i] = rhs[i];
  for (int k = 0; k < n; ++k) std::swap(c[k], c[rowt[k]]);
  // Unit-lower forward substitution (column oriented, like Eigen's trsv).
  for (int i = 0; i < n; ++i)
    if (c[i] != 0.0)
      for (int r = i + 1; r < n; ++r) c[r] -= c[i] * at(r, i);
  // Upper substitution on the leading rank x rank block.
  for (int i = rank - 1; i >= 0; --i)
    if (c[i] != 0.0) {
      c[i] /= at(i, i);
      for (int r = 0; r < i; ++r) c[r] -= c[i] * at(r, i);
    }
  int perm[5];
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) std::swap(perm[k], perm[colt[k]]);
  for (int i = 0; i < n; ++i) sol[perm[i]] = i < rank ? c[i] : 0.0;
}

struct SimplexSolve {
  double dist2 = kInf;
  V3 v;
  int keep[4];
  double weights[4];
  int nkeep = 0;
  bool contains_origin = false;
};

// geometry.cpp:58-95.
SimplexSolve closest_on_simplex(const SupportPoint* simp, int n) {
  SimplexSolve best;
  for (int mask = 1; mask < (1 << n); ++mask) {
    int idx[4];
    int k = 0;
    for (int i = 0; i < n; ++i)
      if (mask & (1 << i)) idx[k++] = i;
    double M[25];
    double rhs[5] = {0, 0, 0, 0, 0};
    const int s = k + 1;
    for (int i = 0; i < k; ++i) {
      for (int j = 0; j < k; ++j) M[j * s + i] = dot(simp[idx[i]].w, simp[idx[j]].w);
      M[k * s + i] = 1.0;
      M[i * s + k] = 1.0;
    }
    M[k * s + k] = 0.0;
    rhs[k] = 1.0;
    double sol[5];
    fullpiv_solve(s, M, rhs, sol);
    bool ok = true;
    for (int i = 0; i < s; ++i) ok = ok && std::isfinite(sol[i]);
    for (int i = 0; ok && i < k; ++i)
      if (sol[i] < -1e-12) ok = false;
    if (!ok) continue;
    V3 v;
    for (int i = 0; i < k; ++i) v += sol[i] * simp[idx[i]].w;
    const double d2 = sqnorm(v);
    if (d2 < best.dist2 - 1e-300 || (k < best.nkeep && d2 <= best.dist2 * (1.0 + 1e-12))) {
      best.dist2 = d2;
      best.v = v;
      best.nkeep = k;
      for (int i = 0; i < k; ++i) {
        best.keep[i] = idx[i];
        best.weights[i] = sol[i];
      }
      if (k == 4) best.contains_origin = true;
    }
  }
  return best;
}

struct GjkOut {
  double distance = 0.0;
  V3 wa, wb;
  bool overlap = false;
  std::vector<SupportPoint> simplex;
};

// geometry.cpp:105-164.
GjkOut gjk_run(const Support& support, double scale) {
  if (g_stats) ++g_stats->gjk_calls;
  GjkOut res;
  SupportPoint simp[4];
  int ns = 1;
  simp[0] = support(V3(1, 0, 0));
  auto witnesses = [&](const SimplexSolve& s, const SupportPoint* pts, bool use_keep) {
    V3 wa, wb;
    for (int i = 0; i < s.nkeep; ++i) {
      const SupportPoint& p = use_keep ? pts[s.keep[i]] : pts[i];
      wa += s.weights[i] * p.a;
      wb += s.weights[i] * p.b;
    }
    res.wa = wa;
    res.wb = wb;
  };
  for (int iter = 0; iter < kGjkMaxIters; ++iter) {
    if (g_stats) ++g_stats->gjk_iters;
    const SimplexSolve s = closest_on_simplex(simp, ns);
    const V3 v = s.v;
    SupportPoint reduced[4];
    for (int i = 0; i < s.nkeep; ++i) reduced[i] = simp[s.keep[i]];
    ns = s.nkeep;
    for (int i = 0; i < ns; ++i) simp[i] = reduced[i];

    if (s.contains_origin || std::sqrt(s.dist2) < kTouchTol * scale) {
      res.overlap = true;
      res.distance = 0.0;
      witnesses(s, simp, false);
      res.simplex.assign(simp, simp + ns);
      return res;
    }
    const SupportPoint w = support(-v);
    const double gap = s.dist2 - dot(v, w.w);
    bool repeat = false;
    for (int i = 0; i < ns; ++i)
      if (norm(simp[i].w - w.w) < 1e-14 * scale) repeat = true;
    if (gap <= kGjkRelTol * s.dist2 + 1e-300 || repeat || ns == 4) {
      res.distance = std::sqrt(s.dist2);
      witnesses(s, simp, false);
      res.simplex.assign(simp, simp + ns);
      return res;
    }
    simp[ns++] = w;
  }
  const SimplexSolve s = closest_on_simplex(simp, ns);
  res.distance = std::sqrt(s.dist2);
  witnesses(s, simp, true);
  res.simplex.assign(simp, simp + ns);
  return res;
}

// geometry.cpp:168-205.
bool pad_to_tetrahedron(std::vector<SupportPoint>& simp, const Support& support, double scale) {
  const double tol = 1e-12 * scale;
  auto independent = [&](const SupportPoint& cand) {
    if (simp.empty()) return true;
    if (simp.size() == 1) return norm(cand.w - simp[0].w) > tol;
    if (simp.size() == 2) {
      const V3 d = normalized(simp[1].w - simp[0].w);
      const V3 r = cand.w - simp[0].w;
      return norm(r - d * dot(d, r)) > tol;
    }
    const V3 n = normalized(cross(simp[1].w - simp[0].w, simp[2].w - simp[0].w));
    return std::abs(dot(n, cand.w - simp[0].w)) > tol;
  };
  std::vector<V3> dirs = {V3(1, 0, 0), V3(-1, 0, 0), V3(0, 1, 0), V3(0, -1, 0), V3(0, 0, 1), V3(0, 0, -1)};
  if (simp.size() == 2) {
    const V3 d = normalized(simp[1].w - simp[0].w);
    const V3 t = std::abs(d.x()) < 0.9 ? V3(1, 0, 0) : V3(0, 1, 0);
    const V3 e1 = normalized(cross(d, t));
    const V3 e2 = cross(d, e1);
    dirs.insert(dirs.begin(), {e1, -e1, e2, -e2});
  }
  if (simp.size() == 3) {
    const V3 n = normalized(cross(simp[1].w - simp[0].w, simp[2].w - simp[0].w));
    dirs.insert(dirs.begin(), {n, -n});
  }
  for (const V3& d : dirs) {
    if (simp.size() == 4) break;
    const SupportPoint cand = support(d);
    if (independent(cand)) simp.push_back(cand);
  }
  return simp.size() == 4;
}

struct EpaFace {
  int v[3];
  V3 n;
  double d = 0.0;
  bool alive = true;
};

bool lex_less(const V3& a, const V3& b) {
  if (a.x() != b.x()) return a.x() < b.x();
  if (a.y() != b.y()) return a.y() < b.y();
  return a.z() < b.z();
}

struct EpaOut {
  double depth = 0.0;
  V3 direction = V3(0, 0, 1);
  V3 wa, wb;
};

// geometry.cpp:227-324.
EpaOut epa_run(std::vector<SupportPoint> simp, const Support& support, double scale) {
  if (g_stats) ++g_stats->epa_calls;
  if (!pad_to_tetrahedron(simp, support, scale)) throw GeometryError("penetration query on a degenerate shape pair");
  std::vector<SupportPoint> verts = std::move(simp);
  const V3 interior = (verts[0].w + verts[1].w + verts[2].w + verts[3].w) / 4.0;
  std::vector<EpaFace> faces;
  auto make_face = [&](int i0, int i1, int i2) {
    EpaFace f;
    f.v[0] = i0; f.v[1] = i1; f.v[2] = i2;
    const V3 n = cross(verts[i1].w - verts[i0].w, verts[i2].w - verts[i0].w);
    const double len = norm(n);
    f.n = len > 0 ? n / len : V3(0, 0, 1);
    f.d = dot(f.n, verts[i0].w);
    if (dot(f.n, interior) > f.d) {
      std::swap(f.v[1], f.v[2]);
      f.n = -f.n;
      f.d = -f.d;
    }
    return f;
  };
  faces.push_back(make_face(0, 1, 2));
  faces.push_back(make_face(0, 2, 3));
  faces.push_back(make_face(0, 3, 1));
  faces.push_back(make_face(1, 3, 2));

  const double grow_tol = 1e-10 * scale;
  int best_face = -1;
  for (int iter = 0; iter < kEpaMaxIters; ++iter) {
    if (g_stats) { ++g_stats->epa_iters; g_stats->epa_face_scans += static_cast<long long>(faces.size()); }
    best_face = -1;
    double best_d = kInf;
    for (int i = 0; i < static_cast<int>(faces.size()); ++i) {
      if (!faces[i].alive) continue;
      const double di = faces[i].d;
      if (di < best_d - 1e-12 * scale ||
          (di < best_d + 1e-12 * scale && best_face >= 0 && lex_less(-faces[i].n, -faces[best_face].n))) {
        best_d = std::min(best_d, di);
        best_face = i;
      }
    }
    if (best_face < 0) throw GeometryError("penetration polytope lost all faces");
    const EpaFace f = faces[best_face];
    const SupportPoint w = support(f.n);
    if (dot(f.n, w.w) - f.d <= grow_tol) break;
    const int wi = static_cast<int>(verts.size());
    verts.push_back(w);
    std::vector<std::pair<int, int>> horizon;
    for (EpaFace& g : faces) {
      if (!g.alive) continue;
      if (dot(g.n, w.w) - g.d > 1e-12 * scale) {
        g.alive = false;
        for (int e = 0; e < 3; ++e) horizon.push_back({g.v[e], g.v[(e + 1) % 3]});
      }
    }
    std::vector<std::pair<int, int>> boundary;
    for (const auto& e : horizon) {
      bool paired = false;
      for (const auto& o : horizon)
        if (o.first == e.second && o.second == e.first) paired = true;
      if (!paired) boundary.push_back(e);
    }
    if (boundary.empty()) break;
    for (const auto& e : boundary) faces.push_back(make_face(e.first, e.second, wi));
  }

  const EpaFace& f = faces[best_face];
  EpaOut out;
  out.depth = std::max(f.d, 0.0);
  out.direction = -f.n;
  const SupportPoint tri[3] = {verts[f.v[0]], verts[f.v[1]], verts[f.v[2]]};
  const SimplexSolve s = closest_on_simplex(tri, 3);
  V3 wa, wb;
  double wsum = 0.0;
  for (int i = 0; i < s.nkeep; ++i) {
    wa += s.weights[i] * tri[s.keep[i]].a;
    wb += s.weights[i] * tri[s.keep[i]].b;
    wsum += s.weights[i];
  }
  if (wsum > 0.5) {
    out.wa = wa;
    out.wb = wb;
  } else {
    out.wa = tri[0].a;
    out.wb = tri[0].b;
  }
  return out;
}

}  // namespace

Nearest point_to_mesh(const V3& p, const std::vector<Part>& parts) {
  if (parts.empty()) throw GeometryError("point query against an empty part list");
  if (g_stats) ++g_stats->point_queries;
  Nearest best;
  best.distance = kInf;
  for (int i = 0; i < static_cast<int>(parts.size()); ++i) {
    const PartHit q = query_part(p, parts[i]);
    if (q.sdist < best.distance) {
      best.distance = q.sdist;
      best.b = q.point;
      best.normal = q.normal;
      best.part = i;
    }
  }
  best.a = p;
  return best;
}

Nearest gjk_distance(const Part& a, const Rigid& pa, const Part& b, const Rigid& pb) {
  const Support support{&a, &b, pa, pb};
  const GjkOut r = gjk_run(support, cloud_scale(a, pa, b, pb));
  Nearest out;
  out.a = r.wa;
  out.b = r.wb;
  out.distance = r.distance;
  out.normal = r.distance > 1e-14 ? (r.wa - r.wb) / r.distance : V3(0, 0, 1);
  return out;
}

std::pair<double, V3> epa_depth(const Part& a, const Rigid& pa, const Part& b, const Rigid& pb) {
  const Support support{&a, &b, pa, pb};
  const double scale = cloud_scale(a, pa, b, pb);
  GjkOut g = gjk_run(support, scale);
  if (!g.overlap) throw GeometryError("penetration depth queried on disjoint parts");
  const EpaOut r = epa_run(std::move(g.simplex), support, scale);
  return {r.depth, r.direction};
}

double signed_distance(const Part& a, const Rigid& pa, const Part& b, const Rigid& pb, Nearest* out, bool* used_epa) {
  const Support support{&a, &b, pa, pb};
  const double scale = cloud_scale(a, pa, b, pb);
  GjkOut g = gjk_run(support, scale);
  if (used_epa) *used_epa = g.overlap;
  if (!g.overlap) {
    if (out) {
      out->a = g.wa;
      out->b = g.wb;
      out->distance = g.distance;
      out->normal = g.distance > 1e-14 ? (g.wa - g.wb) / g.distance : V3(0, 0, 1);
    }
    return g.distance;
  }
  const EpaOut r = epa_run(std::move(g.simplex), support, scale);
  if (out) {
    out->a = r.wa;
    out->b = r.wb;
    out->distance = -r.depth;
    out->normal = r.direction;
  }
  return -r.depth;
}

// geometry.cpp:544-557 with an identity part pose (object frame).
double obb_sphere_distance(const Part& part, const V3& center, double radius) {
  if (g_stats) ++g_stats->obb_tests;
  const V3 q = part.obb_rot.t() * (center - part.obb_center);
  V3 excess;
  for (int i = 0; i < 3; ++i) excess[i] = std::abs(q[i]) - part.obb_half[i];
  double dist;
  if (excess[0] <= 0 && excess[1] <= 0 && excess[2] <= 0) {
    dist = std::max(excess[0], std::max(excess[1], excess[2]));
  } else {
    V3 pos;
    for (int i = 0; i < 3; ++i) pos[i] = std::max(excess[i], 0.0);
    dist = norm(pos);
  }
  return dist - radius;
}

// geometry.cpp:559-572.
std::vector<int> broadphase_cull(const V3& center, double radius, const std::vector<Part>& parts, double reference) {
  std::vector<int> keep;
  for (int i = 0; i < static_cast<int>(parts.size()); ++i)
    if (obb_sphere_distance(parts[i], center, radius) < reference + 1e-9) keep.push_back(i);
  return keep;
}

}  // namespace oracle

// Load-time convex part construction (reference proj/src/geometry.cpp:414-475).
#include "grasp/geometry.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

namespace grasp::geom {
namespace {

// Cyclic Jacobi eigen-decomposition of a symmetric 3x3 matrix; eigenvalues
// ascending with the first-minimum selection swap Eigen's
// SelfAdjointEigenSolver uses to sort (Eigenvalues/SelfAdjointEigenSolver.h).
// The OBB only feeds the broad-phase lower bound, whose soundness makes the
// axis choice result-neutral (reference test_pipeline.cpp:218-260).
void symmetric_eigen(const Mat3& a_in, Vec3& evals, Mat3& evecs) {
  double a[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a[r][c] = a_in(r, c);
  double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = std::abs(a[0][1]) + std::abs(a[0][2]) + std::abs(a[1][2]);
    const double diag = std::abs(a[0][0]) + std::abs(a[1][1]) + std::abs(a[2][2]);
    if (off == 0.0 || off <= 1e-20 * diag) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0);
        const double s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  double ev[3] = {a[0][0], a[1][1], a[2][2]};
  int order[3] = {0, 1, 2};
  for (int i = 0; i < 2; ++i) {
    int k = i;
    for (int j = i + 1; j < 3; ++j)
      if (ev[order[j]] < ev[order[k]]) k = j;
    if (k != i) std::swap(order[i], order[k]);
  }
  for (int i = 0; i < 3; ++i) {
    evals[i] = ev[order[i]];
    evecs.set_col(i, Vec3(v[0][order[i]], v[1][order[i]], v[2][order[i]]));
  }
}

}  // namespace

ConvexPart make_convex_part(std::span<const Vec3> points, double merge_tol) {
  detail::HullMesh mesh = detail::convex_hull(points, merge_tol);
  ConvexPart part;
  part.vertices = std::move(mesh.vertices);
  part.faces = std::move(mesh.faces);

  // Divergence theorem over origin-based tetrahedra (geometry.cpp:421-434).
  double vol = 0.0;
  Vec3 cw = Vec3::Zero();
  for (const auto& t : part.faces) {
    const Vec3& a = part.vertices[t[0]];
    const Vec3& b = part.vertices[t[1]];
    const Vec3& c = part.vertices[t[2]];
    const double v6 = dot(a, cross(b, c));
    vol += v6;
    cw += v6 * (a + b + c);
  }
  part.volume = vol / 6.0;
  if (part.volume <= 0) throw GeometryError("hull volume is not positive; input nearly degenerate");
  part.centroid = cw / (4.0 * vol);

  // PCA box with pinned axis order/sign/handedness (geometry.cpp:438-464).
  Vec3 mean = Vec3::Zero();
  for (const Vec3& v : part.vertices) mean += v;
  mean /= static_cast<double>(part.vertices.size());
  Mat3 cov = Mat3::Zero();
  for (const Vec3& v : part.vertices) cov = cov + outer(v - mean, v - mean);
  Vec3 evals;
  Mat3 evecs;
  symmetric_eigen(cov, evals, evecs);
  Mat3 axes;
  axes.set_col(0, evecs.col(2));
  axes.set_col(1, evecs.col(1));
  axes.set_col(2, evecs.col(0));
  for (int c = 0; c < 3; ++c) {
    const Vec3 col = axes.col(c);
    int arg = 0;
    double best = std::abs(col[0]);
    for (int r = 1; r < 3; ++r)
      if (std::abs(col[r]) > best) { best = std::abs(col[r]); arg = r; }
    if (col[arg] < 0) axes.set_col(c, -col);
  }
  if (axes.determinant() < 0) axes.set_col(2, -axes.col(2));

  Vec3 lo = Vec3::Constant(std::numeric_limits<double>::infinity());
  Vec3 hi = -lo;
  const Mat3 at = axes.transpose();
  for (const Vec3& v : part.vertices) {
    const Vec3 q = at * v;
    lo = cwise_min(lo, q);
    hi = cwise_max(hi, q);
  }
  part.obb.rotation = axes;
  part.obb.center = axes * ((lo + hi) / 2.0);
  part.obb.half_extents = (hi - lo) / 2.0;
  return part;
}

ConvexPart transformed(const ConvexPart& part, const RigidTransform& pose) {
  ConvexPart out = part;
  for (Vec3& v : out.vertices) v = pose.apply(v);
  out.centroid = pose.apply(part.centroid);
  out.obb.center = pose.apply(part.obb.center);
  out.obb.rotation = pose.R * part.obb.rotation;
  return out;
}

}  // namespace grasp::geom

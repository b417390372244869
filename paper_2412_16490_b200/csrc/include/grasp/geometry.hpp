// Convex geometry value types and load-time construction. The per-query
// functions of the reference (point_to_mesh, gjk_distance, epa_depth,
// signed_distance, broadphase_cull; proj/include/grasp/geometry.hpp:74-121)
// run as batched sm_100a kernels behind include/grasp_b200.h.
#pragma once

#include "grasp/la.hpp"

#include <array>
#include <span>
#include <stdexcept>
#include <vector>

namespace grasp::geom {

using Vector3d = Vec3;
using Matrix3d = Mat3;
using grasp::RigidTransform;

/// Oriented bounding box in the part's local frame (geometry.hpp:31-35).
struct Obb {
  Vec3 center = Vec3::Zero();
  Vec3 half_extents = Vec3::Zero();
  Mat3 rotation = Mat3::Identity();  // columns are box axes
};

/// Hulled convex piece (geometry.hpp:40-46).
struct ConvexPart {
  std::vector<Vec3> vertices;
  std::vector<std::array<int, 3>> faces;  // outward-oriented triangles
  Obb obb;
  double volume = 0.0;
  Vec3 centroid = Vec3::Zero();
};

struct SphereProxy {
  Vec3 center_local = Vec3::Zero();
  double radius = 0.0;
  int link_id = -1;
};

/// Signed nearest-point result; normal points from b toward a (geometry.hpp:54-63).
struct NearestPointResult {
  Vec3 point_a = Vec3::Zero();
  Vec3 point_b = Vec3::Zero();
  double distance = 0.0;
  Vec3 normal = Vec3::UnitZ();
  int part_index = -1;
};

struct GeometryError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline constexpr double kVertexMergeTol = 1e-9;

/// Dedup + quickhull + volume/centroid + PCA OBB (geometry.cpp:414-466).
ConvexPart make_convex_part(std::span<const Vec3> points, double merge_tol = kVertexMergeTol);

/// Moves vertices, centroid and OBB by a rigid transform (geometry.cpp:468-475).
ConvexPart transformed(const ConvexPart& part, const RigidTransform& pose);

namespace detail {
struct HullMesh {
  std::vector<Vec3> vertices;
  std::vector<std::array<int, 3>> faces;
};
/// Incremental quickhull with vertex merge (hull3d.cpp:291-303).
HullMesh convex_hull(std::span<const Vec3> points, double merge_tol);
}  // namespace detail

}  // namespace grasp::geom

// Host-side start states and squeeze poses (reference proj/src/pipeline.cpp:388-434).
// The same libstdc++ <random> engine and distributions as the reference give
// identical draws for a seed; Eigen's quaternion arithmetic is restated below.
#include "grasp/pipeline.hpp"

#include <algorithm>
#include <cmath>
#include <numbers>
#include <random>

namespace grasp::pipeline {
namespace {

struct Quat {
  double x, y, z, w;
};

// Eigen QuaternionBase::setFromTwoVectors (Eigen/src/Geometry/Quaternion.h).
Quat from_two_vectors(const Vec3& a, const Vec3& b) {
  const Vec3 v0 = normalized(a);
  const Vec3 v1 = normalized(b);
  double c = dot(v1, v0);
  if (c < -1.0 + 1e-12) {
    // Nearly opposite: any unit axis orthogonal to both (Eigen takes the SVD
    // null vector; the case has probability zero for Gaussian draws).
    c = std::max(c, -1.0);
    Vec3 axis = cross(v0, std::abs(v0.x) < 0.9 ? Vec3::UnitX() : Vec3::UnitY());
    axis = normalized(axis);
    const double w2 = (1.0 + c) * 0.5;
    const double sv = std::sqrt(1.0 - w2);
    return {axis.x * sv, axis.y * sv, axis.z * sv, std::sqrt(w2)};
  }
  const Vec3 axis = cross(v0, v1);
  const double s = std::sqrt((1.0 + c) * 2.0);
  const double invs = 1.0 / s;
  return {axis.x * invs, axis.y * invs, axis.z * invs, s * 0.5};
}

// Quaternion(AngleAxis): w = cos(a/2), vec = sin(a/2) * axis.
Quat from_angle_axis(double angle, const Vec3& axis) {
  const double ha = 0.5 * angle;
  const double s = std::sin(ha);
  return {s * axis.x, s * axis.y, s * axis.z, std::cos(ha)};
}

// Eigen's SSE2 quat_product association (Eigen/src/Geometry/arch/Geometry_SIMD.h).
Quat multiply(const Quat& a, const Quat& b) {
  Quat r;
  r.x = (a.w * b.x + a.y * b.z) - (a.z * b.y - a.x * b.w);
  r.y = (a.w * b.y + a.y * b.w) + (a.z * b.x - a.x * b.z);
  r.z = (a.w * b.z - a.y * b.x) + (a.z * b.w + a.x * b.y);
  r.w = (a.w * b.w - a.y * b.y) - (a.z * b.z + a.x * b.x);
  return r;
}

// QuaternionBase::toRotationMatrix.
Mat3 to_matrix(const Quat& q) {
  const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  Mat3 r;
  r(0, 0) = 1.0 - (tyy + tzz);
  r(0, 1) = txy - twz;
  r(0, 2) = txz + twy;
  r(1, 0) = txy + twz;
  r(1, 1) = 1.0 - (txx + tzz);
  r(1, 2) = tyz - twx;
  r(2, 0) = txz - twy;
  r(2, 1) = tyz + twx;
  r(2, 2) = 1.0 - (txx + tyy);
  return r;
}

}  // namespace

std::vector<VectorXd> init_poses(const hand::HandModel& model, const object::ObjectModel& object, int n,
                                 std::uint64_t seed, const InitParams& params) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  std::uniform_real_distribution<double> roll_draw(0.0, 2.0 * std::numbers::pi);
  std::uniform_real_distribution<double> jitter(-0.5, 0.5);

  const double ring = object::bounding_radius(object) + params.standoff;
  const VectorXd lo = model.lower_limits();
  const VectorXd hi = model.upper_limits();

  std::vector<VectorXd> states;
  states.reserve(n);
  for (int i = 0; i < n; ++i) {
    Vec3 u;
    do {
      // The reference writes Vector3d(gauss(rng), gauss(rng), gauss(rng));
      // GCC evaluates those arguments right to left, so the first draw lands
      // in z. Drawing explicitly keeps that order on any compiler.
      const double g_first = gauss(rng);
      const double g_second = gauss(rng);
      const double g_third = gauss(rng);
      u = Vec3(g_third, g_second, g_first);
    } while (norm(u) < 1e-9);
    u = normalized(u);
    const double roll = roll_draw(rng);

    hand::HandPose pose;
    pose.R = to_matrix(multiply(from_two_vectors(Vec3::UnitZ(), -u), from_angle_axis(roll, Vec3::UnitZ())));
    pose.t = ring * u;
    pose.q.resize(model.dof());
    for (int j = 0; j < model.dof(); ++j) {
      const double mid = 0.5 * (lo[j] + hi[j]);
      const double q = mid + params.joint_span_fraction * (hi[j] - lo[j]) * jitter(rng);
      pose.q[j] = std::clamp(q, lo[j], hi[j]);
    }
    states.push_back(hand::state_from_pose(model, pose));
  }
  return states;
}

VectorXd squeeze_pose(const hand::HandModel& model, const VectorXd& x, const VectorXd& x_p) {
  const hand::HandPose grasp = hand::pose_from_state(model, x);
  const hand::HandPose pre = hand::pose_from_state(model, x_p);
  hand::HandPose out;
  out.R = grasp.R * (pre.R.transpose() * grasp.R);
  out.t = 2.0 * grasp.t - pre.t;
  out.q.resize(model.dof());
  const VectorXd lo = model.lower_limits(), hi = model.upper_limits();
  for (int j = 0; j < model.dof(); ++j) {
    const double v = 2.0 * grasp.q[j] - pre.q[j];
    out.q[j] = std::min(std::max(v, lo[j]), hi[j]);
  }
  return hand::state_from_pose(model, out);
}

}  // namespace grasp::pipeline

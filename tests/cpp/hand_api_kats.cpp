// The reference's hand-API tests (proj/tests/test_hand.cpp:62-252 and the surrogate case of
// test_energy.cpp:516-564), written against this repo's drop-in C++ headers
// (csrc/include/grasp/hand.hpp, energy.hpp) and linked to libgrasp_b200.so. Host only: these
// are the reference's single-state API functions, not the batched device path.
#include "grasp/energy.hpp"
#include "grasp/hand.hpp"

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

using namespace grasp;
using namespace grasp::hand;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      ++failures;                                                     \
      std::printf("CHECK failed line %d: %s\n", __LINE__, #cond);     \
    }                                                                 \
  } while (0)

static Mat3 quat_rotation(std::mt19937_64& rng) {
  std::normal_distribution<double> g(0.0, 1.0);
  double w = g(rng), x = g(rng), y = g(rng), z = g(rng);
  const double n = std::sqrt(w * w + x * x + y * y + z * z);
  w /= n, x /= n, y /= n, z /= n;
  Mat3 R;
  R(0, 0) = 1 - 2 * (y * y + z * z), R(0, 1) = 2 * (x * y - w * z), R(0, 2) = 2 * (x * z + w * y);
  R(1, 0) = 2 * (x * y + w * z), R(1, 1) = 1 - 2 * (x * x + z * z), R(1, 2) = 2 * (y * z - w * x);
  R(2, 0) = 2 * (x * z - w * y), R(2, 1) = 2 * (y * z + w * x), R(2, 2) = 1 - 2 * (x * x + y * y);
  return R;
}

static VectorXd random_state(const HandModel& m, std::mt19937_64& rng) {
  HandPose pose;
  pose.R = quat_rotation(rng);
  std::normal_distribution<double> g(0.0, 0.1);
  pose.t = Vec3(g(rng), g(rng), g(rng));
  for (int j = 0; j < m.dof(); ++j) {
    std::uniform_real_distribution<double> u(m.joints[j].lower, m.joints[j].upper);
    pose.q.push_back(u(rng));
  }
  return state_from_pose(m, pose);
}

static Mat3 raw_of(const VectorXd& x) {
  Mat3 r;
  for (int i = 0; i < 9; ++i) r.m[i] = x[i];
  return r;
}

template <class F>
static MatrixXd fd_jacobian3(F&& f, const VectorXd& x, double h = 1e-6) {
  MatrixXd j(3, static_cast<int>(x.size()));
  VectorXd xp = x;
  for (size_t i = 0; i < x.size(); ++i) {
    xp[i] = x[i] + h;
    const Vec3 fp = f(xp);
    xp[i] = x[i] - h;
    const Vec3 fm = f(xp);
    xp[i] = x[i];
    for (int r = 0; r < 3; ++r) j(r, static_cast<int>(i)) = (fp[r] - fm[r]) / (2 * h);
  }
  return j;
}

template <class F>
static VectorXd fd_gradient(F&& f, const VectorXd& x, double h = 1e-6) {
  VectorXd g(x.size());
  VectorXd xp = x;
  for (size_t i = 0; i < x.size(); ++i) {
    xp[i] = x[i] + h;
    const double fp = f(xp);
    xp[i] = x[i] - h;
    const double fm = f(xp);
    xp[i] = x[i];
    g[i] = (fp - fm) / (2 * h);
  }
  return g;
}

static double max_abs_diff(const MatrixXd& a, const MatrixXd& b) {
  double m = 0.0;
  for (size_t i = 0; i < a.data.size(); ++i) m = std::fmax(m, std::fabs(a.data[i] - b.data[i]));
  return m;
}

int main() {
  const HandModel& m = builtin_hand();
  // test_hand.cpp:112-135: tangent Jacobian vs numeric projection derivatives.
  {
    std::mt19937_64 rng(47);
    std::normal_distribution<double> g(0.0, 0.15);
    int checked = 0;
    for (int k = 0; k < 200; ++k) {
      Mat3 raw = quat_rotation(rng);
      for (double& v : raw.m) v += g(rng);
      const PoseState ps = make_pose_state(raw);
      if (ps.degenerate) continue;
      ++checked;
      const MatrixXd j = rotation_tangent_jacobian(ps);
      const double h = 1e-6;
      for (int c = 0; c < 9; ++c) {
        Mat3 rp = raw, rm = raw;
        rp.m[c] += h;
        rm.m[c] -= h;
        const Mat3 dr = (1.0 / (2 * h)) * (project_rotation(rp).R - project_rotation(rm).R);
        const Mat3 s = ps.R.transpose() * dr;
        const Vec3 w(0.5 * (s(2, 1) - s(1, 2)), 0.5 * (s(0, 2) - s(2, 0)), 0.5 * (s(1, 0) - s(0, 1)));
        CHECK(norm(j.col3(c) - w) < 1e-5 * (1.0 + norm(w)));
      }
    }
    CHECK(checked >= 150);
  }
  // test_hand.cpp:152-183: point and direction Jacobians vs finite differences.
  {
    std::mt19937_64 rng(59);
    std::normal_distribution<double> g(0.0, 0.02);
    for (int k = 0; k < 30; ++k) {
      const VectorXd x = random_state(m, rng);
      const int link = static_cast<int>(rng() % m.links.size());
      const Vec3 p_local(g(rng), g(rng), g(rng));
      auto world_point = [&](const VectorXd& xs) {
        return forward_kinematics(m, pose_from_state(m, xs)).world[link].apply(p_local);
      };
      auto world_dir = [&](const VectorXd& xs) {
        return forward_kinematics(m, pose_from_state(m, xs)).world[link].rotate(Vec3::UnitZ());
      };
      const HandPose pose = pose_from_state(m, x);
      const FkResult fk = forward_kinematics(m, pose);
      const PoseState ps = make_pose_state(raw_of(x));
      CHECK(max_abs_diff(point_jacobian(m, ps, pose, fk, link, world_point(x)), fd_jacobian3(world_point, x)) < 5e-6);
      CHECK(max_abs_diff(direction_jacobian(m, ps, pose, fk, link, world_dir(x)), fd_jacobian3(world_dir, x)) < 5e-6);
    }
  }
  // test_hand.cpp:185-212: limit energy KAT and gradient.
  {
    HandPose pose;
    pose.q.assign(m.dof(), 0.0);
    CHECK(limit_energy(m, pose) == 0.0);
    pose.q[0] = m.joints[0].upper + 0.2;
    pose.q[3] = m.joints[3].lower - 0.1;
    VectorXd grad;
    CHECK(std::fabs(limit_energy(m, pose, &grad) - 0.05) <= 1e-12 * 0.05);
    CHECK(std::fabs(grad[kStateJoints + 0] - 0.4) <= 1e-12);
    CHECK(std::fabs(grad[kStateJoints + 3] + 0.2) <= 1e-12);
  }
  // test_hand.cpp:214-252: self-penetration zero at rest, engaged when curled, FD gradient.
  {
    HandPose rest;
    rest.q.assign(m.dof(), 0.0);
    const PoseState ps = make_pose_state(Mat3::Identity());
    CHECK(self_penetration_energy(m, ps, rest, forward_kinematics(m, rest)) == 0.0);
    CHECK(self_penetration_proxy_depth(m, forward_kinematics(m, rest)) == 0.0);
    HandPose curled;
    for (int j = 0; j < m.dof(); ++j) curled.q.push_back(m.joints[j].upper);
    CHECK(self_penetration_energy(m, ps, curled, forward_kinematics(m, curled)) > 0.0);
    CHECK(self_penetration_proxy_depth(m, forward_kinematics(m, curled)) > 0.0);
    std::mt19937_64 rng(67);
    int checked = 0;
    for (int trial = 0; trial < 40 && checked < 5; ++trial) {
      VectorXd x = random_state(m, rng);
      for (int j = 0; j < m.dof(); ++j) x[kStateJoints + j] = 0.75 * m.joints[j].upper + 0.25 * x[kStateJoints + j];
      const HandPose pose = pose_from_state(m, x);
      VectorXd grad;
      const double e = self_penetration_energy(m, make_pose_state(raw_of(x)), pose, forward_kinematics(m, pose), &grad);
      if (e < 1e-8) continue;
      ++checked;
      const VectorXd gn = fd_gradient(
          [&](const VectorXd& xs) {
            const HandPose pp = pose_from_state(m, xs);
            return self_penetration_energy(m, make_pose_state(raw_of(xs)), pp, forward_kinematics(m, pp));
          },
          x);
      double err = 0.0, nrm = 0.0;
      for (size_t i = 0; i < x.size(); ++i) err = std::fmax(err, std::fabs(grad[i] - gn[i])), nrm += gn[i] * gn[i];
      CHECK(err < 1e-5 * (1.0 + std::sqrt(nrm)));
    }
    CHECK(checked == 5);
  }
  // fingertip spheres follow fingertip_links (hand.cpp:185-198)
  {
    HandPose rest;
    rest.q.assign(m.dof(), 0.0);
    const FkResult fk = forward_kinematics(m, rest);
    const auto spheres = fingertip_spheres(m, fk);
    CHECK(spheres.size() == m.fingertip_links.size());
    for (size_t f = 0; f < spheres.size(); ++f) {
      CHECK(spheres[f].link_id == m.fingertip_links[f]);
      CHECK(norm(spheres[f].center_local - fingertip_center(m, fk, static_cast<int>(f))) == 0.0);
    }
  }
  // test_energy.cpp:516-531: surrogate value KATs.
  {
    const std::vector<Vec3> same(3, Vec3(0.2, -0.1, 0.4));
    CHECK(energy::fine_stage_surrogate(same, same, {}).value == 0.0);
    std::vector<Vec3> moved = same;
    moved[1] += Vec3::UnitZ();
    CHECK(std::fabs(energy::fine_stage_surrogate(moved, same, {}).value - 1.0) < 1e-15);
  }
  std::printf("hand api kats: %d failures\n", failures);
  return failures == 0 ? 0 : 1;
}

// Single-state differential kinematics of the reference's hand API
// (proj/include/grasp/hand.hpp:67-132, proj/src/hand.cpp:75-257): pose state,
// rotation tangent Jacobian, point / direction Jacobians, fingertip spheres,
// limit and self-penetration energies. The batched per-iteration versions of
// these run fused on the GPU inside synthesize (kernels.cuh: warp_fk,
// limit_and_self, expand_gradient); these host functions serve callers that
// evaluate one pose at a time, like the reference's tests and eval tooling.
#include "grasp/hand.hpp"

#include <algorithm>
#include <cmath>

namespace grasp::hand {
namespace {

// hand.cpp:20-29: joint j moves `link` iff it lies on the link's root path.
bool is_ancestor_joint(const HandModel& model, int joint, int link) {
  for (int l = link; l >= 0;) {
    const int j = model.links[l].parent_joint;
    if (j < 0) return false;
    if (j == joint) return true;
    l = model.joints[j].parent_link;
  }
  return false;
}

// -R [v]x J_tan into the 9 rotation columns of J (hand.cpp:163-164, 178-179).
void rotation_columns(const PoseState& ps, const HandPose& pose, const Vec3& v, MatrixXd& J) {
  const MatrixXd T = rotation_tangent_jacobian(ps);
  const Mat3 A = pose.R * skew(v);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 9; ++c) J(r, c) = -(A(r, 0) * T(0, c) + A(r, 1) * T(1, c) + A(r, 2) * T(2, c));
}

void add_jt(VectorXd& g, const MatrixXd& J, const Vec3& f) {
  for (int c = 0; c < J.cols(); ++c) g[c] += J(0, c) * f.x + J(1, c) * f.y + J(2, c) * f.z;
}

}  // namespace

PoseState make_pose_state(const Mat3& raw) {
  PoseState ps;
  ps.raw = raw;
  const RotationProjection proj = project_rotation(raw);
  ps.R = proj.R;
  ps.degenerate = proj.fallback;
  if (ps.degenerate) return ps;
  const Mat3 sf = ps.R.transpose() * raw;
  const Mat3 s = 0.5 * (sf + sf.transpose());
  const double tr = s(0, 0) + s(1, 1) + s(2, 2);
  const Mat3 a = tr * Mat3::Identity() - s;
  const double det = a.determinant();
  if (std::abs(det) < 1e-12) {
    ps.degenerate = true;
    return ps;
  }
  // adjugate / determinant (Eigen's 3x3 inverse is cofactor based)
  Mat3 inv;
  inv(0, 0) = (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) / det;
  inv(0, 1) = (a(0, 2) * a(2, 1) - a(0, 1) * a(2, 2)) / det;
  inv(0, 2) = (a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1)) / det;
  inv(1, 0) = (a(1, 2) * a(2, 0) - a(1, 0) * a(2, 2)) / det;
  inv(1, 1) = (a(0, 0) * a(2, 2) - a(0, 2) * a(2, 0)) / det;
  inv(1, 2) = (a(0, 2) * a(1, 0) - a(0, 0) * a(1, 2)) / det;
  inv(2, 0) = (a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0)) / det;
  inv(2, 1) = (a(0, 1) * a(2, 0) - a(0, 0) * a(2, 1)) / det;
  inv(2, 2) = (a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0)) / det;
  ps.a_inv = inv;
  return ps;
}

MatrixXd rotation_tangent_jacobian(const PoseState& ps) {
  MatrixXd j(3, 9);
  if (ps.degenerate) return j;
  for (int l = 0; l < 3; ++l) {
    const Vec3 e = l == 0 ? Vec3::UnitX() : (l == 1 ? Vec3::UnitY() : Vec3::UnitZ());
    for (int i = 0; i < 3; ++i) {
      const Vec3 col = ps.a_inv * cross(e, ps.R.row(i));
      for (int r = 0; r < 3; ++r) j(r, 3 * l + i) = col[r];
    }
  }
  return j;
}

MatrixXd point_jacobian(const HandModel& model, const PoseState& ps, const HandPose& pose, const FkResult& fk,
                        int link, const Vec3& point_world) {
  MatrixXd j(3, 12 + model.dof());
  const Vec3 v = pose.R.transpose() * (point_world - pose.t);  // chain frame
  rotation_columns(ps, pose, v, j);
  for (int r = 0; r < 3; ++r) j(r, kStateTranslation + r) = 1.0;
  for (int jo = 0; jo < model.dof(); ++jo) {
    if (!is_ancestor_joint(model, jo, link)) continue;
    const Vec3 col = pose.R * cross(fk.joint_axis[jo], v - fk.joint_origin[jo]);
    for (int r = 0; r < 3; ++r) j(r, kStateJoints + jo) = col[r];
  }
  return j;
}

MatrixXd direction_jacobian(const HandModel& model, const PoseState& ps, const HandPose& pose, const FkResult& fk,
                            int link, const Vec3& dir_world) {
  MatrixXd j(3, 12 + model.dof());
  const Vec3 v = pose.R.transpose() * dir_world;
  rotation_columns(ps, pose, v, j);
  for (int jo = 0; jo < model.dof(); ++jo) {
    if (!is_ancestor_joint(model, jo, link)) continue;
    const Vec3 col = pose.R * cross(fk.joint_axis[jo], v);
    for (int r = 0; r < 3; ++r) j(r, kStateJoints + jo) = col[r];
  }
  return j;
}

std::vector<geom::SphereProxy> fingertip_spheres(const HandModel& model, const FkResult& fk) {
  std::vector<geom::SphereProxy> out;
  out.reserve(model.fingertip_links.size());
  for (int l : model.fingertip_links) {
    const HandModel::Link& link = model.links[l];
    const geom::SphereProxy& tip = link.proxies[link.tip_proxy];
    out.push_back({fk.world[l].apply(tip.center_local), tip.radius, l});
  }
  return out;
}

double limit_energy(const HandModel& model, const HandPose& pose, VectorXd* grad) {
  double e = 0.0;
  if (grad) grad->assign(12 + model.dof(), 0.0);
  for (int j = 0; j < model.dof(); ++j) {
    const double over = std::max(pose.q[j] - model.joints[j].upper, 0.0);
    const double under = std::max(model.joints[j].lower - pose.q[j], 0.0);
    e += over * over + under * under;
    if (grad) (*grad)[kStateJoints + j] = 2.0 * over - 2.0 * under;
  }
  return e;
}

double self_penetration_energy(const HandModel& model, const PoseState& ps, const HandPose& pose, const FkResult& fk,
                               VectorXd* grad) {
  double e = 0.0;
  if (grad) grad->assign(12 + model.dof(), 0.0);
  for (const auto& [la, lb] : model.collision_pairs)
    for (const geom::SphereProxy& pa : model.links[la].proxies) {
      const Vec3 ca = fk.world[la].apply(pa.center_local);
      for (const geom::SphereProxy& pb : model.links[lb].proxies) {
        const Vec3 cb = fk.world[lb].apply(pb.center_local);
        const double dist = norm(ca - cb);
        const double overlap = pa.radius + pb.radius - dist;
        if (overlap <= 0) continue;
        e += overlap * overlap;
        if (grad && dist > 1e-12) {
          const Vec3 dir = (ca - cb) / dist;
          add_jt(*grad, point_jacobian(model, ps, pose, fk, la, ca), (-2.0 * overlap) * dir);
          add_jt(*grad, point_jacobian(model, ps, pose, fk, lb, cb), (2.0 * overlap) * dir);
        }
      }
    }
  return e;
}

double self_penetration_proxy_depth(const HandModel& model, const FkResult& fk) {
  double depth = 0.0;
  for (const auto& [la, lb] : model.collision_pairs)
    for (const geom::SphereProxy& pa : model.links[la].proxies)
      for (const geom::SphereProxy& pb : model.links[lb].proxies) {
        const Vec3 ca = fk.world[la].apply(pa.center_local);
        const Vec3 cb = fk.world[lb].apply(pb.center_local);
        depth = std::max(depth, pa.radius + pb.radius - norm(ca - cb));
      }
  return depth;
}

}  // namespace grasp::hand

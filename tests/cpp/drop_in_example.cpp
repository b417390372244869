// A reference-style C++ caller: same calls as proj/tests/test_pipeline.cpp
// (builtin_hand, make_primitive, RunConfig, synthesize, fine_contact_query,
// coarse_distance_energy, fine_grasp_surrogate), linked against
// libgrasp_b200.so instead of the reference's static library.
#include "grasp/config.hpp"
#include "grasp/eval.hpp"
#include "grasp/hand.hpp"
#include "grasp/object.hpp"
#include "grasp/pipeline.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <numbers>
#include <string>
#include <vector>

using namespace grasp;
using VectorXd = std::vector<double>;

static int fails = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    if (!(cond)) {                                                \
      ++fails;                                                    \
      std::printf("CHECK failed line %d: %s\n", __LINE__, #cond); \
    }                                                             \
  } while (0)

static bool same_records(const std::vector<records::GraspRecord>& a, const std::vector<records::GraspRecord>& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    if (a[i].x != b[i].x || a[i].x_s != b[i].x_s || a[i].failed != b[i].failed) return false;
    const bool both_nan = std::isnan(a[i].energy_total) && std::isnan(b[i].energy_total);
    if (!both_nan && a[i].energy_total != b[i].energy_total) return false;
  }
  return true;
}

int main() {
  const hand::HandModel& model = hand::builtin_hand();
  const object::ObjectModel sphere = object::make_primitive("sphere", 0.1);
  RunConfig cfg;
  cfg.batch = 6;
  cfg.seed = 17;
  cfg.pipeline.coarse.iters = 120;
  cfg.pipeline.fine.iters = 50;
  cfg.pipeline.final_stage.iters = 50;
  const auto recs = pipeline::synthesize(model, sphere, cfg);
  int ok = 0;
  for (const auto& r : recs) {
    if (r.failed) continue;
    ++ok;
    if (r.contacts.size() != 3 || r.per_direction.size() != 6 || !std::isfinite(r.energy_total)) return 2;
    const auto xs = pipeline::squeeze_pose(model, r.x, r.x_p);
    for (size_t i = 0; i < xs.size(); ++i)
      if (std::abs(xs[i] - r.x_s[i]) > 1e-9) return 3;
  }
  std::printf("records %zu ok %d stages %zu object %s\n", recs.size(), ok, recs[0].stages.size(),
              recs[0].object_id.c_str());
  // grasp evaluation (eval.hpp): one device pass over all records
  const auto evals = eval::quasi_static_check(model, recs, sphere, cfg);
  if (evals.size() != recs.size()) return 5;
  for (const auto& e : evals)
    if (!(e.pd_mm >= 0.0) || !(e.spd_mm >= 0.0) || !(e.cdc_mm >= 0.0) || e.contact_count < 0 || e.contact_count > 3)
      return 6;
  std::printf("eval: success %d contacts %d pd %.3f mm notes '%s'\n", (int)evals[0].success, evals[0].contact_count,
              evals[0].pd_mm, evals[0].notes.c_str());
  try {
    RunConfig bad = cfg;
    bad.qp.alpha = 2.5;
    pipeline::synthesize(model, sphere, bad);
    return 4;
  } catch (const std::invalid_argument&) {
  }

  // Multi-device synthesize (two shards on device 0): identical records.
  {
    const int devs[2] = {0, 0};
    const auto sharded = pipeline::synthesize(model, sphere, cfg, std::span<const int>(devs, 2));
    CHECK(same_records(sharded, recs));
    std::printf("sharded over 2 contexts: %s\n", same_records(sharded, recs) ? "identical" : "DIFFERENT");
  }

  // Different objects through the same local variable, one per loop pass (a new object
  // at a recycled address must be uploaded, not served from the previous call's upload).
  {
    const char* names[3] = {"box", "cylinder", "capsule"};
    for (const char* name : names) {
      const object::ObjectModel obj = object::make_primitive(name, 0.09);
      RunConfig c2 = cfg;
      c2.batch = 2;
      const auto looped = pipeline::synthesize(model, obj, c2);
      // reference answer from a fresh thread-local context: a copy of the object elsewhere
      const object::ObjectModel copy = obj;
      const auto fresh = pipeline::synthesize(model, copy, c2);
      CHECK(same_records(looped, fresh));
      CHECK(looped[0].object_id == obj.source);
    }
    // and the sphere again: must not reuse the capsule
    CHECK(same_records(pipeline::synthesize(model, sphere, cfg), recs));
  }

  // fine_contact_query from a host FkResult (test_pipeline.cpp:176-216, sphere witnesses).
  {
    const double radius = object::bounding_radius(sphere);
    hand::HandPose pose;
    pose.R = angle_axis_matrix(std::numbers::pi, Vec3::UnitX());
    pose.q.assign(model.dof(), 0.0);
    for (double drop : {0.175, 0.160, 0.148}) {
      pose.t = Vec3(0.0, 0.0, drop);
      const hand::FkResult fk = hand::forward_kinematics(model, pose);
      const auto ws = pipeline::fine_contact_query(model, fk, sphere);
      CHECK(ws.size() == model.fingertip_links.size());
      for (size_t f = 0; f < ws.size(); ++f) {
        const Vec3 c = hand::fingertip_center(model, fk, static_cast<int>(f));
        CHECK(ws[f].link == model.fingertip_links[f]);
        CHECK(std::abs(ws[f].distance - (norm(c) - radius - 0.010)) <= 0.004);
        const Vec3 dir = normalized(c);
        CHECK(norm(ws[f].p_w - dot(ws[f].p_w, dir) * dir) <= 0.008);
        CHECK(dot(ws[f].n, dir) >= 0.9);
        CHECK(std::abs(norm(ws[f].c_w - ws[f].p_w) - std::abs(ws[f].distance)) <= 1e-9 * std::abs(ws[f].distance));
      }
    }
  }

  // coarse_distance_energy gradient vs central differences (test_pipeline.cpp:136-174).
  {
    const object::ObjectModel box = object::make_primitive("box", 0.1);
    const auto [lo, hi] = object::bounding_box(box);
    hand::HandPose pose;
    for (int j = 0; j < model.dof(); ++j) pose.q.push_back(0.5 * (model.joints[j].lower + model.joints[j].upper));
    const hand::FkResult fk0 = hand::forward_kinematics(model, pose);
    const Vec3 tip0 = hand::fingertip_center(model, fk0, 0);
    pose.t = Vec3(0.002, -0.001, hi.z + 0.02) - tip0;
    const VectorXd x = hand::state_from_pose(model, pose);
    VectorXd grad;
    const double e = pipeline::coarse_distance_energy(model, x, box, 0.01, 1e-6, &grad);
    double err = 0.0, nrm = 0.0;
    VectorXd xp = x;
    for (size_t i = 0; i < x.size(); ++i) {
      xp[i] = x[i] + 1e-6;
      const double fp = pipeline::coarse_distance_energy(model, xp, box, 0.01, 1e-6);
      xp[i] = x[i] - 1e-6;
      const double fm = pipeline::coarse_distance_energy(model, xp, box, 0.01, 1e-6);
      xp[i] = x[i];
      const double fd = (fp - fm) / 2e-6;
      err += (grad[i] - fd) * (grad[i] - fd);
      nrm += fd * fd;
    }
    CHECK(e > 0.0);
    CHECK(std::sqrt(err) <= 1e-3 * std::fmax(1.0, std::sqrt(nrm)));
    std::printf("coarse_distance_energy %.6e grad err %.2e\n", e, std::sqrt(err));
  }

  // fine_grasp_surrogate: value and detached gradient (test_pipeline.cpp:262-311, oracle 1).
  {
    const double radius = object::bounding_radius(sphere);
    hand::HandPose pose;
    pose.R = angle_axis_matrix(0.5 * std::numbers::pi, Vec3::UnitX());
    pose.q.assign(model.dof(), 0.0);
    pose.t = Vec3(0.0, -(radius + 0.020), -0.06);
    const VectorXd x = hand::state_from_pose(model, pose);
    const hand::FkResult fk = hand::forward_kinematics(model, pose);
    const auto ws = pipeline::fine_contact_query(model, fk, sphere);
    std::vector<Vec3> anchors, frozen;
    for (const auto& w : ws) {
      anchors.push_back(w.p_w + Vec3(0.02, 0.01, -0.015));
      const RigidTransform& t = fk.world[w.link];
      frozen.push_back(t.R.transpose() * (w.c_w - t.t));
    }
    const energy::SurrogateResult sr = pipeline::fine_grasp_surrogate(model, x, ws, anchors);
    auto fixed_value = [&](const VectorXd& xx) {
      const hand::FkResult f2 = hand::forward_kinematics(model, hand::pose_from_state(model, xx));
      double v = 0.0;
      for (size_t i = 0; i < ws.size(); ++i) v += squared_norm(f2.world[ws[i].link].apply(frozen[i]) - anchors[i]);
      return v;
    };
    CHECK(std::abs(fixed_value(x) - sr.value) <= 1e-12 * std::fmax(1.0, sr.value));
    double err = 0.0, nrm = 0.0;
    VectorXd xp = x;
    for (size_t i = 0; i < x.size(); ++i) {
      xp[i] = x[i] + 1e-6;
      const double fp = fixed_value(xp);
      xp[i] = x[i] - 1e-6;
      const double fm = fixed_value(xp);
      xp[i] = x[i];
      const double fd = (fp - fm) / 2e-6;
      err += (sr.gradient[i] - fd) * (sr.gradient[i] - fd);
      nrm += fd * fd;
    }
    CHECK(std::sqrt(err) <= 1e-5 * std::fmax(1.0, std::sqrt(nrm)));
  }
  std::printf("drop-in checks: %d failures\n", fails);
  if (fails) return 7;
  return ok >= 4 ? 0 : 1;
}

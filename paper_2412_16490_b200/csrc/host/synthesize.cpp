// C++ drop-in for grasp::pipeline::synthesize (reference pipeline.cpp:436-457):
// validate -> init_poses (host, one RNG stream) -> GPU three-stage loop via
// the C ABI -> std::vector<GraspRecord> in input order.
#include "../../../include/grasp_b200.h"

#include "capi_common.hpp"
#include "grasp/eval.hpp"
#include "grasp/pipeline.hpp"

#include <cmath>
#include <limits>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>

namespace grasp::pipeline {
namespace {

struct CtxDeleter {
  void operator()(grasp_ctx* c) const { grasp_ctx_destroy(c); }
};

// One device context per (thread, device). The packed copy of the models last
// uploaded is kept, and a model is re-uploaded whenever its packed content
// differs: a new model at a recycled address, or one changed in place, is
// never served from the previous upload (packing is a few vector copies,
// nothing next to a synthesis run).
struct CachedCtx {
  std::unique_ptr<grasp_ctx, CtxDeleter> ctx;
  bool has_hand = false, has_object = false;
  capi::PackedHand packed_hand;
  capi::PackedObject packed_object;
};

bool same_content(const capi::PackedHand& a, const capi::PackedHand& b) {
  return a.link_parent_joint == b.link_parent_joint && a.link_tip_proxy == b.link_tip_proxy &&
         a.link_vert_begin == b.link_vert_begin && a.link_face_begin == b.link_face_begin &&
         a.link_proxy_begin == b.link_proxy_begin && a.verts == b.verts && a.faces == b.faces &&
         a.link_obb == b.link_obb && a.link_centroid == b.link_centroid && a.link_volume == b.link_volume &&
         a.proxies == b.proxies && a.joint_parent_link == b.joint_parent_link &&
         a.joint_child_link == b.joint_child_link && a.joint_origin == b.joint_origin &&
         a.joint_axis == b.joint_axis && a.joint_lower == b.joint_lower && a.joint_upper == b.joint_upper &&
         a.tip_links == b.tip_links && a.collision_pairs == b.collision_pairs;
}

bool same_content(const capi::PackedObject& a, const capi::PackedObject& b) {
  return a.part_vert_begin == b.part_vert_begin && a.part_face_begin == b.part_face_begin && a.verts == b.verts &&
         a.faces == b.faces && a.part_obb == b.part_obb && a.part_centroid == b.part_centroid &&
         a.part_volume == b.part_volume && a.source == b.source && a.desc.scale == b.desc.scale &&
         a.desc.bbox_diagonal == b.desc.bbox_diagonal && a.desc.mass_center[0] == b.desc.mass_center[0] &&
         a.desc.mass_center[1] == b.desc.mass_center[1] && a.desc.mass_center[2] == b.desc.mass_center[2];
}

void check(int status) {
  if (status == GRASP_OK) return;
  const std::string msg = grasp_last_error();
  switch (status) {
    case GRASP_EINVAL: throw std::invalid_argument(msg);
    case GRASP_EGEOM: throw geom::GeometryError(msg);
    case GRASP_EHAND: throw hand::HandError(msg);
    case GRASP_EOBJECT: throw object::ObjectError(msg);
    default: throw std::runtime_error(msg);
  }
}

// One context per (thread, device list): a single device, or a multi-device
// group (grasp_ctx_create_devices) for the sharded overload of synthesize.
CachedCtx& context_for(const std::vector<int>& devices) {
  thread_local std::map<std::vector<int>, CachedCtx> cache;
  CachedCtx& c = cache[devices];
  if (!c.ctx) {
    grasp_ctx* raw = nullptr;
    if (devices.size() == 1)
      check(grasp_ctx_create(devices[0], &raw));
    else
      check(grasp_ctx_create_devices(devices.data(), static_cast<int>(devices.size()), &raw));
    c.ctx.reset(raw);
  }
  return c;
}

}  // namespace

CachedCtx& bound_context(const hand::HandModel& model, const object::ObjectModel& object,
                         const std::vector<int>& devices) {
  CachedCtx& c = context_for(devices);
  capi::PackedHand ph = capi::pack_hand(model);
  if (!c.has_hand || !same_content(ph, c.packed_hand)) {
    c.has_hand = false;
    c.packed_hand = std::move(ph);  // vector buffers (and the desc's pointers into them) move along
    check(grasp_ctx_set_hand(c.ctx.get(), &c.packed_hand.desc));
    c.has_hand = true;
  }
  capi::PackedObject po = capi::pack_object(object);
  if (!c.has_object || !same_content(po, c.packed_object)) {
    c.has_object = false;
    c.packed_object = std::move(po);
    c.packed_object.desc.source = c.packed_object.source.c_str();  // SSO strings do not move their buffer
    check(grasp_ctx_set_object(c.ctx.get(), &c.packed_object.desc));
    c.has_object = true;
  }
  return c;
}

CachedCtx& bound_context(const hand::HandModel& model, const object::ObjectModel& object, int device) {
  return bound_context(model, object, std::vector<int>{device});
}

namespace {

std::vector<records::GraspRecord> synthesize_on(const hand::HandModel& model, const object::ObjectModel& object,
                                                const RunConfig& cfg, const std::vector<int>& devices) {
  validate(cfg);
  if (devices.empty()) throw std::invalid_argument("synthesize: empty device list");
  CachedCtx& c = bound_context(model, object, devices);
  const int B = cfg.batch, D = 12 + model.dof(), m = static_cast<int>(model.fingertip_links.size());
  const int n = m * cfg.contact.n_edges;
  const std::vector<VectorXd> starts = init_poses(model, object, B, cfg.seed, cfg.init);
  std::vector<double> x0(static_cast<size_t>(B) * D);
  for (int g = 0; g < B; ++g) std::copy(starts[g].begin(), starts[g].end(), x0.begin() + static_cast<size_t>(g) * D);

  std::vector<double> x_p(x0.size()), x(x0.size()), x_s(x0.size()), energy(B), per(6 * B),
      forces(static_cast<size_t>(B) * n * 6), contacts(static_cast<size_t>(B) * m * 12), stage(6 * B);
  std::vector<int> failed(B), conv(6 * B);
  grasp_out out{x_p.data(), x.data(), x_s.data(), energy.data(), per.data(), forces.data(),
                contacts.data(), stage.data(), failed.data(), conv.data()};
  grasp_run_params p;
  capi::from_config(cfg, &p);
  check(grasp_synthesize(c.ctx.get(), &p, B, x0.data(), &out));

  static const char* kNames[3] = {"coarse", "fine", "final"};
  const int iters[3] = {cfg.pipeline.coarse.iters, cfg.pipeline.fine.iters, cfg.pipeline.final_stage.iters};
  const int n_stages = cfg.pipeline.skip_fine_stages ? 1 : 3;
  std::vector<records::GraspRecord> recs(B);
  for (int g = 0; g < B; ++g) {
    records::GraspRecord& r = recs[g];
    auto slice = [&](const std::vector<double>& v) {
      return VectorXd(v.begin() + static_cast<size_t>(g) * D, v.begin() + static_cast<size_t>(g + 1) * D);
    };
    r.x_p = slice(x_p);
    r.x = slice(x);
    r.x_s = slice(x_s);
    r.index = g;
    r.seed = cfg.seed;
    r.object_id = object.source;
    r.object_scale = object.scale;
    r.failed = failed[g] != 0;
    r.note = failed[g] == 1 ? "non-finite energy" : (failed[g] == 2 ? "diverged" : "");
    for (int s = 0; s < n_stages; ++s)
      r.stages.push_back({kNames[s], iters[s], stage[6 * g + 2 * s], stage[6 * g + 2 * s + 1]});
    if (r.failed) {
      r.energy_total = std::numeric_limits<double>::quiet_NaN();
      continue;
    }
    r.energy_total = energy[g];
    r.per_direction.assign(per.begin() + 6 * g, per.begin() + 6 * g + 6);
    r.contact_force_rows = n;
    r.contact_force_cols = 6;
    r.contact_forces.assign(forces.begin() + static_cast<size_t>(g) * n * 6,
                            forces.begin() + static_cast<size_t>(g + 1) * n * 6);
    for (int f = 0; f < m; ++f) {
      const double* cf = contacts.data() + (static_cast<size_t>(g) * m + f) * 12;
      contact::ContactFrame fr;
      fr.p = Vec3(cf[0], cf[1], cf[2]);
      fr.n = Vec3(cf[3], cf[4], cf[5]);
      fr.d = Vec3(cf[6], cf[7], cf[8]);
      fr.e = Vec3(cf[9], cf[10], cf[11]);
      r.contacts.push_back(fr);
    }
  }
  return recs;
}

}  // namespace

std::vector<records::GraspRecord> synthesize(const hand::HandModel& model, const object::ObjectModel& object,
                                             const RunConfig& cfg, int device) {
  return synthesize_on(model, object, cfg, {device});
}

std::vector<records::GraspRecord> synthesize(const hand::HandModel& model, const object::ObjectModel& object,
                                             const RunConfig& cfg, std::span<const int> devices) {
  return synthesize_on(model, object, cfg, std::vector<int>(devices.begin(), devices.end()));
}

std::vector<ContactWitness> fine_contact_query(const hand::HandModel& model, const hand::FkResult& fk,
                                               const object::ObjectModel& object, int device) {
  const int L = static_cast<int>(model.links.size()), m = static_cast<int>(model.fingertip_links.size());
  if (static_cast<int>(fk.world.size()) != L) throw std::invalid_argument("fine_contact_query: FkResult size");
  CachedCtx& c = bound_context(model, object, device);
  std::vector<double> world(static_cast<size_t>(L) * 12), out(static_cast<size_t>(m) * 11);
  for (int l = 0; l < L; ++l) {
    std::copy(fk.world[l].R.m, fk.world[l].R.m + 9, world.begin() + 12 * l);  // column-major
    world[12 * l + 9] = fk.world[l].t.x;
    world[12 * l + 10] = fk.world[l].t.y;
    world[12 * l + 11] = fk.world[l].t.z;
  }
  check(grasp_fine_contact_query_world(c.ctx.get(), 1, world.data(), out.data()));
  std::vector<ContactWitness> ws(m);
  for (int f = 0; f < m; ++f) {
    const double* o = out.data() + 11 * f;
    ws[f].c_w = Vec3(o[0], o[1], o[2]);
    ws[f].p_w = Vec3(o[3], o[4], o[5]);
    ws[f].n = Vec3(o[6], o[7], o[8]);
    ws[f].distance = o[9];
    ws[f].link = static_cast<int>(o[10]);
  }
  return ws;
}

double coarse_distance_energy(const hand::HandModel& model, const VectorXd& x, const object::ObjectModel& object,
                              double offset, double fd_step, VectorXd* grad, int device) {
  const int D = 12 + model.dof();
  if (static_cast<int>(x.size()) != D) throw hand::HandError("state vector has wrong size for this hand");
  CachedCtx& c = bound_context(model, object, device);
  // The coarse-stage total_energy with every weight but the distance term's at
  // zero is exactly coarse_distance_energy (pipeline.cpp:133-163 vs :355-380):
  // the other terms enter as 0 * finite = +0 and the tip force is 2 r (n - dp^T n).
  grasp_run_params p;
  grasp_run_params_default(&p);
  p.w_grasp = p.w_joint_limit = p.w_self_penetration = p.w_object_penetration = 0.0;
  p.w_distance = 1.0;
  p.contact_offset = offset;
  p.fd_step = fd_step;
  double e = 0.0;
  std::vector<double> g(D);
  check(grasp_total_energy(c.ctx.get(), &p, 0, 1, x.data(), nullptr, nullptr, nullptr, &e, g.data()));
  if (grad) *grad = g;
  return e;
}

energy::SurrogateResult fine_grasp_surrogate(const hand::HandModel& model, const VectorXd& x,
                                             std::span<const ContactWitness> witnesses,
                                             std::span<const Vec3> anchors) {
  Mat3 raw;
  for (int i = 0; i < 9; ++i) raw.m[i] = x.at(i);
  const hand::PoseState ps = hand::make_pose_state(raw);
  const hand::HandPose pose = hand::pose_from_state(model, x);
  const hand::FkResult fk = hand::forward_kinematics(model, pose);
  std::vector<Vec3> points;
  std::vector<MatrixXd> jac;
  for (const ContactWitness& w : witnesses) {
    points.push_back(w.c_w);
    jac.push_back(hand::point_jacobian(model, ps, pose, fk, w.link, w.c_w));
  }
  return energy::fine_stage_surrogate(points, anchors, jac);
}

}  // namespace grasp::pipeline

namespace grasp::energy {

SurrogateResult fine_stage_surrogate(std::span<const Vec3> points, std::span<const Vec3> anchors,
                                     std::span<const MatrixXd> jacobians) {
  if (points.size() != anchors.size()) throw std::invalid_argument("point and anchor counts differ");
  if (!jacobians.empty() && jacobians.size() != points.size())
    throw std::invalid_argument("need one Jacobian per point when given");
  SurrogateResult out;
  const int dims = jacobians.empty() ? 0 : jacobians[0].cols();
  out.gradient.assign(dims, 0.0);
  for (size_t i = 0; i < points.size(); ++i) {
    const Vec3 diff = points[i] - anchors[i];
    out.value += squared_norm(diff);
    if (jacobians.empty()) continue;
    if (jacobians[i].rows() != 3 || jacobians[i].cols() != dims)
      throw std::invalid_argument("point Jacobians must be 3 x dims");
    for (int c = 0; c < dims; ++c)
      out.gradient[c] += 2.0 * (jacobians[i](0, c) * diff.x + jacobians[i](1, c) * diff.y + jacobians[i](2, c) * diff.z);
  }
  return out;
}

}  // namespace grasp::energy

namespace grasp::eval {
namespace {

// One device pass over (x, x_s) pairs; notes joined like eval.cpp:139-156.
std::vector<EvalResult> run_eval(const hand::HandModel& model, const object::ObjectModel& object, const RunConfig& cfg,
                                 const std::vector<const VectorXd*>& xs, const std::vector<const VectorXd*>& xss,
                                 int device) {
  const int n = static_cast<int>(xs.size()), D = 12 + model.dof();
  for (int g = 0; g < n; ++g)
    if (static_cast<int>(xs[g]->size()) != D || static_cast<int>(xss[g]->size()) != D)
      throw std::invalid_argument("quasi_static_check: record poses do not match the hand");
  pipeline::CachedCtx& c = pipeline::bound_context(model, object, device);
  std::vector<double> x(static_cast<size_t>(n) * D), x_s(x.size()), real(static_cast<size_t>(n) * 9);
  std::vector<int> ints(static_cast<size_t>(n) * 3);
  for (int g = 0; g < n; ++g) {
    std::copy(xs[g]->begin(), xs[g]->end(), x.begin() + static_cast<size_t>(g) * D);
    std::copy(xss[g]->begin(), xss[g]->end(), x_s.begin() + static_cast<size_t>(g) * D);
  }
  grasp_run_params p;
  capi::from_config(cfg, &p);
  grasp_eval_params e{cfg.eval.mass, cfg.eval.gravity, cfg.eval.residual_rel_tol, cfg.eval.force_budget_factor,
                      cfg.eval.contact_tol, cfg.eval.penetration_tol, cfg.eval.qp_eps};
  if (n > 0) pipeline::check(grasp_eval(c.ctx.get(), &p, &e, n, x.data(), x_s.data(), real.data(), ints.data()));
  std::vector<EvalResult> out(n);
  for (int g = 0; g < n; ++g) {
    EvalResult& r = out[g];
    const double* o = real.data() + static_cast<size_t>(g) * 9;
    r.pd_mm = o[0];
    r.spd_mm = o[1];
    r.cdc_mm = o[2];
    for (int j = 0; j < 6; ++j) r.per_direction_residuals[j] = o[3 + j];
    r.contact_count = ints[3 * g];
    r.success = ints[3 * g + 1] != 0;
    const int f = ints[3 * g + 2];
    std::vector<std::string> notes;
    if (f & 1) notes.push_back("no contacts at the squeeze pose");
    if (f & 2) notes.push_back("resistance qp unconverged");
    if (f & 4) notes.push_back("gravity wrench residual above tolerance");
    if (f & 8) notes.push_back("fewer than two contacts");
    if (f & 16) {
      std::ostringstream msg;
      msg << "penetration " << r.pd_mm << " mm above tolerance";
      notes.push_back(msg.str());
    }
    for (const auto& s : notes) {
      if (!r.notes.empty()) r.notes += "; ";
      r.notes += s;
    }
  }
  return out;
}

}  // namespace

std::vector<EvalResult> quasi_static_check(const hand::HandModel& model,
                                           const std::vector<records::GraspRecord>& records,
                                           const object::ObjectModel& object, const RunConfig& cfg, int device) {
  std::vector<const VectorXd*> xs, xss;
  for (const auto& r : records) {
    xs.push_back(&r.x);
    xss.push_back(&r.x_s);
  }
  return run_eval(model, object, cfg, xs, xss, device);
}

EvalResult quasi_static_check(const hand::HandModel& model, const records::GraspRecord& record,
                              const object::ObjectModel& object, const RunConfig& cfg, int device) {
  return run_eval(model, object, cfg, {&record.x}, {&record.x_s}, device)[0];
}

double penetration_depth(const hand::HandModel& model, const VectorXd& x, const object::ObjectModel& object,
                         int device) {
  return run_eval(model, object, RunConfig{}, {&x}, {&x}, device)[0].pd_mm;
}

double self_penetration_depth(const hand::HandModel& model, const VectorXd& x, const object::ObjectModel& object,
                              int device) {
  return run_eval(model, object, RunConfig{}, {&x}, {&x}, device)[0].spd_mm;
}

double contact_distance_consistency(const hand::HandModel& model, const VectorXd& x,
                                    const object::ObjectModel& object, int device) {
  return run_eval(model, object, RunConfig{}, {&x}, {&x}, device)[0].cdc_mm;
}

}  // namespace grasp::eval

// Oracle (test infrastructure only): restatement of the reference's grasp
// evaluation, proj/src/eval.cpp:51-158 (penetration_depth :51-61,
// self_penetration_depth :63-72, fingertip_distances + contact_distance_consistency
// :74-89, quasi_static_check :91-158). The notes string is returned as flags
// (1 no contacts, 2 resistance qp unconverged, 4 gravity residual above
// tolerance, 8 fewer than two contacts, 16 penetration above tolerance).
#include <algorithm>
#include <cmath>

#include "oracle_impl.hpp"

namespace oracle {

namespace {
Fk fk_of(const Hand& h, const VecX& x) { return forward_kinematics(h, pose_from_state(h, x)); }
}  // namespace

// eval.cpp:51-61
double penetration_depth(const Hand& h, const VecX& x, const Object& obj) {
  const Fk fk = fk_of(h, x);
  double depth = 0.0;
  for (size_t l = 0; l < h.links.size(); ++l)
    for (const Part& part : obj.parts) {
      const double d = signed_distance(h.links[l].part, fk.world[l], part, Rigid{M3::identity(), V3()}, nullptr, nullptr);
      depth = std::max(depth, -d);
    }
  return 1000.0 * depth;
}

// eval.cpp:63-72
double self_penetration_depth(const Hand& h, const VecX& x) {
  const Fk fk = fk_of(h, x);
  double depth = 0.0;
  for (const auto& [i, j] : h.pairs) {
    const double d = signed_distance(h.links[i].part, fk.world[i], h.links[j].part, fk.world[j], nullptr, nullptr);
    depth = std::max(depth, -d);
  }
  return 1000.0 * depth;
}

// eval.cpp:74-89
double contact_distance_consistency(const Hand& h, const VecX& x, const Object& obj) {
  const auto ws = fine_contact_query(h, fk_of(h, x), obj);
  if (ws.empty()) return 0.0;
  double lo = ws[0].distance, hi = ws[0].distance;
  for (const Witness& w : ws) {  // std::minmax_element: first min, last max (values only matter)
    lo = std::min(lo, w.distance);
    hi = std::max(hi, w.distance);
  }
  return 1000.0 * (hi - lo);
}

// eval.cpp:91-158
EvalResult quasi_static_check(const Hand& h, const Object& obj, const Config& cfg, const EvalParams& ep,
                              const VecX& x, const VecX& x_s) {
  EvalResult out;
  out.pd_mm = penetration_depth(h, x, obj);
  out.spd_mm = self_penetration_depth(h, x);
  out.cdc_mm = contact_distance_consistency(h, x, obj);
  const double mg = ep.mass * ep.gravity;
  const double tau = ep.residual_rel_tol * mg;
  std::vector<Frame> frames;
  for (const Witness& w : fine_contact_query(h, fk_of(h, x_s), obj))
    if (w.distance <= ep.contact_tol) frames.push_back(build_frame(w.p_w, -w.n));
  out.contact_count = static_cast<int>(frames.size());
  bool resisted = false;
  if (frames.empty()) {
    for (double& r : out.residuals) r = mg;
    out.note_flags |= 1;
  } else {
    const double cap = ep.force_budget_factor * mg / static_cast<double>(frames.size());
    MatX targets(6, 6);
    for (int j = 0; j < 6; ++j) targets(j / 2, j) = (j % 2 == 0) ? -1.0 : 1.0;  // minus gravity
    QpParams qp = cfg.qp;
    qp.eps_primal = ep.qp_eps;
    qp.eps_dual = ep.qp_eps;
    const EnergyReport rep =
        grasp_energy(frames, mg / cap, cfg.gamma_per_contact, cfg.mu, cfg.n_edges, qp, nullptr, nullptr, &targets);
    bool all_conv = true;
    for (char c : rep.converged) all_conv = all_conv && c;
    for (int j = 0; j < 6; ++j) out.residuals[j] = cap * std::sqrt(std::max(rep.per_direction[j], 0.0));
    if (!all_conv) out.note_flags |= 2;
    resisted = true;
    for (double r : out.residuals) resisted = resisted && r <= tau;
    if (!resisted) out.note_flags |= 4;
  }
  if (out.contact_count < 2) out.note_flags |= 8;
  const bool shallow = out.pd_mm <= 1000.0 * ep.penetration_tol;
  if (!shallow) out.note_flags |= 16;
  out.success = resisted && out.contact_count >= 2 && shallow;
  return out;
}

}  // namespace oracle

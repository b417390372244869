// ORACLE (test infrastructure only). fp64 restatement of
// /root/reference/proj/src/pipeline.cpp:36-434 (total_energy, apply_step,
// run_grasp, fine_contact_query, coarse_distance_energy, squeeze) and
// energy.cpp:208-229 (fine-stage surrogate).
#include "oracle_impl.hpp"

#include <cmath>
#include <limits>
#include <numbers>

namespace oracle {
namespace {

constexpr double kNan = std::numeric_limits<double>::quiet_NaN();

struct Posed {
  PoseState ps;
  Pose pose;
  Fk fk;
};

// Teacher forcing of the kinematics (tests only): when set, the world link
// transforms of the next pose_hand calls on this thread are taken from here
// ([L*12], R column-major, t) instead of this oracle's own FK, so the rest of
// total_energy runs on exactly the device's link poses.
thread_local const double* tl_world_override = nullptr;

// pipeline.cpp:36-42 (projection is done twice, as in the reference).
Posed pose_hand(const Hand& h, const VecX& x) {
  Posed p;
  p.ps = make_pose_state(raw_block(x));
  p.pose = pose_from_state(h, x);
  p.fk = forward_kinematics(h, p.pose);
  if (tl_world_override)
    for (size_t l = 0; l < p.fk.world.size(); ++l) {
      const double* w = tl_world_override + 12 * l;
      for (int c = 0; c < 3; ++c)
        for (int i = 0; i < 3; ++i) p.fk.world[l].R(i, c) = w[3 * c + i];
      p.fk.world[l].t = V3(w[9], w[10], w[11]);
    }
  return p;
}

// pipeline.cpp:47-52.
double envelope_radius(const Link& link) {
  const V3& tip = link.proxies[link.tip_proxy].c;
  double r = 0.0;
  for (const V3& v : link.part.verts) r = std::max(r, norm(v - tip));
  return r;
}

void add_scaled(VecX& g, const VecX& v, double s) {
  for (size_t i = 0; i < g.size(); ++i) g[i] += s * v[i];
}

// J^T f for a 3xD Jacobian.
void add_jt(VecX& g, const MatX& J, const V3& f, double s) {
  for (int c = 0; c < J.cols; ++c) g[c] += s * (J(0, c) * f[0] + J(1, c) * f[1] + J(2, c) * f[2]);
}

// energy.cpp:208-229 via pipeline.cpp:54-65.
double surrogate_at(const Hand& h, const Posed& ph, const std::vector<Witness>& ws, const std::vector<V3>& anchors,
                    VecX* grad) {
  double value = 0.0;
  for (size_t i = 0; i < ws.size(); ++i) {
    const V3 diff = ws[i].c_w - anchors[i];
    value += sqnorm(diff);
    if (grad) {
      const MatX J = point_jacobian(h, ph.ps, ph.pose, ph.fk, ws[i].link, ws[i].c_w);
      add_jt(*grad, J, diff, 2.0);
    }
  }
  return value;
}

V3 tip_center(const Hand& h, const Fk& fk, int f) {
  const int link = h.tips[f];
  const Link& ln = h.links[link];
  return fk.world[link].apply(ln.proxies[ln.tip_proxy].c);
}

}  // namespace

void set_world_override(const double* world) { tl_world_override = world; }

// pipeline.cpp:320-353.
std::vector<Witness> fine_contact_query(const Hand& h, const Fk& fk, const Object& obj) {
  std::vector<Witness> out;
  for (int link : h.tips) {
    const Link& ln = h.links[link];
    const Proxy& tip = ln.proxies[ln.tip_proxy];
    const Rigid& lp = fk.world[link];
    const V3 center = lp.apply(tip.c);
    const double reference = point_to_mesh(center, obj.parts).distance - tip.r;
    const std::vector<int> keep = broadphase_cull(lp.apply(tip.c), envelope_radius(ln), obj.parts, reference);
    Witness w;
    w.link = link;
    w.distance = std::numeric_limits<double>::infinity();
    for (int pi : keep) {
      Nearest r;
      const double d = signed_distance(ln.part, lp, obj.parts[pi], Rigid{M3::identity(), V3()}, &r, nullptr);
      if (d < w.distance) {
        w.distance = d;
        w.c_w = r.a;
        w.p_w = r.b;
        w.n = r.normal;
      }
    }
    out.push_back(w);
  }
  return out;
}

// pipeline.cpp:96-210.
double total_energy(const Hand& h, const Object& obj, const Config& cfg, int stage, const std::vector<V3>& anchors,
                    const VecX& x, QpScratch& scratch, VecX* grad) {
  const Posed ph = pose_hand(h, x);
  const int dims = h.dims();
  if (grad) grad->assign(dims, 0.0);
  VecX g;
  double total = 0.0;
  const double offset = stage == 2 ? 0.0 : cfg.contact_offset;

  double e = limit_energy(h, ph.pose, grad ? &g : nullptr);
  total += cfg.w_limit * e;
  if (grad) add_scaled(*grad, g, cfg.w_limit);

  e = self_penetration_energy(h, ph.ps, ph.pose, ph.fk, grad ? &g : nullptr);
  total += cfg.w_self * e;
  if (grad) add_scaled(*grad, g, cfg.w_self);

  if (stage == 0) {
    for (size_t l = 0; l < h.links.size(); ++l)
      for (const Proxy& pr : h.links[l].proxies) {
        const V3 c = ph.fk.world[l].apply(pr.c);
        const Nearest q = point_to_mesh(c, obj.parts);
        const double sd = q.distance - pr.r;
        if (sd >= 0.0) continue;
        total += cfg.w_pen * sd * sd;
        if (grad) {
          const MatX jc = point_jacobian(h, ph.ps, ph.pose, ph.fk, static_cast<int>(l), c);
          add_jt(*grad, jc, q.normal, cfg.w_pen * 2.0 * sd);
        }
      }
    const int m = static_cast<int>(h.tips.size());
    std::vector<Frame> frames(m);
    std::vector<MatX> jac_p(m), jac_n(m);
    const double hstep = cfg.fd_step;
    for (int f = 0; f < m; ++f) {
      const int link = h.tips[f];
      const Proxy& tip = h.links[link].proxies[h.links[link].tip_proxy];
      const V3 c = ph.fk.world[link].apply(tip.c);
      const Nearest q0 = point_to_mesh(c, obj.parts);
      frames[f] = build_frame(q0.b, -q0.normal);
      const double r = q0.distance - tip.r - offset;
      total += cfg.w_distance * r * r;
      if (grad) {
        M3 dp = M3::zero(), dn = M3::zero();
        for (int k = 0; k < 3; ++k) {
          const V3 step = hstep * V3::unit(k);
          const Nearest qp = point_to_mesh(c + step, obj.parts);
          const Nearest qm = point_to_mesh(c - step, obj.parts);
          dp.set_col(k, (qp.b - qm.b) / (2.0 * hstep));
          dn.set_col(k, (qp.normal - qm.normal) / (2.0 * hstep));
        }
        const MatX jc = point_jacobian(h, ph.ps, ph.pose, ph.fk, link, c);
        const V3 dd = (M3::identity() - dp).t() * q0.normal;  // row vector n^T (I - dp)
        add_jt(*grad, jc, dd, cfg.w_distance * 2.0 * r);
        jac_p[f] = MatX(3, dims);
        jac_n[f] = MatX(3, dims);
        for (int col = 0; col < dims; ++col)
          for (int rr = 0; rr < 3; ++rr) {
            double sp = 0.0, sn = 0.0;
            for (int kk = 0; kk < 3; ++kk) {
              sp += dp(rr, kk) * jc(kk, col);
              sn += dn(rr, kk) * jc(kk, col);
            }
            jac_p[f](rr, col) = sp;
            jac_n[f](rr, col) = -sn;
          }
      }
    }
    EnergyReport rep = grasp_energy(frames, cfg.beta, cfg.gamma_per_contact, cfg.mu, cfg.n_edges, cfg.qp,
                                    scratch.ready ? &scratch.forces : nullptr, scratch.ready ? &scratch.duals : nullptr);
    scratch.forces = rep.forces;
    scratch.duals = rep.duals;
    scratch.ready = true;
    scratch.iters = rep.iters;
    scratch.converged = rep.converged;
    total += cfg.w_grasp * rep.total;
    if (grad) add_scaled(*grad, grasp_energy_gradient(frames, rep, cfg.mu, cfg.n_edges, jac_p, jac_n), cfg.w_grasp);
  } else {
    for (size_t l = 0; l < h.links.size(); ++l)
      for (const Part& part : obj.parts) {
        Nearest r;
        const double d = signed_distance(h.links[l].part, ph.fk.world[l], part, Rigid{M3::identity(), V3()}, &r, nullptr);
        if (d >= 0.0) continue;
        total += cfg.w_pen * d * d;
        if (grad) {
          const MatX jc = point_jacobian(h, ph.ps, ph.pose, ph.fk, static_cast<int>(l), r.a);
          add_jt(*grad, jc, r.normal, cfg.w_pen * 2.0 * d);
        }
      }
    const std::vector<Witness> ws = fine_contact_query(h, ph.fk, obj);
    for (const Witness& w : ws) {
      const double r = w.distance - offset;
      total += cfg.w_distance * r * r;
      if (grad) {
        const MatX jc = point_jacobian(h, ph.ps, ph.pose, ph.fk, w.link, w.c_w);
        add_jt(*grad, jc, w.n, cfg.w_distance * 2.0 * r);
      }
    }
    VecX sg(dims, 0.0);
    const double sv = surrogate_at(h, ph, ws, anchors, grad ? &sg : nullptr);
    total += cfg.w_grasp * sv;
    if (grad) add_scaled(*grad, sg, cfg.w_grasp);
  }
  return total;
}

// pipeline.cpp:214-231.
void apply_step(const Hand& h, const Stage& s, int it, const VecX& grad, VecX& x) {
  const double t = s.iters > 1 ? static_cast<double>(it) / s.iters : 0.0;
  const double decay = s.step_floor + (1.0 - s.step_floor) * 0.5 * (1.0 + std::cos(std::numbers::pi * t));
  auto move = [&](int start, int len, double step) {
    double n2 = 0.0;
    for (int i = 0; i < len; ++i) n2 += grad[start + i] * grad[start + i];
    const double scale = step * decay / std::max(1.0, std::sqrt(n2));
    for (int i = 0; i < len; ++i) x[start + i] -= scale * grad[start + i];
  };
  move(0, 9, s.step_rotation);
  move(9, 3, s.step_translation);
  if (h.dof() > 0) {
    move(12, h.dof(), s.step_joints);
    for (int j = 0; j < h.dof(); ++j) x[12 + j] = std::min(std::max(x[12 + j], h.joints[j].lower), h.joints[j].upper);
  }
}

// pipeline.cpp:355-380.
double coarse_distance_energy(const Hand& h, const VecX& x, const Object& obj, double offset, double fd, VecX* grad) {
  const Posed ph = pose_hand(h, x);
  if (grad) grad->assign(h.dims(), 0.0);
  double total = 0.0;
  for (int f = 0; f < static_cast<int>(h.tips.size()); ++f) {
    const int link = h.tips[f];
    const Proxy& tip = h.links[link].proxies[h.links[link].tip_proxy];
    const V3 c = ph.fk.world[link].apply(tip.c);
    const Nearest q0 = point_to_mesh(c, obj.parts);
    const double r = q0.distance - tip.r - offset;
    total += r * r;
    if (!grad) continue;
    M3 dp = M3::zero();
    for (int k = 0; k < 3; ++k) {
      const V3 step = fd * V3::unit(k);
      dp.set_col(k, (point_to_mesh(c + step, obj.parts).b - point_to_mesh(c - step, obj.parts).b) / (2.0 * fd));
    }
    const MatX jc = point_jacobian(h, ph.ps, ph.pose, ph.fk, link, c);
    const V3 dd = (M3::identity() - dp).t() * q0.normal;
    add_jt(*grad, jc, dd, 2.0 * r);
  }
  return total;
}

// pipeline.cpp:426-434.
VecX squeeze_pose(const Hand& h, const VecX& x, const VecX& xp) {
  const Pose g = pose_from_state(h, x);
  const Pose p = pose_from_state(h, xp);
  const M3 R = g.R * (p.R.t() * g.R);
  VecX out(h.dims());
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) out[3 * c + i] = R(i, c);
  for (int i = 0; i < 3; ++i) out[9 + i] = 2.0 * g.t[i] - p.t[i];
  for (int j = 0; j < h.dof(); ++j)
    out[12 + j] = std::min(std::max(2.0 * g.q[j] - p.q[j], h.joints[j].lower), h.joints[j].upper);
  return out;
}

// pipeline.cpp:233-316.
Record run_grasp(const Hand& h, const Object& obj, const Config& cfg, const VecX& x0) {
  Record rec;
  for (auto& s : rec.stage_energy) s[0] = s[1] = kNan;
  const Stage* scheds[3] = {&cfg.coarse, &cfg.fine, &cfg.final_stage};
  const int n_stages = cfg.skip_fine ? 1 : 3;
  const double travel_limit = 1e3;
  VecX x = x0;
  std::vector<V3> anchors;
  QpScratch scratch;
  bool failed = false;
  bool have_pregrasp = false;
  for (int s = 0; s < n_stages; ++s) {
    const Stage& st = *scheds[s];
    if (!failed) {
      VecX grad;
      for (int it = 0; it < st.iters; ++it) {
        const double e = total_energy(h, obj, cfg, s, anchors, x, scratch, &grad);
        if (it == 0) rec.stage_energy[s][0] = e;
        bool finite = std::isfinite(e);
        for (double gv : grad) finite = finite && std::isfinite(gv);
        if (!finite) {
          failed = true;
          rec.failed = 1;
          break;
        }
        const VecX before = x;
        apply_step(h, st, it, grad, x);
        bool xf = true;
        for (double v : x) xf = xf && std::isfinite(v);
        const double tn = std::sqrt(x[9] * x[9] + x[10] * x[10] + x[11] * x[11]);
        if (!xf || tn > travel_limit) {
          x = before;
          failed = true;
          rec.failed = 2;
          break;
        }
      }
      if (!failed) rec.stage_energy[s][1] = total_energy(h, obj, cfg, s, anchors, x, scratch, nullptr);
    }
    if (failed) continue;
    if (s == 0) {
      const Posed ph = pose_hand(h, x);
      anchors.clear();
      for (int f = 0; f < static_cast<int>(h.tips.size()); ++f)
        anchors.push_back(point_to_mesh(tip_center(h, ph.fk, f), obj.parts).b);
      if (cfg.skip_fine) {
        rec.x_p = x;
        have_pregrasp = true;
      }
    } else if (s == 1) {
      rec.x_p = x;
      have_pregrasp = true;
    }
  }
  rec.x = x;
  if (!have_pregrasp) rec.x_p = x;
  rec.x_s = failed ? x : squeeze_pose(h, x, rec.x_p);
  if (!failed) {
    const Posed ph = pose_hand(h, x);
    const std::vector<Witness> ws = fine_contact_query(h, ph.fk, obj);
    for (const Witness& w : ws) rec.contacts.push_back(build_frame(w.p_w, -w.n));
    const EnergyReport rep =
        grasp_energy(rec.contacts, cfg.beta, cfg.gamma_per_contact, cfg.mu, cfg.n_edges, cfg.qp, nullptr, nullptr);
    rec.energy_total = rep.total;
    rec.per_direction = rep.per_direction;
    rec.forces = rep.forces;
    rec.converged = rep.converged;
  } else {
    rec.energy_total = kNan;
  }
  return rec;
}

}  // namespace oracle

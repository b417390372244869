// ORACLE (test infrastructure only). C entry points over the fp64
// restatement, taking the same packed descriptors as the product C ABI
// (include/grasp_b200.h) so tests feed both sides identical inputs.
#include "oracle_impl.hpp"

#include "../../include/grasp_b200.h"

#include <algorithm>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>

using namespace oracle;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const GeometryError& e) {
    g_err = e.what();
    return GRASP_EGEOM;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return GRASP_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GRASP_EINVAL;
  }
}

V3 v3(const double* p) { return V3(p[0], p[1], p[2]); }

M3 m3_colmajor(const double* p) {
  M3 r;
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) r(i, c) = p[3 * c + i];
  return r;
}

Part make_part(const double* verts, int v0, int v1, const int* faces, int f0, int f1, const double* obb,
               const double* centroid, double volume) {
  Part p;
  for (int v = v0; v < v1; ++v) p.verts.push_back(v3(verts + 3 * v));
  for (int f = f0; f < f1; ++f) p.faces.push_back({faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]});
  p.obb_center = v3(obb);
  p.obb_half = v3(obb + 3);
  p.obb_rot = m3_colmajor(obb + 6);
  p.centroid = v3(centroid);
  p.volume = volume;
  return p;
}

Hand make_hand(const grasp_hand_desc* d) {
  Hand h;
  h.links.resize(d->n_links);
  for (int l = 0; l < d->n_links; ++l) {
    Link& ln = h.links[l];
    ln.parent_joint = d->link_parent_joint[l];
    ln.tip_proxy = d->link_tip_proxy[l];
    ln.part = make_part(d->verts, d->link_vert_begin[l], d->link_vert_begin[l + 1], d->faces, d->link_face_begin[l],
                        d->link_face_begin[l + 1], d->link_obb + 15 * l, d->link_centroid + 3 * l, d->link_volume[l]);
    for (int p = d->link_proxy_begin[l]; p < d->link_proxy_begin[l + 1]; ++p)
      ln.proxies.push_back(Proxy{v3(d->proxies + 4 * p), d->proxies[4 * p + 3]});
  }
  h.joints.resize(d->dof);
  for (int j = 0; j < d->dof; ++j) {
    Joint& jt = h.joints[j];
    jt.parent_link = d->joint_parent_link[j];
    jt.child_link = d->joint_child_link[j];
    jt.origin = v3(d->joint_origin + 3 * j);
    jt.axis = v3(d->joint_axis + 3 * j);
    jt.lower = d->joint_lower[j];
    jt.upper = d->joint_upper[j];
  }
  h.tips.assign(d->tip_links, d->tip_links + d->n_tips);
  for (int i = 0; i < d->n_pairs; ++i) h.pairs.push_back({d->collision_pairs[2 * i], d->collision_pairs[2 * i + 1]});
  return h;
}

Object make_object(const grasp_object_desc* d) {
  Object o;
  for (int p = 0; p < d->n_parts; ++p)
    o.parts.push_back(make_part(d->verts, d->part_vert_begin[p], d->part_vert_begin[p + 1], d->faces,
                                d->part_face_begin[p], d->part_face_begin[p + 1], d->part_obb + 15 * p,
                                d->part_centroid + 3 * p, d->part_volume[p]));
  return o;
}

Config make_config(const grasp_run_params* p) {
  Config c;
  c.qp.rho = p->qp_rho;
  c.qp.sigma = p->qp_sigma;
  c.qp.alpha = p->qp_alpha;
  c.qp.max_iters = p->qp_max_iters;
  c.qp.eps_primal = p->qp_eps_primal;
  c.qp.eps_dual = p->qp_eps_dual;
  c.qp.check_interval = p->qp_check_interval;
  c.mu = p->mu;
  c.n_edges = p->n_edges;
  c.beta = p->beta;
  c.gamma_per_contact = p->gamma_per_contact;
  c.w_grasp = p->w_grasp;
  c.w_distance = p->w_distance;
  c.w_limit = p->w_joint_limit;
  c.w_self = p->w_self_penetration;
  c.w_pen = p->w_object_penetration;
  auto stage = [](const grasp_stage_params& s) {
    return Stage{s.iters, s.step_rotation, s.step_translation, s.step_joints, s.step_floor};
  };
  c.coarse = stage(p->coarse);
  c.fine = stage(p->fine);
  c.final_stage = stage(p->final_stage);
  c.contact_offset = p->contact_offset;
  c.fd_step = p->fd_step;
  c.skip_fine = p->skip_fine_stages != 0;
  return c;
}

Rigid rigid12(const double* p) { return Rigid{m3_colmajor(p), v3(p + 9)}; }

std::vector<Frame> frames_from(const double* f, int m) {
  std::vector<Frame> out(m);
  for (int i = 0; i < m; ++i) {
    out[i].p = v3(f + 12 * i);
    out[i].n = v3(f + 12 * i + 3);
    out[i].d = v3(f + 12 * i + 6);
    out[i].e = v3(f + 12 * i + 9);
  }
  return out;
}

Stats g_total_stats;
std::mutex g_stats_mu;

void write_record(const Record& r, int g, int D, int n, int m, grasp_out* out) {
  auto copy = [&](double* dst, const VecX& src) {
    if (dst) std::memcpy(dst + static_cast<size_t>(g) * D, src.data(), sizeof(double) * D);
  };
  copy(out->x_p, r.x_p);
  copy(out->x, r.x);
  copy(out->x_s, r.x_s);
  if (out->energy_total) out->energy_total[g] = r.energy_total;
  const double nan = std::numeric_limits<double>::quiet_NaN();
  if (out->per_direction)
    for (int j = 0; j < 6; ++j) out->per_direction[6 * g + j] = r.per_direction.empty() ? nan : r.per_direction[j];
  if (out->contact_forces)
    for (int i = 0; i < n * 6; ++i) out->contact_forces[static_cast<size_t>(g) * n * 6 + i] = r.forces.empty() ? nan : r.forces.d[i];
  if (out->contacts)
    for (int i = 0; i < m; ++i) {
      double* c = out->contacts + (static_cast<size_t>(g) * m + i) * 12;
      if (r.contacts.empty()) {
        for (int k = 0; k < 12; ++k) c[k] = nan;
        continue;
      }
      const Frame& f = r.contacts[i];
      for (int k = 0; k < 3; ++k) {
        c[k] = f.p[k];
        c[3 + k] = f.n[k];
        c[6 + k] = f.d[k];
        c[9 + k] = f.e[k];
      }
    }
  if (out->stage_energy)
    for (int s = 0; s < 3; ++s) {
      out->stage_energy[6 * g + 2 * s] = r.stage_energy[s][0];
      out->stage_energy[6 * g + 2 * s + 1] = r.stage_energy[s][1];
    }
  if (out->failed) out->failed[g] = r.failed;
  if (out->qp_converged)
    for (int j = 0; j < 6; ++j) out->qp_converged[6 * g + j] = r.converged.empty() ? 0 : r.converged[j];
}

// Runs fn(g) for g in [0, n) on `threads` std::threads (strided, like
// pipeline.cpp:443-455); rethrows the first exception on the caller.
template <class F>
void parallel_grasps(int n, int threads, F&& fn) {
  const int nw = std::max(1, std::min(threads, n));
  if (nw == 1) {
    for (int g = 0; g < n; ++g) fn(g);
    return;
  }
  std::mutex mu;
  std::exception_ptr first;
  std::vector<std::thread> pool;
  for (int w = 0; w < nw; ++w)
    pool.emplace_back([&, w] {
      try {
        for (int g = w; g < n; g += nw) fn(g);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!first) first = std::current_exception();
      }
    });
  for (auto& t : pool) t.join();
  if (first) std::rethrow_exception(first);
}

}  // namespace

namespace oracle {
Hand make_hand_desc(const grasp_hand_desc* d) { return make_hand(d); }
Config make_config_params(const grasp_run_params* p) { return make_config(p); }
int set_error(int code, const char* what) {
  g_err = what;
  return code;
}
}  // namespace oracle

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

int oracle_point_to_mesh(const grasp_object_desc* od, int n, const double* pts, double* out) {
  return guarded([&] {
    const Object obj = make_object(od);
    for (int i = 0; i < n; ++i) {
      const Nearest r = point_to_mesh(v3(pts + 3 * i), obj.parts);
      double* o = out + 8 * i;
      o[0] = r.distance;
      for (int k = 0; k < 3; ++k) { o[1 + k] = r.b[k]; o[4 + k] = r.normal[k]; }
      o[7] = r.part;
    }
  });
}

// Pairs of object parts (od_a[ia[i]] posed by poses_a vs od_b[ib[i]] posed
// by poses_b). kind 0: signed_distance, 1: gjk_distance, 2: epa_depth.
int oracle_part_pairs(const grasp_object_desc* oa, const grasp_object_desc* ob, int n, const int* ia, const int* ib,
                      const double* poses_a, const double* poses_b, int kind, double* out) {
  return guarded([&] {
    const Object A = make_object(oa), B = make_object(ob);
    for (int i = 0; i < n; ++i) {
      const Rigid pa = rigid12(poses_a + 12 * i), pb = rigid12(poses_b + 12 * i);
      double* o = out + 11 * i;
      Nearest r;
      bool epa = false;
      if (kind == 0) {
        signed_distance(A.parts[ia[i]], pa, B.parts[ib[i]], pb, &r, &epa);
      } else if (kind == 1) {
        r = gjk_distance(A.parts[ia[i]], pa, B.parts[ib[i]], pb);
      } else {
        const auto de = epa_depth(A.parts[ia[i]], pa, B.parts[ib[i]], pb);
        r.distance = de.first;
        r.normal = de.second;
        epa = true;
      }
      o[0] = r.distance;
      for (int k = 0; k < 3; ++k) { o[1 + k] = r.a[k]; o[4 + k] = r.b[k]; o[7 + k] = r.normal[k]; }
      o[10] = epa ? 1.0 : 0.0;
    }
  });
}

int oracle_signed_distance(const grasp_hand_desc* hd, const grasp_object_desc* od, int n, const int* link_ids,
                           const int* part_ids, const double* poses, double* out) {
  return guarded([&] {
    const Hand h = make_hand(hd);
    const Object obj = make_object(od);
    for (int i = 0; i < n; ++i) {
      Nearest r;
      bool epa = false;
      signed_distance(h.links[link_ids[i]].part, rigid12(poses + 12 * i), obj.parts[part_ids[i]],
                      Rigid{M3::identity(), V3()}, &r, &epa);
      double* o = out + 11 * i;
      o[0] = r.distance;
      for (int k = 0; k < 3; ++k) { o[1 + k] = r.a[k]; o[4 + k] = r.b[k]; o[7 + k] = r.normal[k]; }
      o[10] = epa ? 1.0 : 0.0;
    }
  });
}

// total_energy (pipeline.cpp:96-210) per grasp, grasps spread over `threads`
// std::threads. warm_ready[g] (NULL = all) selects which grasps start the
// coarse QP from warm_x/warm_y; those are updated in place like the
// reference's QpScratch. qp_iters/qp_conv receive the coarse QP's per-column
// sweep counts and convergence flags. world (optional, [n*L*12]) teacher-forces
// the link transforms (set_world_override).
int oracle_total_energy(const grasp_hand_desc* hd, const grasp_object_desc* od, const grasp_run_params* p, int stage,
                        int n, const double* x, const double* anchors, double* warm_x, double* warm_y,
                        const int* warm_ready, const double* world, double* energy, double* grad, int* qp_iters,
                        int* qp_conv, int threads) {
  return guarded([&] {
    const Hand h = make_hand(hd);
    const Object obj = make_object(od);
    const Config cfg = make_config(p);
    const int D = h.dims(), m = static_cast<int>(h.tips.size()), nv = m * cfg.n_edges, M = m + 1 + nv;
    auto one = [&](int g) {
      VecX xv(x + static_cast<size_t>(g) * D, x + static_cast<size_t>(g + 1) * D);
      std::vector<V3> anc;
      if (anchors)
        for (int f = 0; f < m; ++f) anc.push_back(v3(anchors + (static_cast<size_t>(g) * m + f) * 3));
      QpScratch scratch;
      if (warm_x && warm_y && (!warm_ready || warm_ready[g])) {
        scratch.forces = MatX(nv, 6);
        scratch.duals = MatX(M, 6);
        std::memcpy(scratch.forces.d.data(), warm_x + static_cast<size_t>(g) * nv * 6, sizeof(double) * nv * 6);
        std::memcpy(scratch.duals.d.data(), warm_y + static_cast<size_t>(g) * M * 6, sizeof(double) * M * 6);
        scratch.ready = true;
      }
      VecX gr;
      set_world_override(world ? world + static_cast<size_t>(g) * h.links.size() * 12 : nullptr);
      try {
        energy[g] = total_energy(h, obj, cfg, stage, anc, xv, scratch, grad ? &gr : nullptr);
      } catch (...) {
        set_world_override(nullptr);
        throw;
      }
      set_world_override(nullptr);
      if (grad) std::memcpy(grad + static_cast<size_t>(g) * D, gr.data(), sizeof(double) * D);
      if (stage == 0)
        for (int j = 0; j < 6; ++j) {
          if (qp_iters) qp_iters[6 * g + j] = scratch.iters[j];
          if (qp_conv) qp_conv[6 * g + j] = scratch.converged[j];
        }
      if (warm_x && warm_y && stage == 0) {
        std::memcpy(warm_x + static_cast<size_t>(g) * nv * 6, scratch.forces.d.data(), sizeof(double) * nv * 6);
        std::memcpy(warm_y + static_cast<size_t>(g) * M * 6, scratch.duals.d.data(), sizeof(double) * M * 6);
      }
    };
    parallel_grasps(n, threads, one);
  });
}

// forward_kinematics(pose_from_state(x)) (hand.cpp:108-153): out[n*L*12] world R (column-major) t.
int oracle_forward_kinematics(const grasp_hand_desc* hd, int n, const double* x, double* out) {
  return guarded([&] {
    const Hand h = make_hand(hd);
    const int D = h.dims(), L = static_cast<int>(h.links.size());
    for (int g = 0; g < n; ++g) {
      VecX xv(x + static_cast<size_t>(g) * D, x + static_cast<size_t>(g + 1) * D);
      const Fk fk = forward_kinematics(h, pose_from_state(h, xv));
      for (int l = 0; l < L; ++l) {
        double* o = out + (static_cast<size_t>(g) * L + l) * 12;
        for (int c = 0; c < 3; ++c)
          for (int i = 0; i < 3; ++i) o[3 * c + i] = fk.world[l].R(i, c);
        for (int i = 0; i < 3; ++i) o[9 + i] = fk.world[l].t[i];
      }
    }
  });
}

int oracle_apply_step(const grasp_hand_desc* hd, const grasp_stage_params* s, int it, int n, const double* grad,
                      double* x) {
  return guarded([&] {
    const Hand h = make_hand(hd);
    const Stage st{s->iters, s->step_rotation, s->step_translation, s->step_joints, s->step_floor};
    const int D = h.dims();
    for (int g = 0; g < n; ++g) {
      VecX xv(x + static_cast<size_t>(g) * D, x + static_cast<size_t>(g + 1) * D);
      VecX gv(grad + static_cast<size_t>(g) * D, grad + static_cast<size_t>(g + 1) * D);
      apply_step(h, st, it, gv, xv);
      std::memcpy(x + static_cast<size_t>(g) * D, xv.data(), sizeof(double) * D);
    }
  });
}

int oracle_coarse_distance_energy(const grasp_hand_desc* hd, const grasp_object_desc* od, int n, const double* x,
                                  double offset, double fd, double* energy, double* grad) {
  return guarded([&] {
    const Hand h = make_hand(hd);
    const Object obj = make_object(od);
    const int D = h.dims();
    for (int g = 0; g < n; ++g) {
      VecX xv(x + static_cast<size_t>(g) * D, x + static_cast<size_t>(g + 1) * D);
      VecX gr;
      energy[g] = coarse_distance_energy(h, xv, obj, offset, fd, grad ? &gr : nullptr);
      if (grad) std::memcpy(grad + static_cast<size_t>(g) * D, gr.data(), sizeof(double) * D);
    }
  });
}

int oracle_fine_contact_query(const grasp_hand_desc* hd, const grasp_object_desc* od, int n, const double* x,
                              double* out) {
  return guarded([&] {
    const Hand h = make_hand(hd);
    const Object obj = make_object(od);
    const int D = h.dims(), m = static_cast<int>(h.tips.size());
    for (int g = 0; g < n; ++g) {
      VecX xv(x + static_cast<size_t>(g) * D, x + static_cast<size_t>(g + 1) * D);
      const Fk fk = forward_kinematics(h, pose_from_state(h, xv));
      const auto ws = fine_contact_query(h, fk, obj);
      for (int f = 0; f < m; ++f) {
        double* o = out + (static_cast<size_t>(g) * m + f) * 11;
        for (int k = 0; k < 3; ++k) { o[k] = ws[f].c_w[k]; o[3 + k] = ws[f].p_w[k]; o[6 + k] = ws[f].n[k]; }
        o[9] = ws[f].distance;
        o[10] = ws[f].link;
      }
    }
  });
}

// Grasp evaluation (eval.cpp:51-158). ev = {mass, gravity, residual_rel_tol,
// force_budget_factor, contact_tol, penetration_tol, qp_eps}. Per grasp:
// out_real[9] = pd_mm, spd_mm, cdc_mm, residuals[6]; out_int[3] =
// contact_count, success, note_flags.
int oracle_eval(const grasp_hand_desc* hd, const grasp_object_desc* od, const grasp_run_params* p, const double* ev,
                int n, const double* x, const double* x_s, double* out_real, int* out_int) {
  return guarded([&] {
    const Hand h = make_hand(hd);
    const Object obj = make_object(od);
    const Config cfg = make_config(p);
    EvalParams e;
    e.mass = ev[0], e.gravity = ev[1], e.residual_rel_tol = ev[2], e.force_budget_factor = ev[3];
    e.contact_tol = ev[4], e.penetration_tol = ev[5], e.qp_eps = ev[6];
    const int D = h.dims();
    for (int g = 0; g < n; ++g) {
      const VecX xv(x + static_cast<size_t>(g) * D, x + static_cast<size_t>(g + 1) * D);
      const VecX xs(x_s + static_cast<size_t>(g) * D, x_s + static_cast<size_t>(g + 1) * D);
      const EvalResult r = quasi_static_check(h, obj, cfg, e, xv, xs);
      double* o = out_real + static_cast<size_t>(g) * 9;
      o[0] = r.pd_mm;
      o[1] = r.spd_mm;
      o[2] = r.cdc_mm;
      for (int j = 0; j < 6; ++j) o[3 + j] = r.residuals[j];
      int* oi = out_int + static_cast<size_t>(g) * 3;
      oi[0] = r.contact_count;
      oi[1] = r.success ? 1 : 0;
      oi[2] = r.note_flags;
    }
  });
}

// Lower QP batch, one 6-column batch per grasp (energy.cpp:60-92).
int oracle_qp_batch(const grasp_run_params* p, int n_grasps, int m, const double* frames, const double* warm_x,
                    const double* warm_y, double* X, double* Y, double* Z, int* iters, int* converged,
                    double* per_direction, int threads) {
  return guarded([&] {
    const Config cfg = make_config(p);
    const int nv = m * cfg.n_edges, M = m + 1 + nv;
    auto work = [&](int t) {
      for (int g = t; g < n_grasps; g += threads) {
        const auto fr = frames_from(frames + static_cast<size_t>(g) * m * 12, m);
        MatX wx, wy;
        if (warm_x && warm_y) {
          wx = MatX(nv, 6);
          wy = MatX(M, 6);
          std::memcpy(wx.d.data(), warm_x + static_cast<size_t>(g) * nv * 6, sizeof(double) * nv * 6);
          std::memcpy(wy.d.data(), warm_y + static_cast<size_t>(g) * M * 6, sizeof(double) * M * 6);
        }
        const MatX dirs = closure_directions();
        const MatX W = wrench_basis(fr, cfg.mu, cfg.n_edges);
        const SharedBatch b = assemble_lower_qp(W, m, dirs, cfg.beta, cfg.gamma_per_contact * m);
        const BatchSolution s = solve_shared(b, cfg.qp, warm_x ? &wx : nullptr, warm_y ? &wy : nullptr);
        if (X) std::memcpy(X + static_cast<size_t>(g) * nv * 6, s.X.d.data(), sizeof(double) * nv * 6);
        if (Y) std::memcpy(Y + static_cast<size_t>(g) * M * 6, s.Y.d.data(), sizeof(double) * M * 6);
        if (Z) std::memcpy(Z + static_cast<size_t>(g) * M * 6, s.Z.d.data(), sizeof(double) * M * 6);
        for (int j = 0; j < 6; ++j) {
          if (iters) iters[6 * g + j] = s.iters[j];
          if (converged) converged[6 * g + j] = s.converged[j];
          if (per_direction) {
            double e = 0.0;
            for (int r = 0; r < 6; ++r) {
              double wl = 0.0;
              for (int c = 0; c < nv; ++c) wl += W(r, c) * s.X(c, j);
              const double res = cfg.beta * dirs(r, j) - wl;
              e += res * res;
            }
            per_direction[6 * g + j] = e;
          }
        }
      }
    };
    if (threads <= 1) {
      threads = 1;
      work(0);
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
      for (auto& th : pool) th.join();
    }
  });
}

// synthesize (pipeline.cpp:436-457) over caller-provided x0, strided over
// `workers` std::threads like the reference. stats (optional) receives the
// 15 op counters of Stats in declaration order.
int oracle_synthesize(const grasp_hand_desc* hd, const grasp_object_desc* od, const grasp_run_params* p, int batch,
                      const double* x0, int workers, grasp_out* out, long long* stats) {
  return guarded([&] {
    const Hand h = make_hand(hd);
    const Object obj = make_object(od);
    const Config cfg = make_config(p);
    const int D = h.dims(), m = static_cast<int>(h.tips.size()), nv = m * cfg.n_edges;
    Stats total;
    std::mutex mu;
    std::string first_error;
    const int nw = std::min(std::max(workers, 1), batch);
    auto slice = [&](int w) {
      Stats local;
      if (stats) set_stats_sink(&local);
      try {
        for (int g = w; g < batch; g += nw) {
          VecX xv(x0 + static_cast<size_t>(g) * D, x0 + static_cast<size_t>(g + 1) * D);
          const Record r = run_grasp(h, obj, cfg, xv);
          write_record(r, g, D, nv, m, out);
        }
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(mu);
        if (first_error.empty()) first_error = e.what();
      }
      set_stats_sink(nullptr);
      std::lock_guard<std::mutex> lk(mu);
      total.add(local);
    };
    if (nw == 1) {
      slice(0);
    } else {
      std::vector<std::thread> pool;
      for (int w = 0; w < nw; ++w) pool.emplace_back(slice, w);
      for (auto& t : pool) t.join();
    }
    if (!first_error.empty()) throw std::runtime_error(first_error);
    if (stats) {
      const long long v[15] = {total.point_queries, total.inside_faces, total.outside_faces, total.gjk_calls,
                               total.gjk_iters, total.gjk_support_verts, total.epa_calls, total.epa_iters,
                               total.epa_face_scans, total.qp_solves, total.qp_sweeps, total.qp_column_sweeps,
                               total.jacobians, total.self_pairs, total.obb_tests};
      std::memcpy(stats, v, sizeof(v));
    }
  });
}

}  // extern "C"

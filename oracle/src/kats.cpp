// ORACLE (test infrastructure only). Fine-grained C entry points into the
// fp64 restatement so tests/test_oracle_kats.py can run the reference's own
// known-answer tests (proj/tests/test_hand.cpp, test_contact.cpp,
// test_qpsolve.cpp, test_energy.cpp, test_pipeline.cpp) against it. Layouts:
// 3x3 blocks column-major (the state layout, hand.hpp:56-61), Jacobians
// 3 x D row-major, general matrices column-major (Eigen's default).
#include "oracle_impl.hpp"

#include "../../include/grasp_b200.h"

#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

namespace oracle {
// capi.cpp
Hand make_hand_desc(const grasp_hand_desc* d);
Config make_config_params(const grasp_run_params* p);
int set_error(int code, const char* what);
}  // namespace oracle

using namespace oracle;

namespace {

template <class F>
int kat_guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const GeometryError& e) {
    return set_error(GRASP_EGEOM, e.what());
  } catch (const std::exception& e) {
    return set_error(GRASP_EINVAL, e.what());
  }
}

M3 colmajor(const double* p) {
  M3 r;
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) r(i, c) = p[3 * c + i];
  return r;
}

void store_colmajor(const M3& m, double* p) {
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) p[3 * c + i] = m(i, c);
}

V3 v3p(const double* p) { return V3(p[0], p[1], p[2]); }

MatX matx(const double* p, int rows, int cols) {
  MatX m(rows, cols);
  std::memcpy(m.d.data(), p, sizeof(double) * rows * cols);
  return m;
}

std::vector<Frame> frames_of(const double* f, int m) {
  std::vector<Frame> out(m);
  for (int i = 0; i < m; ++i) out[i] = Frame{v3p(f + 12 * i), v3p(f + 12 * i + 3), v3p(f + 12 * i + 6), v3p(f + 12 * i + 9)};
  return out;
}

QpParams qp_of(const grasp_run_params* p) {
  QpParams q;
  q.rho = p->qp_rho;
  q.sigma = p->qp_sigma;
  q.alpha = p->qp_alpha;
  q.max_iters = p->qp_max_iters;
  q.eps_primal = p->qp_eps_primal;
  q.eps_dual = p->qp_eps_dual;
  q.check_interval = p->qp_check_interval;
  return q;
}

}  // namespace

extern "C" {

// project_rotation (hand.cpp:45-73) for n raw blocks.
int oracle_project_rotation(int n, const double* raw, double* R, int* fallback) {
  return kat_guard([&] {
    for (int i = 0; i < n; ++i) {
      bool fb = false;
      store_colmajor(project_rotation(colmajor(raw + 9 * i), &fb), R + 9 * i);
      if (fallback) fallback[i] = fb ? 1 : 0;
    }
  });
}

// make_pose_state + rotation_tangent_jacobian (hand.cpp:75-106): R, a_inv (column-major),
// degenerate flag, tangent Jacobian 3 x 9 row-major.
int oracle_pose_state(int n, const double* raw, double* R, double* a_inv, int* degenerate, double* tangent) {
  return kat_guard([&] {
    for (int i = 0; i < n; ++i) {
      const PoseState ps = make_pose_state(colmajor(raw + 9 * i));
      if (R) store_colmajor(ps.R, R + 9 * i);
      if (a_inv) store_colmajor(ps.a_inv, a_inv + 9 * i);
      if (degenerate) degenerate[i] = ps.degenerate ? 1 : 0;
      if (tangent) {
        double J[3][9];
        tangent_jacobian(ps, J);
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 9; ++c) tangent[27 * i + 9 * r + c] = J[r][c];
      }
    }
  });
}

// point_jacobian (kind 0, hand.cpp:155-169) / direction_jacobian (kind 1, :171-183) of a world
// point / direction attached to `link` at state x: J[3*D] row-major.
int oracle_hand_jacobian(const grasp_hand_desc* hd, const double* x, int link, const double* vec, int kind, double* J) {
  return kat_guard([&] {
    const Hand h = make_hand_desc(hd);
    if (link < 0 || link >= static_cast<int>(h.links.size())) throw std::invalid_argument("link out of range");
    const int D = h.dims();
    const VecX xv(x, x + D);
    const PoseState ps = make_pose_state(raw_block(xv));
    const Pose pose = pose_from_state(h, xv);
    const Fk fk = forward_kinematics(h, pose);
    const MatX M = kind == 0 ? point_jacobian(h, ps, pose, fk, link, v3p(vec))
                             : direction_jacobian(h, ps, pose, fk, link, v3p(vec));
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < D; ++c) J[r * D + c] = M(r, c);
  });
}

// limit_energy (hand.cpp:207-218, which = 0) / self_penetration_energy (:220-245, which = 1)
// for n states; grad[n*D] optional.
int oracle_hand_energy(const grasp_hand_desc* hd, int which, int n, const double* x, double* e, double* grad) {
  return kat_guard([&] {
    const Hand h = make_hand_desc(hd);
    const int D = h.dims();
    for (int g = 0; g < n; ++g) {
      const VecX xv(x + static_cast<size_t>(g) * D, x + static_cast<size_t>(g + 1) * D);
      const Pose pose = pose_from_state(h, xv);
      VecX gr;
      if (which == 0) {
        e[g] = limit_energy(h, pose, grad ? &gr : nullptr);
      } else {
        const PoseState ps = make_pose_state(raw_block(xv));
        e[g] = self_penetration_energy(h, ps, pose, forward_kinematics(h, pose), grad ? &gr : nullptr);
      }
      if (grad) std::memcpy(grad + static_cast<size_t>(g) * D, gr.data(), sizeof(double) * D);
    }
  });
}

// build_frame (contact.cpp:13-21) for n (p, n) pairs: out[n*12] = p n d e.
int oracle_build_frame(int n, const double* p, const double* nrm, double* out) {
  return kat_guard([&] {
    for (int i = 0; i < n; ++i) {
      const Frame f = build_frame(v3p(p + 3 * i), v3p(nrm + 3 * i));
      for (int k = 0; k < 3; ++k) {
        out[12 * i + k] = f.p[k];
        out[12 * i + 3 + k] = f.n[k];
        out[12 * i + 6 + k] = f.d[k];
        out[12 * i + 9 + k] = f.e[k];
      }
    }
  });
}

// wrench_basis (contact.cpp:47-53): W[6 * m*k] column-major.
int oracle_wrench_basis(int m, const double* frames, double mu, int k, double* W) {
  return kat_guard([&] {
    if (k < 3) throw std::invalid_argument("friction pyramid needs >= 3 edges");
    if (!(mu > 0)) throw std::invalid_argument("friction coefficient must be positive");
    const MatX w = wrench_basis(frames_of(frames, m), mu, k);
    std::memcpy(W, w.d.data(), sizeof(double) * w.d.size());
  });
}

// assemble_lower_qp (qpsolve.cpp:193-235) from W[6*nv] (column-major) and targets[6*B].
int oracle_assemble_lower_qp(const double* W, int m, int nv, const double* targets, int B, double beta,
                             double gamma_total, double* P, double* A, double* Q, double* L, double* U) {
  return kat_guard([&] {
    const SharedBatch b = assemble_lower_qp(matx(W, 6, nv), m, matx(targets, 6, B), beta, gamma_total);
    const int M = b.A.rows;
    std::memcpy(P, b.P.d.data(), sizeof(double) * nv * nv);
    std::memcpy(A, b.A.d.data(), sizeof(double) * M * nv);
    std::memcpy(Q, b.Q.d.data(), sizeof(double) * nv * B);
    std::memcpy(L, b.L.d.data(), sizeof(double) * M * B);
    std::memcpy(U, b.U.d.data(), sizeof(double) * M * B);
  });
}

// solve_shared (qpsolve.cpp:45-120) on a general shared-structure batch: P[n*n], A[M*n],
// Q[n*B], L/U[M*B] column-major; QP settings from p's qp_* fields.
// rows[3] = row counts of Q, L, U as given (checked against n and M like qpsolve.cpp:14-25).
int oracle_solve_shared(int n, int M, int B, const double* P, const double* A, const double* Q, const double* L,
                        const double* U, const int* rows, const grasp_run_params* p, const double* warm_x,
                        const double* warm_y, double* X, double* Y, double* Z, int* iters, int* converged) {
  return kat_guard([&] {
    SharedBatch b;
    b.P = matx(P, n, n);
    b.A = matx(A, M, n);
    b.Q = matx(Q, rows[0], B);
    b.L = matx(L, rows[1], B);
    b.U = matx(U, rows[2], B);
    MatX wx, wy;
    if (warm_x && warm_y) {
      wx = matx(warm_x, n, B);
      wy = matx(warm_y, M, B);
    }
    const BatchSolution s = solve_shared(b, qp_of(p), warm_x ? &wx : nullptr, warm_y ? &wy : nullptr);
    if (X) std::memcpy(X, s.X.d.data(), sizeof(double) * n * B);
    if (Y) std::memcpy(Y, s.Y.d.data(), sizeof(double) * M * B);
    if (Z) std::memcpy(Z, s.Z.d.data(), sizeof(double) * M * B);
    for (int c = 0; c < B; ++c) {
      if (iters) iters[c] = s.iters[c];
      if (converged) converged[c] = s.converged[c];
    }
  });
}

// grasp_energy (energy.cpp:60-92) with arbitrary targets[6*B] (NULL = the six closure
// directions, B = 6): total, per_direction[B], forces[nv*B], residuals[6*B], duals[M*B],
// converged[B], iters[B].
int oracle_grasp_energy(const grasp_run_params* p, int m, const double* frames, int B, const double* targets,
                        const double* warm_x, const double* warm_y, double* total, double* per_direction,
                        double* forces, double* residuals, double* duals, int* converged, int* iters) {
  return kat_guard([&] {
    const int k = p->n_edges, nv = m * k, M = m + 1 + nv;
    const MatX tg = targets ? matx(targets, 6, B) : closure_directions();
    MatX wx, wy;
    if (warm_x && warm_y) {
      wx = matx(warm_x, nv, tg.cols);
      wy = matx(warm_y, M, tg.cols);
    }
    const EnergyReport r = grasp_energy(frames_of(frames, m), p->beta, p->gamma_per_contact, p->mu, k, qp_of(p),
                                        warm_x ? &wx : nullptr, warm_y ? &wy : nullptr, &tg);
    if (total) *total = r.total;
    for (int j = 0; j < tg.cols; ++j) {
      if (per_direction) per_direction[j] = r.per_direction[j];
      if (converged) converged[j] = r.converged[j];
      if (iters) iters[j] = r.iters[j];
    }
    if (forces) std::memcpy(forces, r.forces.d.data(), sizeof(double) * r.forces.d.size());
    if (residuals) std::memcpy(residuals, r.residuals.d.data(), sizeof(double) * r.residuals.d.size());
    if (duals) std::memcpy(duals, r.duals.d.data(), sizeof(double) * r.duals.d.size());
  });
}

// grasp_energy_gradient (energy.cpp:94-145) from a closure-direction report (forces[nv*6],
// residuals[6*6]) and contact Jacobians jac_p/jac_n[m*3*D] (3 x D row-major each).
int oracle_grasp_energy_gradient(const grasp_run_params* p, int m, const double* frames, const double* forces,
                                 const double* residuals, int D, const double* jac_p, const double* jac_n,
                                 double* grad) {
  return kat_guard([&] {
    const int k = p->n_edges, nv = m * k;
    EnergyReport r;
    r.forces = matx(forces, nv, 6);
    r.residuals = matx(residuals, 6, 6);
    std::vector<MatX> jp(m), jn(m);
    for (int i = 0; i < m; ++i) {
      jp[i] = MatX(3, D);
      jn[i] = MatX(3, D);
      for (int rr = 0; rr < 3; ++rr)
        for (int c = 0; c < D; ++c) {
          jp[i](rr, c) = jac_p[(static_cast<size_t>(i) * 3 + rr) * D + c];
          jn[i](rr, c) = jac_n[(static_cast<size_t>(i) * 3 + rr) * D + c];
        }
    }
    const VecX g = grasp_energy_gradient(frames_of(frames, m), r, p->mu, k, jp, jn);
    std::memcpy(grad, g.data(), sizeof(double) * D);
  });
}

// fine_stage_surrogate (energy.cpp:208-229) on n points with optional Jacobians jac[n*3*D].
int oracle_stage_surrogate(int n, const double* points, const double* anchors, int D, const double* jac,
                           double* value, double* grad) {
  return kat_guard([&] {
    std::vector<V3> pts, anc;
    std::vector<MatX> js;
    for (int i = 0; i < n; ++i) {
      pts.push_back(v3p(points + 3 * i));
      anc.push_back(v3p(anchors + 3 * i));
      if (jac) {
        MatX J(3, D);
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < D; ++c) J(r, c) = jac[(static_cast<size_t>(i) * 3 + r) * D + c];
        js.push_back(J);
      }
    }
    VecX g;
    *value = fine_stage_surrogate(pts, anc, js, grad ? &g : nullptr);
    if (grad && jac) std::memcpy(grad, g.data(), sizeof(double) * D);
  });
}

// fine_grasp_surrogate (pipeline.cpp:54-65, 382-386): witnesses c_w[m*3] on links[m],
// anchors[m*3], state x -> value, grad[D] (witnesses rigid on their links).
int oracle_fine_grasp_surrogate(const grasp_hand_desc* hd, const double* x, int m, const double* c_w,
                                const int* links, const double* anchors, double* value, double* grad) {
  return kat_guard([&] {
    const Hand h = make_hand_desc(hd);
    const int D = h.dims();
    const VecX xv(x, x + D);
    const PoseState ps = make_pose_state(raw_block(xv));
    const Pose pose = pose_from_state(h, xv);
    const Fk fk = forward_kinematics(h, pose);
    std::vector<V3> pts, anc;
    std::vector<MatX> js;
    for (int i = 0; i < m; ++i) {
      pts.push_back(v3p(c_w + 3 * i));
      anc.push_back(v3p(anchors + 3 * i));
      js.push_back(point_jacobian(h, ps, pose, fk, links[i], pts.back()));
    }
    VecX g;
    *value = fine_stage_surrogate(pts, anc, js, grad ? &g : nullptr);
    if (grad) std::memcpy(grad, g.data(), sizeof(double) * D);
  });
}

}  // extern "C"

// ORACLE (test infrastructure only). fp64 restatement of
// /root/reference/proj/src/hand.cpp:14-245 (projection, pose state, FK,
// point Jacobian, limit + self-penetration energies), contact.cpp:9-53,
// qpsolve.cpp:45-120 + 193-235 (dense LLT ADMM) and energy.cpp:49-145.
#include "oracle_impl.hpp"

#include <cmath>
#include <numbers>

namespace oracle {

// ------------------------------------------------------------ rotations
namespace {

// One-sided Jacobi SVD of a 3x3 (stands in for Eigen::JacobiSVD, hand.cpp:47).
void svd3(const M3& a, M3& U, V3& s, M3& V) {
  double col[3][3], v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) col[j][i] = a(i, j);
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool changed = false;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double al = 0, be = 0, ga = 0;
        for (int i = 0; i < 3; ++i) {
          al += col[p][i] * col[p][i];
          be += col[q][i] * col[q][i];
          ga += col[p][i] * col[q][i];
        }
        if (ga == 0.0 || std::abs(ga) <= 1e-15 * std::sqrt(al * be)) continue;
        changed = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        for (int i = 0; i < 3; ++i) {
          const double x = col[p][i], y = col[q][i];
          col[p][i] = c * x - sn * y;
          col[q][i] = sn * x + c * y;
          const double vx = v[p][i], vy = v[q][i];
          v[p][i] = c * vx - sn * vy;
          v[q][i] = sn * vx + c * vy;
        }
      }
    if (!changed) break;
  }
  double sv[3];
  for (int j = 0; j < 3; ++j) sv[j] = std::sqrt(col[j][0] * col[j][0] + col[j][1] * col[j][1] + col[j][2] * col[j][2]);
  int ord[3] = {0, 1, 2};
  for (int i = 0; i < 2; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (sv[ord[j]] > sv[ord[i]]) std::swap(ord[i], ord[j]);
  for (int k = 0; k < 3; ++k) {
    s[k] = sv[ord[k]];
    for (int i = 0; i < 3; ++i) {
      V(i, k) = v[ord[k]][i];
      U(i, k) = sv[ord[k]] > 0 ? col[ord[k]][i] / sv[ord[k]] : 0.0;
    }
  }
}

}  // namespace

// hand.cpp:45-73.
M3 project_rotation(const M3& raw, bool* fallback) {
  M3 U, V;
  V3 s;
  svd3(raw, U, s, V);
  if (!(s[0] > 0) || s[2] < 1e-9 * s[0]) {
    if (fallback) *fallback = true;
    V3 c0 = raw.col(0);
    if (norm(c0) < 1e-12) c0 = V3(1, 0, 0);
    c0 = normalized(c0);
    V3 c1 = raw.col(1) - c0 * dot(c0, raw.col(1));
    if (norm(c1) < 1e-12) {
      c1 = V3(0, 1, 0) - c0 * c0.y();
      if (norm(c1) < 1e-12) c1 = V3(0, 0, 1) - c0 * c0.z();
    }
    c1 = normalized(c1);
    M3 R;
    R.set_col(0, c0);
    R.set_col(1, c1);
    R.set_col(2, cross(c0, c1));
    return R;
  }
  if (fallback) *fallback = false;
  const M3 uvt = U * V.t();
  M3 fix;
  fix(2, 2) = uvt.det() < 0 ? -1.0 : 1.0;
  return U * fix * V.t();
}

// hand.cpp:75-95.
PoseState make_pose_state(const M3& raw) {
  PoseState ps;
  ps.raw = raw;
  bool fb = false;
  ps.R = project_rotation(raw, &fb);
  ps.degenerate = fb;
  if (!ps.degenerate) {
    const M3 sf = ps.R.t() * raw;
    const M3 s = 0.5 * (sf + sf.t());
    const M3 a = s.trace() * M3::identity() - s;
    const double det = a.det();
    if (std::abs(det) < 1e-12) {
      ps.degenerate = true;
    } else {
      M3 inv;  // adjugate / determinant
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
    }
  }
  return ps;
}

M3 raw_block(const VecX& x) {
  M3 r;
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 3; ++i) r(i, c) = x[3 * c + i];  // column-major state
  return r;
}

// hand.cpp:108-116.
Pose pose_from_state(const Hand& h, const VecX& x) {
  if (static_cast<int>(x.size()) != h.dims()) throw std::invalid_argument("state vector has wrong size for this hand");
  Pose p;
  p.R = project_rotation(raw_block(x), nullptr);
  p.t = V3(x[9], x[10], x[11]);
  p.q.assign(x.begin() + 12, x.end());
  return p;
}

// hand.cpp:126-153.
Fk forward_kinematics(const Hand& h, const Pose& pose) {
  Fk fk;
  const int L = static_cast<int>(h.links.size());
  fk.chain.resize(L);
  fk.world.resize(L);
  fk.joint_origin.resize(h.dof());
  fk.joint_axis.resize(h.dof());
  const Rigid base{pose.R, pose.t};
  for (int l = 0; l < L; ++l) {
    const int j = h.links[l].parent_joint;
    if (j < 0) {
      fk.chain[l] = Rigid{M3::identity(), V3()};
    } else {
      const Joint& jt = h.joints[j];
      const Rigid parent = fk.chain[jt.parent_link];
      const Rigid step{angle_axis(pose.q[j], jt.axis), jt.origin};
      fk.chain[l] = parent * step;
      fk.joint_origin[j] = parent.apply(jt.origin);
      fk.joint_axis[j] = fk.chain[l].R * jt.axis;
    }
    fk.world[l] = base * fk.chain[l];
  }
  return fk;
}

namespace {

// hand.cpp:20-29.
bool is_ancestor_joint(const Hand& h, int joint, int link) {
  int l = link;
  while (l >= 0) {
    const int j = h.links[l].parent_joint;
    if (j < 0) return false;
    if (j == joint) return true;
    l = h.joints[j].parent_link;
  }
  return false;
}

// hand.cpp:97-106: 3x9, column 3l+i = a_inv (e_l x R.row(i)).
void rotation_tangent_jacobian(const PoseState& ps, double J[3][9]) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 9; ++c) J[r][c] = 0.0;
  if (ps.degenerate) return;
  for (int l = 0; l < 3; ++l)
    for (int i = 0; i < 3; ++i) {
      const V3 col = ps.a_inv * cross(V3::unit(l), ps.R.row(i));
      for (int r = 0; r < 3; ++r) J[r][3 * l + i] = col[r];
    }
}

}  // namespace

// hand.cpp:155-169.
MatX point_jacobian(const Hand& h, const PoseState& ps, const Pose& pose, const Fk& fk, int link, const V3& pw) {
  if (Stats* st = stats_sink()) ++st->jacobians;
  MatX J(3, h.dims());
  const V3 v = pose.R.t() * (pw - pose.t);
  double T[3][9];
  rotation_tangent_jacobian(ps, T);
  const M3 A = pose.R * skew(v);  // J_rot = -A * T
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 9; ++c) J(r, c) = -(A(r, 0) * T[0][c] + A(r, 1) * T[1][c] + A(r, 2) * T[2][c]);
  for (int r = 0; r < 3; ++r) J(r, 9 + r) = 1.0;
  for (int jo = 0; jo < h.dof(); ++jo) {
    if (!is_ancestor_joint(h, jo, link)) continue;
    const V3 col = pose.R * cross(fk.joint_axis[jo], v - fk.joint_origin[jo]);
    for (int r = 0; r < 3; ++r) J(r, 12 + jo) = col[r];
  }
  return J;
}

// hand.cpp:171-183: like point_jacobian for a direction (no translation columns).
MatX direction_jacobian(const Hand& h, const PoseState& ps, const Pose& pose, const Fk& fk, int link, const V3& dw) {
  MatX J(3, h.dims());
  const V3 v = pose.R.t() * dw;
  double T[3][9];
  rotation_tangent_jacobian(ps, T);
  const M3 A = pose.R * skew(v);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 9; ++c) J(r, c) = -(A(r, 0) * T[0][c] + A(r, 1) * T[1][c] + A(r, 2) * T[2][c]);
  for (int jo = 0; jo < h.dof(); ++jo) {
    if (!is_ancestor_joint(h, jo, link)) continue;
    const V3 col = pose.R * cross(fk.joint_axis[jo], v);
    for (int r = 0; r < 3; ++r) J(r, 12 + jo) = col[r];
  }
  return J;
}

void tangent_jacobian(const PoseState& ps, double J[3][9]) { rotation_tangent_jacobian(ps, J); }

// hand.cpp:207-218.
double limit_energy(const Hand& h, const Pose& pose, VecX* grad) {
  double e = 0.0;
  if (grad) grad->assign(h.dims(), 0.0);
  for (int j = 0; j < h.dof(); ++j) {
    const double over = std::max(pose.q[j] - h.joints[j].upper, 0.0);
    const double under = std::max(h.joints[j].lower - pose.q[j], 0.0);
    e += over * over + under * under;
    if (grad) (*grad)[12 + j] = 2.0 * over - 2.0 * under;
  }
  return e;
}

// hand.cpp:220-245.
double self_penetration_energy(const Hand& h, const PoseState& ps, const Pose& pose, const Fk& fk, VecX* grad) {
  double e = 0.0;
  if (grad) grad->assign(h.dims(), 0.0);
  for (const auto& [la, lb] : h.pairs) {
    for (const Proxy& pa : h.links[la].proxies) {
      const V3 ca = fk.world[la].apply(pa.c);
      for (const Proxy& pb : h.links[lb].proxies) {
        if (Stats* st = stats_sink()) ++st->self_pairs;
        const V3 cb = fk.world[lb].apply(pb.c);
        const double dist = norm(ca - cb);
        const double overlap = pa.r + pb.r - dist;
        if (overlap <= 0) continue;
        e += overlap * overlap;
        if (grad && dist > 1e-12) {
          const V3 dir = (ca - cb) / dist;
          const MatX ja = point_jacobian(h, ps, pose, fk, la, ca);
          const MatX jb = point_jacobian(h, ps, pose, fk, lb, cb);
          for (int c = 0; c < h.dims(); ++c) {
            double s = 0.0;
            for (int r = 0; r < 3; ++r) s += ja(r, c) * (-2.0 * overlap * dir[r]) + jb(r, c) * (2.0 * overlap * dir[r]);
            (*grad)[c] += s;
          }
        }
      }
    }
  }
  return e;
}

// ------------------------------------------------------------- contact
// contact.cpp:9-21.
V3 frame_seed(const V3& n) { return std::abs(n.x()) > 0.99 ? V3(0, 1, 0) : V3(1, 0, 0); }

Frame build_frame(const V3& p, const V3& n) {
  Frame f;
  f.p = p;
  f.n = n;
  f.d = normalized(cross(n, frame_seed(n)));
  f.e = cross(n, f.d);
  return f;
}

// contact.cpp:30-53: column (i*k + j) = [edge; p x edge].
MatX wrench_basis(const std::vector<Frame>& frames, double mu, int k) {
  const int m = static_cast<int>(frames.size());
  MatX W(6, m * k);
  for (int i = 0; i < m; ++i) {
    const Frame& f = frames[i];
    for (int j = 0; j < k; ++j) {
      const double th = 2.0 * std::numbers::pi * j / k;
      const V3 edge = f.n + mu * (std::cos(th) * f.d + std::sin(th) * f.e);
      const V3 tq = cross(f.p, edge);
      for (int r = 0; r < 3; ++r) {
        W(r, i * k + j) = edge[r];
        W(3 + r, i * k + j) = tq[r];
      }
    }
  }
  return W;
}

// ------------------------------------------------------------------ QP
namespace {

MatX matmul(const MatX& a, const MatX& b) {
  MatX r(a.rows, b.cols);
  for (int j = 0; j < b.cols; ++j)
    for (int k = 0; k < a.cols; ++k) {
      const double bkj = b(k, j);
      if (bkj == 0.0) continue;
      for (int i = 0; i < a.rows; ++i) r(i, j) += a(i, k) * bkj;
    }
  return r;
}

MatX transpose(const MatX& a) {
  MatX r(a.cols, a.rows);
  for (int j = 0; j < a.cols; ++j)
    for (int i = 0; i < a.rows; ++i) r(j, i) = a(i, j);
  return r;
}

// Dense Cholesky K = L L^T (stands in for Eigen::LLT, qpsolve.cpp:55).
bool cholesky(const MatX& K, MatX& L) {
  const int n = K.rows;
  L = MatX(n, n);
  for (int j = 0; j < n; ++j) {
    double d = K(j, j);
    for (int k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
    if (!(d > 0.0)) return false;
    const double ljj = std::sqrt(d);
    L(j, j) = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = K(i, j);
      for (int k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
      L(i, j) = s / ljj;
    }
  }
  return true;
}

void chol_solve(const MatX& L, MatX& B) {
  const int n = L.rows;
  for (int c = 0; c < B.cols; ++c) {
    for (int i = 0; i < n; ++i) {
      double s = B(i, c);
      for (int k = 0; k < i; ++k) s -= L(i, k) * B(k, c);
      B(i, c) = s / L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = B(i, c);
      for (int k = i + 1; k < n; ++k) s -= L(k, i) * B(k, c);
      B(i, c) = s / L(i, i);
    }
  }
}

}  // namespace

// qpsolve.cpp:193-235.
SharedBatch assemble_lower_qp(const MatX& W, int m, const MatX& targets, double beta, double gamma_total) {
  if (W.rows != 6) throw std::invalid_argument("wrench basis must have 6 rows");
  if (m < 1) throw std::invalid_argument("need at least one contact");
  const int n = W.cols;
  if (n % m != 0) throw std::invalid_argument("wrench basis width must split evenly across contacts");
  const int k = n / m;
  if (gamma_total > static_cast<double>(m) + 1e-12)
    throw std::invalid_argument("total-weight floor exceeds the per-contact caps; lower QP infeasible");
  if (gamma_total < 0) throw std::invalid_argument("total-weight floor must be >= 0");
  const double inf = std::numeric_limits<double>::infinity();
  const int B = targets.cols;
  SharedBatch b;
  const MatX Wt = transpose(W);
  MatX P = matmul(Wt, W);
  b.P = MatX(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) b.P(i, j) = 0.5 * (2.0 * P(i, j) + 2.0 * P(j, i));
  b.Q = MatX(n, B);
  const MatX WtT = matmul(Wt, targets);
  for (int c = 0; c < B; ++c)
    for (int i = 0; i < n; ++i) b.Q(i, c) = -2.0 * beta * WtT(i, c);
  const int rows = m + 1 + n;
  b.A = MatX(rows, n);
  b.L = MatX(rows, B);
  b.U = MatX(rows, B);
  for (int i = 0; i < m; ++i) {
    for (int j = 0; j < k; ++j) b.A(i, i * k + j) = 1.0;
    for (int c = 0; c < B; ++c) { b.L(i, c) = 0.0; b.U(i, c) = 1.0; }
  }
  for (int j = 0; j < n; ++j) b.A(m, j) = 1.0;
  for (int c = 0; c < B; ++c) { b.L(m, c) = gamma_total; b.U(m, c) = inf; }
  for (int j = 0; j < n; ++j) {
    b.A(m + 1 + j, j) = 1.0;
    for (int c = 0; c < B; ++c) { b.L(m + 1 + j, c) = 0.0; b.U(m + 1 + j, c) = inf; }
  }
  return b;
}

// qpsolve.cpp:14-25.
void check_dims(const SharedBatch& b) {
  const int n = b.P.rows, m = b.A.rows;
  if (b.P.cols != n || b.A.cols != n) throw std::invalid_argument("qp: P/A dimension mismatch");
  if (b.Q.rows != n || b.L.rows != m || b.U.rows != m)
    throw std::invalid_argument("qp: vector block dimension mismatch");
  if (b.Q.cols != b.L.cols || b.Q.cols != b.U.cols || b.Q.cols < 1)
    throw std::invalid_argument("qp: batch width mismatch");
  double asym = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) asym = std::max(asym, std::abs(b.P(i, j) - b.P(j, i)));
  if (asym > 1e-9) throw std::invalid_argument("qp: P must be symmetric");
}

// qpsolve.cpp:45-120 (OSQP-form ADMM, lockstep columns, freeze at checks).
BatchSolution solve_shared(const SharedBatch& b, const QpParams& p, const MatX* warm_x, const MatX* warm_y) {
  check_dims(b);
  const int n = b.P.rows, M = b.A.rows, B = b.Q.cols;
  const double rho = p.rho, sigma = p.sigma, alpha = p.alpha;
  const MatX At = transpose(b.A);
  MatX K = matmul(At, b.A);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) K(i, j) = b.P(i, j) + (i == j ? sigma : 0.0) + rho * K(i, j);
  MatX L;
  if (!cholesky(K, L)) throw std::invalid_argument("qp: P + sigma I + rho A'A is not positive definite");
  MatX x = warm_x ? *warm_x : MatX(n, B);
  MatX y = warm_y ? *warm_y : MatX(M, B);
  if (x.rows != n || x.cols != B || y.rows != M || y.cols != B)
    throw std::invalid_argument("qp: warm start dimension mismatch");
  MatX z = matmul(b.A, x);
  BatchSolution out;
  out.X = MatX(n, B);
  out.Z = MatX(M, B);
  out.Y = MatX(M, B);
  out.iters.assign(B, p.max_iters);
  out.converged.assign(B, 0);
  std::vector<char> frozen(B, 0);
  int n_frozen = 0;
  Stats* st = stats_sink();
  if (st) ++st->qp_solves;
  auto snapshot = [&](int c, int iter, bool ok) {
    for (int i = 0; i < n; ++i) out.X(i, c) = x(i, c);
    for (int i = 0; i < M; ++i) { out.Z(i, c) = z(i, c); out.Y(i, c) = y(i, c); }
    out.iters[c] = iter;
    out.converged[c] = ok ? 1 : 0;
  };
  MatX rhs(n, B);
  for (int iter = 1; iter <= p.max_iters; ++iter) {
    if (st) { ++st->qp_sweeps; st->qp_column_sweeps += B; }
    MatX v(M, B);
    for (int c = 0; c < B; ++c)
      for (int i = 0; i < M; ++i) v(i, c) = rho * z(i, c) - y(i, c);
    rhs = matmul(At, v);
    for (int c = 0; c < B; ++c)
      for (int i = 0; i < n; ++i) rhs(i, c) += sigma * x(i, c) - b.Q(i, c);
    MatX xt = rhs;
    chol_solve(L, xt);
    const MatX zt = matmul(b.A, xt);
    for (int c = 0; c < B; ++c) {
      for (int i = 0; i < n; ++i) x(i, c) = alpha * xt(i, c) + (1.0 - alpha) * x(i, c);
      for (int i = 0; i < M; ++i) {
        const double zbar = alpha * zt(i, c) + (1.0 - alpha) * z(i, c);
        const double zn = std::min(std::max(zbar + y(i, c) / rho, b.L(i, c)), b.U(i, c));
        y(i, c) += rho * (zbar - zn);
        z(i, c) = zn;
      }
    }
    if (iter % p.check_interval == 0 || iter == p.max_iters) {
      const MatX ax = matmul(b.A, x);
      MatX dual = matmul(b.P, x);
      const MatX aty = matmul(At, y);
      for (int c = 0; c < B; ++c) {
        if (frozen[c]) continue;
        double rp = 0.0, rd = 0.0;
        for (int i = 0; i < M; ++i) rp = std::max(rp, std::abs(ax(i, c) - z(i, c)));
        for (int i = 0; i < n; ++i) rd = std::max(rd, std::abs(dual(i, c) + aty(i, c) + b.Q(i, c)));
        if (rp <= p.eps_primal && rd <= p.eps_dual) {
          frozen[c] = 1;
          ++n_frozen;
          snapshot(c, iter, true);
        } else if (iter == p.max_iters) {
          snapshot(c, iter, false);
        }
      }
      if (n_frozen == B) break;
    }
  }
  return out;
}

// -------------------------------------------------------------- energy
// energy.cpp:49-58.
MatX closure_directions() {
  MatX d(6, 6);
  for (int axis = 0; axis < 3; ++axis) {
    d(axis, 2 * axis) = 1.0;
    d(axis, 2 * axis + 1) = -1.0;
  }
  return d;
}

// energy.cpp:60-92.
EnergyReport grasp_energy(const std::vector<Frame>& frames, double beta, double gamma_per_contact, double mu, int k,
                          const QpParams& qp, const MatX* warm_x, const MatX* warm_y, const MatX* targets) {
  const int m = static_cast<int>(frames.size());
  if (m < 1) throw std::invalid_argument("grasp energy needs at least one contact");
  const MatX dirs = targets ? *targets : closure_directions();
  const MatX W = wrench_basis(frames, mu, k);
  const SharedBatch batch = assemble_lower_qp(W, m, dirs, beta, gamma_per_contact * m);
  const BatchSolution sol = solve_shared(batch, qp, warm_x, warm_y);
  EnergyReport rep;
  rep.forces = sol.X;
  rep.duals = sol.Y;
  rep.converged = sol.converged;
  rep.iters = sol.iters;
  const int B = dirs.cols;  // closure directions (6) or caller targets (energy.cpp:66-70)
  rep.residuals = MatX(6, B);
  rep.per_direction.assign(B, 0.0);
  for (int j = 0; j < B; ++j) {
    double e = 0.0;
    for (int r = 0; r < 6; ++r) {
      double wl = 0.0;
      for (int c = 0; c < W.cols; ++c) wl += W(r, c) * sol.X(c, j);
      const double res = beta * dirs(r, j) - wl;
      rep.residuals(r, j) = res;
      e += res * res;
    }
    rep.per_direction[j] = e;
  }
  rep.total = 0.0;
  for (int j = 0; j < B; ++j) rep.total += rep.per_direction[j];
  return rep;
}

// energy.cpp:208-229.
double fine_stage_surrogate(const std::vector<V3>& points, const std::vector<V3>& anchors,
                            const std::vector<MatX>& jacobians, VecX* grad) {
  if (points.size() != anchors.size()) throw std::invalid_argument("point and anchor counts differ");
  if (!jacobians.empty() && jacobians.size() != points.size())
    throw std::invalid_argument("need one Jacobian per point when given");
  const int dims = jacobians.empty() ? 0 : jacobians[0].cols;
  if (grad) grad->assign(dims, 0.0);
  double value = 0.0;
  for (size_t i = 0; i < points.size(); ++i) {
    const V3 diff = points[i] - anchors[i];
    value += sqnorm(diff);
    if (!jacobians.empty() && grad) {
      if (jacobians[i].rows != 3 || jacobians[i].cols != dims)
        throw std::invalid_argument("point Jacobians must be 3 x dims");
      for (int c = 0; c < dims; ++c)
        (*grad)[c] += 2.0 * (jacobians[i](0, c) * diff[0] + jacobians[i](1, c) * diff[1] + jacobians[i](2, c) * diff[2]);
    }
  }
  return value;
}

// energy.cpp:94-145 (envelope gradient, lambda* fixed).
VecX grasp_energy_gradient(const std::vector<Frame>& frames, const EnergyReport& rep, double mu, int k,
                           const std::vector<MatX>& jac_p, const std::vector<MatX>& jac_n) {
  const int m = static_cast<int>(frames.size());
  const int dims = jac_p[0].cols;
  VecX grad(dims, 0.0);
  for (int i = 0; i < m; ++i) {
    const Frame& c = frames[i];
    const V3 seed = frame_seed(c.n);
    const double cnorm = norm(cross(c.n, seed));
    const M3 md = (-1.0 / cnorm) * ((M3::identity() - outer(c.d, c.d)) * skew(seed));
    const M3 me = skew(c.n) * md - skew(c.d);
    for (int j = 0; j < 6; ++j) {
      const V3 rf(rep.residuals(0, j), rep.residuals(1, j), rep.residuals(2, j));
      const V3 rt(rep.residuals(3, j), rep.residuals(4, j), rep.residuals(5, j));
      double sum = 0, sum_cos = 0, sum_sin = 0;
      V3 f;
      for (int e = 0; e < k; ++e) {
        const double th = 2.0 * std::numbers::pi * e / k;
        const double lam = rep.forces(i * k + e, j);
        sum += lam;
        sum_cos += lam * std::cos(th);
        sum_sin += lam * std::sin(th);
        f += lam * (c.n + mu * (std::cos(th) * c.d + std::sin(th) * c.e));
      }
      const V3 g = rf + cross(rt, c.p);
      const V3 an = sum * g + mu * sum_cos * (md.t() * g) + mu * sum_sin * (me.t() * g);
      const V3 ap = cross(f, rt);
      for (int col = 0; col < dims; ++col) {
        double s = 0.0;
        for (int r = 0; r < 3; ++r) s += jac_n[i](r, col) * an[r] + jac_p[i](r, col) * ap[r];
        grad[col] -= 2.0 * s;
      }
    }
  }
  return grad;
}

}  // namespace oracle

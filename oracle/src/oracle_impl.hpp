// ORACLE (test infrastructure only). fp64 CPU restatement of the reference
// hot path, /root/reference/proj/src/{geometry,hand,contact,qpsolve,energy,pipeline}.cpp.
// Every function cites the reference lines it follows. Consumed only by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference.
#pragma once

#include "dense.hpp"

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

struct GeometryError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Part {
  std::vector<V3> verts;
  std::vector<std::array<int, 3>> faces;
  V3 obb_center, obb_half;
  M3 obb_rot;
  V3 centroid;
  double volume = 0.0;
};

struct Proxy {
  V3 c;
  double r = 0.0;
};

struct Link {
  int parent_joint = -1;
  int tip_proxy = -1;
  Part part;
  std::vector<Proxy> proxies;
};

struct Joint {
  int parent_link = -1, child_link = -1;
  V3 origin, axis;
  double lower = 0.0, upper = 0.0;
};

struct Hand {
  std::vector<Link> links;
  std::vector<Joint> joints;
  std::vector<int> tips;
  std::vector<std::pair<int, int>> pairs;
  int dof() const { return static_cast<int>(joints.size()); }
  int dims() const { return 12 + dof(); }
};

struct Object {
  std::vector<Part> parts;
};

// Op counters for the roofline's algorithmic-flop formula.
struct Stats {
  long long point_queries = 0, inside_faces = 0, outside_faces = 0;
  long long gjk_calls = 0, gjk_iters = 0, gjk_support_verts = 0;
  long long epa_calls = 0, epa_iters = 0, epa_face_scans = 0;
  long long qp_solves = 0, qp_sweeps = 0, qp_column_sweeps = 0;
  long long jacobians = 0, self_pairs = 0, obb_tests = 0;
  void add(const Stats& o);
};
Stats* stats_sink();  // thread-local accumulator (nullptr = off)
void set_stats_sink(Stats* s);

// ---- geometry (geometry.cpp) ------------------------------------------
struct Nearest {
  V3 a, b;
  double distance = 0.0;
  V3 normal = V3(0, 0, 1);
  int part = -1;
};
Nearest point_to_mesh(const V3& p, const std::vector<Part>& parts);
double signed_distance(const Part& a, const Rigid& pa, const Part& b, const Rigid& pb, Nearest* out, bool* used_epa);
Nearest gjk_distance(const Part& a, const Rigid& pa, const Part& b, const Rigid& pb);
std::pair<double, V3> epa_depth(const Part& a, const Rigid& pa, const Part& b, const Rigid& pb);
double obb_sphere_distance(const Part& part, const V3& center, double radius);
std::vector<int> broadphase_cull(const V3& center, double radius, const std::vector<Part>& parts, double reference);

// ---- kinematics (hand.cpp) --------------------------------------------
struct PoseState {
  M3 raw, R, a_inv;
  bool degenerate = false;
};
M3 project_rotation(const M3& raw, bool* fallback);
PoseState make_pose_state(const M3& raw);
struct Pose {
  M3 R;
  V3 t;
  VecX q;
};
struct Fk {
  std::vector<Rigid> chain, world;
  std::vector<V3> joint_origin, joint_axis;
};
M3 raw_block(const VecX& x);
Pose pose_from_state(const Hand& h, const VecX& x);
Fk forward_kinematics(const Hand& h, const Pose& pose);
MatX point_jacobian(const Hand& h, const PoseState& ps, const Pose& pose, const Fk& fk, int link, const V3& pw);
MatX direction_jacobian(const Hand& h, const PoseState& ps, const Pose& pose, const Fk& fk, int link, const V3& dw);
void tangent_jacobian(const PoseState& ps, double J[3][9]);  // hand.cpp:97-106
double limit_energy(const Hand& h, const Pose& pose, VecX* grad);
double self_penetration_energy(const Hand& h, const PoseState& ps, const Pose& pose, const Fk& fk, VecX* grad);

// ---- contact / QP / energy (contact.cpp, qpsolve.cpp, energy.cpp) -----
struct Frame {
  V3 p, n, d, e;
};
V3 frame_seed(const V3& n);
Frame build_frame(const V3& p, const V3& n);
MatX wrench_basis(const std::vector<Frame>& frames, double mu, int k);

struct QpParams {
  double rho = 0.1, sigma = 1e-6, alpha = 1.6;
  int max_iters = 500;
  double eps_primal = 1e-5, eps_dual = 1e-5;
  int check_interval = 10;
};
struct SharedBatch {
  MatX P, A, Q, L, U;
};
struct BatchSolution {
  MatX X, Z, Y;
  std::vector<int> iters;
  std::vector<char> converged;
};
SharedBatch assemble_lower_qp(const MatX& W, int m, const MatX& targets, double beta, double gamma_total);
BatchSolution solve_shared(const SharedBatch& b, const QpParams& p, const MatX* warm_x, const MatX* warm_y);

struct EnergyReport {
  double total = 0.0;
  VecX per_direction;
  MatX forces, residuals, duals;
  std::vector<char> converged;
  std::vector<int> iters;  // per-column sweep count at the freeze (qpsolve.cpp:99-117)
};
MatX closure_directions();
EnergyReport grasp_energy(const std::vector<Frame>& frames, double beta, double gamma_per_contact, double mu, int k,
                          const QpParams& qp, const MatX* warm_x, const MatX* warm_y,
                          const MatX* targets = nullptr);
double fine_stage_surrogate(const std::vector<V3>& points, const std::vector<V3>& anchors,
                            const std::vector<MatX>& jacobians, VecX* grad);
VecX grasp_energy_gradient(const std::vector<Frame>& frames, const EnergyReport& rep, double mu, int k,
                           const std::vector<MatX>& jac_p, const std::vector<MatX>& jac_n);

// ---- pipeline (pipeline.cpp) -------------------------------------------
struct Stage {
  int iters = 300;
  double step_rotation = 0.010, step_translation = 0.0025, step_joints = 0.010, step_floor = 0.1;
};
struct Config {
  QpParams qp;
  double mu = 0.6;
  int n_edges = 8;
  double beta = 10.0, gamma_per_contact = 0.1;
  double w_grasp = 1.0, w_distance = 100.0, w_limit = 10.0, w_self = 10.0, w_pen = 10.0;
  Stage coarse{300, 0.010, 0.0025, 0.010, 0.1};
  Stage fine{100, 0.004, 0.0010, 0.004, 0.1};
  Stage final_stage{100, 0.004, 0.0010, 0.004, 0.1};
  double contact_offset = 0.01, fd_step = 1e-6;
  bool skip_fine = false;
};

struct Witness {
  V3 c_w, p_w, n = V3(0, 0, 1);
  double distance = 0.0;
  int link = -1;
};
std::vector<Witness> fine_contact_query(const Hand& h, const Fk& fk, const Object& obj);

// ---- eval (eval.cpp:51-158) --------------------------------------------
struct EvalParams {
  double mass = 0.03, gravity = 9.8, residual_rel_tol = 1e-3, force_budget_factor = 20.0;
  double contact_tol = 0.002, penetration_tol = 0.003, qp_eps = 1e-8;
};
struct EvalResult {
  bool success = false;
  double residuals[6] = {0, 0, 0, 0, 0, 0};
  double pd_mm = 0.0, spd_mm = 0.0, cdc_mm = 0.0;
  int contact_count = 0;
  int note_flags = 0;  // 1 no contacts, 2 qp unconverged, 4 residual, 8 < 2 contacts, 16 penetration
};
double penetration_depth(const Hand& h, const VecX& x, const Object& obj);
double self_penetration_depth(const Hand& h, const VecX& x);
double contact_distance_consistency(const Hand& h, const VecX& x, const Object& obj);
struct Config;
EvalResult quasi_static_check(const Hand& h, const Object& obj, const Config& cfg, const EvalParams& ep,
                              const VecX& x, const VecX& x_s);

struct QpScratch {
  MatX forces, duals;
  bool ready = false;
  std::vector<int> iters;        // last solve's per-column sweep counts (instrumentation)
  std::vector<char> converged;
};
// stage: 0 coarse, 1 fine, 2 final
double total_energy(const Hand& h, const Object& obj, const Config& cfg, int stage, const std::vector<V3>& anchors,
                    const VecX& x, QpScratch& scratch, VecX* grad);
// Test-only teacher forcing: world link transforms for this thread's next
// pose_hand calls ([L*12] R column-major, t), nullptr = own FK.
void set_world_override(const double* world);
void apply_step(const Hand& h, const Stage& s, int it, const VecX& grad, VecX& x);
double coarse_distance_energy(const Hand& h, const VecX& x, const Object& obj, double offset, double fd, VecX* grad);

struct Record {
  VecX x_p, x, x_s;
  double energy_total = 0.0;
  VecX per_direction;
  MatX forces;
  std::vector<Frame> contacts;
  std::vector<char> converged;
  int failed = 0;  // 0 ok, 1 non-finite energy, 2 diverged
  double stage_energy[3][2];
};
VecX squeeze_pose(const Hand& h, const VecX& x, const VecX& xp);
Record run_grasp(const Hand& h, const Object& obj, const Config& cfg, const VecX& x0);

}  // namespace oracle

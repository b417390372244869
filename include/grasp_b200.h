/*
 * grasp_b200.h -- C ABI of the B200-native bilevel grasp-synthesis engine.
 *
 * The reference (arxiv 2412.16490, /root/reference/proj) is a static C++20
 * library, not a plugin: its hot path is
 *   grasp::pipeline::synthesize(const HandModel&, const ObjectModel&, const RunConfig&)
 *   (proj/include/grasp/pipeline.hpp:69-71, proj/src/pipeline.cpp:436-457).
 * This header is the thin, exception-free boundary a foreign caller binds
 * (ctypes / cgo / JNI); the C++ API in paper_2412_16490_b200/csrc/include/grasp/
 * keeps the reference's names and types on top of it.
 *
 * Conventions: plain pointers and sizes, fp64 everywhere (the reference's
 * arithmetic type), caller-owned outputs, int status (0 = ok). On failure
 * grasp_last_error() returns a thread-local message. Nothing here throws.
 */
#ifndef GRASP_B200_H
#define GRASP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------- */
#define GRASP_OK 0
#define GRASP_EINVAL 1 /* std::invalid_argument in the reference (validate, QP/energy checks) */
#define GRASP_EGEOM 2  /* geom::GeometryError (geometry.hpp:64-66) */
#define GRASP_EHAND 3  /* hand::HandError (hand.hpp:134-136) */
#define GRASP_EOBJECT 4 /* object::ObjectError (object.hpp:27-29) */
#define GRASP_ECUDA 5  /* device/driver failure (no reference analogue) */
#define GRASP_ENOMEM 6

/* Per-grasp failure codes (data, not errors; pipeline.cpp:264-277). */
#define GRASP_OK_GRASP 0
#define GRASP_FAIL_NONFINITE 1 /* note "non-finite energy" */
#define GRASP_FAIL_DIVERGED 2  /* note "diverged" */

const char* grasp_last_error(void);
const char* grasp_version(void);

/* ---- host models (load-time, C++) ------------------------------------- */
typedef struct grasp_hand grasp_hand;
typedef struct grasp_object grasp_object;

/* hand::builtin_hand() (hand.hpp:141-143). Returned handle is owned by the caller. */
int grasp_hand_builtin(grasp_hand** out);
/* hand::parse_hand_spec(json) (hand.hpp:139). */
int grasp_hand_parse(const char* json_text, grasp_hand** out);
void grasp_hand_free(grasp_hand* h);
/* Copies hand::builtin_hand_json() into buf (returns the required size incl. NUL). */
int64_t grasp_hand_builtin_json(char* buf, int64_t cap);

/* object::make_primitive(name, scale) (object.hpp:45). */
int grasp_object_primitive(const char* name, double scale, grasp_object** out);
/* object::parse_object_text(text, scale, source) (object.hpp:41-42). */
int grasp_object_parse(const char* obj_text, double scale, const char* source, grasp_object** out);
/* Raw convex parts via geom::make_convex_part (geometry.cpp:414-466), no
 * normalization or recentering: counts[n_parts], points[sum(counts)*3]. */
int grasp_object_from_points(int n_parts, const int* counts, const double* points, grasp_object** out);
void grasp_object_free(grasp_object* o);
double grasp_object_bounding_radius(const grasp_object* o);
/* geom::make_convex_part for many point clouds on the device (
 * geometry.cpp:414-466 with the quickhull of hull3d.cpp:291-303), one thread
 * per part, bit-identical to the host builder (grasp_object_from_points).
 * Part p's points are points[3 * point_begin[p] .. 3 * point_begin[p + 1]).
 * Outputs per part p: out_n_verts[p] hull vertices at out_verts[3 *
 * point_begin[p] ...], out_n_faces[p] faces (local vertex triples) at
 * out_faces[6 * point_begin[p] ...] (room for 2 faces per point),
 * out_volume[p], out_centroid[3p..], out_obb[15p..] (center, half extents,
 * rotation column-major), out_status[p] (0 ok, 1 degenerate: fewer than 4
 * non-coplanar points or non-positive volume, 2 workspace overflow). */
int grasp_build_convex_parts(int device, const double* points, const int* point_begin, int n_parts, double merge_tol,
                             double* out_verts, int* out_n_verts, int* out_faces, int* out_n_faces,
                             double* out_volume, double* out_centroid, double* out_obb, int* out_status);

/* Packed, read-only views of a model (pointers stay valid while the handle lives). */
typedef struct grasp_hand_desc {
  int n_links, dof, n_tips, n_proxies, n_pairs, n_verts, n_faces;
  const int* link_parent_joint; /* [n_links], -1 for the base */
  const int* link_tip_proxy;    /* [n_links], index into the link's proxies or -1 */
  const int* link_vert_begin;   /* [n_links+1] */
  const int* link_face_begin;   /* [n_links+1] */
  const int* link_proxy_begin;  /* [n_links+1] */
  const double* verts;          /* [n_verts*3] link-local hull vertices */
  const int* faces;             /* [n_faces*3] indices local to the link's vertex range */
  const double* link_obb;       /* [n_links*15] center(3) half_extents(3) rotation(9, column-major) */
  const double* link_centroid;  /* [n_links*3] */
  const double* link_volume;    /* [n_links] */
  const double* proxies;        /* [n_proxies*4] center_local(3), radius */
  const int* joint_parent_link; /* [dof] */
  const int* joint_child_link;  /* [dof] */
  const double* joint_origin;   /* [dof*3] parent frame */
  const double* joint_axis;     /* [dof*3] unit, child frame */
  const double* joint_lower;    /* [dof] */
  const double* joint_upper;    /* [dof] */
  const int* tip_links;         /* [n_tips] = fingertip_links */
  const int* collision_pairs;   /* [n_pairs*2] */
} grasp_hand_desc;

typedef struct grasp_object_desc {
  int n_parts, n_verts, n_faces;
  const int* part_vert_begin;   /* [n_parts+1] */
  const int* part_face_begin;   /* [n_parts+1] */
  const double* verts;          /* [n_verts*3] object frame */
  const int* faces;             /* [n_faces*3] indices local to the part's vertex range */
  const double* part_obb;       /* [n_parts*15] */
  const double* part_centroid;  /* [n_parts*3] */
  const double* part_volume;    /* [n_parts] */
  double scale;
  double bbox_diagonal;
  double mass_center[3];
  const char* source;
} grasp_object_desc;

int grasp_hand_describe(const grasp_hand* h, grasp_hand_desc* out);
int grasp_object_describe(const grasp_object* o, grasp_object_desc* out);

/* ---- run configuration (config.hpp:8-88; same fields, same defaults) --- */
typedef struct grasp_stage_params {
  int iters;
  double step_rotation, step_translation, step_joints, step_floor;
} grasp_stage_params;

typedef struct grasp_run_params {
  /* QpParams */
  double qp_rho, qp_sigma, qp_alpha;
  int qp_max_iters;
  double qp_eps_primal, qp_eps_dual;
  int qp_check_interval;
  /* ContactParams */
  double mu;
  int n_edges;
  /* EnergyParams */
  double beta, gamma_per_contact;
  /* ObjectiveWeights */
  double w_grasp, w_distance, w_joint_limit, w_self_penetration, w_object_penetration;
  /* PipelineParams */
  grasp_stage_params coarse, fine, final_stage;
  double contact_offset, fd_step;
  int skip_fine_stages;
  /* InitParams */
  double standoff, joint_span_fraction;
  /* run */
  uint64_t seed;
  int batch;
  int workers;
} grasp_run_params;

/* Fills the reference defaults (config.hpp:9-87). */
void grasp_run_params_default(grasp_run_params* p);
/* parse_run_config(json) -> params (strict: unknown keys rejected). */
int grasp_run_params_parse(const char* json_text, grasp_run_params* out);
/* validate(cfg) (config.cpp:196-229). */
int grasp_run_params_validate(const grasp_run_params* p);

/* init_poses(model, object, n, seed, init) (pipeline.cpp:388-424): out[n*D]. */
int grasp_init_poses(const grasp_hand* h, const grasp_object* o, int n, uint64_t seed, double standoff,
                     double joint_span_fraction, double* out);
/* squeeze_pose(model, x, x_p) (pipeline.cpp:426-434): out[D]. */
int grasp_squeeze_pose(const grasp_hand* h, const double* x, const double* x_p, double* out);
/* forward_kinematics(model, pose_from_state(model, x)) (hand.hpp:100, hand.cpp:126-153) for n
 * states x[n*D]: world link transforms out[n*n_links*12] = R (9, column-major), t (3). Host. */
int grasp_forward_kinematics(const grasp_hand* h, int n, const double* x, double* out);

/* ---- device engine ------------------------------------------------------ */
typedef struct grasp_ctx grasp_ctx;

/* One context drives one CUDA device on one stream. */
int grasp_ctx_create(int device, grasp_ctx** out);
/* A context over several devices: models are uploaded to every
 * device, and grasp_synthesize splits the batch into contiguous shards
 * [k*B/n, (k+1)*B/n), each run by its own host thread and stream, writing its
 * rows of the caller's outputs (results equal the single-device run's).
 * Repeated device ids are allowed (several streams on one GPU). The other
 * entry points use the first device; grasp_synthesize_device is single-device only. */
int grasp_ctx_create_devices(const int* devices, int n, grasp_ctx** out);
void grasp_ctx_destroy(grasp_ctx* ctx);
/* Uploads the packed hand / object (replaces any previous one). */
int grasp_ctx_set_hand(grasp_ctx* ctx, const grasp_hand_desc* hand);
int grasp_ctx_set_object(grasp_ctx* ctx, const grasp_object_desc* object);

/* Several objects in one context (object.hpp:19-25): their convex parts are
 * packed back to back on the device, replacing the context's object(s).
 * grasp_ctx_set_object(ctx, o) is grasp_ctx_set_objects(ctx, 1, &o). */
int grasp_ctx_set_objects(grasp_ctx* ctx, int n, const grasp_object_desc* const* objects);

/* Caller-owned per-grasp outputs of synthesize (records.hpp:29-44 as SoA).
 * D = 12 + dof, m = n_tips, n = m * n_edges. Any pointer may be NULL. */
typedef struct grasp_out {
  double* x_p;            /* [batch*D] */
  double* x;              /* [batch*D] */
  double* x_s;            /* [batch*D] */
  double* energy_total;   /* [batch] NaN if failed */
  double* per_direction;  /* [batch*6] */
  double* contact_forces; /* [batch*n*6] per grasp column-major (n x 6) */
  double* contacts;       /* [batch*m*12] per contact p(3) n(3) d(3) e(3) */
  double* stage_energy;   /* [batch*3*2] (energy_start, energy_end) per stage, NaN if skipped */
  int* failed;            /* [batch] GRASP_OK_GRASP / GRASP_FAIL_* */
  int* qp_converged;      /* [batch*6] final-record QP convergence flags */
} grasp_out;

/* synthesize over grasps [0, batch) whose start states x0[batch*D] the
 * caller produced with grasp_init_poses (the reference's single RNG stream).
 * Per-grasp failure is reported in out->failed, never as an error. */
int grasp_synthesize(grasp_ctx* ctx, const grasp_run_params* p, int batch, const double* x0, grasp_out* out);

/* One synthesis over grasps of several objects (the objects of grasp_ctx_set_objects):
 * grasp g grasps object object_index[g] from start state x0[g] (grasp_init_poses of that
 * object). Every kernel launch covers the whole batch; each record equals the one a
 * single-object grasp_synthesize of that grasp gives. Single-device contexts only. */
int grasp_synthesize_objects(grasp_ctx* ctx, const grasp_run_params* p, int batch, const double* x0,
                             const int* object_index, grasp_out* out);

/* Same, but x0 and every output pointer are DEVICE pointers on ctx's device
 * (no host copies; used to time the kernels with inputs resident in HBM). */
int grasp_synthesize_device(grasp_ctx* ctx, const grasp_run_params* p, int batch, const double* x0_dev,
                            grasp_out* out_dev);

/* Batched lower-level QP, the config-5 micro-bench surface
 * (energy.cpp:60-92 -> qpsolve.cpp:45-120, 193-235): one 6-column batch per
 * grasp built from m contact frames (frames[g*m*12]: p n d e), cold start
 * unless warm_x/warm_y are given ([g*n*6], [g*M*6], M = m + 1 + n).
 * Outputs: X[g*n*6], Y[g*M*6], Z[g*M*6], iters[g*6], converged[g*6],
 * per_direction[g*6]. Device or host pointers per `device_ptrs`. */
int grasp_qp_batch(grasp_ctx* ctx, const grasp_run_params* p, int n_grasps, int m, const double* frames,
                   const double* warm_x, const double* warm_y, double* X, double* Y, double* Z, int* iters,
                   int* converged, double* per_direction, int device_ptrs);

/* ---- evaluation (eval.cpp:51-158) ------------------ */
typedef struct grasp_eval_params {
  double mass, gravity, residual_rel_tol, force_budget_factor, contact_tol, penetration_tol, qp_eps;
} grasp_eval_params;
/* EvalParams{} defaults (config.hpp:66-74). */
void grasp_eval_params_default(grasp_eval_params* e);
/* quasi_static_check(model, {x, x_s}, object, cfg) (eval.cpp:91-158) for n grasps on the
 * device: penetration_depth over every (link, part) pair, self_penetration_depth over the
 * collision pairs, contact_distance_consistency of the fingertip witnesses at x, and the six
 * gravity-resistance QPs on the witnesses within contact_tol at x_s. out_real[n*9] = pd_mm,
 * spd_mm, cdc_mm, per_direction_residuals[6]; out_int[n*3] = contact_count, success,
 * note flags (1 no contacts, 2 resistance qp unconverged, 4 gravity residual above
 * tolerance, 8 fewer than two contacts, 16 penetration above tolerance). */
int grasp_eval(grasp_ctx* ctx, const grasp_run_params* p, const grasp_eval_params* e, int n, const double* x,
               const double* x_s, double* out_real, int* out_int);

/* ---- teacher-forced surfaces (parity tests call the kernels piecewise) -- */
/* point_to_mesh(p, object.parts) for n points: out[n*8] = distance, point_b(3),
 * normal(3), part_index (geometry.cpp:527-542). */
int grasp_point_to_mesh(grasp_ctx* ctx, int n, const double* points, double* out);
/* signed_distance(link part, pose, object part, identity) for n pairs
 * (geometry.cpp:500-525): poses[n*12] = R(9, column-major) t(3);
 * out[n*11] = distance, point_a(3), point_b(3), normal(3), epa_flag. */
int grasp_signed_distance(grasp_ctx* ctx, int n, const int* link_ids, const int* part_ids, const double* poses,
                          double* out);
/* total_energy(x) with gradient for each grasp, stage 0 = coarse (spheres,
 * QP warm-started from warm_x/warm_y which are updated in place, pass
 * NULL for cold), 1 = fine, 2 = final (anchors[g*m*3] used).
 * (pipeline.cpp:96-210). energy[g], grad[g*D]. */
int grasp_total_energy(grasp_ctx* ctx, const grasp_run_params* p, int stage, int n, const double* x,
                       const double* anchors, double* warm_x, double* warm_y, double* energy, double* grad);
/* forward_kinematics(pose_from_state(x)) on the device, the FK every iteration of
 * synthesize runs (hand.cpp:108-153): out[n*n_links*12] = R (9, column-major), t (3). */
int grasp_device_forward_kinematics(grasp_ctx* ctx, int n, const double* x, double* out);
/* fine_contact_query(model, fk, object) (pipeline.hpp:32-34) from given world link
 * transforms world[n*n_links*12] (R column-major, t), e.g. a host FkResult: out as below. */
int grasp_fine_contact_query_world(grasp_ctx* ctx, int n, const double* world, double* out);
/* fine_contact_query at states x (pipeline.cpp:320-353): out[g*m*11] =
 * c_w(3) p_w(3) n(3) distance link. */
int grasp_fine_contact_query(grasp_ctx* ctx, int n, const double* x, double* out);

/* ---- instrumentation (bench.py; not part of the reference API) ---------- */
/* The cudaStream_t the context launches on (for CUDA-event timing). */
void* grasp_ctx_stream(grasp_ctx* ctx);
/* Enables per-kernel-class CUDA-event timing and algorithmic op counters;
 * resets the accumulators. Classes: 0 point_query, 1 qp, 2 step_coarse,
 * 3 pairs, 4 step_mesh, 5 fk, 6 finalize, 7 pairs_big. Ops: 0 plane tests,
 * 1 triangle tests, 2 ADMM column-sweeps, 3 QP solves, 4 GJK iterations,
 * 5 support vertices scanned, 6 EPA iterations, 7 point queries, 8 pairs
 * not culled, 9 EPA overflows. */
int grasp_ctx_set_profiling(grasp_ctx* ctx, int on);
int grasp_ctx_profile(grasp_ctx* ctx, double* ms /*[8]*/, long long* launches /*[8]*/,
                      unsigned long long* ops /*[20]*/);
/* Engine options (defaults are the product settings; results never depend on
 * them except "pair_cull"): "query_buckets" (1: the coarse stage's point
 * queries listed by spatial bucket, 0: slot order), "query_lanes" (lanes per
 * point query in all-slot launches, 1 = thread per query; 2..32) and
 * "tip_query_lanes" (tip-only launches, default 4), "pair_cull" (0: every
 * (link, part) pair through GJK like the reference; 1: the opt-in separation
 * cull, exact for the true geometry only) with "pair_sat" (its
 * link-box vs part-box test, default 1), "pair_early" (pairs whose last EPA
 * ran more than this many iterations run GJK + EPA on a side stream next to
 * the GJK pass; default 24, >= 255 off), "graphs" (1: a synthesis runs as a
 * captured CUDA graph, cached per models, buffers and parameters; 0, the
 * default: eager launches, better when several contexts share a device).
 * GRASP_EINVAL for unknown names. */
int grasp_ctx_set_option(grasp_ctx* ctx, const char* name, int value);

/* Kernels launched by synthesis on this context so far (every kernel, all of
 * a launch group: the pair pass counts its six kernels). */
long long grasp_ctx_launch_count(grasp_ctx* ctx);

/* Per-iteration trace of the next grasp_synthesize* calls (teacher-forced parity:
 * the reference's run_grasp loop, pipeline.cpp:254-281, restarted from any
 * recorded state). Snapshot k is taken at iteration iter[k] of stage stage[k]
 * (0 coarse, 1 fine, 2 final) for every grasp of the batch: the iteration's
 * inputs before it runs (x_in, the device FK of x_in, the QP warm start and its
 * ready flag, the anchors) and its outputs after the step (total_energy and its
 * gradient, the stepped state, the QP snapshot and per-column sweep counts /
 * convergence flags of that iteration's lower QP, the failure code). Buffers
 * are HOST memory, snapshot-major ([n_snap][batch][...]), any may be NULL, and
 * must stay valid until the synthesize call returns. Snapshots of grasps that
 * failed earlier hold stale values (check `failed`). D = 12 + dof,
 * n = m * n_edges, M = m + 1 + n. */
typedef struct grasp_trace {
  int n_snap;
  const int* stage;   /* [n_snap] */
  const int* iter;    /* [n_snap] */
  double* x_in;       /* [n_snap*batch*D] */
  double* world_in;   /* [n_snap*batch*n_links*12] R (9, row-major: the device layout), t (3) */
  double* warm_x_in;  /* [n_snap*batch*n*6] column-major n x 6 */
  double* warm_y_in;  /* [n_snap*batch*M*6] */
  int* warm_ready_in; /* [n_snap*batch] */
  double* anchors;    /* [n_snap*batch*m*3] */
  double* energy;     /* [n_snap*batch] */
  double* grad;       /* [n_snap*batch*D] */
  double* x_out;      /* [n_snap*batch*D] */
  double* warm_x_out; /* [n_snap*batch*n*6] */
  double* warm_y_out; /* [n_snap*batch*M*6] */
  int* qp_iters;      /* [n_snap*batch*6] */
  int* qp_converged;  /* [n_snap*batch*6] */
  int* failed;        /* [n_snap*batch] */
} grasp_trace;
/* Arms (trace != NULL, copied) or disarms (NULL) the trace. */
int grasp_ctx_set_trace(grasp_ctx* ctx, const grasp_trace* trace);
/* Measured dense fp64 FMA throughput of the device (TFLOP/s). */
int grasp_measure_fp64_peak(int device, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* GRASP_B200_H */

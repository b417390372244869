// Device-resident hand / object / run parameters and per-grasp state layout.
#pragma once

#include <cstdint>

namespace gdev {

constexpr int kMaxLinks = 32;    // one lane per link in the warp-per-grasp kernels
constexpr int kMaxDof = 32;
constexpr int kMaxTips = 5;      // QP lanes = 6 directions x tips <= 30
constexpr int kMaxEdges = 8;
constexpr int kMaxDims = 12 + kMaxDof;
constexpr int kMaxDepth = 12;    // kinematic chain depth
constexpr int kMaxProxies = 128;
constexpr int kMaxParts = 64;

// Object face record for point queries (query_part, geometry.cpp:355-395):
// a, b, c vertices, unit normal n (cross/len as the reference forms it),
// nd = n.a, valid = (len >= 1e-30). 16 doubles = 128 B per face.
constexpr int kFaceStride = 16;

// Absolute slack on every conservative culling bound (metres). Bounds are
// computed in fp64 from quantities of size ~0.1-1, so their rounding error is
// ~1e-16; the slack only has to dominate that.
constexpr double kCullSlack = 1e-9;

struct DevHand {
  int L, dof, m, S, nsp, D;
  int cull;                         // opt-in (option "pair_cull") separation cull of (link, part) pairs, see pair_needed
  const int* link_parent_joint;     // [L]
  const int* link_depth;            // [L] path length root..l
  const int* link_path;             // [L*kMaxDepth] links from root to l
  const int* joint_parent_link;     // [dof]
  const double* joint_origin;       // [dof*3]
  const double* joint_axis;         // [dof*3]
  const double* joint_lower;        // [dof]
  const double* joint_upper;        // [dof]
  const unsigned* joint_subtree;    // [dof] bitmask of links moved by the joint
  const double* proxy;              // [S*4] center_local, radius
  const int* proxy_link;            // [S]
  const int* tip_link;              // [m]
  const int* tip_proxy;             // [m] global proxy index
  const double* tip_envelope;       // [m] envelope_radius (pipeline.cpp:47-52)
  int ncp;                          // collision link pairs (eval self-penetration depth)
  const int* cp_a;                  // [ncp]
  const int* cp_b;
  const int* sp_a;                  // [nsp] self-penetration proxy pairs, reference order
  const int* sp_b;
  const int* link_vbeg;             // [L+1]
  const double* link_verts;         // [nv*3]
  const double* link_centroid;      // [L*3]
  const double* link_halfnorm;      // [L] |obb.half_extents|
  const int* link_tip;              // [L] fingertip index of the link, -1 if none
  const double* link_bsphere;       // [L*4] bounding sphere of the link hull (link frame): center, radius
  const double* link_box;           // [L*15] box containing the link hull (link frame): center, half, axes (col-major)
  const int* link_cm;               // [L] base of the link hull's support map in cm_off, -1 = full scan
  const int* cm_off;                // support-map cell offsets into cm_idx (kSupportCells + 1 per map)
  const unsigned short* cm_idx;     // candidate vertex indices per cell, ascending
};

struct DevObject {
  int P, F;                   // parts and faces of all objects in the context
  int NO, Pmax;               // objects; most parts of one object (pair-slot stride per link)
  const int* obj_pbeg;        // [NO+1] first part of each object
  const int* part_fbeg;       // [P+1]
  const int* part_vbeg;       // [P+1]
  const double* faces;        // [F*kFaceStride]
  const double* verts;        // [nv*3]
  const double* part_centroid;  // [P*3]
  const double* part_halfnorm;  // [P]
  const double* part_obb;       // [P*15] center, half, rotation (column-major)
  const double* part_sphere;    // [P*4] bounding sphere of the part: center, radius
  const double* part_box;       // [P*15] box containing the part hull: center, half, axes (col-major)
  const double* face_sphere;    // [F*4] bounding sphere of each triangle: center, radius
  // Point-query order: within each part the faces are permuted into spatially
  // compact runs (engine.cu set_object); face_sphere32, face_box32, the
  // clusters and pq_faces are indexed by position, pq_fid maps a position to
  // the face index (the scans compare (distance, face index) pairs).
  const double* pq_faces;       // [F*kFaceStride] face records in point-query order
  const int* pq_fid;            // [F] face index of each position
  const float4* face_sphere32;  // [F] (point-query order) face spheres in fp32, radius rounded up (culling bounds only)
  const double4* face_plane;    // [F] (n, n.a) in fp64; degenerate faces (0, 0, 0, +inf)
  const float4* face_box32;     // [4F] (point-query order) thin box per face: (o, hu), (u, hv), (v, hn), (n, 0); fp32, bounds only
  const int* part_cbeg;         // [P+1] face clusters of each part
  const int* cluster_fbeg;      // [NC+1] first position of each cluster (point-query order)
  const float4* cluster_sphere32;  // [NC] fp32 sphere bounding the cluster's face spheres
  const float4* cluster_box32;     // [NC*4] fp32 oriented box of the cluster's vertices (face-box layout)
  const int* part_cm;              // [P] base of the part hull's support map in cm_off, -1 = full scan
  const int* cm_off;
  const unsigned short* cm_idx;
  int NC;                          // face clusters
  const int* face_cluster;         // [F] cluster of each face (point-query bucketing)
  // Plane groups (inside test): each part's non-degenerate face planes grouped
  // by normal direction, with a lower bound on the group's plane depths;
  // groups of neighbouring directions form super-groups with their own bound.
  const int* part_gbeg;            // [P+1] plane super-groups of each part
  const int* sup_gbeg;             // [NS+1] first group of each super-group
  const float4* sup_bound;         // [NS*2] super-group bounds (grp_bound layout)
  const int* grp_beg;              // [NG+1] first entry of each group in grp_plane / grp_face
  const float4* grp_bound;         // [NG*2] (n_g, h_g), (C_g, delta_g): fp32, h_g <= min (w_f - n_f.C_g), delta_g >= max |n_f - n_g|
  const double4* grp_plane;        // planes in group order (copies of face_plane)
  const int* grp_face;             // face index of each entry
};


// Support maps (cube map of directions -> candidate support vertices). A hull
// with at least kSupportMapMinVerts vertices gets, for each of the 6 * N * N
// cells of a cube map of directions, the ascending list of every vertex that
// can be the fp64-computed argmax of dir . v for some direction in the cell
// (exclusion needs a provable margin over the rounding of the dot products),
// so scanning the list in index order returns exactly the full scan's first
// maximum (geometry.cpp:399-412). Built on the host at upload.
#ifndef GDEV_SUPPORT_MAP_N
#define GDEV_SUPPORT_MAP_N 16
#endif
#ifndef GDEV_SUPPORT_MAP_MIN_VERTS
#define GDEV_SUPPORT_MAP_MIN_VERTS 24
#endif
constexpr int kSupportMapN = GDEV_SUPPORT_MAP_N;
#ifndef GDEV_PQ_REBUCKET
#define GDEV_PQ_REBUCKET 4
#endif
constexpr int kPqRebucket = GDEV_PQ_REBUCKET;  // coarse point-query list rebuilt every this many iterations
constexpr int kSupportCells = 6 * kSupportMapN * kSupportMapN;
constexpr int kSupportMapMinVerts = GDEV_SUPPORT_MAP_MIN_VERTS;

// Cell of direction d: face = dominant axis and sign (x+, x-, y+, y-, z+, z-),
// (u, v) = the other two components in axis order over |d_face|, binned in
// [-1, 1]. Returns -1 for zero, tiny, huge or NaN directions (full scan).
__host__ __device__ __forceinline__ int support_cell(double dx, double dy, double dz) {
  const double ax = fabs(dx), ay = fabs(dy), az = fabs(dz);
  int face;
  double m, pu, pv;
  if (ax >= ay && ax >= az) {
    face = dx >= 0 ? 0 : 1;
    m = ax, pu = dy, pv = dz;
  } else if (ay >= az) {
    face = dy >= 0 ? 2 : 3;
    m = ay, pu = dx, pv = dz;
  } else {
    face = dz >= 0 ? 4 : 5;
    m = az, pu = dx, pv = dy;
  }
  if (!(m > 1e-200 && m < 1e200)) return -1;
  const double sc = 0.5 * kSupportMapN / m;
  int iu = (int)((pu + m) * sc), iv = (int)((pv + m) * sc);
  iu = iu < 0 ? 0 : (iu >= kSupportMapN ? kSupportMapN - 1 : iu);
  iv = iv < 0 ? 0 : (iv >= kSupportMapN ? kSupportMapN - 1 : iv);
  return (face * kSupportMapN + iv) * kSupportMapN + iu;
}

#ifndef GDEV_FACE_CLUSTER
#define GDEV_FACE_CLUSTER 8  // with the spatial face order: 8: 150, 16: 153, 32: 165 ms point queries
#endif
constexpr int kFaceCluster = GDEV_FACE_CLUSTER;  // faces per point-query cluster

// Slack on the fp32 culling bounds: fp32 distances of <= 1 m carry < 1e-7 m
// rounding error, so 1e-5 m keeps every bound conservative.
constexpr float kCullSlack32 = 1e-5f;

struct DevParams {
  double rho, sigma, alpha;
  int max_iters;
  double eps_primal, eps_dual;
  int check_interval;
  double mu;
  int k;  // n_edges
  double beta, gamma_total;
  double w_grasp, w_distance, w_limit, w_self, w_pen;
  double fd_step;
  double target_sign;  // QP targets beta * target_sign * (+-e_axis); -1 for the eval gravity wrenches
  double cos_t[kMaxEdges], sin_t[kMaxEdges];  // host libm cos/sin(2 pi j / k)
};

struct StageArgs {
  int stage;  // 0 coarse, 1 fine, 2 final
  int iters;
  int it;
  double step_rot, step_trans, step_joints, step_floor;
  double offset;
  int mode;  // 0: energy + gradient + step, 1: energy only (stage end)
  double decay;  // host-computed cosine decay for `it`
};

// Per-grasp device buffers (all [G][...] contiguous).
struct DevState {
  int G;       // grasps in this launch
  int NQ;      // query slots per grasp = S + 6m
  int NP;      // pair slots per grasp = L*P
  double* x;        // [G*D]
  double* pose;     // [G*24]: R(9 row-major), t(3), a_inv(9 row-major), degenerate, pad
  double* world;    // [G*L*12]: R(9 row-major), t(3)
  double* joints;   // [G*dof*6]: chain-frame origin(3), axis(3)
  double* qpts;     // [G*NQ*3]
  double* qres;     // [G*NQ*8]: d, pb(3), n(3), part
  int* qface;       // [G*NQ] closest face of the slot's last query (warm-start seed), -1 if none
  int* qsep;        // [G*NQ] face whose plane put the last query outside its winning part, -1 if none
  int early_pred;   // k_pairs_early takes slots whose last EPA ran more iterations (option "pair_early")
  const int* obj;   // [G] object of each grasp (multi-object contexts), nullptr = object 0
  int* pq_key;      // [G*NQ] bucket of each query slot (its last closest face's cluster, ...)
  int* pq_count;    // [NC + P + 1] queries per bucket, then the fill cursor
  int* pq_total;    // [1] listed queries
  int* pq_list;     // [G*NQ] query slots (g * NQ + slot) grouped by bucket
  double* pairs;    // [G*NP*12]: d, pa(3), pb(3), n(3), flags, pad
  double* warm_x;   // [G*n*6] column-major n x 6
  double* warm_y;   // [G*M*6]
  double* out_z;    // [G*M*6]
  int* qp_iters;    // [G*6]
  int* qp_conv;     // [G*6]
  int* qp_ready;    // [G]
  double* qp_force;   // [G*m*3]
  double* qp_energy;  // [G]
  double* qp_perdir;  // [G*6]
  double* frames;     // [G*m*12]
  double* anchors;    // [G*m*3]
  double* energy;     // [G]
  double* grad;       // [G*D]
  int* failed;        // [G]
  double* stage_energy;  // [G*6]
  double* x_p;        // [G*D]
  int* have_pregrasp; // [G]
  int* err;           // [4]: 0 epa-degenerate, 1 epa-overflow, 2 unused, 3 unused
  unsigned long long* ops;  // [kNumOps] algorithmic op counters, nullptr unless profiling
  int* ovf_count;      // pairs whose EPA outgrew the per-thread polytope this launch
  int* ovf_list;       // [ovf_cap] their slots: (g * NP + link * P + part)
  int ovf_cap;
  void* big_scratch;   // [big_slots] EpaScratchBig in global memory
  int big_slots;
  int* pair_count;     // compacted list of pair slots that need GJK
  int* pair_list;      // [G*NP]
  unsigned char* pair_need;  // [G*NP-slot order of the launch] 0, or 1 + bucket when the pair needs GJK
  unsigned char* pair_hist;  // [G*NP] GJK closest-point calls of the slot's last evaluation (bucketing)
  int* seg_count;      // [NP] needed pairs per (link, part) segment, then the fill cursor
  int* seg_offset;     // [NP] exclusive scan of seg_count
  int* epa_count;       // overlapping pairs handed from GJK to the EPA kernel
  int* epa_long_count;  // ... of them predicted long (epa_hist), stored from epa_cap on
  double* epa_jobs;     // [2 * epa_cap * kEpaJobStride]: slot, ns, 4 x (w, a, b)
  unsigned char* epa_hist;  // [G*NP] EPA iterations of the slot's last EPA run (job split)
  int epa_cap;
};

constexpr int kEpaJobStride = 18;  // slot, ns, 4 x (w, support key)
// The GJK list is segmented by (link, part) and, inside a segment, by the
// slot's previous GJK length (kPairBuckets buckets), so a warp's pairs tend
// to need the same number of iterations.
constexpr int kPairBuckets = 16;
#ifndef GDEV_EPA_EARLY_PRED
#define GDEV_EPA_EARLY_PRED 24  // 8: 354, 16: 346, 24: 340, 32: 342, 40: 346 ms pairs; off: 346
#endif
constexpr int kEpaEarlyPred = GDEV_EPA_EARLY_PRED;  // k_pairs_early: slots whose last EPA took more iterations
__host__ __device__ inline int pair_bucket(int calls) { return calls < 1 ? 0 : (calls > 16 ? 15 : calls - 1); }

// Op counters (profiling mode) for the roofline's algorithmic flop count
// (SURVEY.md 8(d) constants are applied on the host).
enum OpCounter {
  kOpPlaneTests = 0,     // inside-test face planes evaluated
  kOpTriangleTests = 1,  // closest_on_triangle evaluations
  kOpQpColumnSweeps = 2, // ADMM column-sweeps
  kOpQpSolves = 3,
  kOpGjkIters = 4,
  kOpSupportVerts = 5,   // vertices scanned by support (GJK + EPA)
  kOpEpaIters = 6,
  kOpPointQueries = 7,
  kOpPairsNeeded = 8,    // (link, part) pairs that needed GJK (not culled)
  kOpEpaOverflow = 9,    // pairs redone with the large EPA buffer
  kOpGjkHist = 10,       // 10..15: pairs by GJK iterations <=4, <=8, <=16, <=32, <=64, >64
  kOpGjkCycleJumps = 16, // pairs whose GJK state cycle was fast-forwarded to the iteration cap
  kOpGjkItersSkipped = 17,
  kOpEpaMaxIters = 18,  // max EPA iterations of one job (atomicMax)
  kOpEpaLongJobs = 19,  // EPA jobs with more than 8 iterations
  kNumOps = 20
};

}  // namespace gdev

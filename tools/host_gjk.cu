// Debug harness: runs the device GJK/EPA code (gjk.cuh, __host__ __device__)
// on the CPU so it can be compared with the oracle without a GPU.
#include "../include/grasp_b200.h"
#include "../paper_2412_16490_b200/csrc/cuda/gjk.cuh"

#include <cmath>
#include <vector>

using namespace gdev;

extern "C" int host_signed_distance(const grasp_hand_desc* H, const grasp_object_desc* O, int n, const int* links,
                                    const int* parts, const double* poses, double* out, EpaDebug* dbg) {
  static EpaScratch scratch;
  for (int t = 0; t < n; ++t) {
    const int link = links[t], part = parts[t];
    M33 Rw;
    for (int c = 0; c < 3; ++c)
      for (int i = 0; i < 3; ++i) Rw.m[i * 3 + c] = poses[12 * t + 3 * c + i];
    const D3 tw = ld3(poses + 12 * t + 9);
    Hull A;
    A.verts = H->verts + 3 * H->link_vert_begin[link];
    A.nv = H->link_vert_begin[link + 1] - H->link_vert_begin[link];
    A.posed = true;
    A.R = Rw;
    A.t = tw;
    Hull B;
    B.verts = O->verts + 3 * O->part_vert_begin[part];
    B.nv = O->part_vert_begin[part + 1] - O->part_vert_begin[part];
    B.posed = false;
    B.R = eye();
    B.t = mk(0, 0, 0);
    const double* lo = H->link_obb + 15 * link;
    const double* po = O->part_obb + 15 * part;
    const double lh = std::sqrt(lo[3] * lo[3] + lo[4] * lo[4] + lo[5] * lo[5]);
    const double ph = std::sqrt(po[3] * po[3] + po[4] * po[4] + po[5] * po[5]);
    double scale = 1.0;
    scale = std::fmax(scale, nrm(mul(Rw, ld3(H->link_centroid + 3 * link)) + tw) + 2.0 * lh);
    scale = std::fmax(scale, nrm(ld3(O->part_centroid + 3 * part)) + 2.0 * ph);
    const PairResult r = signed_distance(A, B, scale, scratch, dbg ? dbg + t : nullptr);
    double* o = out + 11 * t;
    o[0] = r.d;
    st3(o + 1, r.pa);
    st3(o + 4, r.pb);
    st3(o + 7, r.n);
    o[10] = r.flags;
  }
  return 0;
}

// Load-time convex parts on the device: the reference's
// make_convex_part (proj/src/geometry.cpp:414-466) with its quickhull
// (proj/src/hull3d.cpp:15-303) for many point clouds at once, one thread per
// part. It follows the host builder (csrc/host/hull3d.cpp, geometry_build.cpp)
// operation for operation - the same lexicographic sort and suffix merge, seed
// tetrahedron, LIFO face stack, BFS visibility flood, horizon fan, orphan
// reassignment and compaction in face-creation order, the same divergence-
// theorem volume and Jacobi PCA box - and this translation unit is compiled
// with --fmad=false, so vertex order, face order and every double are the
// host's bit for bit (the hull's order feeds every downstream tie-break).
// Lists live in per-part global-memory workspaces (face records, outside
// lists as linked points, visibility stamps instead of per-apex vectors).
#include "../../../include/grasp_b200.h"
#include "../host/capi_common.hpp"
#include "dmath.cuh"

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <vector>

namespace gdev {
namespace {

struct HullWs {
  // points (merged, sorted) and their outside-list links
  D3* pts;
  int* next;
  // faces
  int* fv;     // [fc][3]
  int* fnb;    // [fc][3]
  D3* fn;
  double* fd;
  unsigned char* alive;
  int* head;   // outside list
  int* tail;
  int* far_idx;
  double* far_dist;
  int* stamp;  // visibility stamp (add_apex's `seen`)
  // temporaries
  int* lit;
  int* rim_u;
  int* rim_v;
  int* rim_o;
  int* fresh;
  int* orphans;
  int* stack;
  int* remap;
  int fc;  // face capacity
  int n;   // points after the merge
  int nf;  // faces created
};

// the host's cwise_min / cwise_max (la.hpp), signed zeros included
__device__ D3 cw_min(D3 a, D3 b) { return {b.x < a.x ? b.x : a.x, b.y < a.y ? b.y : a.y, b.z < a.z ? b.z : a.z}; }
__device__ D3 cw_max(D3 a, D3 b) { return {a.x < b.x ? b.x : a.x, a.y < b.y ? b.y : a.y, a.z < b.z ? b.z : a.z}; }

__device__ bool lex_less3(D3 a, D3 b) {
  if (a.x != b.x) return a.x < b.x;
  if (a.y != b.y) return a.y < b.y;
  return a.z < b.z;
}

// Heap sort (any sort gives the same sequence: the order is total up to exact
// duplicates, which are identical values).
__device__ void sort_points(D3* a, int n) {
  auto sift = [&](int root, int end) {
    while (2 * root + 1 < end) {
      int child = 2 * root + 1;
      if (child + 1 < end && lex_less3(a[child], a[child + 1])) ++child;
      if (!lex_less3(a[root], a[child])) return;
      const D3 t = a[root];
      a[root] = a[child];
      a[child] = t;
      root = child;
    }
  };
  for (int s = n / 2 - 1; s >= 0; --s) sift(s, n);
  for (int e = n - 1; e > 0; --e) {
    const D3 t = a[0];
    a[0] = a[e];
    a[e] = t;
    sift(0, e);
  }
}

// merge_close (hull3d.cpp:15-31): sorted, then a point within tol of a kept
// point (scanning back while the x gap allows) is dropped. In place.
__device__ int merge_close(D3* pts, int n, double tol) {
  sort_points(pts, n);
  int kept = 0;
  for (int i = 0; i < n; ++i) {
    const D3 p = pts[i];
    bool duplicate = false;
    for (int k = kept - 1; k >= 0; --k) {
      if (p.x - pts[k].x > tol) break;
      if (nrm(p - pts[k]) <= tol) {
        duplicate = true;
        break;
      }
    }
    if (!duplicate) pts[kept++] = p;
  }
  return kept;
}

__device__ void plane(HullWs& w, int f) {
  const int* v = w.fv + 3 * f;
  const D3 a = w.pts[v[0]];
  const D3 c = cross(w.pts[v[1]] - a, w.pts[v[2]] - a);
  const double len = nrm(c);
  w.fn[f] = len > 0 ? c / len : mk(0, 0, 1);
  w.fd[f] = dot(w.fn[f], a);
}

__device__ double above(const HullWs& w, int f, int p) { return dot(w.fn[f], w.pts[p]) - w.fd[f]; }

__device__ int new_face(HullWs& w, int a, int b, int c) {
  if (w.nf >= w.fc) return -1;
  const int f = w.nf++;
  w.fv[3 * f] = a;
  w.fv[3 * f + 1] = b;
  w.fv[3 * f + 2] = c;
  w.fnb[3 * f] = w.fnb[3 * f + 1] = w.fnb[3 * f + 2] = 0;
  w.alive[f] = 1;
  w.head[f] = w.tail[f] = -1;
  w.far_idx[f] = -1;
  w.far_dist[f] = 0.0;
  w.stamp[f] = -1;
  return f;
}

__device__ void push_outside(HullWs& w, int f, int p, double eps) {
  const double d = above(w, f, p);
  if (d <= eps) return;
  w.next[p] = -1;
  if (w.tail[f] < 0) {
    w.head[f] = p;
  } else {
    w.next[w.tail[f]] = p;
  }
  w.tail[f] = p;
  if (d > w.far_dist[f]) {
    w.far_dist[f] = d;
    w.far_idx[f] = p;
  }
}

// Gives p to the candidate face it lies farthest above (first wins ties).
__device__ void assign(HullWs& w, int p, const int* cand, int nc, double eps) {
  int target = -1;
  double best = eps;
  for (int i = 0; i < nc; ++i) {
    const double d = above(w, cand[i], p);
    if (d > best) {
      best = d;
      target = cand[i];
    }
  }
  if (target >= 0) push_outside(w, target, p, eps);
}

// 0 ok, 1 degenerate, 2 workspace overflow
__device__ int seed_tetrahedron(HullWs& w, double eps, D3& interior) {
  const int n = w.n;
  if (n < 4) return 1;
  int a = 0;
  for (int i = 1; i < n; ++i)
    if (w.pts[i].x < w.pts[a].x) a = i;
  int b = -1;
  double best = -1;
  for (int i = 0; i < n; ++i) {
    const double d = nrm(w.pts[i] - w.pts[a]);
    if (d > best) {
      best = d;
      b = i;
    }
  }
  if (best <= eps) return 1;
  const D3 axis = normalized(w.pts[b] - w.pts[a]);
  int c = -1;
  best = -1;
  for (int i = 0; i < n; ++i) {
    const D3 r = w.pts[i] - w.pts[a];
    const double d = nrm(r - axis * dot(axis, r));
    if (d > best) {
      best = d;
      c = i;
    }
  }
  if (best <= eps) return 1;
  const D3 nrm3 = normalized(cross(w.pts[b] - w.pts[a], w.pts[c] - w.pts[a]));
  int d4 = -1;
  best = -1;
  for (int i = 0; i < n; ++i) {
    const double d = fabs(dot(nrm3, w.pts[i] - w.pts[a]));
    if (d > best) {
      best = d;
      d4 = i;
    }
  }
  if (best <= eps) return 1;
  interior = (((w.pts[a] + w.pts[b]) + w.pts[c]) + w.pts[d4]) / 4.0;
  const int tris[4][3] = {{a, b, c}, {a, c, d4}, {a, d4, b}, {b, d4, c}};
  for (int t = 0; t < 4; ++t) {
    const int f = new_face(w, tris[t][0], tris[t][1], tris[t][2]);
    if (f < 0) return 2;
    plane(w, f);
    if (dot(w.fn[f], interior) > w.fd[f]) {
      const int tmp = w.fv[3 * f + 1];
      w.fv[3 * f + 1] = w.fv[3 * f + 2];
      w.fv[3 * f + 2] = tmp;
      plane(w, f);
    }
  }
  for (int fa = 0; fa < 4; ++fa)
    for (int e = 0; e < 3; ++e) {
      const int u = w.fv[3 * fa + e], x = w.fv[3 * fa + (e + 1) % 3];
      for (int fb = 0; fb < 4; ++fb) {
        if (fb == fa) continue;
        for (int k = 0; k < 3; ++k)
          if (w.fv[3 * fb + k] == x && w.fv[3 * fb + (k + 1) % 3] == u) w.fnb[3 * fa + e] = fb;
      }
    }
  return 0;
}

// add_apex (hull3d.cpp Builder::add_apex); returns the number of fresh faces
// (in w.fresh), or -1 on workspace overflow.
__device__ int add_apex(HullWs& w, int seed, double eps, D3 interior, int call) {
  const int apex = w.far_idx[seed];
  const D3 ap = w.pts[apex];
  int n_lit = 1, n_rim = 0;
  w.lit[0] = seed;
  const int old_nf = w.nf;
  w.stamp[seed] = call;
  auto seen = [&](int f) { return f < old_nf && w.stamp[f] == call; };
  for (int k = 0; k < n_lit; ++k) {
    const int fi = w.lit[k];
    for (int e = 0; e < 3; ++e) {
      const int nb = w.fnb[3 * fi + e];
      if (seen(nb)) continue;
      if (dot(w.fn[nb], ap) - w.fd[nb] > eps) {
        w.stamp[nb] = call;
        if (n_lit >= w.fc) return -1;
        w.lit[n_lit++] = nb;
      } else {
        if (n_rim >= w.fc) return -1;
        w.rim_u[n_rim] = w.fv[3 * fi + e];
        w.rim_v[n_rim] = w.fv[3 * fi + (e + 1) % 3];
        w.rim_o[n_rim] = nb;
        ++n_rim;
      }
    }
  }
  // a rim entry can be recorded before its outer face turned visible
  int kept = 0;
  for (int h = 0; h < n_rim; ++h) {
    if (seen(w.rim_o[h])) continue;
    w.rim_u[kept] = w.rim_u[h];
    w.rim_v[kept] = w.rim_v[h];
    w.rim_o[kept] = w.rim_o[h];
    ++kept;
  }
  n_rim = kept;
  int n_orph = 0;
  for (int k = 0; k < n_lit; ++k) {
    const int fi = w.lit[k];
    w.alive[fi] = 0;
    for (int p = w.head[fi]; p >= 0; p = w.next[p])
      if (p != apex) w.orphans[n_orph++] = p;
    w.head[fi] = w.tail[fi] = -1;
  }
  for (int h = 0; h < n_rim; ++h) {
    const int f = new_face(w, w.rim_u[h], w.rim_v[h], apex);
    if (f < 0) return -1;
    plane(w, f);
    if (dot(w.fn[f], interior) > w.fd[f]) {
      const int tmp = w.fv[3 * f];
      w.fv[3 * f] = w.fv[3 * f + 1];
      w.fv[3 * f + 1] = tmp;
      plane(w, f);
    }
    w.fnb[3 * f] = w.rim_o[h];
    w.fresh[h] = f;
    const int outer = w.rim_o[h];
    for (int e = 0; e < 3; ++e)
      if (seen(w.fnb[3 * outer + e])) {
        const int a = w.fv[3 * outer + e], b = w.fv[3 * outer + (e + 1) % 3];
        if ((a == w.rim_v[h] && b == w.rim_u[h]) || (a == w.rim_u[h] && b == w.rim_v[h])) w.fnb[3 * outer + e] = f;
      }
  }
  for (int h = 0; h < n_rim; ++h) {
    const int f = w.fresh[h];
    int next = -1;
    for (int g = 0; g < n_rim; ++g)
      if (w.fv[3 * w.fresh[g]] == w.fv[3 * f + 1]) {
        next = w.fresh[g];
        break;
      }
    w.fnb[3 * f + 1] = next >= 0 ? next : f;
    int prev = -1;
    for (int g = 0; g < n_rim; ++g)
      if (w.fv[3 * w.fresh[g] + 1] == w.fv[3 * f]) prev = w.fresh[g];
    w.fnb[3 * f + 2] = prev >= 0 ? prev : f;
  }
  for (int i = 0; i < n_orph; ++i) assign(w, w.orphans[i], w.fresh, n_rim, eps);
  return n_rim;
}

// Cyclic Jacobi eigen-decomposition, eigenvalues ascending (geometry_build.cpp).
__device__ void symmetric_eigen(const double (&a_in)[3][3], double (&evals)[3], double (&evecs)[3][3]) {
  double a[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a[r][c] = a_in[r][c];
  double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = (fabs(a[0][1]) + fabs(a[0][2])) + fabs(a[1][2]);
    const double diag = (fabs(a[0][0]) + fabs(a[1][1])) + fabs(a[2][2]);
    if (off == 0.0 || off <= 1e-20 * diag) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  const double ev[3] = {a[0][0], a[1][1], a[2][2]};
  int order[3] = {0, 1, 2};
  for (int i = 0; i < 2; ++i) {
    int k = i;
    for (int j = i + 1; j < 3; ++j)
      if (ev[order[j]] < ev[order[k]]) k = j;
    if (k != i) {
      const int t = order[i];
      order[i] = order[k];
      order[k] = t;
    }
  }
  for (int i = 0; i < 3; ++i) {
    evals[i] = ev[order[i]];
    for (int r = 0; r < 3; ++r) evecs[r][i] = v[r][order[i]];
  }
}

struct BuildArgs {
  const double* points;
  const int* point_begin;
  int n_parts;
  double merge_tol;
  // workspace
  char* ws;
  const long long* ws_off;  // [n_parts] byte offset of each part's workspace
  const int* fc;            // [n_parts] face capacity
  // outputs
  double* verts;     // slot of part p at 3 * point_begin[p]
  int* n_verts;
  int* faces;        // slot of part p at 3 * 2 * point_begin[p]
  int* n_faces;
  double* volume;
  double* centroid;  // [3]
  double* obb;       // [15] center, half extents, rotation (column-major)
  int* status;
};

template <class T>
__device__ T* carve(char*& p, long long count) {
  T* r = reinterpret_cast<T*>(p);
  p += ((count * (long long)sizeof(T) + 15) / 16) * 16;
  return r;
}

__global__ void k_build_parts(BuildArgs A) {
  const int part = blockIdx.x * blockDim.x + threadIdx.x;
  if (part >= A.n_parts) return;
  const int p0 = A.point_begin[part], n_in = A.point_begin[part + 1] - p0;
  const int fc = A.fc[part];
  char* cur = A.ws + A.ws_off[part];
  HullWs w;
  w.pts = carve<D3>(cur, n_in);
  w.next = carve<int>(cur, n_in);
  w.fv = carve<int>(cur, 3LL * fc);
  w.fnb = carve<int>(cur, 3LL * fc);
  w.fn = carve<D3>(cur, fc);
  w.fd = carve<double>(cur, fc);
  w.alive = carve<unsigned char>(cur, fc);
  w.head = carve<int>(cur, fc);
  w.tail = carve<int>(cur, fc);
  w.far_idx = carve<int>(cur, fc);
  w.far_dist = carve<double>(cur, fc);
  w.stamp = carve<int>(cur, fc);
  w.lit = carve<int>(cur, fc);
  w.rim_u = carve<int>(cur, fc);
  w.rim_v = carve<int>(cur, fc);
  w.rim_o = carve<int>(cur, fc);
  w.fresh = carve<int>(cur, fc);
  w.orphans = carve<int>(cur, n_in);
  w.stack = carve<int>(cur, fc);
  w.remap = carve<int>(cur, n_in);
  w.fc = fc;
  w.nf = 0;
  A.status[part] = 0;
  A.n_verts[part] = A.n_faces[part] = 0;
  for (int i = 0; i < n_in; ++i) w.pts[i] = mk(A.points[3 * (p0 + i)], A.points[3 * (p0 + i) + 1], A.points[3 * (p0 + i) + 2]);
  // convex_hull (hull3d.cpp:291-303)
  w.n = merge_close(w.pts, n_in, A.merge_tol);
  if (w.n < 4) {
    A.status[part] = 1;
    return;
  }
  D3 lo = w.pts[0], hi = w.pts[0];
  for (int i = 0; i < w.n; ++i) {
    lo = cw_min(lo, w.pts[i]);
    hi = cw_max(hi, w.pts[i]);
  }
  const double eps = fmax(64.0 * 2.220446049250313e-16 * nrm(hi - lo), 1e-300);
  D3 interior;
  const int s = seed_tetrahedron(w, eps, interior);
  if (s) {
    A.status[part] = s;
    return;
  }
  {
    const int all[4] = {0, 1, 2, 3};
    for (int p = 0; p < w.n; ++p) assign(w, p, all, 4, eps);
  }
  int n_stack = 0;
  for (int f = 0; f < 4; ++f)
    if (w.head[f] >= 0) w.stack[n_stack++] = f;
  int call = 0;
  while (n_stack > 0) {
    const int f = w.stack[--n_stack];
    if (!w.alive[f] || w.head[f] < 0) continue;
    const int nr = add_apex(w, f, eps, interior, call++);
    if (nr < 0) {
      A.status[part] = 2;
      return;
    }
    for (int h = 0; h < nr; ++h) {
      const int g = w.fresh[h];
      if (w.head[g] >= 0) {
        if (n_stack >= w.fc) {
          A.status[part] = 2;
          return;
        }
        w.stack[n_stack++] = g;
      }
    }
  }
  // emit: vertices in first-use order of the live faces (creation order)
  for (int i = 0; i < w.n; ++i) w.remap[i] = -1;
  double* V = A.verts + 3LL * p0;
  int* Fo = A.faces + 6LL * p0;
  int nv = 0, nfo = 0;
  for (int f = 0; f < w.nf; ++f) {
    if (!w.alive[f]) continue;
    if (nfo >= 2 * n_in) {
      A.status[part] = 2;
      return;
    }
    for (int k = 0; k < 3; ++k) {
      int& r = w.remap[w.fv[3 * f + k]];
      if (r < 0) {
        r = nv++;
        const D3 q = w.pts[w.fv[3 * f + k]];
        V[3 * r] = q.x;
        V[3 * r + 1] = q.y;
        V[3 * r + 2] = q.z;
      }
      Fo[3 * nfo + k] = r;
    }
    ++nfo;
  }
  A.n_verts[part] = nv;
  A.n_faces[part] = nfo;
  // make_convex_part (geometry.cpp:414-466; geometry_build.cpp)
  auto vert = [&](int i) { return mk(V[3 * i], V[3 * i + 1], V[3 * i + 2]); };
  double vol = 0.0;
  D3 cw = mk(0, 0, 0);
  for (int f = 0; f < nfo; ++f) {
    const D3 a = vert(Fo[3 * f]), b = vert(Fo[3 * f + 1]), c = vert(Fo[3 * f + 2]);
    const double v6 = dot(a, cross(b, c));
    vol += v6;
    cw += v6 * ((a + b) + c);
  }
  const double volume = vol / 6.0;
  if (volume <= 0) {
    A.status[part] = 1;
    return;
  }
  const D3 centroid = cw / (4.0 * vol);
  D3 mean = mk(0, 0, 0);
  for (int i = 0; i < nv; ++i) mean += vert(i);
  mean = mean / static_cast<double>(nv);
  double cov[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int i = 0; i < nv; ++i) {
    const D3 d = vert(i) - mean;
    const double dv[3] = {d.x, d.y, d.z};
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) cov[r][c] = cov[r][c] + dv[r] * dv[c];
  }
  double evals[3], evecs[3][3];
  symmetric_eigen(cov, evals, evecs);
  double axes[3][3];  // columns: evecs 2, 1, 0
  for (int r = 0; r < 3; ++r) {
    axes[r][0] = evecs[r][2];
    axes[r][1] = evecs[r][1];
    axes[r][2] = evecs[r][0];
  }
  for (int c = 0; c < 3; ++c) {
    int arg = 0;
    double best = fabs(axes[0][c]);
    for (int r = 1; r < 3; ++r)
      if (fabs(axes[r][c]) > best) {
        best = fabs(axes[r][c]);
        arg = r;
      }
    if (axes[arg][c] < 0)
      for (int r = 0; r < 3; ++r) axes[r][c] = -axes[r][c];
  }
  const double det = axes[0][0] * (axes[1][1] * axes[2][2] - axes[1][2] * axes[2][1]) -
                     axes[0][1] * (axes[1][0] * axes[2][2] - axes[1][2] * axes[2][0]) +
                     axes[0][2] * (axes[1][0] * axes[2][1] - axes[1][1] * axes[2][0]);
  if (det < 0)
    for (int r = 0; r < 3; ++r) axes[r][2] = -axes[r][2];
  double blo[3] = {INFINITY, INFINITY, INFINITY}, bhi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = 0; i < nv; ++i) {
    const D3 v = vert(i);
    for (int c = 0; c < 3; ++c) {
      const double q = (axes[0][c] * v.x + axes[1][c] * v.y) + axes[2][c] * v.z;
      blo[c] = q < blo[c] ? q : blo[c];  // (the host's cwise_min / cwise_max)
      bhi[c] = bhi[c] < q ? q : bhi[c];
    }
  }
  double mid[3], half[3];
  for (int c = 0; c < 3; ++c) {
    mid[c] = (blo[c] + bhi[c]) / 2.0;
    half[c] = (bhi[c] - blo[c]) / 2.0;
  }
  double* ob = A.obb + 15LL * part;
  for (int r = 0; r < 3; ++r) ob[r] = (axes[r][0] * mid[0] + axes[r][1] * mid[1]) + axes[r][2] * mid[2];
  for (int c = 0; c < 3; ++c) ob[3 + c] = half[c];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) ob[6 + 3 * c + r] = axes[r][c];
  A.volume[part] = volume;
  A.centroid[3 * part] = centroid.x;
  A.centroid[3 * part + 1] = centroid.y;
  A.centroid[3 * part + 2] = centroid.z;
}

struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return GRASP_OK;
  } catch (const DeviceError& e) {
    return grasp::capi::fail(GRASP_ECUDA, e.what());
  } catch (const std::invalid_argument& e) {
    return grasp::capi::fail(GRASP_EINVAL, e.what());
  } catch (const std::bad_alloc&) {
    return grasp::capi::fail(GRASP_ENOMEM, "out of host memory");
  } catch (const std::exception& e) {
    return grasp::capi::fail(GRASP_EINVAL, e.what());
  }
}

template <class T>
struct Buf {
  T* p = nullptr;
  explicit Buf(size_t n) { ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
  ~Buf() { cudaFree(p); }
};

}  // namespace
}  // namespace gdev

extern "C" int grasp_build_convex_parts(int device, const double* points, const int* point_begin, int n_parts,
                                        double merge_tol, double* out_verts, int* out_n_verts, int* out_faces,
                                        int* out_n_faces, double* out_volume, double* out_centroid, double* out_obb,
                                        int* out_status) {
  using namespace gdev;
  return guard([&] {
    if (n_parts < 0 || (n_parts > 0 && (!points || !point_begin || !out_verts || !out_n_verts || !out_faces ||
                                        !out_n_faces || !out_volume || !out_centroid || !out_obb || !out_status)))
      throw std::invalid_argument("null argument");
    if (n_parts == 0) return;
    if (!(merge_tol >= 0.0)) throw std::invalid_argument("merge_tol must be nonnegative");
    for (int p = 0; p < n_parts; ++p)
      if (point_begin[p + 1] < point_begin[p] || point_begin[p] < 0)
        throw std::invalid_argument("point_begin must be nondecreasing from 0");
    ck(cudaSetDevice(device), "cudaSetDevice");
    const int n_pts = point_begin[n_parts];
    // workspace per part: face capacity 16 n + 64
    std::vector<long long> off(n_parts);
    std::vector<int> fc(n_parts);
    long long total = 0;
    auto bytes = [](long long count, long long size) { return ((count * size + 15) / 16) * 16; };
    for (int p = 0; p < n_parts; ++p) {
      const long long n = point_begin[p + 1] - point_begin[p];
      const long long f = 16 * n + 64;
      fc[p] = static_cast<int>(f);
      off[p] = total;
      total += bytes(n, 24) + 3 * bytes(n, 4) + 2 * bytes(3 * f, 4) + bytes(f, 24) + 2 * bytes(f, 8) + bytes(f, 1) +
               11 * bytes(f, 4);
    }
    cudaStream_t s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    Buf<double> d_pts(3LL * n_pts), d_verts(3LL * n_pts), d_vol(n_parts), d_cen(3LL * n_parts), d_obb(15LL * n_parts);
    Buf<int> d_beg(n_parts + 1), d_nv(n_parts), d_faces(6LL * n_pts), d_nf(n_parts), d_status(n_parts), d_fc(n_parts);
    Buf<long long> d_off(n_parts);
    Buf<char> d_ws(total);
    ck(cudaMemcpyAsync(d_pts.p, points, sizeof(double) * 3 * n_pts, cudaMemcpyHostToDevice, s), "copy");
    ck(cudaMemcpyAsync(d_beg.p, point_begin, sizeof(int) * (n_parts + 1), cudaMemcpyHostToDevice, s), "copy");
    ck(cudaMemcpyAsync(d_off.p, off.data(), sizeof(long long) * n_parts, cudaMemcpyHostToDevice, s), "copy");
    ck(cudaMemcpyAsync(d_fc.p, fc.data(), sizeof(int) * n_parts, cudaMemcpyHostToDevice, s), "copy");
    BuildArgs a{d_pts.p, d_beg.p, n_parts, merge_tol, d_ws.p, d_off.p, d_fc.p, d_verts.p, d_nv.p, d_faces.p, d_nf.p,
                d_vol.p, d_cen.p, d_obb.p, d_status.p};
    k_build_parts<<<(n_parts + 63) / 64, 64, 0, s>>>(a);
    ck(cudaGetLastError(), "k_build_parts");
    ck(cudaMemcpyAsync(out_verts, d_verts.p, sizeof(double) * 3 * n_pts, cudaMemcpyDeviceToHost, s), "copy");
    ck(cudaMemcpyAsync(out_faces, d_faces.p, sizeof(int) * 6 * n_pts, cudaMemcpyDeviceToHost, s), "copy");
    ck(cudaMemcpyAsync(out_n_verts, d_nv.p, sizeof(int) * n_parts, cudaMemcpyDeviceToHost, s), "copy");
    ck(cudaMemcpyAsync(out_n_faces, d_nf.p, sizeof(int) * n_parts, cudaMemcpyDeviceToHost, s), "copy");
    ck(cudaMemcpyAsync(out_volume, d_vol.p, sizeof(double) * n_parts, cudaMemcpyDeviceToHost, s), "copy");
    ck(cudaMemcpyAsync(out_centroid, d_cen.p, sizeof(double) * 3 * n_parts, cudaMemcpyDeviceToHost, s), "copy");
    ck(cudaMemcpyAsync(out_obb, d_obb.p, sizeof(double) * 15 * n_parts, cudaMemcpyDeviceToHost, s), "copy");
    ck(cudaMemcpyAsync(out_status, d_status.p, sizeof(int) * n_parts, cudaMemcpyDeviceToHost, s), "copy");
    ck(cudaStreamSynchronize(s), "k_build_parts");
  });
}

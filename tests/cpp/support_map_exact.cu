// Host check of the GJK support maps (model.cuh, support_map.cuh), compiled as host code
// from the same headers as the kernels (run by tests/test_device_math_host.py): for every
// hull and direction the map-accelerated support() returns the same vertex index as the
// reference's full first-maximum scan (geometry.cpp:399-412), bit for bit -- on round
// hulls, boxes and lattices full of exact ties, for random, axis-aligned, face-normal,
// cell-boundary, tiny and huge directions, posed and unposed.
#include "../../paper_2412_16490_b200/csrc/cuda/gjk.cuh"
#include "../../paper_2412_16490_b200/csrc/cuda/support_map.cuh"

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

using namespace gdev;

static std::vector<double> ball(int n, double r, double jitter, std::mt19937_64& rng) {
  std::normal_distribution<double> g(0.0, 1.0);
  std::vector<double> v;
  const double golden = 3.14159265358979323846 * (3.0 - std::sqrt(5.0));
  for (int k = 0; k < n; ++k) {
    const double z = 1.0 - 2.0 * (k + 0.5) / n, rr = std::sqrt(std::fmax(0.0, 1.0 - z * z));
    v.push_back(r * rr * std::cos(golden * k) + jitter * g(rng));
    v.push_back(r * rr * std::sin(golden * k) + jitter * g(rng));
    v.push_back(r * z + jitter * g(rng));
  }
  return v;
}

int main(int argc, char** argv) {
  std::mt19937_64 rng(11);
  std::vector<std::vector<double>> hulls;
  hulls.push_back(ball(386, 0.05, 0.0, rng));
  hulls.push_back(ball(242, 0.03, 2e-4, rng));
  hulls.push_back(ball(64, 1.0, 0.0, rng));
  {  // lattice cube: many exact ties on faces, edges and corners
    std::vector<double> v;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        for (int k = 0; k < 4; ++k) {
          v.push_back(-0.03 + 0.02 * i);
          v.push_back(-0.03 + 0.02 * j);
          v.push_back(-0.03 + 0.02 * k);
        }
    hulls.push_back(v);
  }
  {  // cylinder-like: two rings (flat caps) of 32
    std::vector<double> v;
    for (int h = 0; h < 2; ++h)
      for (int k = 0; k < 32; ++k) {
        const double a = 2.0 * 3.14159265358979323846 * k / 32;
        v.push_back(0.02 * std::cos(a));
        v.push_back(0.02 * std::sin(a));
        v.push_back(h ? 0.04 : -0.04);
      }
    hulls.push_back(v);
  }
  // Extra hulls from argv: files of "x y z" lines (e.g. the drill parts dumped by the test).
  for (int a = 1; a < argc; ++a) {
    FILE* f = std::fopen(argv[a], "r");
    if (!f) continue;
    std::vector<double> v;
    double x, y, z;
    while (std::fscanf(f, "%lf %lf %lf", &x, &y, &z) == 3) v.insert(v.end(), {x, y, z});
    std::fclose(f);
    if (v.size() >= 3 * static_cast<size_t>(kSupportMapMinVerts)) hulls.push_back(v);
  }

  std::uniform_real_distribution<double> U(-1, 1);
  long mismatches = 0, calls = 0, scanned_full = 0, scanned_map = 0;
  for (const auto& V : hulls) {
    const int nv = static_cast<int>(V.size() / 3);
    std::vector<int> base, off;
    std::vector<unsigned short> idx;
    const int beg[2] = {0, nv};
    build_support_maps(V.data(), beg, 1, base, off, idx);
    if (base[0] < 0) {
      std::printf("hull without map (nv %d)\n", nv);
      return 2;
    }
    Hull plain, fast;
    plain.verts = fast.verts = V.data();
    plain.nv = fast.nv = nv;
    fast.cm_off = off.data() + base[0];
    fast.cm_idx = idx.data();
    scanned_map += static_cast<long>(idx.size());
    scanned_full += static_cast<long>(nv) * kSupportCells;
    for (int posed = 0; posed < 2; ++posed) {
      M33 R = eye();
      if (posed) {  // a random rotation (Gram-Schmidt of a random matrix)
        D3 c0 = mk(U(rng), U(rng), U(rng)), c1 = mk(U(rng), U(rng), U(rng));
        c0 = c0 / nrm(c0);
        c1 = c1 - dot(c0, c1) * c0;
        c1 = c1 / nrm(c1);
        const D3 c2 = cross(c0, c1);
        R = {{c0.x, c1.x, c2.x, c0.y, c1.y, c2.y, c0.z, c1.z, c2.z}};
      }
      plain.posed = fast.posed = posed != 0;
      plain.R = fast.R = R;
      plain.t = fast.t = mk(0.01, -0.02, 0.03);
      auto check = [&](D3 d) {
        int ia = -1, ib = -2;
        const D3 a = support(plain, d, ia);
        const D3 b = support(fast, d, ib);
        ++calls;
        if (ia != ib || a.x != b.x || a.y != b.y || a.z != b.z) ++mismatches;
      };
      for (int t = 0; t < 200000; ++t) check(mk(U(rng), U(rng), U(rng)));
      for (int ax = 0; ax < 3; ++ax)
        for (int sg = -1; sg <= 1; sg += 2) {
          D3 d = mk(0, 0, 0);
          if (ax == 0) d.x = sg;
          if (ax == 1) d.y = sg;
          if (ax == 2) d.z = sg;
          check(d);
          check(1e-190 * d);
          check(1e190 * d);
        }
      // directions on cube-map cell boundaries and face diagonals
      for (int t = 0; t < 20000; ++t) {
        const double b = -1.0 + 2.0 * static_cast<double>(rng() % (kSupportMapN + 1)) / kSupportMapN;
        const double eps = (rng() % 3 == 0) ? 0.0 : std::ldexp(U(rng), -50);
        const double s = std::ldexp(1.0, static_cast<int>(rng() % 40) - 20);
        D3 d = mk(1.0, b + eps, U(rng));
        if (t % 3 == 1) d = mk(U(rng), 1.0, b + eps);
        if (t % 3 == 2) d = mk(b + eps, U(rng), -1.0);
        if (t % 7 == 0) d = mk(1.0, 1.0, b);
        check(s * d);
      }
      // edge and face normals of the hull (exact ties): differences of vertex pairs, crossed
      for (int t = 0; t < 20000; ++t) {
        const int i = static_cast<int>(rng() % nv), j = static_cast<int>(rng() % nv), k = static_cast<int>(rng() % nv);
        const D3 p = ldg3(V.data() + 3 * i), q = ldg3(V.data() + 3 * j), r = ldg3(V.data() + 3 * k);
        check(cross(q - p, r - p));
        check(-cross(q - p, r - p));
      }
    }
  }
  std::printf("support maps: %ld calls, %ld mismatches, candidates %.2f%% of a full scan\n", calls, mismatches,
              100.0 * static_cast<double>(scanned_map) / static_cast<double>(scanned_full));
  return mismatches == 0 ? 0 : 1;
}

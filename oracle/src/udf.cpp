// ORACLE (test infrastructure only) — stage 1a: voxel-grid-hierarchy narrow-band UDF
// and UDF->SDF, restated from SPEC.md:157-236 / PAPER.md:55-74,93.
//
// Pinned semantics (SURVEY §7 pins P1-P4):
//   levels r = 8, 16, ..., R; cell centre c = ((i+0.5)/r, ...);
//   thr_r = 3/R + kHalfSqrt3/r  (band + cell bounding-sphere radius);
//   a (cell, tri) pair survives level r iff its parent pair survived level r/2 (level 8: all
//   pairs are tested) AND  box_d2(c, aabb(tri)) <= (thr_r + 1e-9)^2
//                     AND  sqrt(point_triangle_sq(c, tri)) <= thr_r        (P4, FP64)
//   (the box test is a conservative pre-check — the true distance is >= the box distance);
//   compute_udf: vertex v (lattice point (i/R, j/R, k/R), P1) takes
//   min over the UNION of the candidate triangles of its surviving owning finest cells (P2)
//   of point_triangle_sq(v, tri); no candidate -> +INF.  udf = (float)sqrt(min d2).
//   udf_to_sdf: s = (float)((double)udf - eps); +INF -> +1.0f.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

#include "geom.hpp"
#include "par.hpp"

namespace orc {

int& worker_count_ref() {
  static int n = 0;
  return n;
}

constexpr double kHalfSqrt3 = 0.8660254037844386;

struct Tri {
  V3 a, b, c, lo, hi;
};

static inline double box_d2(V3 p, V3 lo, V3 hi) {
  const double dx = std::max(std::max(lo.x - p.x, p.x - hi.x), 0.0);
  const double dy = std::max(std::max(lo.y - p.y, p.y - hi.y), 0.0);
  const double dz = std::max(std::max(lo.z - p.z, p.z - hi.z), 0.0);
  return (dx * dx + dy * dy) + dz * dz;
}

static inline bool survives(const Tri& t, V3 c, double thr) {
  const double tb = thr + 1e-9;
  if (box_d2(c, t.lo, t.hi) > tb * tb) return false;
  return std::sqrt(point_triangle_sq(c, t.a, t.b, t.c)) <= thr;
}

static inline double level_thr(int R, int r) { return 3.0 / R + kHalfSqrt3 / r; }

static std::vector<Tri> load_tris(const double* v, const int32_t* f, int64_t nf) {
  std::vector<Tri> tris(nf);
  for (int64_t i = 0; i < nf; ++i) {
    Tri t;
    const int32_t* fi = f + 3 * i;
    t.a = v3(v[3 * fi[0]], v[3 * fi[0] + 1], v[3 * fi[0] + 2]);
    t.b = v3(v[3 * fi[1]], v[3 * fi[1] + 1], v[3 * fi[1] + 2]);
    t.c = v3(v[3 * fi[2]], v[3 * fi[2] + 1], v[3 * fi[2] + 2]);
    t.lo = v3(std::min(std::min(t.a.x, t.b.x), t.c.x), std::min(std::min(t.a.y, t.b.y), t.c.y),
              std::min(std::min(t.a.z, t.b.z), t.c.z));
    t.hi = v3(std::max(std::max(t.a.x, t.b.x), t.c.x), std::max(std::max(t.a.y, t.b.y), t.c.y),
              std::max(std::max(t.a.z, t.b.z), t.c.z));
    tris[i] = t;
  }
  return tris;
}

// Per-triangle coarse-to-fine descent.  Returns the surviving cells of every level
// (level index l: r = 8 << l), each as linear index x-fastest at that level.
static void descend(const Tri& t, int R, std::vector<std::vector<int64_t>>& levels) {
  const int nlev = static_cast<int>(std::log2(R / 8)) + 1;
  levels.assign(nlev, {});
  // level 0: every cell of the 8^3 grid is a candidate; iterate a conservative index box
  {
    const int r = 8;
    const double thr = level_thr(R, r);
    const double tb = thr + 1e-9;
    int lo[3], hi[3];
    const double los[3] = {t.lo.x, t.lo.y, t.lo.z}, his[3] = {t.hi.x, t.hi.y, t.hi.z};
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::max(0, static_cast<int>(std::floor((los[k] - tb) * r - 0.5)) - 1);
      hi[k] = std::min(r - 1, static_cast<int>(std::ceil((his[k] + tb) * r - 0.5)) + 1);
    }
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x) {
          const V3 c = v3((x + 0.5) / r, (y + 0.5) / r, (z + 0.5) / r);
          if (survives(t, c, thr)) levels[0].push_back(x + static_cast<int64_t>(r) * (y + static_cast<int64_t>(r) * z));
        }
  }
  for (int l = 1; l < nlev; ++l) {
    const int rp = 8 << (l - 1), r = 8 << l;
    const double thr = level_thr(R, r);
    for (int64_t pc : levels[l - 1]) {
      const int px = static_cast<int>(pc % rp), py = static_cast<int>((pc / rp) % rp),
                pz = static_cast<int>(pc / (static_cast<int64_t>(rp) * rp));
      for (int ch = 0; ch < 8; ++ch) {
        const int x = 2 * px + (ch & 1), y = 2 * py + ((ch >> 1) & 1), z = 2 * pz + ((ch >> 2) & 1);
        const V3 c = v3((x + 0.5) / r, (y + 0.5) / r, (z + 0.5) / r);
        if (survives(t, c, thr)) levels[l].push_back(x + static_cast<int64_t>(r) * (y + static_cast<int64_t>(r) * z));
      }
    }
    std::sort(levels[l].begin(), levels[l].end());
  }
}

}  // namespace orc

using namespace orc;

extern "C" {

void orc_set_workers(int n) { worker_count_ref() = n; }

// build_hierarchy debug view: surviving (cell, tri) pairs of level r,
// sorted by (cell, tri).  Count-then-fill: pairs == nullptr returns the count.
int64_t orc_hierarchy_pairs(const double* v, const int32_t* f, int64_t nf, int R, int r,
                            int64_t* pairs, int64_t cap) {
  const std::vector<Tri> tris = load_tris(v, f, nf);
  int lvl = 0;
  while ((8 << lvl) < r) ++lvl;
  std::vector<std::vector<int64_t>> per_tri(nf);
  parallel_for(nf, [&](int64_t i) {
    std::vector<std::vector<int64_t>> levels;
    descend(tris[i], R, levels);
    per_tri[i] = levels[lvl];
  }, 64);
  std::vector<std::pair<int64_t, int64_t>> all;
  for (int64_t i = 0; i < nf; ++i)
    for (int64_t c : per_tri[i]) all.emplace_back(c, i);
  std::sort(all.begin(), all.end());
  const int64_t n = static_cast<int64_t>(all.size());
  if (pairs)
    for (int64_t i = 0; i < std::min(n, cap); ++i) {
      pairs[2 * i] = all[i].first;
      pairs[2 * i + 1] = all[i].second;
    }
  return n;
}

// compute_udf + udf_to_sdf.  udf/sdf: (R+1)^3 floats, x-fastest
// (either may be null).  Returns the number of finite samples.
int64_t orc_compute_udf_sdf(const double* v, const int32_t* f, int64_t nf, int R, double eps,
                            float* udf, float* sdf) {
  const std::vector<Tri> tris = load_tris(v, f, nf);
  const int64_t n1 = R + 1;
  const int64_t nvert = n1 * n1 * n1;
  std::vector<std::atomic<uint64_t>> d2(nvert);
  for (auto& a : d2) a.store(~0ull, std::memory_order_relaxed);
  const int nlev = static_cast<int>(std::log2(R / 8)) + 1;
  parallel_for(nf, [&](int64_t ti) {
    std::vector<std::vector<int64_t>> levels;
    descend(tris[ti], R, levels);
    const std::vector<int64_t>& fin = levels[nlev - 1];
    std::vector<int64_t> verts;
    verts.reserve(fin.size() * 8);
    for (int64_t c : fin) {
      const int64_t x = c % R, y = (c / R) % R, z = c / (static_cast<int64_t>(R) * R);
      for (int k = 0; k < 8; ++k)
        verts.push_back((x + (k & 1)) + n1 * ((y + ((k >> 1) & 1)) + n1 * (z + ((k >> 2) & 1))));
    }
    std::sort(verts.begin(), verts.end());
    verts.erase(std::unique(verts.begin(), verts.end()), verts.end());
    const Tri& t = tris[ti];
    for (int64_t vi : verts) {
      const int64_t x = vi % n1, y = (vi / n1) % n1, z = vi / (n1 * n1);
      const V3 p = v3(static_cast<double>(x) / R, static_cast<double>(y) / R, static_cast<double>(z) / R);
      const double d = point_triangle_sq(p, t.a, t.b, t.c);
      uint64_t bits;
      std::memcpy(&bits, &d, 8);
      atomic_min_u64(d2[vi], bits);
    }
  }, 16);
  int64_t finite = 0;
  for (int64_t i = 0; i < nvert; ++i) {
    const uint64_t b = d2[i].load(std::memory_order_relaxed);
    float u, s;
    if (b == ~0ull) {
      u = std::numeric_limits<float>::infinity();
      s = 1.0f;
    } else {
      double d;
      std::memcpy(&d, &b, 8);
      u = static_cast<float>(std::sqrt(d));
      s = static_cast<float>(static_cast<double>(u) - eps);
      ++finite;
    }
    if (udf) udf[i] = u;
    if (sdf) sdf[i] = s;
  }
  return finite;
}

// Reference-style brute force for the SPEC oracle equivalence:
// min over ALL triangles of point_triangle_sq at every vertex (small inputs only).
void orc_brute_udf(const double* v, const int32_t* f, int64_t nf, int R, float* udf) {
  const std::vector<Tri> tris = load_tris(v, f, nf);
  const int64_t n1 = R + 1;
  parallel_for(n1 * n1 * n1, [&](int64_t vi) {
    const int64_t x = vi % n1, y = (vi / n1) % n1, z = vi / (n1 * n1);
    const V3 p = v3(static_cast<double>(x) / R, static_cast<double>(y) / R, static_cast<double>(z) / R);
    double best = std::numeric_limits<double>::infinity();
    for (const Tri& t : tris) best = std::min(best, point_triangle_sq(p, t.a, t.b, t.c));
    udf[vi] = static_cast<float>(std::sqrt(best));
  });
}

double orc_point_triangle_sq(const double* p, const double* a, const double* b, const double* c) {
  return point_triangle_sq(v3(p[0], p[1], p[2]), v3(a[0], a[1], a[2]), v3(b[0], b[1], b[2]),
                           v3(c[0], c[1], c[2]));
}

void orc_point_triangle_sq_batch(const double* p, const double* a, const double* b,
                                 const double* c, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_point_triangle_sq(p + 3 * i, a + 3 * i, b + 3 * i, c + 3 * i);
}

double orc_det_exp(double x) { return det_exp(x); }
double orc_sigmoid(double t, double beta) { return sigmoid_t(t, beta); }

}  // extern "C"

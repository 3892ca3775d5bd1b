// ORACLE — TEST INFRASTRUCTURE ONLY.  CPU restatement of the certification / quality-metric
// operations beside the hot path:
//   * analyze_topology (mesh.cpp:113-150, TopologySummary mesh.hpp:44-51): edge incidence
//     counts, boundary edges, non-manifold edges (count not in {1,2}), non-manifold vertices
//     (the one-ring is not a single fan: some incident face has > 2 fan neighbours across
//     2-face edges at v, or the fan graph is disconnected), Euler characteristic over used
//     vertices.  Restated with sorted edge keys instead of std::map.
//   * nearest_primitive (lbvh.cpp:192-237): exact nearest face by brute force, ties to the lower
//     face id, closest point of the face (distance.cpp:26-79 region order).
//   * quality_metrics (SPEC.md quality_metrics: chamfer, hausdorff, min_internal_angle) on the
//     pinned sampler below.
// Pinned sampler (the SPEC leaves it open): area_f = |cross(b-a, c-a)|/2; w_f =
// floor(area_f / max_area * 2^32) (integers, so the cumulative weights are order-free);
// sample i uses h_k = mix(seed + (3i+k+1)*0x9E3779B97F4A7C15) (SplitMix64 finaliser), face =
// first f with cum_f > mulhi(h_0, W), s = sqrt(u1), p = (a(1-s) + b(s(1-u2))) + c(s u2) with
// u = (h >> 11) 2^-53.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#include "geom.hpp"
#include "par.hpp"

namespace orc {
namespace metrics {

inline V3 P(const double* v, int64_t i) { return v3(v[3 * i], v[3 * i + 1], v[3 * i + 2]); }

// -------------------------------------------------------------------------- topology
struct Topo {
  int64_t manifold = 0, watertight = 0, euler = 0, boundary = 0;
  std::vector<int64_t> nm_edges;  // (a<<32|b), ascending
  std::vector<int32_t> nm_verts;  // ascending
};

inline uint64_t ekey(int32_t u, int32_t v) {
  const uint32_t a = static_cast<uint32_t>(std::min(u, v)), b = static_cast<uint32_t>(std::max(u, v));
  return (static_cast<uint64_t>(a) << 32) | b;
}

void topology(const int32_t* F, int64_t nf, int64_t nv, Topo& out) {
  // (edge key, face) for every face side, sorted: runs = EdgeInfo::faces lists
  std::vector<std::pair<uint64_t, int32_t>> ent;
  ent.reserve(3 * nf);
  for (int64_t f = 0; f < nf; ++f)
    for (int k = 0; k < 3; ++k) ent.push_back({ekey(F[3 * f + k], F[3 * f + (k + 1) % 3]), static_cast<int32_t>(f)});
  std::sort(ent.begin(), ent.end());
  std::vector<uint64_t> keys;
  std::vector<int64_t> start;
  for (int64_t i = 0; i < static_cast<int64_t>(ent.size()); ++i)
    if (i == 0 || ent[i].first != ent[i - 1].first) {
      keys.push_back(ent[i].first);
      start.push_back(i);
    }
  start.push_back(static_cast<int64_t>(ent.size()));
  const int64_t ne = static_cast<int64_t>(keys.size());
  bool edges_ok = true;
  for (int64_t e = 0; e < ne; ++e) {
    const int64_t c = start[e + 1] - start[e];
    if (c == 1) ++out.boundary;
    if (c != 1 && c != 2) {
      out.nm_edges.push_back(static_cast<int64_t>(keys[e]));
      edges_ok = false;
    }
  }
  // unique incident faces per vertex, ascending
  std::vector<std::vector<int32_t>> inc(nv);
  for (int64_t f = 0; f < nf; ++f)
    for (int k = 0; k < 3; ++k) {
      const int32_t v = F[3 * f + k];
      if ((k >= 1 && v == F[3 * f]) || (k == 2 && v == F[3 * f + 1])) continue;
      inc[v].push_back(static_cast<int32_t>(f));
    }
  std::vector<uint8_t> bad(nv, 0);
  parallel_for(nv, [&](int64_t v) {
    const auto& L = inc[v];
    const int m = static_cast<int>(L.size());
    if (m == 0) return;
    std::vector<std::array<int, 3>> nb(m, {-1, -1, -1});
    std::vector<int> deg(m, 0);
    for (int i = 0; i < m; ++i) {
      const int32_t* t = F + 3 * static_cast<int64_t>(L[i]);
      for (int k = 0; k < 3; ++k) {
        const int32_t a = t[k], b = t[(k + 1) % 3];
        if (a != v && b != v) continue;
        const int64_t e = std::lower_bound(keys.begin(), keys.end(), ekey(a, b)) - keys.begin();
        if (start[e + 1] - start[e] != 2) continue;
        for (int64_t j = start[e]; j < start[e + 1]; ++j) {
          const int32_t g = ent[j].second;
          if (g == L[i]) continue;
          const int li = static_cast<int>(std::lower_bound(L.begin(), L.end(), g) - L.begin());
          bool seen = false;
          for (int q = 0; q < std::min(deg[i], 3); ++q) seen |= nb[i][q] == li;
          if (!seen) {
            if (deg[i] < 3) nb[i][deg[i]] = li;
            ++deg[i];
          }
        }
      }
      if (deg[i] > 2) {
        bad[v] = 1;
        return;
      }
    }
    std::vector<char> seen(m, 0);
    std::vector<int> st = {0};
    seen[0] = 1;
    int cnt = 1;
    while (!st.empty()) {
      const int i = st.back();
      st.pop_back();
      for (int q = 0; q < deg[i]; ++q)
        if (!seen[nb[i][q]]) {
          seen[nb[i][q]] = 1;
          ++cnt;
          st.push_back(nb[i][q]);
        }
    }
    if (cnt != m) bad[v] = 1;
  });
  int64_t used = 0;
  for (int64_t v = 0; v < nv; ++v) {
    if (bad[v]) out.nm_verts.push_back(static_cast<int32_t>(v));
    used += !inc[v].empty();
  }
  out.manifold = edges_ok && out.nm_verts.empty();
  out.watertight = out.manifold && out.boundary == 0;
  out.euler = used - ne + nf;
}

// --------------------------------------------------------------------------- nearest
// point_triangle_sq_distance with the closest point (distance.cpp:26-79)
double ptri_closest(V3 p, V3 a, V3 b, V3 c, V3& q) {
  const V3 n = cross(b - a, c - a);
  const double nn = sqnorm(n);
  double best = std::numeric_limits<double>::infinity();
  q = a;
  if (nn > 0.0) {
    const V3 ap = p - a;
    const double dist_n = dot(ap, n);
    const V3 proj = p - (dist_n / nn) * n;
    const V3 v0 = b - a, v1 = c - a, v2 = proj - a;
    const double d00 = sqnorm(v0), d01 = dot(v0, v1), d11 = sqnorm(v1);
    const double d20 = dot(v2, v0), d21 = dot(v2, v1);
    const double denom = d00 * d11 - d01 * d01;
    if (denom > 0.0) {
      const double v = (d11 * d20 - d01 * d21) / denom;
      const double w = (d00 * d21 - d01 * d20) / denom;
      if (v >= 0.0 && w >= 0.0 && v + w <= 1.0) {
        best = dist_n * dist_n / nn;
        q = proj;
      }
    }
  }
  const V3 E[3][2] = {{a, b}, {b, c}, {c, a}};
  for (int k = 0; k < 3; ++k) {
    const V3 u = E[k][0], ab = E[k][1] - E[k][0];
    const double denom = sqnorm(ab);
    double t = denom > 0.0 ? dot(p - u, ab) / denom : 0.0;
    t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);
    const V3 s = u + t * ab;
    const double d2 = sqnorm(p - s);
    if (d2 < best) {
      best = d2;
      q = s;
    }
  }
  return best;
}

void nearest(const double* V, const int32_t* F, int64_t nf, const double* pts, int64_t n, int32_t* face,
             double* dist, double* closest) {
  parallel_for(n, [&](int64_t i) {
    const V3 p = P(pts, i);
    double best = std::numeric_limits<double>::infinity();
    int32_t bf = -1;
    for (int64_t f = 0; f < nf; ++f) {
      const double d2 = point_triangle_sq(p, P(V, F[3 * f]), P(V, F[3 * f + 1]), P(V, F[3 * f + 2]));
      if (d2 < best) {  // ascending f: ties keep the lower id
        best = d2;
        bf = static_cast<int32_t>(f);
      }
    }
    V3 q = v3(0, 0, 0);
    if (bf >= 0) ptri_closest(p, P(V, F[3 * bf]), P(V, F[3 * bf + 1]), P(V, F[3 * bf + 2]), q);
    if (face) face[i] = bf;
    if (dist) dist[i] = std::sqrt(best);
    if (closest) {
      closest[3 * i] = q.x;
      closest[3 * i + 1] = q.y;
      closest[3 * i + 2] = q.z;
    }
  }, 16);
}

// ---------------------------------------------------------------------------- sampler
inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t hash_k(uint64_t seed, uint64_t k) { return mix64(seed + (k + 1) * 0x9E3779B97F4A7C15ull); }
inline double unit53(uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }

double face_area(const double* V, const int32_t* t) {
  const V3 a = P(V, t[0]), b = P(V, t[1]), c = P(V, t[2]);
  return 0.5 * std::sqrt(sqnorm(cross(b - a, c - a)));
}

// returns false for a zero-area mesh
bool sample(const double* V, const int32_t* F, int64_t nf, int64_t n, uint64_t seed, double* pts, int32_t* fid,
            double* total_area) {
  std::vector<double> area(nf);
  double amax = 0.0, tot = 0.0;
  for (int64_t f = 0; f < nf; ++f) {
    area[f] = face_area(V, F + 3 * f);
    amax = std::max(amax, area[f]);
    tot += area[f];
  }
  if (!(amax > 0.0)) return false;
  std::vector<uint64_t> cum(nf);
  uint64_t W = 0;
  for (int64_t f = 0; f < nf; ++f) {
    W += static_cast<uint64_t>(std::floor(area[f] / amax * 4294967296.0));
    cum[f] = W;
  }
  if (total_area) *total_area = tot;
  parallel_for(n, [&](int64_t i) {
    const uint64_t h0 = hash_k(seed, 3 * i), h1 = hash_k(seed, 3 * i + 1), h2 = hash_k(seed, 3 * i + 2);
    const uint64_t t = static_cast<uint64_t>((static_cast<unsigned __int128>(h0) * W) >> 64);
    const int64_t f = std::upper_bound(cum.begin(), cum.end(), t) - cum.begin();
    const double u1 = unit53(h1), u2 = unit53(h2);
    const double s = std::sqrt(u1);
    const double wa = 1.0 - s, wb = s * (1.0 - u2), wc = s * u2;
    const V3 a = P(V, F[3 * f]), b = P(V, F[3 * f + 1]), c = P(V, F[3 * f + 2]);
    pts[3 * i] = (a.x * wa + b.x * wb) + c.x * wc;
    pts[3 * i + 1] = (a.y * wa + b.y * wb) + c.y * wc;
    pts[3 * i + 2] = (a.z * wa + b.z * wb) + c.z * wc;
    if (fid) fid[i] = static_cast<int32_t>(f);
  }, 64);
  return true;
}

// max corner cosine over the mesh; a zero-area face counts as cos = 1 (angle 0)
double max_corner_cos(const double* V, const int32_t* F, int64_t nf) {
  double m = -1.0;
  for (int64_t f = 0; f < nf; ++f) {
    const V3 p[3] = {P(V, F[3 * f]), P(V, F[3 * f + 1]), P(V, F[3 * f + 2])};
    if (!(sqnorm(cross(p[1] - p[0], p[2] - p[0])) > 0.0)) return 1.0;
    for (int k = 0; k < 3; ++k) {
      const V3 u = p[(k + 1) % 3] - p[k], w = p[(k + 2) % 3] - p[k];
      double c = dot(u, w) / std::sqrt(sqnorm(u) * sqnorm(w));
      c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
      m = std::max(m, c);
    }
  }
  return m;
}

}  // namespace metrics
}  // namespace orc

using namespace orc::metrics;

extern "C" {

static Topo g_topo;

// out = {manifold, watertight, euler, boundary_edges, n_nonmanifold_edges, n_nonmanifold_vertices}
void orc_topology(const int32_t* F, int64_t nf, int64_t nv, int64_t* out) {
  g_topo = Topo();
  topology(F, nf, nv, g_topo);
  out[0] = g_topo.manifold;
  out[1] = g_topo.watertight;
  out[2] = g_topo.euler;
  out[3] = g_topo.boundary;
  out[4] = static_cast<int64_t>(g_topo.nm_edges.size());
  out[5] = static_cast<int64_t>(g_topo.nm_verts.size());
}

void orc_topology_lists(int64_t* edges, int32_t* verts) {
  if (edges) std::memcpy(edges, g_topo.nm_edges.data(), g_topo.nm_edges.size() * 8);
  if (verts) std::memcpy(verts, g_topo.nm_verts.data(), g_topo.nm_verts.size() * 4);
}

void orc_nearest(const double* V, const int32_t* F, int64_t nf, const double* pts, int64_t n, int32_t* face,
                 double* dist, double* closest) {
  nearest(V, F, nf, pts, n, face, dist, closest);
}

// returns 0, or -1 for a zero-area mesh
int orc_sample(const double* V, const int32_t* F, int64_t nf, int64_t n, uint64_t seed, double* pts, int32_t* fid,
               double* total_area) {
  return sample(V, F, nf, n, seed, pts, fid, total_area) ? 0 : -1;
}

double orc_max_corner_cos(const double* V, const int32_t* F, int64_t nf) { return max_corner_cos(V, F, nf); }

}  // extern "C"

// ORACLE (test infrastructure only) — self-intersection detection restated from
// SPEC.md:399-471 and PAPER.md:196-217,811-919.
//
// Pinned verdict.  Faces f1,f2 (f1 != f2):
//   candidates: inflated (1e-7, lbvh.hpp:72) closed AABB overlap (types.hpp:43-45) —
//               exactly the pairs the reference LBVH broad phase returns (lbvh.cpp:182-190);
//   duplicate (3 shared indices) or degenerate (exactly collinear) face -> intersecting
//               (SPEC.md:443);
//   shared s = index intersection count; coplanar <=> T2's three vertices
//               have exact orientation 0 w.r.t. T1's plane (exact predicates: every verdict
//               is exact, so there are no false negatives by construction);
//   non-coplanar: s=0 Guigue-Devillers closed test (touching counts);
//                 s=1 true iff the intersection is longer than the shared point
//                     (positive-length rule of SPEC.md:422 evaluated exactly, delta -> 0);
//                 s=2 false;
//   coplanar:     s=0 closed 2D test; s=1 angular-sector overlap beyond the apex
//                 (zero cross products resolved by dot signs);
//                 s=2 apexes strictly on the same side of the shared edge.
#include <algorithm>
#include <atomic>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "geom.hpp"
#include "par.hpp"

namespace orc {
namespace isect {


// ---- non-coplanar, no shared vertex: Guigue & Devillers (2003), closed, exact -------
static int o3(V3 a, V3 b, V3 c, V3 d) { return orient3d(a, b, c, d); }

static bool check_min_max(V3 p1, V3 q1, V3 r1, V3 p2, V3 q2, V3 r2) {
  if (o3(q2, p2, p1, q1) > 0) return false;
  if (o3(r2, p2, r1, p1) > 0) return false;
  return true;
}

static bool tri_tri_3d(V3 p1, V3 q1, V3 r1, V3 p2, V3 q2, V3 r2, int dp2, int dq2, int dr2) {
  if (dp2 > 0) {
    if (dq2 > 0) return check_min_max(p1, r1, q1, r2, p2, q2);
    if (dr2 > 0) return check_min_max(p1, r1, q1, q2, r2, p2);
    return check_min_max(p1, q1, r1, p2, q2, r2);
  }
  if (dp2 < 0) {
    if (dq2 < 0) return check_min_max(p1, q1, r1, r2, p2, q2);
    if (dr2 < 0) return check_min_max(p1, q1, r1, q2, r2, p2);
    return check_min_max(p1, r1, q1, p2, q2, r2);
  }
  if (dq2 < 0) {
    if (dr2 >= 0) return check_min_max(p1, r1, q1, q2, r2, p2);
    return check_min_max(p1, q1, r1, p2, q2, r2);
  }
  if (dq2 > 0) {
    if (dr2 > 0) return check_min_max(p1, r1, q1, p2, q2, r2);
    return check_min_max(p1, q1, r1, q2, r2, p2);
  }
  if (dr2 > 0) return check_min_max(p1, q1, r1, r2, p2, q2);
  if (dr2 < 0) return check_min_max(p1, r1, q1, r2, p2, q2);
  return true;  // unreachable (coplanar handled by the caller)
}

static bool noncoplanar_disjoint_vertices(V3 p1, V3 q1, V3 r1, V3 p2, V3 q2, V3 r2) {
  const int dp1 = o3(p1, p2, q2, r2), dq1 = o3(q1, p2, q2, r2), dr1 = o3(r1, p2, q2, r2);
  if (dp1 * dq1 > 0 && dp1 * dr1 > 0) return false;
  const int dp2 = o3(p2, p1, q1, r1), dq2 = o3(q2, p1, q1, r1), dr2 = o3(r2, p1, q1, r1);
  if (dp2 * dq2 > 0 && dp2 * dr2 > 0) return false;
  if (dp1 > 0) {
    if (dq1 > 0) return tri_tri_3d(r1, p1, q1, p2, r2, q2, dp2, dr2, dq2);
    if (dr1 > 0) return tri_tri_3d(q1, r1, p1, p2, r2, q2, dp2, dr2, dq2);
    return tri_tri_3d(p1, q1, r1, p2, q2, r2, dp2, dq2, dr2);
  }
  if (dp1 < 0) {
    if (dq1 < 0) return tri_tri_3d(r1, p1, q1, p2, q2, r2, dp2, dq2, dr2);
    if (dr1 < 0) return tri_tri_3d(q1, r1, p1, p2, q2, r2, dp2, dq2, dr2);
    return tri_tri_3d(p1, q1, r1, p2, r2, q2, dp2, dr2, dq2);
  }
  if (dq1 < 0) {
    if (dr1 >= 0) return tri_tri_3d(q1, r1, p1, p2, r2, q2, dp2, dr2, dq2);
    return tri_tri_3d(p1, q1, r1, p2, q2, r2, dp2, dq2, dr2);
  }
  if (dq1 > 0) {
    if (dr1 > 0) return tri_tri_3d(p1, q1, r1, p2, r2, q2, dp2, dr2, dq2);
    return tri_tri_3d(q1, r1, p1, p2, q2, r2, dp2, dq2, dr2);
  }
  if (dr1 > 0) return tri_tri_3d(r1, p1, q1, p2, q2, r2, dp2, dq2, dr2);
  if (dr1 < 0) return tri_tri_3d(r1, p1, q1, p2, r2, q2, dp2, dr2, dq2);
  return true;  // unreachable
}

// ---- non-coplanar, one shared vertex A: T1=(A,B,C), T2=(A,D,E) ----------------------
static bool noncoplanar_shared_vertex(V3 A, V3 B, V3 C, V3 D, V3 E) {
  const int oB = o3(B, A, D, E), oC = o3(C, A, D, E);
  if (oB * oC > 0) return false;
  const int oD = o3(D, A, B, C), oE = o3(E, A, B, C);
  if (oD * oE > 0) return false;
  // P2 = DE ∩ plane(T1); test P2 inside the closed sector (AB, AC) using Z off the plane
  int sP, sC, tP, tB;
  if (oD != 0) {  // Z = D, P2 = D + s(E-D), s in (0,1]
    sP = o3(A, B, E, D);
    sC = o3(A, B, C, D);
    tP = o3(A, C, E, D);
    tB = o3(A, C, B, D);
  } else {  // P2 = D, Z = E
    sP = o3(A, B, D, E);
    sC = o3(A, B, C, E);
    tP = o3(A, C, D, E);
    tB = o3(A, C, B, E);
  }
  return sP * sC >= 0 && tP * tB >= 0;
}

// ---- coplanar helpers (projection dropping axis `drop`) --------------------------------
struct P2 {
  double x, y;
};
static P2 proj(V3 p, int drop) {
  if (drop == 0) return P2{p.y, p.z};
  if (drop == 1) return P2{p.z, p.x};
  return P2{p.x, p.y};
}
static int o2(P2 a, P2 b, P2 c) { return orient2d(a.x, a.y, b.x, b.y, c.x, c.y); }

// closed segment intersection in 2D
static bool on_seg_collinear(P2 p, P2 a, P2 b) {
  return std::min(a.x, b.x) <= p.x && p.x <= std::max(a.x, b.x) && std::min(a.y, b.y) <= p.y &&
         p.y <= std::max(a.y, b.y);
}
static bool seg_seg(P2 a, P2 b, P2 c, P2 d) {
  const int d1 = o2(a, b, c), d2 = o2(a, b, d), d3 = o2(c, d, a), d4 = o2(c, d, b);
  if (d1 * d2 < 0 && d3 * d4 < 0) return true;
  if (d1 == 0 && on_seg_collinear(c, a, b)) return true;
  if (d2 == 0 && on_seg_collinear(d, a, b)) return true;
  if (d3 == 0 && on_seg_collinear(a, c, d)) return true;
  if (d4 == 0 && on_seg_collinear(b, c, d)) return true;
  return false;
}
static bool point_in_tri(P2 p, P2 a, P2 b, P2 c) {
  const int s1 = o2(a, b, p), s2 = o2(b, c, p), s3 = o2(c, a, p);
  const bool has_neg = s1 < 0 || s2 < 0 || s3 < 0;
  const bool has_pos = s1 > 0 || s2 > 0 || s3 > 0;
  return !(has_neg && has_pos);
}
static bool coplanar_disjoint_vertices(const P2* t1, const P2* t2) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (seg_seg(t1[i], t1[(i + 1) % 3], t2[j], t2[(j + 1) % 3])) return true;
  if (point_in_tri(t1[0], t2[0], t2[1], t2[2])) return true;
  if (point_in_tri(t2[0], t1[0], t1[1], t1[2])) return true;
  return false;
}

// sign of dot(U-A, V-A) for collinear (A,U,V) with U,V != A: compare a nonzero coordinate
static int collinear_dot_sign(P2 A, P2 U, P2 V) {
  if (U.x != A.x) return ((U.x > A.x) == (V.x > A.x)) ? 1 : -1;
  return ((U.y > A.y) == (V.y > A.y)) ? 1 : -1;
}
// ray A->U inside the closed sector from ray A->P (ccw) to ray A->Q (angle < pi)
static bool ray_in_sector(P2 A, P2 P, P2 Q, P2 U) {
  const int s1 = o2(A, P, U), s2 = o2(A, U, Q);
  if (s1 < 0 || s2 < 0) return false;
  if (s1 == 0 && collinear_dot_sign(A, P, U) < 0) return false;
  if (s2 == 0 && collinear_dot_sign(A, Q, U) < 0) return false;
  return true;
}
static bool coplanar_shared_vertex(P2 A, P2 B, P2 C, P2 D, P2 E) {
  if (o2(A, B, C) < 0) std::swap(B, C);
  if (o2(A, D, E) < 0) std::swap(D, E);
  return ray_in_sector(A, B, C, D) || ray_in_sector(A, B, C, E) || ray_in_sector(A, D, E, B) ||
         ray_in_sector(A, D, E, C);
}

}  // namespace isect

// degenerate <=> the exact normal is the zero vector (all three projections collinear)
static bool degenerate(V3 a, V3 b, V3 c) {
  return orient2d(a.y, a.z, b.y, b.z, c.y, c.z) == 0 && orient2d(a.z, a.x, b.z, b.x, c.z, c.x) == 0 &&
         orient2d(a.x, a.y, b.x, b.y, c.x, c.y) == 0;
}

bool tri_tri_verdict(const int32_t* t1, const int32_t* t2, const double* v) {
  using namespace isect;
  auto P = [&](int i) { return v3(v[3 * i], v[3 * i + 1], v[3 * i + 2]); };
  int shared = 0;
  int s1[3] = {-1, -1, -1}, s2[3] = {-1, -1, -1};  // s1[k]: index in t2 equal to t1[k]
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (t1[i] == t2[j]) {
        s1[i] = j;
        s2[j] = i;
        ++shared;
      }
  if (shared == 3) return true;
  const V3 a = P(t1[0]), b = P(t1[1]), c = P(t1[2]);
  const V3 d = P(t2[0]), e = P(t2[1]), f = P(t2[2]);
  if (degenerate(a, b, c) || degenerate(d, e, f)) return true;
  // shared vertices lie on T1's plane by definition: only the unshared ones are tested
  const V3 T2v[3] = {d, e, f};
  bool coplanar = true;
  for (int j = 0; j < 3 && coplanar; ++j)
    if (s2[j] < 0 && orient3d(T2v[j], a, b, c) != 0) coplanar = false;
  if (!coplanar) {
    if (shared == 2) return false;
    if (shared == 0) return noncoplanar_disjoint_vertices(a, b, c, d, e, f);
    // one shared vertex: rotate so it comes first in both
    int i1 = 0;
    while (s1[i1] < 0) ++i1;
    const int j1 = s1[i1];
    const V3 T1[3] = {a, b, c}, T2[3] = {d, e, f};
    return noncoplanar_shared_vertex(T1[i1], T1[(i1 + 1) % 3], T1[(i1 + 2) % 3], T2[(j1 + 1) % 3],
                                     T2[(j1 + 2) % 3]);
  }
  // coplanar: projection axis = first (by decreasing |n_i| of the double normal, ties low i)
  // whose exact 2D orientation of T1 is nonzero
  const V3 n = cross(b - a, c - a);
  const double an[3] = {std::fabs(n.x), std::fabs(n.y), std::fabs(n.z)};
  int order[3] = {0, 1, 2};
  std::stable_sort(order, order + 3, [&](int x, int y) { return an[x] > an[y]; });
  int drop = order[0];
  for (int k = 0; k < 3; ++k) {
    const P2 pa = proj(a, order[k]), pb = proj(b, order[k]), pc = proj(c, order[k]);
    if (o2(pa, pb, pc) != 0) {
      drop = order[k];
      break;
    }
  }
  const V3 T1[3] = {a, b, c}, T2[3] = {d, e, f};
  P2 p1[3], p2[3];
  for (int k = 0; k < 3; ++k) {
    p1[k] = proj(T1[k], drop);
    p2[k] = proj(T2[k], drop);
  }
  if (shared == 0) return coplanar_disjoint_vertices(p1, p2);
  if (shared == 1) {
    int i1 = 0;
    while (s1[i1] < 0) ++i1;
    const int j1 = s1[i1];
    return coplanar_shared_vertex(p1[i1], p1[(i1 + 1) % 3], p1[(i1 + 2) % 3], p2[(j1 + 1) % 3],
                                  p2[(j1 + 2) % 3]);
  }
  // shared == 2: apex of each triangle = its unshared vertex
  int ia = 0, ja = 0;
  while (s1[ia] >= 0) ++ia;
  while (s2[ja] >= 0) ++ja;
  const int sa = (ia + 1) % 3, sb = (ia + 2) % 3;  // the shared edge A,B in T1
  const int oc = o2(p1[sa], p1[sb], p1[ia]), odd = o2(p1[sa], p1[sb], p2[ja]);
  return oc * odd > 0;
}

struct Box {
  V3 lo, hi;
};
Box face_box(const int32_t* t, const double* v) {
  Box b;
  const double inf = std::numeric_limits<double>::infinity();
  b.lo = v3(inf, inf, inf);
  b.hi = v3(-inf, -inf, -inf);
  for (int k = 0; k < 3; ++k) {
    const V3 p = v3(v[3 * t[k]], v[3 * t[k] + 1], v[3 * t[k] + 2]);
    b.lo = v3(p.x < b.lo.x ? p.x : b.lo.x, p.y < b.lo.y ? p.y : b.lo.y, p.z < b.lo.z ? p.z : b.lo.z);
    b.hi = v3(b.hi.x < p.x ? p.x : b.hi.x, b.hi.y < p.y ? p.y : b.hi.y, b.hi.z < p.z ? p.z : b.hi.z);
  }
  const double r = 1e-7;
  b.lo = v3(b.lo.x - r, b.lo.y - r, b.lo.z - r);
  b.hi = v3(b.hi.x + r, b.hi.y + r, b.hi.z + r);
  return b;
}
bool box_overlap(const Box& a, const Box& b) {
  return a.lo.x <= b.hi.x && a.lo.y <= b.hi.y && a.lo.z <= b.hi.z && a.hi.x >= b.lo.x &&
         a.hi.y >= b.lo.y && a.hi.z >= b.lo.z;
}

// Intersecting pairs (i<j) among `alive` faces where at least one of i,j has query[i]!=0
// (query == nullptr: every alive face).  The candidate set is the closed inflated-AABB overlap
// set (lbvh.cpp:182-190 semantics): a uniform hashed grid over the query faces (cell edge 1.5x
// their mean box extent) is probed by every alive face, each pair examined in the first common
// cell of the two cell ranges; faces covering more than kMaxCells cells are paired by a direct
// scan.  Only the set matters (it is sorted and deduplicated), never the grid.
std::vector<std::pair<int32_t, int32_t>> detect_pairs(const double* v, const int32_t* f, int64_t nf,
                                                      const uint8_t* alive, const uint8_t* query) {
  constexpr int64_t kMaxCells = 64, kChunk = 4096;
  struct Range {
    int64_t lo[3], hi[3];
    int64_t count() const { return (hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1); }
  };
  const int64_t nchunk = (nf + kChunk - 1) / kChunk;
  auto live = [&](int64_t i) { return !alive || alive[i]; };
  auto in_build = [&](int64_t i) { return live(i) && (!query || query[i]); };
  std::vector<Box> boxes(nf);
  // boxes, and the build set (ascending ids) by a chunked count / scan / fill
  std::vector<int64_t> coff(nchunk + 1, 0);
  parallel_for(nchunk, [&](int64_t c) {
    int64_t n = 0;
    for (int64_t i = c * kChunk; i < std::min(nf, (c + 1) * kChunk); ++i) {
      if (!live(i)) continue;
      boxes[i] = face_box(f + 3 * i, v);
      n += in_build(i);
    }
    coff[c + 1] = n;
  }, 1);
  for (int64_t c = 0; c < nchunk; ++c) coff[c + 1] += coff[c];
  std::vector<int32_t> build(coff[nchunk]);
  parallel_for(nchunk, [&](int64_t c) {
    int64_t k = coff[c];
    for (int64_t i = c * kChunk; i < std::min(nf, (c + 1) * kChunk); ++i)
      if (in_build(i)) build[k++] = static_cast<int32_t>(i);
  }, 1);
  if (build.empty()) return {};
  const int64_t nb_ = static_cast<int64_t>(build.size());
  const int64_t nbc = (nb_ + kChunk - 1) / kChunk;
  std::vector<double> ext_part(nbc, 0.0);
  parallel_for(nbc, [&](int64_t c) {
    double e = 0.0;
    for (int64_t k = c * kChunk; k < std::min(nb_, (c + 1) * kChunk); ++k) {
      const Box& x = boxes[build[k]];
      e += std::max(std::max(x.hi.x - x.lo.x, x.hi.y - x.lo.y), x.hi.z - x.lo.z);
    }
    ext_part[c] = e;
  }, 1);
  double ext = 0.0;
  for (double e : ext_part) ext += e;
  const double mean = ext / static_cast<double>(nb_);
  const double inv_h = 1.0 / (1.5 * (mean > 0.0 ? mean : 1e-3));
  auto range_of = [&](const Box& b) {
    Range r;
    const double lo[3] = {b.lo.x, b.lo.y, b.lo.z}, hi[3] = {b.hi.x, b.hi.y, b.hi.z};
    for (int k = 0; k < 3; ++k) {
      r.lo[k] = static_cast<int64_t>(std::floor(lo[k] * inv_h));
      r.hi[k] = static_cast<int64_t>(std::floor(hi[k] * inv_h));
    }
    return r;
  };
  auto hash = [](int64_t x, int64_t y, int64_t z, uint64_t mask) {
    uint64_t h = static_cast<uint64_t>(x) * 0x9E3779B97F4A7C15ull ^ static_cast<uint64_t>(y) * 0xC2B2AE3D27D4EB4Full ^
                 static_cast<uint64_t>(z) * 0x165667B19E3779F9ull;
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 32;
    return h & mask;
  };
  // hashed uniform grid over the build set: counting sort of (cell, face) entries into buckets
  // (parallel count with atomics, serial scan, parallel fill; the order inside a bucket does not
  // matter: the emitted pair set is sorted and deduplicated at the end)
  std::vector<Range> brange(nb_);
  std::vector<int64_t> ncell_part(nbc, 0);
  parallel_for(nbc, [&](int64_t c) {
    int64_t n = 0;
    for (int64_t k = c * kChunk; k < std::min(nb_, (c + 1) * kChunk); ++k) {
      brange[k] = range_of(boxes[build[k]]);
      const int64_t cc = brange[k].count();
      if (cc <= kMaxCells) n += cc;
    }
    ncell_part[c] = n;
  }, 1);
  int64_t nent = 0;
  for (int64_t n : ncell_part) nent += n;
  std::vector<int32_t> big;
  for (int64_t k = 0; k < nb_; ++k)
    if (brange[k].count() > kMaxCells) big.push_back(build[k]);
  uint64_t nbk = 1024;
  while (nbk < static_cast<uint64_t>(2 * nent + 1)) nbk <<= 1;
  const uint64_t mask = nbk - 1;
  struct Entry {
    int32_t face;
    int64_t lo[3];
  };
  std::vector<std::atomic<uint32_t>> bcnt(nbk);
  for (auto& x : bcnt) x.store(0, std::memory_order_relaxed);
  auto for_cells = [&](const Range& r, auto&& fn) {
    for (int64_t z = r.lo[2]; z <= r.hi[2]; ++z)
      for (int64_t y = r.lo[1]; y <= r.hi[1]; ++y)
        for (int64_t x = r.lo[0]; x <= r.hi[0]; ++x) fn(x, y, z);
  };
  parallel_for(nbc, [&](int64_t c) {
    for (int64_t k = c * kChunk; k < std::min(nb_, (c + 1) * kChunk); ++k) {
      if (brange[k].count() > kMaxCells) continue;
      for_cells(brange[k], [&](int64_t x, int64_t y, int64_t z) {
        bcnt[hash(x, y, z, mask)].fetch_add(1, std::memory_order_relaxed);
      });
    }
  }, 1);
  std::vector<uint32_t> boff(nbk + 1, 0);
  for (uint64_t h = 0; h < nbk; ++h) {
    boff[h + 1] = boff[h] + bcnt[h].load(std::memory_order_relaxed);
    bcnt[h].store(boff[h], std::memory_order_relaxed);  // reused as the fill cursor
  }
  std::vector<Entry> ent(static_cast<size_t>(nent));
  parallel_for(nbc, [&](int64_t c) {
    for (int64_t k = c * kChunk; k < std::min(nb_, (c + 1) * kChunk); ++k) {
      const Range& r = brange[k];
      if (r.count() > kMaxCells) continue;
      for_cells(r, [&](int64_t x, int64_t y, int64_t z) {
        ent[bcnt[hash(x, y, z, mask)].fetch_add(1, std::memory_order_relaxed)] =
            Entry{build[k], {r.lo[0], r.lo[1], r.lo[2]}};
      });
    }
  }, 1);
  std::vector<uint8_t> is_build(nf, 0);
  parallel_for(nb_, [&](int64_t k) { is_build[build[k]] = 1; }, kChunk);
  // probe: every alive face walks its cells; a pair is examined in the first common cell of the
  // two ranges; (p, b) with both in the build set only from p < b
  std::vector<std::vector<std::pair<int32_t, int32_t>>> found(nchunk);
  parallel_for(nchunk, [&](int64_t ch) {
    auto& out = found[ch];
    for (int64_t pi = ch * kChunk; pi < std::min(nf, (ch + 1) * kChunk); ++pi) {
      if (!live(pi)) continue;
      const int32_t p = static_cast<int32_t>(pi);
      const Box& bp = boxes[p];
      auto consider = [&](int32_t b) {
        if (b == p || (is_build[p] && b < p)) return;
        if (!box_overlap(bp, boxes[b])) return;
        if (tri_tri_verdict(f + 3 * p, f + 3 * b, v)) out.emplace_back(std::min(p, b), std::max(p, b));
      };
      const Range rp = range_of(bp);
      if (rp.count() > kMaxCells) {  // huge probe: scan the build set (big build faces below)
        for (int64_t j = 0; j < nb_; ++j)
          if (brange[j].count() <= kMaxCells) consider(build[j]);
      } else {
        for_cells(rp, [&](int64_t x, int64_t y, int64_t z) {
          const uint64_t h = hash(x, y, z, mask);
          for (uint32_t e = boff[h]; e < boff[h + 1]; ++e) {
            const Entry& en = ent[e];
            if (x == std::max(rp.lo[0], en.lo[0]) && y == std::max(rp.lo[1], en.lo[1]) &&
                z == std::max(rp.lo[2], en.lo[2]))
              consider(en.face);
          }
        });
      }
      for (int32_t b : big) consider(b);
    }
  }, 1);
  std::vector<std::pair<int32_t, int32_t>> out;
  for (auto& x : found) out.insert(out.end(), x.begin(), x.end());
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

}  // namespace orc

using namespace orc;

extern "C" {

int orc_tri_tri(const double* tri1, const double* tri2, int shared_mask_dummy) {
  (void)shared_mask_dummy;
  // geometry-only entry: six distinct vertex ids (0-shared)
  double v[18];
  std::memcpy(v, tri1, 9 * 8);
  std::memcpy(v + 9, tri2, 9 * 8);
  const int32_t t1[3] = {0, 1, 2}, t2[3] = {3, 4, 5};
  return tri_tri_verdict(t1, t2, v) ? 1 : 0;
}

// verdict for a list of face-index pairs of a mesh
void orc_tri_tri_pairs(const double* v, const int32_t* f, const int32_t* pairs, int64_t n,
                       int32_t* out) {
  parallel_for(n, [&](int64_t i) {
    out[i] = tri_tri_verdict(f + 3 * pairs[2 * i], f + 3 * pairs[2 * i + 1], v) ? 1 : 0;
  });
}

int orc_orient3d(const double* a, const double* b, const double* c, const double* d) {
  return orient3d(v3(a[0], a[1], a[2]), v3(b[0], b[1], b[2]), v3(c[0], c[1], c[2]), v3(d[0], d[1], d[2]));
}

// detect_self_intersections: sorted (f1<f2) pairs.  Count-then-fill.
int64_t orc_self_intersections(const double* v, int64_t nv, const int32_t* f, int64_t nf,
                               int32_t* pairs, int64_t cap) {
  (void)nv;
  const auto out = detect_pairs(v, f, nf, nullptr, nullptr);
  const int64_t n = static_cast<int64_t>(out.size());
  if (pairs)
    for (int64_t i = 0; i < std::min(n, cap); ++i) {
      pairs[2 * i] = out[i].first;
      pairs[2 * i + 1] = out[i].second;
    }
  return n;
}

// all candidate pairs (closed inflated-AABB overlap), for broad-phase equivalence tests
int64_t orc_overlap_pairs(const double* v, const int32_t* f, int64_t nf, int32_t* pairs, int64_t cap) {
  std::vector<Box> boxes(nf);
  for (int64_t i = 0; i < nf; ++i) boxes[i] = face_box(f + 3 * i, v);
  int64_t n = 0;
  for (int64_t i = 0; i < nf; ++i)
    for (int64_t j = i + 1; j < nf; ++j)
      if (box_overlap(boxes[i], boxes[j])) {
        if (pairs && n < cap) {
          pairs[2 * n] = static_cast<int32_t>(i);
          pairs[2 * n + 1] = static_cast<int32_t>(j);
        }
        ++n;
      }
  return n;
}

}  // extern "C"

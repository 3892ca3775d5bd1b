// isect.cu — fully parallel self-intersection detection (PAPER.md:196-217,
// 811-919): uniform hashed-grid broad phase + exact triangle-triangle narrow phase.
//
// Broad phase.  The reference uses an LBVH over 1e-7-inflated boxes (lbvh.cpp:159-190,
// lbvh.hpp:72).  Here: boxes of a build set A are binned (counting sort into a hashed uniform
// grid, cell size = mean box extent) and every probe face of set B walks the cells its box
// covers; a pair is examined exactly once per probe, in the cell max(lo_a, lo_b) of the two
// cell ranges.  The candidate set is a superset of the closed inflated-AABB overlap pairs and
// the exact box test then reduces it to exactly the reference's set, so the output does not
// depend on the grid.  Faces covering more than kMaxCells cells are kept in a "big" list that
// every probe scans directly.
//
// Narrow phase: duplicate / degenerate faces intersect; shared-vertex count by
// index; coplanarity by exact orientation; non-coplanar: 0 shared -> Guigue-Devillers closed
// test, 1 shared -> positive-length rule, 2 shared -> false; coplanar: 0 shared -> closed 2D
// test, 1 shared -> angular-sector overlap, 2 shared -> apexes on the same side.  All
// predicates are exact (exact.cuh), so every verdict is exact.
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"
#include "exact.cuh"
#include "kernels.cuh"

namespace pcu {

struct IsectScratch {
  DevBuf<double> boxes;      // 6 per build entry
  DevBuf<uint32_t> bcount, boff, bcur;
  DevBuf<int32_t> entries;   // face ids by bucket
  DevBuf<int32_t> big;
  DevBuf<unsigned long long> counters;  // [0] entries, [1] big, [2] pairs
  DevBuf<double> ext_sum;
  DevBuf<uint8_t> in_build;
  DevBuf<uint64_t> cand;
  DevBuf<float> fbox;  // 6 floats per face
};

IsectScratch* isect_scratch_create() { return new IsectScratch(); }
void isect_scratch_destroy(IsectScratch* s) { delete s; }

namespace {

constexpr int kMaxCells = 64;

struct Box {
  double lo[3], hi[3];
};

__device__ __forceinline__ D3 vtx(const double* V, int i) { return D3{V[3 * i], V[3 * i + 1], V[3 * i + 2]}; }

__device__ __forceinline__ Box face_box(const double* V, const int32_t* t) {
  Box b;
  const D3 p0 = vtx(V, t[0]), p1 = vtx(V, t[1]), p2 = vtx(V, t[2]);
  b.lo[0] = fmin(fmin(p0.x, p1.x), p2.x) - 1e-7;
  b.lo[1] = fmin(fmin(p0.y, p1.y), p2.y) - 1e-7;
  b.lo[2] = fmin(fmin(p0.z, p1.z), p2.z) - 1e-7;
  b.hi[0] = fmax(fmax(p0.x, p1.x), p2.x) + 1e-7;
  b.hi[1] = fmax(fmax(p0.y, p1.y), p2.y) + 1e-7;
  b.hi[2] = fmax(fmax(p0.z, p1.z), p2.z) + 1e-7;
  return b;
}

__device__ __forceinline__ bool overlap(const Box& a, const Box& b) {
  return a.lo[0] <= b.hi[0] && a.lo[1] <= b.hi[1] && a.lo[2] <= b.hi[2] && a.hi[0] >= b.lo[0] &&
         a.hi[1] >= b.lo[1] && a.hi[2] >= b.lo[2];
}

// conservative float copy of the inflated box (lo rounded down, hi rounded up): the float
// overlap test admits a superset of the double-box pairs; the exact test runs in k_narrow
struct FBox {
  float lo[3], hi[3];
};

__device__ __forceinline__ bool overlap(const FBox& a, const FBox& b) {
  return a.lo[0] <= b.hi[0] && a.lo[1] <= b.hi[1] && a.lo[2] <= b.hi[2] && a.hi[0] >= b.lo[0] &&
         a.hi[1] >= b.lo[1] && a.hi[2] >= b.lo[2];
}

struct CellRange {
  int64_t lo[3], hi[3];
  __device__ int64_t count() const { return (hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1); }
};

__device__ __forceinline__ CellRange cells_of(const Box& b, double inv_h) {
  CellRange r;
  for (int k = 0; k < 3; ++k) {
    r.lo[k] = static_cast<int64_t>(floor(b.lo[k] * inv_h));
    r.hi[k] = static_cast<int64_t>(floor(b.hi[k] * inv_h));
  }
  return r;
}

__device__ __forceinline__ CellRange cells_of(const FBox& b, double inv_h) {
  CellRange r;
  for (int k = 0; k < 3; ++k) {
    r.lo[k] = static_cast<int64_t>(floor(static_cast<double>(b.lo[k]) * inv_h));
    r.hi[k] = static_cast<int64_t>(floor(static_cast<double>(b.hi[k]) * inv_h));
  }
  return r;
}

__device__ __forceinline__ uint32_t cell_hash(int64_t x, int64_t y, int64_t z, uint32_t mask) {
  uint64_t h = static_cast<uint64_t>(x) * 0x9E3779B97F4A7C15ull ^ static_cast<uint64_t>(y) * 0xC2B2AE3D27D4EB4Full ^
               static_cast<uint64_t>(z) * 0x165667B19E3779F9ull;
  h ^= h >> 29;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 32;
  return static_cast<uint32_t>(h) & mask;
}

// ------------------------------------------------------------------ narrow phase (device)
__device__ __forceinline__ bool check_min_max(D3 p1, D3 q1, D3 r1, D3 p2, D3 q2, D3 r2) {
  if (orient3d(q2, p2, p1, q1) > 0) return false;
  if (orient3d(r2, p2, r1, p1) > 0) return false;
  return true;
}

__device__ bool gd_3d(D3 p1, D3 q1, D3 r1, D3 p2, D3 q2, D3 r2, int dp2, int dq2, int dr2) {
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
  return true;
}

__device__ bool gd_disjoint(D3 p1, D3 q1, D3 r1, D3 p2, D3 q2, D3 r2) {
  const int dp1 = orient3d(p1, p2, q2, r2), dq1 = orient3d(q1, p2, q2, r2), dr1 = orient3d(r1, p2, q2, r2);
  if (dp1 * dq1 > 0 && dp1 * dr1 > 0) return false;
  const int dp2 = orient3d(p2, p1, q1, r1), dq2 = orient3d(q2, p1, q1, r1), dr2 = orient3d(r2, p1, q1, r1);
  if (dp2 * dq2 > 0 && dp2 * dr2 > 0) return false;
  if (dp1 > 0) {
    if (dq1 > 0) return gd_3d(r1, p1, q1, p2, r2, q2, dp2, dr2, dq2);
    if (dr1 > 0) return gd_3d(q1, r1, p1, p2, r2, q2, dp2, dr2, dq2);
    return gd_3d(p1, q1, r1, p2, q2, r2, dp2, dq2, dr2);
  }
  if (dp1 < 0) {
    if (dq1 < 0) return gd_3d(r1, p1, q1, p2, q2, r2, dp2, dq2, dr2);
    if (dr1 < 0) return gd_3d(q1, r1, p1, p2, q2, r2, dp2, dq2, dr2);
    return gd_3d(p1, q1, r1, p2, r2, q2, dp2, dr2, dq2);
  }
  if (dq1 < 0) {
    if (dr1 >= 0) return gd_3d(q1, r1, p1, p2, r2, q2, dp2, dr2, dq2);
    return gd_3d(p1, q1, r1, p2, q2, r2, dp2, dq2, dr2);
  }
  if (dq1 > 0) {
    if (dr1 > 0) return gd_3d(p1, q1, r1, p2, r2, q2, dp2, dr2, dq2);
    return gd_3d(q1, r1, p1, p2, q2, r2, dp2, dq2, dr2);
  }
  if (dr1 > 0) return gd_3d(r1, p1, q1, p2, q2, r2, dp2, dq2, dr2);
  if (dr1 < 0) return gd_3d(r1, p1, q1, p2, r2, q2, dp2, dr2, dq2);
  return true;
}

// T1=(A,B,C), T2=(A,D,E) non-coplanar: intersection longer than the shared point?
__device__ bool shared_vertex_3d(D3 A, D3 B, D3 C, D3 D, D3 E) {
  if (orient3d(B, A, D, E) * orient3d(C, A, D, E) > 0) return false;
  const int oD = orient3d(D, A, B, C), oE = orient3d(E, A, B, C);
  if (oD * oE > 0) return false;
  const D3 Z = oD != 0 ? D : E;   // a vertex of T2 off the plane of T1
  const D3 P = oD != 0 ? E : D;   // the side of the crossing point of DE with that plane
  const int sP = orient3d(A, B, P, Z), sC = orient3d(A, B, C, Z);
  const int tP = orient3d(A, C, P, Z), tB = orient3d(A, C, B, Z);
  return sP * sC >= 0 && tP * tB >= 0;
}

struct P2 {
  double x, y;
};
__device__ __forceinline__ P2 proj2(D3 p, int drop) {
  return drop == 0 ? P2{p.y, p.z} : (drop == 1 ? P2{p.z, p.x} : P2{p.x, p.y});
}
__device__ __forceinline__ int o2(P2 a, P2 b, P2 c) { return orient2d(a.x, a.y, b.x, b.y, c.x, c.y); }

__device__ __forceinline__ bool in_span(P2 p, P2 a, P2 b) {
  return fmin(a.x, b.x) <= p.x && p.x <= fmax(a.x, b.x) && fmin(a.y, b.y) <= p.y && p.y <= fmax(a.y, b.y);
}
__device__ bool seg_seg2(P2 a, P2 b, P2 c, P2 d) {
  const int d1 = o2(a, b, c), d2 = o2(a, b, d), d3 = o2(c, d, a), d4 = o2(c, d, b);
  if (d1 * d2 < 0 && d3 * d4 < 0) return true;
  return (d1 == 0 && in_span(c, a, b)) || (d2 == 0 && in_span(d, a, b)) || (d3 == 0 && in_span(a, c, d)) ||
         (d4 == 0 && in_span(b, c, d));
}
__device__ bool inside2(P2 p, P2 a, P2 b, P2 c) {
  const int s1 = o2(a, b, p), s2 = o2(b, c, p), s3 = o2(c, a, p);
  return !((s1 < 0 || s2 < 0 || s3 < 0) && (s1 > 0 || s2 > 0 || s3 > 0));
}
__device__ int collinear_dot(P2 A, P2 U, P2 V) {
  if (U.x != A.x) return ((U.x > A.x) == (V.x > A.x)) ? 1 : -1;
  return ((U.y > A.y) == (V.y > A.y)) ? 1 : -1;
}
__device__ bool ray_in(P2 A, P2 P, P2 Q, P2 U) {
  const int s1 = o2(A, P, U), s2 = o2(A, U, Q);
  if (s1 < 0 || s2 < 0) return false;
  if (s1 == 0 && collinear_dot(A, P, U) < 0) return false;
  if (s2 == 0 && collinear_dot(A, Q, U) < 0) return false;
  return true;
}

// degenerate <=> the exact normal is zero (all three projected orientations are zero).  The
// filtered determinants certify most faces non-degenerate without any exact evaluation.
__device__ __forceinline__ bool certainly_nonzero2(double ax, double ay, double bx, double by, double cx, double cy) {
  const double l = (ax - cx) * (by - cy), r = (ay - cy) * (bx - cx);
  const double det = l - r;
  return fabs(det) > (3.0 + 16.0 * 1.1102230246251565e-16) * 1.1102230246251565e-16 * (fabs(l) + fabs(r));
}
__device__ bool degenerate(D3 a, D3 b, D3 c) {
  if (certainly_nonzero2(a.x, a.y, b.x, b.y, c.x, c.y) || certainly_nonzero2(a.y, a.z, b.y, b.z, c.y, c.z) ||
      certainly_nonzero2(a.z, a.x, b.z, b.x, c.z, c.x))
    return false;
  return orient2d(a.y, a.z, b.y, b.z, c.y, c.z) == 0 && orient2d(a.z, a.x, b.z, b.x, c.z, c.x) == 0 &&
         orient2d(a.x, a.y, b.x, b.y, c.x, c.y) == 0;
}

__device__ bool verdict(const double* __restrict__ V, const int32_t* t1, const int32_t* t2) {
  int s1[3] = {-1, -1, -1}, s2[3] = {-1, -1, -1}, shared = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (t1[i] == t2[j]) {
        s1[i] = j;
        s2[j] = i;
        ++shared;
      }
  if (shared == 3) return true;
  const D3 T1[3] = {vtx(V, t1[0]), vtx(V, t1[1]), vtx(V, t1[2])};
  const D3 T2[3] = {vtx(V, t2[0]), vtx(V, t2[1]), vtx(V, t2[2])};
  if (degenerate(T1[0], T1[1], T1[2]) || degenerate(T2[0], T2[1], T2[2])) return true;
  // coplanar <=> every vertex of T2 lies on T1's plane (shared vertices trivially do)
  bool coplanar = true;
  for (int j = 0; j < 3 && coplanar; ++j)
    if (s2[j] < 0 && orient3d(T2[j], T1[0], T1[1], T1[2]) != 0) coplanar = false;
  if (!coplanar) {
    if (shared == 2) return false;
    if (shared == 0) return gd_disjoint(T1[0], T1[1], T1[2], T2[0], T2[1], T2[2]);
    int i1 = 0;
    while (s1[i1] < 0) ++i1;
    const int j1 = s1[i1];
    return shared_vertex_3d(T1[i1], T1[(i1 + 1) % 3], T1[(i1 + 2) % 3], T2[(j1 + 1) % 3], T2[(j1 + 2) % 3]);
  }
  // projection: decreasing |n_i| of the double normal (ties -> lower axis), first with a
  // nonzero exact 2D orientation of T1
  const D3 n = cross(sub(T1[1], T1[0]), sub(T1[2], T1[0]));
  const double an[3] = {fabs(n.x), fabs(n.y), fabs(n.z)};
  int ord[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i)  // stable insertion sort, descending
    for (int j = i; j > 0 && an[ord[j]] > an[ord[j - 1]]; --j) {
      const int t = ord[j];
      ord[j] = ord[j - 1];
      ord[j - 1] = t;
    }
  int drop = ord[0];
  for (int k = 0; k < 3; ++k)
    if (o2(proj2(T1[0], ord[k]), proj2(T1[1], ord[k]), proj2(T1[2], ord[k])) != 0) {
      drop = ord[k];
      break;
    }
  P2 p1[3], p2[3];
  for (int k = 0; k < 3; ++k) {
    p1[k] = proj2(T1[k], drop);
    p2[k] = proj2(T2[k], drop);
  }
  if (shared == 0) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        if (seg_seg2(p1[i], p1[(i + 1) % 3], p2[j], p2[(j + 1) % 3])) return true;
    return inside2(p1[0], p2[0], p2[1], p2[2]) || inside2(p2[0], p1[0], p1[1], p1[2]);
  }
  if (shared == 1) {
    int i1 = 0;
    while (s1[i1] < 0) ++i1;
    const int j1 = s1[i1];
    const P2 A = p1[i1];
    P2 B = p1[(i1 + 1) % 3], C = p1[(i1 + 2) % 3], D = p2[(j1 + 1) % 3], E = p2[(j1 + 2) % 3];
    if (o2(A, B, C) < 0) {
      const P2 t = B;
      B = C;
      C = t;
    }
    if (o2(A, D, E) < 0) {
      const P2 t = D;
      D = E;
      E = t;
    }
    return ray_in(A, B, C, D) || ray_in(A, B, C, E) || ray_in(A, D, E, B) || ray_in(A, D, E, C);
  }
  int ia = 0, ja = 0;
  while (s1[ia] >= 0) ++ia;
  while (s2[ja] >= 0) ++ja;
  const P2 A = p1[(ia + 1) % 3], B = p1[(ia + 2) % 3];
  return o2(A, B, p1[ia]) * o2(A, B, p2[ja]) > 0;
}

// ------------------------------------------------------------------------ grid kernels
__global__ void k_fboxes(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t nf,
                         const uint8_t* __restrict__ alive, FBox* __restrict__ out) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  FBox fb;
  if (alive && !alive[f]) {
    for (int k = 0; k < 3; ++k) {
      fb.lo[k] = __int_as_float(0x7f800000);
      fb.hi[k] = __int_as_float(0xff800000);
    }
  } else {
    const Box b = face_box(V, F + 3 * f);
    for (int k = 0; k < 3; ++k) {
      fb.lo[k] = __double2float_rd(b.lo[k]);
      fb.hi[k] = __double2float_ru(b.hi[k]);
    }
  }
  out[f] = fb;
}

__global__ void k_ext_sum(const FBox* __restrict__ B, const int32_t* __restrict__ ids, int64_t n,
                          const uint8_t* __restrict__ alive, double* __restrict__ out) {
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  double s = 0.0;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t f = ids ? ids[k] : k;
    if (alive && !alive[f]) continue;
    const FBox& b = B[f];
    s += fmax(fmax(b.hi[0] - b.lo[0], b.hi[1] - b.lo[1]), b.hi[2] - b.lo[2]);
  }
  const double t = BR(tmp).Sum(s);
  if (threadIdx.x == 0) atomicAdd(out, t);
}

// pass 0: count bucket entries (or big); pass 1: fill
__global__ void k_bin(const FBox* __restrict__ B, const int32_t* __restrict__ ids, int64_t n,
                      const uint8_t* __restrict__ alive, double inv_h, uint32_t mask, int pass,
                      uint32_t* __restrict__ bcount, const uint32_t* __restrict__ boff, uint32_t* __restrict__ bcur,
                      int32_t* __restrict__ entries, int32_t* __restrict__ big, unsigned long long* counters) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const int32_t f = ids ? ids[k] : static_cast<int32_t>(k);
  if (alive && !alive[f]) return;
  const CellRange cr = cells_of(B[f], inv_h);
  if (cr.count() > kMaxCells) {
    if (pass == 1) big[atomicAdd(&counters[1], 1ull)] = f;
    return;
  }
  for (int64_t z = cr.lo[2]; z <= cr.hi[2]; ++z)
    for (int64_t y = cr.lo[1]; y <= cr.hi[1]; ++y)
      for (int64_t x = cr.lo[0]; x <= cr.hi[0]; ++x) {
        const uint32_t h = cell_hash(x, y, z, mask);
        if (pass == 0) atomicAdd(&bcount[h], 1u);
        else entries[boff[h] + atomicAdd(&bcur[h], 1u)] = f;
      }
}

// Broad phase: every probe face p walks the cells its box covers and emits candidate pairs
// (p, a) with a in the build grid and overlapping (conservative float) boxes.  `sym` = probe
// set == build set (each unordered pair once); otherwise a pair of two build faces is emitted
// only from its smaller probe.
__global__ void __launch_bounds__(128) k_probe(const FBox* __restrict__ B, int64_t n, const uint8_t* __restrict__ alive,
                                               double inv_h, uint32_t mask, const uint32_t* __restrict__ bcount,
                                               const uint32_t* __restrict__ boff, const int32_t* __restrict__ entries,
                                               const int32_t* __restrict__ big, int64_t nbig, int sym,
                                               const uint8_t* __restrict__ in_build, uint64_t* __restrict__ cand,
                                               uint64_t cap, unsigned long long* __restrict__ ncand,
                                               const int32_t* __restrict__ probe_ids) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const int32_t p = probe_ids ? probe_ids[k] : static_cast<int32_t>(k);
  if (alive && !alive[p]) return;
  const bool p_build = sym || (in_build && in_build[p]);
  const FBox bp = B[p];
  const CellRange cp = cells_of(bp, inv_h);
  auto consider = [&](int32_t a, const FBox& ba) {
    if (a == p) return;
    if (p_build && a < p) return;  // the pair is emitted from probe a instead
    if (!overlap(bp, ba)) return;
    const unsigned long long slot = atomicAdd(ncand, 1ull);
    if (slot < cap) cand[slot] = (static_cast<uint64_t>(static_cast<uint32_t>(p)) << 32) | static_cast<uint32_t>(a);
  };
  if (cp.count() > kMaxCells) {
    // huge probe: scan the whole build set, each entry once (in the bucket of its first cell)
    for (uint32_t h = 0; h <= mask; ++h)
      for (uint32_t e = boff[h]; e < boff[h] + bcount[h]; ++e) {
        const int32_t a = entries[e];
        const FBox ba = B[a];
        const CellRange ca = cells_of(ba, inv_h);
        if (cell_hash(ca.lo[0], ca.lo[1], ca.lo[2], mask) != h) continue;
        consider(a, ba);
      }
  } else {
    for (int64_t z = cp.lo[2]; z <= cp.hi[2]; ++z)
      for (int64_t y = cp.lo[1]; y <= cp.hi[1]; ++y)
        for (int64_t x = cp.lo[0]; x <= cp.hi[0]; ++x) {
          const uint32_t h = cell_hash(x, y, z, mask);
          const uint32_t e1 = boff[h] + bcount[h];
          for (uint32_t e = boff[h]; e < e1; ++e) {
            const int32_t a = entries[e];
            const FBox ba = B[a];
            const CellRange ca = cells_of(ba, inv_h);
            // the entry really covers (x,y,z) and this is the first common cell of the two ranges
            if (x < ca.lo[0] || x > ca.hi[0] || y < ca.lo[1] || y > ca.hi[1] || z < ca.lo[2] || z > ca.hi[2]) continue;
            if (x != max(cp.lo[0], ca.lo[0]) || y != max(cp.lo[1], ca.lo[1]) || z != max(cp.lo[2], ca.lo[2])) continue;
            consider(a, ba);
          }
        }
  }
  for (int64_t b = 0; b < nbig; ++b) consider(big[b], B[big[b]]);
}

// Narrow phase over candidate pairs.  mode 0: append intersecting pairs (min, max);
// mode 1: flag the applied owners of both faces for revert (QEM undo loop).
__global__ void __launch_bounds__(128) k_narrow(const double* __restrict__ V, const int32_t* __restrict__ F,
                                                const uint64_t* __restrict__ cand, int64_t n, int mode,
                                                int32_t* __restrict__ pairs, uint64_t cap,
                                                unsigned long long* __restrict__ npairs,
                                                const int32_t* __restrict__ owner, const uint8_t* __restrict__ applied,
                                                uint8_t* __restrict__ revert) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int32_t p = static_cast<int32_t>(cand[i] >> 32), a = static_cast<int32_t>(cand[i] & 0xffffffffu);
  // the reference candidate set: closed overlap of the 1e-7-inflated double boxes
  if (!overlap(face_box(V, F + 3 * p), face_box(V, F + 3 * a))) return;
  if (mode == 1) {
    // only pairs whose owners can still be reverted matter
    const int32_t op = owner[p], oa = owner[a];
    const bool rp = op >= 0 && applied[op], ra = oa >= 0 && applied[oa];
    if (!rp && !ra) return;
    if (rp && ra && revert[op] && revert[oa]) return;  // both already flagged
    if (!verdict(V, F + 3 * p, F + 3 * a)) return;
    atomicAdd(npairs, 1ull);
    if (rp) revert[op] = 1;
    if (ra) revert[oa] = 1;
  } else {
    if (!verdict(V, F + 3 * p, F + 3 * a)) return;
    const unsigned long long k = atomicAdd(npairs, 1ull);
    if (k < cap) {
      pairs[2 * k] = min(p, a);
      pairs[2 * k + 1] = max(p, a);
    }
  }
}

__global__ void k_verdict_pairs(const double* __restrict__ V, const int32_t* __restrict__ F,
                                const int32_t* __restrict__ pairs, int64_t n, int32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  out[i] = verdict(V, F + 3 * pairs[2 * i], F + 3 * pairs[2 * i + 1]) ? 1 : 0;
}

uint32_t pow2_at_least(uint64_t x) {
  uint32_t p = 1024;
  while (p < x && p < (1u << 30)) p <<= 1;
  return p;
}

// Builds the grid over (ids or all alive faces) from the float boxes; returns (inv_h, mask, nbig).
void build_grid(Ctx& ctx, IsectScratch& S, const int32_t* d_ids, int64_t n, const uint8_t* d_alive, double& inv_h,
                uint32_t& mask, int64_t& nbig, int64_t n_alive_hint) {
  const FBox* B = reinterpret_cast<const FBox*>(S.fbox.get());
  S.ext_sum.ensure(1, ctx.stream);
  S.ext_sum.memset(0, ctx.stream);
  PCU_LAUNCH(ctx, k_ext_sum, static_cast<unsigned>(std::min<int64_t>(grid_for(n, 256), ctx.num_sms * 4)), 256, 0, B,
             d_ids, n, d_alive, S.ext_sum.get());
  const double sum = read_scalar(ctx, S.ext_sum.get());
  const double mean = n_alive_hint > 0 ? sum / static_cast<double>(n_alive_hint) : 1.0;
  const double h = mean > 0.0 ? mean : 1e-3;
  inv_h = 1.0 / h;
  const uint32_t nb = pow2_at_least(static_cast<uint64_t>(n_alive_hint) * 2 + 1);
  mask = nb - 1;
  S.bcount.ensure(nb, ctx.stream);
  S.boff.ensure(nb, ctx.stream);
  S.bcur.ensure(nb, ctx.stream);
  S.counters.ensure(4, ctx.stream);
  PCU_CUDA(cudaMemsetAsync(S.bcount.get(), 0, nb * 4, ctx.stream));
  PCU_CUDA(cudaMemsetAsync(S.bcur.get(), 0, nb * 4, ctx.stream));
  S.counters.memset(0, ctx.stream);
  S.big.ensure(1, ctx.stream);
  PCU_LAUNCH(ctx, k_bin, grid_for(n, 256), 256, 0, B, d_ids, n, d_alive, inv_h, mask, 0, S.bcount.get(), S.boff.get(),
             S.bcur.get(), nullptr, nullptr, S.counters.get());
  exclusive_scan_u32(ctx, S.bcount.get(), S.boff.get(), nb);
  const uint64_t total = static_cast<uint64_t>(read_scalar(ctx, S.boff.get() + nb - 1)) + read_scalar(ctx, S.bcount.get() + nb - 1);
  S.entries.ensure(total ? total : 1, ctx.stream);
  S.big.ensure(static_cast<size_t>(n > 0 ? n : 1), ctx.stream);
  PCU_LAUNCH(ctx, k_bin, grid_for(n, 256), 256, 0, B, d_ids, n, d_alive, inv_h, mask, 1, S.bcount.get(), S.boff.get(),
             S.bcur.get(), S.entries.get(), S.big.get(), S.counters.get());
  unsigned long long nb_big = 0;
  PCU_CUDA(cudaMemcpyAsync(&nb_big, S.counters.get() + 1, 8, cudaMemcpyDeviceToHost, ctx.stream));
  PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  nbig = static_cast<int64_t>(nb_big);
}

void make_fboxes(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf, const uint8_t* d_alive) {
  S.fbox.ensure(6 * static_cast<size_t>(nf > 0 ? nf : 1), ctx.stream);
  PCU_LAUNCH(ctx, k_fboxes, grid_for(nf, 256), 256, 0, dV, dF, nf, d_alive, reinterpret_cast<FBox*>(S.fbox.get()));
}

__global__ void k_flag_ids(const int32_t* __restrict__ ids, int64_t n, uint8_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) flag[ids[i]] = 1;
}

int64_t probe_candidates(Ctx& ctx, IsectScratch& S, int64_t nf, const uint8_t* d_alive, double inv_h, uint32_t mask,
                         int64_t nbig, int sym, const uint8_t* in_build, const int32_t* probe_ids = nullptr) {
  uint64_t cap = std::max<uint64_t>(S.cand.n, static_cast<uint64_t>(nf) * 4 + 1024);
  const FBox* B = reinterpret_cast<const FBox*>(S.fbox.get());
  while (true) {
    S.cand.ensure(cap, ctx.stream);
    PCU_CUDA(cudaMemsetAsync(S.counters.get() + 3, 0, 8, ctx.stream));
    PCU_LAUNCH(ctx, k_probe, grid_for(nf, 128), 128, 0, B, nf, d_alive, inv_h, mask, S.bcount.get(), S.boff.get(),
               S.entries.get(), S.big.get(), nbig, sym, in_build, S.cand.get(), S.cand.n, S.counters.get() + 3,
               probe_ids);
    const uint64_t got = read_scalar(ctx, S.counters.get() + 3);
    if (got <= S.cand.n) return static_cast<int64_t>(got);
    cap = got + got / 4 + 1024;
  }
}

}  // namespace

std::vector<int32_t> self_intersections(Ctx& ctx, const double* dV, int64_t nv, const int32_t* dF, int64_t nf,
                                        const uint8_t* d_alive, const uint8_t* d_query) {
  (void)nv;
  (void)d_query;
  std::vector<int32_t> out;
  if (nf < 2) return out;
  IsectScratch S;
  double inv_h;
  uint32_t mask;
  int64_t nbig;
  make_fboxes(ctx, S, dV, dF, nf, d_alive);
  build_grid(ctx, S, nullptr, nf, d_alive, inv_h, mask, nbig, nf);
  const int64_t ncand = probe_candidates(ctx, S, nf, d_alive, inv_h, mask, nbig, 1, nullptr);
  uint64_t cap = 1024;
  while (true) {
    DevBuf<int32_t> pairs(2 * cap, ctx.stream);
    PCU_CUDA(cudaMemsetAsync(S.counters.get() + 2, 0, 8, ctx.stream));
    if (ncand)
      PCU_LAUNCH(ctx, k_narrow, grid_for(ncand, 128), 128, 0, dV, dF, S.cand.get(), ncand, 0, pairs.get(), cap,
                 S.counters.get() + 2, nullptr, nullptr, nullptr);
    const uint64_t got = read_scalar(ctx, S.counters.get() + 2);
    if (got > cap) {
      cap = got + 1024;
      continue;
    }
    out.resize(2 * got);
    if (got) PCU_CUDA(cudaMemcpyAsync(out.data(), pairs.get(), got * 8, cudaMemcpyDeviceToHost, ctx.stream));
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    break;
  }
  std::vector<std::pair<int32_t, int32_t>> pv(out.size() / 2);
  for (size_t i = 0; i < pv.size(); ++i) pv[i] = {out[2 * i], out[2 * i + 1]};
  std::sort(pv.begin(), pv.end());
  pv.erase(std::unique(pv.begin(), pv.end()), pv.end());
  out.resize(2 * pv.size());
  for (size_t i = 0; i < pv.size(); ++i) {
    out[2 * i] = pv[i].first;
    out[2 * i + 1] = pv[i].second;
  }
  return out;
}

void tri_tri_pairs(Ctx& ctx, const double* dV, const int32_t* dF, const int32_t* d_pairs, int64_t n, int32_t* d_out) {
  if (n == 0) return;
  PCU_LAUNCH(ctx, k_verdict_pairs, grid_for(n, 128), 128, 0, dV, dF, d_pairs, n, d_out);
}

int64_t undo_detect(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf,
                    const uint8_t* d_falive, const int32_t* d_query_faces, int64_t n_query, const int32_t* d_owner,
                    const uint8_t* d_applied, uint8_t* d_revert) {
  if (n_query == 0) return 0;
  double inv_h;
  uint32_t mask;
  int64_t nbig;
  // grid over the (few) query faces, probed by every alive face
  ctx.prof.mark(ctx.stream, "undo_detect:pre");
  make_fboxes(ctx, S, dV, dF, nf, d_falive);
  build_grid(ctx, S, d_query_faces, n_query, d_falive, inv_h, mask, nbig, n_query);
  S.in_build.ensure(nf, ctx.stream);
  PCU_CUDA(cudaMemsetAsync(S.in_build.get(), 0, nf, ctx.stream));
  PCU_LAUNCH(ctx, k_flag_ids, grid_for(n_query, 256), 256, 0, d_query_faces, n_query, S.in_build.get());
  ctx.prof.mark(ctx.stream, "undo_detect:grid");
  const int64_t ncand = probe_candidates(ctx, S, nf, d_falive, inv_h, mask, nbig, 0, S.in_build.get());
  ctx.prof.mark(ctx.stream, "undo_detect:broad");
  if (ncand == 0) return 0;
  PCU_CUDA(cudaMemsetAsync(S.counters.get() + 2, 0, 8, ctx.stream));
  PCU_LAUNCH(ctx, k_narrow, grid_for(ncand, 128), 128, 0, dV, dF, S.cand.get(), ncand, 1, nullptr, 0,
             S.counters.get() + 2, d_owner, d_applied, d_revert);
  return static_cast<int64_t>(read_scalar(ctx, S.counters.get() + 2));
}

// Later undo rounds: only pairs (restored face, face owned by an applied collapse) can be new —
// every other pair is unchanged since the previous round's check.  Grid over the restored
// faces, probed by the owned faces.
int64_t undo_detect_restored(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf,
                             const uint8_t* d_falive, const int32_t* d_restored, int64_t n_restored,
                             const int32_t* d_owned, int64_t n_owned, const int32_t* d_owner,
                             const uint8_t* d_applied, uint8_t* d_revert) {
  if (n_restored == 0 || n_owned == 0) return 0;
  double inv_h;
  uint32_t mask;
  int64_t nbig;
  make_fboxes(ctx, S, dV, dF, nf, d_falive);
  build_grid(ctx, S, d_restored, n_restored, d_falive, inv_h, mask, nbig, n_restored);
  ctx.prof.mark(ctx.stream, "undo_detect:grid");
  const int64_t ncand = probe_candidates(ctx, S, n_owned, d_falive, inv_h, mask, nbig, 0, nullptr, d_owned);
  ctx.prof.mark(ctx.stream, "undo_detect:broad");
  if (ncand == 0) return 0;
  PCU_CUDA(cudaMemsetAsync(S.counters.get() + 2, 0, 8, ctx.stream));
  PCU_LAUNCH(ctx, k_narrow, grid_for(ncand, 128), 128, 0, dV, dF, S.cand.get(), ncand, 1, nullptr, 0,
             S.counters.get() + 2, d_owner, d_applied, d_revert);
  return static_cast<int64_t>(read_scalar(ctx, S.counters.get() + 2));
}

}  // namespace pcu

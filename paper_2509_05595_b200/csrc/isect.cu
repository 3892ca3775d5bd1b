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
#include <cstdlib>

#include "common.cuh"
#include "exact.cuh"
#include "kernels.cuh"

namespace pcu {

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
// Out-of-line orientation: the narrow phase calls it ~20 times; inlining every copy blew the
// instruction cache (ncu: `no_instruction` stalls) and the register budget.
__device__ __noinline__ int o3(D3 a, D3 b, D3 c, D3 d) { return orient3d(a, b, c, d); }
__device__ __forceinline__ bool check_min_max(D3 p1, D3 q1, D3 r1, D3 p2, D3 q2, D3 r2) {
  if (o3(q2, p2, p1, q1) > 0) return false;
  if (o3(r2, p2, r1, p1) > 0) return false;
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

// T1=(A,B,C), T2=(A,D,E) non-coplanar: intersection longer than the shared point?  oD, oE are
// the exact orientations of D and E against T1's plane (the caller's coplanarity test made them;
// a cyclic rotation of T1 keeps their signs), so a same-side pair costs no further predicate.
__device__ bool shared_vertex_3d(D3 A, D3 B, D3 C, D3 D, D3 E, int oD, int oE) {
  if (oD * oE > 0) return false;
  if (o3(B, A, D, E) * o3(C, A, D, E) > 0) return false;
  const D3 Z = oD != 0 ? D : E;   // a vertex of T2 off the plane of T1
  const D3 P = oD != 0 ? E : D;   // the side of the crossing point of DE with that plane
  const int sP = o3(A, B, P, Z), sC = o3(A, B, C, Z);
  const int tP = o3(A, C, P, Z), tB = o3(A, C, B, Z);
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

struct PairInfo {
  int s1[3], s2[3];  // s1[k]: index in t2 of t1's vertex k (or -1); s2 likewise
  int shared;
};

__device__ __forceinline__ PairInfo pair_info(const int32_t* t1, const int32_t* t2) {
  PairInfo I{{-1, -1, -1}, {-1, -1, -1}, 0};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (t1[i] == t2[j]) {
        I.s1[i] = j;
        I.s2[j] = i;
        ++I.shared;
      }
  return I;
}

// projection for coplanar pairs: decreasing |n_i| of T1's double normal (ties -> lower axis),
// the first axis whose exact 2D orientation of T1 is nonzero
__device__ int drop_axis(const D3* T1) {
  const D3 n = cross(sub(T1[1], T1[0]), sub(T1[2], T1[0]));
  const double an[3] = {fabs(n.x), fabs(n.y), fabs(n.z)};
  int ord[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i)
    for (int j = i; j > 0 && an[ord[j]] > an[ord[j - 1]]; --j) {
      const int t = ord[j];
      ord[j] = ord[j - 1];
      ord[j - 1] = t;
    }
  for (int k = 0; k < 3; ++k)
    if (o2(proj2(T1[0], ord[k]), proj2(T1[1], ord[k]), proj2(T1[2], ord[k])) != 0) return ord[k];
  return ord[0];
}

// non-degenerate, 0 shared vertices
__device__ __noinline__ bool verdict0(const double* __restrict__ V, const int32_t* t1, const int32_t* t2) {
  const D3 T1[3] = {vtx(V, t1[0]), vtx(V, t1[1]), vtx(V, t1[2])};
  const D3 T2[3] = {vtx(V, t2[0]), vtx(V, t2[1]), vtx(V, t2[2])};
  const int dp2 = o3(T2[0], T1[0], T1[1], T1[2]), dq2 = o3(T2[1], T1[0], T1[1], T1[2]),
            dr2 = o3(T2[2], T1[0], T1[1], T1[2]);
  if (dp2 != 0 || dq2 != 0 || dr2 != 0) {
    if (dp2 * dq2 > 0 && dp2 * dr2 > 0) return false;
    // Guigue-Devillers (closed), reusing the orientations of T2 w.r.t. T1
    const D3 p1 = T1[0], q1 = T1[1], r1 = T1[2], p2 = T2[0], q2 = T2[1], r2 = T2[2];
    const int dp1 = o3(p1, p2, q2, r2), dq1 = o3(q1, p2, q2, r2), dr1 = o3(r1, p2, q2, r2);
    if (dp1 * dq1 > 0 && dp1 * dr1 > 0) return false;
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
  const int drop = drop_axis(T1);
  P2 p1[3], p2[3];
  for (int k = 0; k < 3; ++k) {
    p1[k] = proj2(T1[k], drop);
    p2[k] = proj2(T2[k], drop);
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (seg_seg2(p1[i], p1[(i + 1) % 3], p2[j], p2[(j + 1) % 3])) return true;
  return inside2(p1[0], p2[0], p2[1], p2[2]) || inside2(p2[0], p1[0], p1[1], p1[2]);
}

// non-degenerate, exactly 1 shared vertex
__device__ __noinline__ bool verdict1(const double* __restrict__ V, const int32_t* t1, const int32_t* t2,
                                      const PairInfo& I) {
  const D3 T1[3] = {vtx(V, t1[0]), vtx(V, t1[1]), vtx(V, t1[2])};
  int i1 = 0;
  while (I.s1[i1] < 0) ++i1;
  const int j1 = I.s1[i1];
  const D3 D3d = vtx(V, t2[(j1 + 1) % 3]), E3d = vtx(V, t2[(j1 + 2) % 3]);  // T2's shared vertex is T1[i1]
  const int oD = o3(D3d, T1[0], T1[1], T1[2]), oE = o3(E3d, T1[0], T1[1], T1[2]);
  if (oD != 0 || oE != 0) return shared_vertex_3d(T1[i1], T1[(i1 + 1) % 3], T1[(i1 + 2) % 3], D3d, E3d, oD, oE);
  const int drop = drop_axis(T1);
  const P2 A = proj2(T1[i1], drop);
  P2 B = proj2(T1[(i1 + 1) % 3], drop), C = proj2(T1[(i1 + 2) % 3], drop);
  P2 D = proj2(D3d, drop), E = proj2(E3d, drop);
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

// verdict1 from filtered orientations only: 0/1 = the verdict (every predicate it needed was
// certified, so it equals verdict1's), 2 = undecided (an uncertain orientation, or a coplanar
// pair) -> the pair is re-run through verdict1 by a second pass.
__device__ __forceinline__ int verdict1_fast(const double* __restrict__ V, const int32_t* t1, const int32_t* t2,
                                             const PairInfo& I) {
  const D3 T1[3] = {vtx(V, t1[0]), vtx(V, t1[1]), vtx(V, t1[2])};
  int i1 = 0;
  while (I.s1[i1] < 0) ++i1;
  const int j1 = I.s1[i1];
  const D3 D = vtx(V, t2[(j1 + 1) % 3]), E = vtx(V, t2[(j1 + 2) % 3]);
  const int oD = orient3d_filtered(D, T1[0], T1[1], T1[2]), oE = orient3d_filtered(E, T1[0], T1[1], T1[2]);
  if (oD == 2 || oE == 2 || (oD == 0 && oE == 0)) return 2;
  // shared_vertex_3d, predicate for predicate
  if (oD * oE > 0) return 0;
  const D3 A = T1[i1], B = T1[(i1 + 1) % 3], C = T1[(i1 + 2) % 3];
  const int b1 = orient3d_filtered(B, A, D, E), c1 = orient3d_filtered(C, A, D, E);
  if (b1 == 2 || c1 == 2) return 2;
  if (b1 * c1 > 0) return 0;
  const D3 Z = oD != 0 ? D : E;
  const D3 P = oD != 0 ? E : D;
  const int sP = orient3d_filtered(A, B, P, Z), sC = orient3d_filtered(A, B, C, Z);
  const int tP = orient3d_filtered(A, C, P, Z), tB = orient3d_filtered(A, C, B, Z);
  if (sP == 2 || sC == 2 || tP == 2 || tB == 2) return 2;
  return sP * sC >= 0 && tP * tB >= 0 ? 1 : 0;
}

// non-degenerate, exactly 2 shared vertices
__device__ __noinline__ bool verdict2(const double* __restrict__ V, const int32_t* t1, const int32_t* t2,
                                      const PairInfo& I) {
  int ia = 0, ja = 0;
  while (I.s1[ia] >= 0) ++ia;
  while (I.s2[ja] >= 0) ++ja;
  const D3 T1[3] = {vtx(V, t1[0]), vtx(V, t1[1]), vtx(V, t1[2])};
  const D3 apex2 = vtx(V, t2[ja]);
  if (o3(apex2, T1[0], T1[1], T1[2]) != 0) return false;  // non-coplanar edge neighbours never cross
  const int drop = drop_axis(T1);
  const P2 A = proj2(T1[(ia + 1) % 3], drop), B = proj2(T1[(ia + 2) % 3], drop);
  return o2(A, B, proj2(T1[ia], drop)) * o2(A, B, proj2(apex2, drop)) > 0;
}

// full verdict (explicit pair API)
__device__ bool verdict(const double* __restrict__ V, const int32_t* t1, const int32_t* t2) {
  const PairInfo I = pair_info(t1, t2);
  if (I.shared == 3) return true;
  if (degenerate(vtx(V, t1[0]), vtx(V, t1[1]), vtx(V, t1[2])) || degenerate(vtx(V, t2[0]), vtx(V, t2[1]), vtx(V, t2[2])))
    return true;
  if (I.shared == 0) return verdict0(V, t1, t2);
  if (I.shared == 1) return verdict1(V, t1, t2, I);
  return verdict2(V, t1, t2, I);
}

// ------------------------------------------------------------------------ grid kernels
// Device-side scalars of one detection round: the launches below read sizes and the cell size
// from here, so a round issues no host synchronisation of its own.
struct DetectScalars {
  double ext_sum;
  double inv_h;
  unsigned long long nbig;
  unsigned long long ncand;
  unsigned long long found;
  unsigned long long npairs;
  unsigned long long ncls[3];
  unsigned long long nhuge;  // probes covering > kMaxCells cells, handed to k_probe_huge
  int redo;  // candidate buffer overflowed: the round's outputs are void, the caller repeats it
  unsigned ext_blocks;  // k_ext_sum blocks finished (the last one sets inv_h)
};

__device__ __forceinline__ FBox fbox_of(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t f,
                                        const uint8_t* __restrict__ alive, uint8_t* __restrict__ degen) {
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
    const int32_t* t = F + 3 * f;
    degen[f] = degenerate(vtx(V, t[0]), vtx(V, t[1]), vtx(V, t[2])) ? 1 : 0;
  }
  return fb;
}

__global__ void k_fboxes(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t n,
                         const uint8_t* __restrict__ alive, FBox* __restrict__ out, uint8_t* __restrict__ degen,
                         const int32_t* __restrict__ ids) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const int64_t f = ids ? ids[k] : k;
  out[f] = fbox_of(V, F, f, alive, degen);
}

// cell size = PCU_CELL_SCALE x the mean box extent of the build set; the block that finishes last
// turns the sum into inv_h (one launch instead of a reduction + a one-thread kernel)
#ifndef PCU_CELL_SCALE
#define PCU_CELL_SCALE 1.5
#endif
// With `fresh` (the QEM undo loop: the build set is exactly the faces a collapse batch or a
// revert just changed), the build faces' boxes and degenerate flags are recomputed here first.
__global__ void k_ext_sum(FBox* __restrict__ B, const int32_t* __restrict__ ids, int64_t n,
                          const uint8_t* __restrict__ alive, DetectScalars* ds, const double* __restrict__ V,
                          const int32_t* __restrict__ F, uint8_t* __restrict__ degen, int fresh) {
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  __shared__ bool last;
  double s = 0.0;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t f = ids ? ids[k] : k;
    FBox b;
    if (fresh) {
      b = fbox_of(V, F, f, alive, degen);
      B[f] = b;
    }
    if (alive && !alive[f]) continue;
    if (!fresh) b = B[f];
    s += fmax(fmax(b.hi[0] - b.lo[0], b.hi[1] - b.lo[1]), b.hi[2] - b.lo[2]);
  }
  const double t = BR(tmp).Sum(s);
  if (threadIdx.x == 0) {
    atomicAdd(&ds->ext_sum, t);
    __threadfence();
    last = atomicAdd(&ds->ext_blocks, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    const double sum = atomicAdd(&ds->ext_sum, 0.0);  // every block's contribution is visible
    const double mean = n > 0 ? sum / static_cast<double>(n) : 1.0;
    ds->inv_h = 1.0 / (PCU_CELL_SCALE * (mean > 0.0 ? mean : 1e-3));
  }
}

// pass 0: count bucket entries (or big); pass 1: fill
__global__ void k_bin(const FBox* __restrict__ B, const int32_t* __restrict__ ids, int64_t n,
                      const uint8_t* __restrict__ alive, DetectScalars* __restrict__ ds, uint32_t mask, int pass,
                      uint32_t* __restrict__ bcount, const uint32_t* __restrict__ boff, uint32_t* __restrict__ bcur,
                      int4* __restrict__ entries, int32_t* __restrict__ big, uint32_t* __restrict__ occ) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const int32_t f = ids ? ids[k] : static_cast<int32_t>(k);
  if (alive && !alive[f]) return;
  const CellRange cr = cells_of(B[f], ds->inv_h);
  if (cr.count() > kMaxCells) {
    if (pass == 1) big[agg_inc(&ds->nbig)] = f;
    return;
  }
  for (int64_t z = cr.lo[2]; z <= cr.hi[2]; ++z)
    for (int64_t y = cr.lo[1]; y <= cr.hi[1]; ++y)
      for (int64_t x = cr.lo[0]; x <= cr.hi[0]; ++x) {
        const uint32_t h = cell_hash(x, y, z, mask);
        if (pass == 0) {
          atomicAdd(&bcount[h], 1u);
          atomicOr(&occ[h >> 5], 1u << (h & 31));
        } else {
          entries[boff[h] + atomicAdd(&bcur[h], 1u)] =
              make_int4(f, static_cast<int>(cr.lo[0]), static_cast<int>(cr.lo[1]), static_cast<int>(cr.lo[2]));
        }
      }
}

// Broad phase: every probe face p walks the cells its box covers and emits candidate pairs
// (p, a) with a in the build grid and overlapping (conservative float) boxes, in the first
// common cell of the two cell ranges only.  `sym` = probe set == build set (each unordered pair
// once); otherwise a pair of two build faces is emitted only from its smaller probe.
// SIMT balance: probes differ wildly in work (0 .. 64 occupied cells), so lanes only enumerate
// their occupied cells into a per-warp queue of (owner lane, cell) records; whenever 32 records
// are queued the whole warp drains them, one cell's entry list per lane.  Probes covering more
// than kMaxCells cells go to k_probe_large.
__global__ void __launch_bounds__(128) k_probe(const FBox* __restrict__ B, int64_t n, const uint8_t* __restrict__ alive,
                                               const DetectScalars* __restrict__ ds, uint32_t mask,
                                               const uint32_t* __restrict__ bcount, const uint32_t* __restrict__ boff,
                                               const int4* __restrict__ entries, const int32_t* __restrict__ big,
                                               const uint32_t* __restrict__ occ, int sym,
                                               const int32_t* __restrict__ in_build, uint64_t* __restrict__ cand,
                                               uint64_t cap, unsigned long long* __restrict__ ncand,
                                               const int32_t* __restrict__ probe_ids, int32_t* __restrict__ huge,
                                               unsigned long long* __restrict__ nhuge,
                                               const uint8_t* __restrict__ in_probe, int ppw) {
  // candidates are staged in shared memory and flushed with one global atomic per block
  // (a single-address counter bumped per candidate serialises in the L2 atomic unit)
  constexpr int kBuf = 1024, kQ = 64;
  __shared__ uint64_t buf[kBuf];
  __shared__ unsigned int nbuf;
  __shared__ unsigned long long gbase;
  __shared__ FBox sbox[4][32];
  __shared__ int32_t sp[4][32];
  __shared__ int32_t slo[4][32][3];
  __shared__ uint8_t sbuild[4][32];
  __shared__ int32_t qc[4][kQ][3];
  __shared__ uint32_t qh[4][kQ];
  __shared__ uint8_t qo[4][kQ];
  __shared__ uint32_t spre[4][32], sbase[4][32];  // drain: inclusive entry-count prefix, first entry
  (void)big;
  if (threadIdx.x == 0) nbuf = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  // ppw probes per warp (lanes >= ppw only help drain): fewer for small probe sets, so a short
  // round spreads its (cell, entry) work over more warps
  const int64_t k = ((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5) * ppw + lane;
  int32_t p = -1;
  if (lane < ppw && k < n) {
    p = probe_ids ? probe_ids[k] : static_cast<int32_t>(k);
    if (alive && !alive[p]) p = -1;
  }
  const double inv_h = ds->inv_h;
  FBox bp{};
  CellRange cp{};
  bool p_build = false;
  int64_t ncell = 0;
  if (p >= 0) {
    p_build = sym || (in_build && in_build[p] >= 0);
    bp = B[p];
    cp = cells_of(bp, inv_h);
    ncell = cp.count();
    if (ncell > kMaxCells) {  // huge probe: k_probe_large scans the build set for it
      huge[agg_inc(nhuge)] = p;
      ncell = 0;
    }
  }
  sbox[warp][lane] = bp;
  sp[warp][lane] = p;
  for (int c = 0; c < 3; ++c) slo[warp][lane][c] = static_cast<int32_t>(cp.lo[c]);
  sbuild[warp][lane] = p_build ? 1 : 0;
  const int64_t nx = cp.hi[0] - cp.lo[0] + 1, ny = cp.hi[1] - cp.lo[1] + 1;
  int64_t ci = 0;
  int qn = 0;  // warp-uniform queue length
  __syncwarp();
  for (;;) {
    // fill: every lane contributes its next occupied cell (empty buckets are skipped via the
    // L2-resident occupancy bitmap)
    bool got = false;
    int32_t cx = 0, cy = 0, cz = 0;
    uint32_t ch = 0;
    while (ci < ncell) {
      cx = static_cast<int32_t>(cp.lo[0] + ci % nx);
      cy = static_cast<int32_t>(cp.lo[1] + (ci / nx) % ny);
      cz = static_cast<int32_t>(cp.lo[2] + ci / (nx * ny));
      ++ci;
      ch = cell_hash(cx, cy, cz, mask);
      if ((occ[ch >> 5] >> (ch & 31)) & 1u) {
        got = true;
        break;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, got);
    if (got) {
      const int pos = qn + __popc(m & lt);
      qc[warp][pos][0] = cx;
      qc[warp][pos][1] = cy;
      qc[warp][pos][2] = cz;
      qh[warp][pos] = ch;
      qo[warp][pos] = static_cast<uint8_t>(lane);
    }
    qn += __popc(m);
    const bool more = __any_sync(0xffffffffu, ci < ncell);
    if (qn >= 32 || (!more && qn > 0)) {
      __syncwarp();
      const int take = min(qn, 32);
      // lane r < take owns record qn - take + r; its cell's entry list is spread over the warp:
      // flattened (record, entry) index t -> record by a 5-step search of the warp's prefix sums
      uint32_t cnt = 0, e0 = 0;
      if (lane < take) {
        const uint32_t h = qh[warp][qn - take + lane];
        e0 = boff[h];
        cnt = bcount[h];
      }
      uint32_t incl = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      spre[warp][lane] = incl;
      sbase[warp][lane] = e0;
      __syncwarp();
      // warp-uniform trip count, so emitting lanes reserve their buffer slots with one shared
      // atomic per warp step instead of one per candidate
      for (uint32_t t0 = 0; t0 < total; t0 += 32) {
        const uint32_t t = t0 + lane;
        bool emit = false;
        uint64_t v = 0;
        if (t < total) {
          int lo = 0, hi = take - 1;  // first record whose inclusive prefix exceeds t
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (spre[warp][mid] > t) hi = mid;
            else lo = mid + 1;
          }
          const int r = qn - take + lo;
          const uint32_t e = sbase[warp][lo] + (t - (lo ? spre[warp][lo - 1] : 0u));
          const int o = qo[warp][r];
          const int32_t op = sp[warp][o];
          const int4 en = entries[e];  // face id + its first cell: the dedup test needs no box load
          // first common cell of the two ranges (a hash collision can at worst duplicate a pair)
          const int32_t a = en.x;
          emit = qc[warp][r][0] == max(slo[warp][o][0], en.y) && qc[warp][r][1] == max(slo[warp][o][1], en.z) &&
                 qc[warp][r][2] == max(slo[warp][o][2], en.w) &&
                 // a pair met from both sides (a also probes, op also in the grid): the smaller probe
                 !(a == op || (sbuild[warp][o] && a < op && (!in_probe || in_probe[a]))) &&
                 overlap(sbox[warp][o], B[a]);
          v = (static_cast<uint64_t>(static_cast<uint32_t>(op)) << 32) | static_cast<uint32_t>(a);
        }
        const unsigned em = __ballot_sync(0xffffffffu, emit);
        if (em == 0u) continue;
        unsigned base = 0;
        if (lane == __ffs(em) - 1) base = atomicAdd(&nbuf, static_cast<unsigned>(__popc(em)));
        base = __shfl_sync(0xffffffffu, base, __ffs(em) - 1);
        if (emit) {
          const unsigned slot = base + __popc(em & lt);
          if (slot < kBuf) {
            buf[slot] = v;
          } else {  // block buffer full: direct global append
            const unsigned long long g = agg_inc(ncand);
            if (g < cap) cand[g] = v;
          }
        }
      }
      __syncwarp();
      qn -= take;
    }
    if (!more && qn == 0) break;
  }
  // pairs with big build faces come from k_probe_large
  __syncthreads();
  const unsigned mm = min(nbuf, static_cast<unsigned>(kBuf));
  if (threadIdx.x == 0 && mm) gbase = atomicAdd(ncand, static_cast<unsigned long long>(mm));
  __syncthreads();
  for (unsigned i = threadIdx.x; i < mm; i += blockDim.x)
    if (gbase + i < cap) cand[gbase + i] = buf[i];
}

// Probes and build faces too large for the grid (their box covers more than kMaxCells cells),
// one warp each, in one launch:
//   * a huge probe p: lanes stride over the build set (ids, or every alive face), skipping the
//     big build faces (handled below);
//   * a big build face b: lanes stride over the probe set, pairs (x, b).
// Each pair is met exactly once, with k_probe's emission rules.
__global__ void __launch_bounds__(128) k_probe_large(const FBox* __restrict__ B, const DetectScalars* __restrict__ ds,
                                                     const int32_t* __restrict__ huge, const int32_t* __restrict__ big,
                                                     const int32_t* __restrict__ build_ids, int64_t n_build,
                                                     const int32_t* __restrict__ probe_ids, int64_t n_probe,
                                                     const uint8_t* __restrict__ alive, int sym,
                                                     const int32_t* __restrict__ in_build, uint64_t* __restrict__ cand,
                                                     uint64_t cap, unsigned long long* __restrict__ ncand,
                                                     const uint8_t* __restrict__ in_probe) {
  const unsigned long long nh = ds->nhuge, nb = ds->nbig;
  const double inv_h = ds->inv_h;
  const int lane = threadIdx.x & 31;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  auto emit = [&](int32_t p, int32_t a) {
    const unsigned long long g = agg_inc(ncand);
    if (g < cap) cand[g] = (static_cast<uint64_t>(static_cast<uint32_t>(p)) << 32) | static_cast<uint32_t>(a);
  };
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); w < nh + nb; w += nw) {
    if (w < nh) {
      const int32_t p = huge[w];
      const bool p_build = sym || (in_build && in_build[p] >= 0);
      const FBox bp = B[p];
      for (int64_t k = lane; k < n_build; k += 32) {
        const int32_t a = build_ids ? build_ids[k] : static_cast<int32_t>(k);
        if (alive && !alive[a]) continue;
        if (a == p || (p_build && a < p && (!in_probe || in_probe[a]))) continue;
        const FBox ba = B[a];
        if (!overlap(bp, ba)) continue;
        if (cells_of(ba, inv_h).count() > kMaxCells) continue;  // big build face: second half
        emit(p, a);
      }
    } else {
      const int32_t b = big[w - nh];
      const FBox bb = B[b];
      for (int64_t k = lane; k < n_probe; k += 32) {
        const int32_t x = probe_ids ? probe_ids[k] : static_cast<int32_t>(k);
        if (alive && !alive[x]) continue;
        if (x == b) continue;
        const bool x_build = sym || (in_build && in_build[x] >= 0);
        if (x_build && b < x && (!in_probe || in_probe[b])) continue;  // emitted from probe b instead
        if (!overlap(B[x], bb)) continue;
        emit(x, b);
      }
    }
  }
}

__device__ __forceinline__ void report(DetectScalars* ds, int mode, int32_t p, int32_t a, int32_t* pairs,
                                       uint64_t pair_cap, const int32_t* owner,
                                       uint8_t* revert) {
  if (mode == 1) {
    atomicAdd(&ds->found, 1ull);
    const int32_t op = owner[p], oa = owner[a];
    // owner[f] >= 0 exactly while its collapse is applied (k_collapse sets it only for applied
    // collapses, k_revert clears it together with applied), so no applied[] lookup is needed
    if (op >= 0) revert[op] = 1;
    if (oa >= 0) revert[oa] = 1;
  } else {
    const unsigned long long k = atomicAdd(&ds->npairs, 1ull);
    if (k < pair_cap) {
      pairs[2 * k] = min(p, a);
      pairs[2 * k + 1] = max(p, a);
    }
  }
}

// Narrow phase, stage 1 (grid-stride over the device-side candidate count): the exact
// inflated double-box test (the reference's candidate set), duplicates and degenerate faces
// (always intersecting) and the 2-shared verdict inline, then bucketing the 0/1-shared pairs so
// stage 2 runs one uniform code path per warp.  mode 1 (QEM undo): stage 2 skips pairs none of
// whose owners can still be reverted.
__device__ __forceinline__ bool deep_overlap(const FBox& a, const FBox& b) {
  bool ok = true;
  for (int k = 0; k < 3; ++k) {
    // shrink each float box by 2 ulps (a superset of the 1-ulp outward rounding) before testing
    const float alo = a.lo[k] + 2.5e-7f * fabsf(a.lo[k]) + 1e-30f, ahi = a.hi[k] - 2.5e-7f * fabsf(a.hi[k]) - 1e-30f;
    const float blo = b.lo[k] + 2.5e-7f * fabsf(b.lo[k]) + 1e-30f, bhi = b.hi[k] - 2.5e-7f * fabsf(b.hi[k]) - 1e-30f;
    ok = ok && alo <= bhi && ahi >= blo;
  }
  return ok;
}

__global__ void __launch_bounds__(256) k_classify(const double* __restrict__ V, const int32_t* __restrict__ F,
                                                  const FBox* __restrict__ B,
                                                  const uint8_t* __restrict__ degen, const uint64_t* __restrict__ cand,
                                                  uint64_t cap, DetectScalars* __restrict__ ds, int mode,
                                                  uint64_t* __restrict__ cls, int32_t* __restrict__ pairs,
                                                  uint64_t pair_cap, const int32_t* __restrict__ owner,
                                                  uint8_t* __restrict__ revert) {
  const unsigned long long n = ds->ncand;
  if (n > cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ds->redo = 1;
    return;
  }
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int32_t p = static_cast<int32_t>(cand[i] >> 32), a = static_cast<int32_t>(cand[i] & 0xffffffffu);
    // (undo mode: every candidate already has an applied-owned face — round 1 builds the grid over
    // the owned faces, later rounds probe with them — so no owner filter is needed here)
    const int32_t* tp = F + 3 * p;
    const int32_t* ta = F + 3 * a;
    int shared = 0;
    for (int u = 0; u < 3; ++u)
      for (int w = 0; w < 3; ++w) shared += tp[u] == ta[w];
    // faces sharing a vertex: both (inflated) double boxes contain it, so they overlap.  Otherwise
    // the float boxes enclose the double boxes within one f32 ulp per side: an overlap deeper
    // than that margin in every axis certifies the double-box overlap without the vertex loads
    if (shared == 0 && !deep_overlap(B[p], B[a]) && !overlap(face_box(V, tp), face_box(V, ta))) continue;
    if (shared == 3 || degen[p] || degen[a]) {
      report(ds, mode, p, a, pairs, pair_cap, owner, revert);
      continue;
    }
    if (shared == 2) {  // edge neighbours: one orientation decides almost every pair, so no bucket
      if (verdict2(V, tp, ta, pair_info(tp, ta))) report(ds, mode, p, a, pairs, pair_cap, owner, revert);
      continue;
    }
    const unsigned long long slot = agg_inc_labeled(&ds->ncls[shared], static_cast<unsigned>(shared));
    cls[shared * cap + slot] = cand[i];
  }
}

// Stage 2a for the 1-shared bucket: certified-filter verdicts only (a small register budget,
// so high occupancy for these latency-bound gathers); undecided pairs go to list 2 (empty:
// 2-shared pairs are decided in k_classify) for the exact k_narrow<1, 2>.
#ifndef PCU_NARROW1_FAST_MINB
#define PCU_NARROW1_FAST_MINB 6
#endif
__global__ void __launch_bounds__(128, PCU_NARROW1_FAST_MINB) k_narrow1_fast(const double* __restrict__ V, const int32_t* __restrict__ F,
                                                      uint64_t* __restrict__ cls, uint64_t cap,
                                                      DetectScalars* __restrict__ ds, int mode,
                                                      int32_t* __restrict__ pairs, uint64_t pair_cap,
                                                      const int32_t* __restrict__ owner, uint8_t* __restrict__ revert) {
  if (ds->redo) return;
  const unsigned long long n = ds->ncls[1];
  const uint64_t* L = cls + cap;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t c = L[i];
    const int32_t p = static_cast<int32_t>(c >> 32), a = static_cast<int32_t>(c & 0xffffffffu);
    if (mode == 1) {
      const int32_t op = owner[p], oa = owner[a];
      if ((op < 0 || revert[op]) && (oa < 0 || revert[oa])) continue;
    }
    const int32_t* tp = F + 3 * p;
    const int32_t* ta = F + 3 * a;
    const int v = verdict1_fast(V, tp, ta, pair_info(tp, ta));
    if (v == 1) {
      report(ds, mode, p, a, pairs, pair_cap, owner, revert);
    } else if (v == 2) {
      const unsigned long long slot = agg_inc_labeled(&ds->ncls[2], 2u);
      cls[2 * cap + slot] = c;
    }
  }
}

template <int SHARED, int LIST = SHARED>
#ifndef PCU_NARROW_MINB
#define PCU_NARROW_MINB 1
#endif
__global__ void __launch_bounds__(128, PCU_NARROW_MINB) k_narrow(const double* __restrict__ V, const int32_t* __restrict__ F,
                                                const uint64_t* __restrict__ cls, uint64_t cap,
                                                DetectScalars* __restrict__ ds, int mode, int32_t* __restrict__ pairs,
                                                uint64_t pair_cap, const int32_t* __restrict__ owner,
                                                uint8_t* __restrict__ revert) {
  if (ds->redo) return;
  const unsigned long long n = ds->ncls[LIST];
  const uint64_t* L = cls + LIST * cap;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int32_t p = static_cast<int32_t>(L[i] >> 32), a = static_cast<int32_t>(L[i] & 0xffffffffu);
    if (mode == 1) {
      const int32_t op = owner[p], oa = owner[a];
      const bool rp = op >= 0, ra = oa >= 0;  // owner >= 0 <=> applied (see report)
      if ((!rp || revert[op]) && (!ra || revert[oa])) continue;  // nothing left to flag
    }
    const int32_t* tp = F + 3 * p;
    const int32_t* ta = F + 3 * a;
    bool hit;
    if (SHARED == 0) {
      hit = verdict0(V, tp, ta);
    } else {
      const PairInfo I = pair_info(tp, ta);
      hit = SHARED == 1 ? verdict1(V, tp, ta, I) : verdict2(V, tp, ta, I);
    }
    if (hit) report(ds, mode, p, a, pairs, pair_cap, owner, revert);
  }
}

// classify_pair: shared count by index; coplanar <=> every unshared vertex of
// T2 has exact orientation 0 w.r.t. T1's plane (a degenerate face counts as coplanar: all its
// orientations vanish).  3 shared = a duplicate face (excluded upstream by the SPEC).
__device__ int pair_coplanar(const double* __restrict__ V, const int32_t* t1, const int32_t* t2, const PairInfo& I) {
  const D3 T1[3] = {vtx(V, t1[0]), vtx(V, t1[1]), vtx(V, t1[2])};
  if (degenerate(T1[0], T1[1], T1[2]) || degenerate(vtx(V, t2[0]), vtx(V, t2[1]), vtx(V, t2[2]))) return 1;
  for (int j = 0; j < 3; ++j)
    if (I.s2[j] < 0 && o3(vtx(V, t2[j]), T1[0], T1[1], T1[2]) != 0) return 0;
  return 1;
}

__global__ void k_pair_class(const double* __restrict__ V, const int32_t* __restrict__ F,
                             const int32_t* __restrict__ pairs, int64_t n, int32_t* __restrict__ shared,
                             int32_t* __restrict__ coplanar) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int32_t* t1 = F + 3 * pairs[2 * i];
  const int32_t* t2 = F + 3 * pairs[2 * i + 1];
  const PairInfo I = pair_info(t1, t2);
  shared[i] = I.shared;
  coplanar[i] = I.shared == 3 ? 1 : pair_coplanar(V, t1, t2, I);
}

// intersect_3d (mode 1) / intersect_coplanar (mode 2) restricted to their class: out = -1 when
// the pair violates the precondition (coplanar for 3D, non-coplanar for coplanar)
__global__ void k_verdict_class(const double* __restrict__ V, const int32_t* __restrict__ F,
                                const int32_t* __restrict__ pairs, int64_t n, int mode, int32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int32_t* t1 = F + 3 * pairs[2 * i];
  const int32_t* t2 = F + 3 * pairs[2 * i + 1];
  const PairInfo I = pair_info(t1, t2);
  const int cop = I.shared == 3 ? 1 : pair_coplanar(V, t1, t2, I);
  if ((mode == 1) == (cop == 1)) {
    out[i] = -1;
    return;
  }
  out[i] = verdict(V, t1, t2) ? 1 : 0;  // the class-dispatching verdict takes exactly this branch
}

__global__ void k_verdict_pairs(const double* __restrict__ V, const int32_t* __restrict__ F,
                                const int32_t* __restrict__ pairs, int64_t n, int32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  out[i] = verdict(V, F + 3 * pairs[2 * i], F + 3 * pairs[2 * i + 1]) ? 1 : 0;
}

#ifndef PCU_PROBE_FULL_WARP
#define PCU_PROBE_FULL_WARP (1 << 17)
#endif
// hash buckets per build face (a face covers ~8 cells: fewer buckets mix cells in one list)
#ifndef PCU_BUCKETS_PER_FACE
#define PCU_BUCKETS_PER_FACE 2
#endif
uint32_t pow2_at_least(uint64_t x) {
  uint32_t p = 1024;
  while (p < x && p < (1u << 30)) p <<= 1;
  return p;
}

}  // namespace

struct IsectScratch {
  DevBuf<uint32_t> bcount, boff, bcur;
  DevBuf<int4> entries;      // (face id, first cell x, y, z) by bucket
  DevBuf<uint32_t> occ;      // non-empty bucket bitmap
  DevBuf<int32_t> big;
  DevBuf<int32_t> huge;      // huge probe ids
  DevBuf<uint64_t> cand;
  DevBuf<float> fbox;        // 6 floats per face
  DevBuf<uint8_t> degen;     // degenerate-face flags
  DevBuf<uint64_t> cls;      // candidate pairs by shared-vertex count (3 x cap)
  DevBuf<DetectScalars> ds;
  uint64_t cand_cap = 0;
};

IsectScratch* isect_scratch_create() { return new IsectScratch(); }
void isect_scratch_destroy(IsectScratch* s) { delete s; }

namespace {

// One detection round, entirely asynchronous (no host sync):
//   boxes of all faces -> grid over `build` (ids, or every alive face) -> probe with `probe`
//   (ids, or every alive face) -> narrow phase.  Results stay in S.ds (found / npairs / redo).
void detect_round(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf, const uint8_t* d_alive,
                  const int32_t* build_ids, int64_t n_build, const int32_t* probe_ids, int64_t n_probe, int sym,
                  int mode, int32_t* pairs, uint64_t pair_cap, const int32_t* owner,
                  uint8_t* revert, bool boxes_current = false, const uint8_t* in_probe = nullptr,
                  std::initializer_list<FillRange> extra_fills = {}, bool fresh_build_boxes = false) {
  cudaStream_t st = ctx.stream;
  S.ds.ensure(1, st);
  const uint32_t nb = pow2_at_least(static_cast<uint64_t>(n_build) * PCU_BUCKETS_PER_FACE + 1);
  const uint32_t mask = nb - 1;
  S.bcount.ensure(nb, st);
  S.boff.ensure(nb, st);
  S.bcur.ensure(nb, st);
  S.occ.ensure(nb / 32 + 1, st);
  // the round's scalars and the grid's bucket counters / occupancy bitmap, zeroed in one launch
  // (plus the caller's resets for the round, in the same launch)
  FillRange fills[kMaxFillRanges] = {{S.ds.get(), sizeof(DetectScalars), 0},
                                     {S.bcount.get(), static_cast<uint64_t>(nb) * 4, 0},
                                     {S.bcur.get(), static_cast<uint64_t>(nb) * 4, 0},
                                     {S.occ.get(), (static_cast<uint64_t>(nb) / 32 + 1) * 4, 0}};
  size_t nfill = 4;
  for (const FillRange& r : extra_fills) {
    PCU_REQUIRE(nfill < kMaxFillRanges, PAMOPT_CU_EINVAL, "detect_round: too many resets");
    fills[nfill++] = r;
  }
  fill_multi(ctx, fills, nfill);
  const FBox* B = reinterpret_cast<const FBox*>(S.fbox.get());
  if (!boxes_current) {
    S.fbox.ensure(6 * static_cast<size_t>(nf > 0 ? nf : 1), st);
    S.degen.ensure(static_cast<size_t>(nf > 0 ? nf : 1), st);
    B = reinterpret_cast<const FBox*>(S.fbox.get());
    PCU_LAUNCH(ctx, k_fboxes, grid_for(nf, 256), 256, 0, dV, dF, nf, d_alive, reinterpret_cast<FBox*>(S.fbox.get()),
               S.degen.get(), nullptr);
  }
  // build-set membership (round 1 of the undo loop): the build set is exactly the faces an applied
  // collapse owns, so owner[f] >= 0 is the flag
  const int32_t* in_build = (!sym && mode == 1 && !probe_ids) ? owner : nullptr;
  PCU_LAUNCH(ctx, k_ext_sum, static_cast<unsigned>(std::min<int64_t>(grid_for(n_build, 256), ctx.num_sms * 4)), 256, 0,
             const_cast<FBox*>(B), build_ids, n_build, d_alive, S.ds.get(), dV, dF, S.degen.get(),
             fresh_build_boxes ? 1 : 0);
  // hard capacity: a non-big face covers at most kMaxCells cells
  S.entries.ensure(static_cast<size_t>(n_build) * kMaxCells + 16, st);
  S.big.ensure(static_cast<size_t>(n_build) + 16, st);
  PCU_LAUNCH(ctx, k_bin, grid_for(n_build, 256), 256, 0, B, build_ids, n_build, d_alive, S.ds.get(), mask, 0,
             S.bcount.get(), S.boff.get(), S.bcur.get(), nullptr, nullptr, S.occ.get());
  exclusive_scan_u32(ctx, S.bcount.get(), S.boff.get(), nb);
  PCU_LAUNCH(ctx, k_bin, grid_for(n_build, 256), 256, 0, B, build_ids, n_build, d_alive, S.ds.get(), mask, 1,
             S.bcount.get(), S.boff.get(), S.bcur.get(), S.entries.get(), S.big.get(), S.occ.get());
  if (S.cand_cap == 0) S.cand_cap = static_cast<uint64_t>(nf) * 4 + 4096;
  S.cand.ensure(S.cand_cap, st);
  S.huge.ensure(static_cast<size_t>(n_probe) + 16, st);
  const int64_t p32 = PCU_PROBE_FULL_WARP;  // probe-set size from which a warp takes 32 probes
  const int ppw = n_probe >= p32 ? 32 : n_probe >= p32 / 2 ? 16 : n_probe >= p32 / 4 ? 8 : 4;
  PCU_LAUNCH(ctx, k_probe, grid_for(n_probe * (32 / ppw), 128), 128, 0, B, n_probe,
             d_alive, S.ds.get(), mask, S.bcount.get(), S.boff.get(), S.entries.get(), S.big.get(), S.occ.get(), sym,
             in_build,
             S.cand.get(), S.cand_cap, &S.ds.get()->ncand, probe_ids, S.huge.get(), &S.ds.get()->nhuge, in_probe, ppw);
  PCU_LAUNCH(ctx, k_probe_large, static_cast<unsigned>(ctx.num_sms * 2), 128, 0, B, S.ds.get(), S.huge.get(),
             S.big.get(), build_ids, n_build, probe_ids, n_probe, d_alive, sym, in_build, S.cand.get(), S.cand_cap,
             &S.ds.get()->ncand, in_probe);
  S.cls.ensure(3 * S.cand_cap, st);
  // narrow-phase grids sized from the expected candidate count (about 10-30 per face of the
  // smaller set): the small rounds of a long QEM tail do not schedule thousands of idle CTAs; the
  // kernels stride over the device-side counts, so any grid is correct
  const uint64_t est = 32 * static_cast<uint64_t>(std::max<int64_t>(std::min(n_build, n_probe), 1));
  const unsigned g = static_cast<unsigned>(
      std::min<uint64_t>(std::max<uint64_t>((est + 255) / 256, static_cast<uint64_t>(ctx.num_sms)),
                         static_cast<uint64_t>(ctx.num_sms) * 16));
  PCU_LAUNCH(ctx, k_classify, g, 256, 0, dV, dF, B, S.degen.get(), S.cand.get(), S.cand_cap, S.ds.get(), mode,
             S.cls.get(), pairs, pair_cap, owner, revert);
  // the 1-shared chain (certified filter, then the exact pass over its few undecided pairs, a
  // latency-bound launch) runs on the aux stream beside the 0-shared bucket: the buckets are
  // independent, and both only add to the found / pair counters and set revert flags
  {
    AuxFork fork(ctx);
    PCU_LAUNCH(ctx, k_narrow1_fast, g, 128, 0, dV, dF, S.cls.get(), S.cand_cap, S.ds.get(), mode, pairs, pair_cap,
               owner, revert);
    // the undecided remainder is a small fraction of the bucket: one CTA per SM
    PCU_LAUNCH(ctx, (k_narrow<1, 2>), static_cast<unsigned>(ctx.num_sms), 128, 0, dV, dF, S.cls.get(), S.cand_cap,
               S.ds.get(), mode, pairs, pair_cap, owner, revert);
    fork.to_main();
    PCU_LAUNCH(ctx, k_narrow<0>, g, 128, 0, dV, dF, S.cls.get(), S.cand_cap, S.ds.get(), mode, pairs, pair_cap, owner,
               revert);
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
  uint64_t pair_cap = static_cast<uint64_t>(nf) + 1024;
  DevBuf<int32_t> pairs(2 * pair_cap, ctx.stream);
  while (true) {
    detect_round(ctx, S, dV, dF, nf, d_alive, nullptr, nf, nullptr, nf, 1, 0, pairs.get(), pair_cap, nullptr, nullptr);
    const DetectScalars ds = read_scalar(ctx, S.ds.get());
    if (ds.redo) {
      S.cand_cap = ds.ncand + ds.ncand / 4 + 4096;
      continue;
    }
    if (ds.npairs > pair_cap) {
      pair_cap = ds.npairs + 1024;
      pairs.alloc(2 * pair_cap, ctx.stream);
      continue;
    }
    out.resize(2 * ds.npairs);
    if (ds.npairs)
      PCU_CUDA(cudaMemcpyAsync(out.data(), pairs.get(), ds.npairs * 8, cudaMemcpyDeviceToHost, ctx.stream));
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

void classify_pairs(Ctx& ctx, const double* dV, const int32_t* dF, const int32_t* d_pairs, int64_t n, int32_t* d_shared,
                    int32_t* d_coplanar) {
  if (n == 0) return;
  PCU_LAUNCH(ctx, k_pair_class, grid_for(n, 128), 128, 0, dV, dF, d_pairs, n, d_shared, d_coplanar);
}

void verdict_by_class(Ctx& ctx, const double* dV, const int32_t* dF, const int32_t* d_pairs, int64_t n, int mode,
                      int32_t* d_out) {
  if (n == 0) return;
  PCU_LAUNCH(ctx, k_verdict_class, grid_for(n, 128), 128, 0, dV, dF, d_pairs, n, mode, d_out);
}

void undo_detect_async(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf,
                       const uint8_t* d_falive, const int32_t* d_query_faces, int64_t n_query, const int32_t* d_owner,
                       uint8_t* d_revert, std::initializer_list<FillRange> resets) {
  // round 1: grid over the faces owned by applied collapses (~0.4 of the alive faces in every
  // iteration), probed by every alive face.  The converse (grid over every alive face, probed by
  // the owned faces, pairs of two owned faces from the smaller probe via in_probe) was measured
  // slower at C3: k_probe 36.0 -> 61.6 ms, k_bin 7.6 -> 19.4 ms (profiles/r02_summary.md).
  detect_round(ctx, S, dV, dF, nf, d_falive, d_query_faces, n_query, nullptr, nf, 0, 1, nullptr, 0, d_owner,
               d_revert, true, nullptr, resets, true);
}

void undo_detect_restored_async(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf,
                                const uint8_t* d_falive, const int32_t* d_restored, int64_t n_restored,
                                const int32_t* d_owned, int64_t n_owned, const int32_t* d_owner,
                                uint8_t* d_revert, std::initializer_list<FillRange> resets) {
  // later rounds: only (restored face, applied-owned face) pairs can be new
  detect_round(ctx, S, dV, dF, nf, d_falive, d_restored, n_restored, d_owned, n_owned, 0, 1, nullptr, 0, d_owner,
               d_revert, true, nullptr, resets, true);
}

// Persistent face boxes for the QEM loop: computed once, then refreshed only for the faces a
// collapse batch or a revert touched (every other face keeps its geometry).
void boxes_init(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, int64_t nf, const uint8_t* d_alive) {
  S.fbox.ensure(6 * static_cast<size_t>(nf > 0 ? nf : 1), ctx.stream);
  S.degen.ensure(static_cast<size_t>(nf > 0 ? nf : 1), ctx.stream);
  PCU_LAUNCH(ctx, k_fboxes, grid_for(nf, 256), 256, 0, dV, dF, nf, d_alive, reinterpret_cast<FBox*>(S.fbox.get()),
             S.degen.get(), nullptr);
}
void boxes_update(Ctx& ctx, IsectScratch& S, const double* dV, const int32_t* dF, const int32_t* ids, int64_t n,
                  const uint8_t* d_alive) {
  if (n <= 0) return;
  PCU_LAUNCH(ctx, k_fboxes, grid_for(n, 256), 256, 0, dV, dF, n, d_alive, reinterpret_cast<FBox*>(S.fbox.get()),
             S.degen.get(), ids);
}

const void* detect_scalars_ptr(IsectScratch& S) { return S.ds.get(); }
size_t detect_scalars_size() { return sizeof(DetectScalars); }
void detect_grow(IsectScratch& S, unsigned long long ncand) { S.cand_cap = ncand + ncand / 4 + 4096; }
void detect_read(const void* host_copy, unsigned long long* found, int* redo, unsigned long long* ncand,
                 unsigned long long* ncls) {
  const DetectScalars* d = static_cast<const DetectScalars*>(host_copy);
  *found = d->found;
  *redo = d->redo;
  *ncand = d->ncand;
  if (ncls)
    for (int k = 0; k < 3; ++k) ncls[k] = d->ncls[k];
}

}  // namespace pcu

// simplify.cu — stage 2: parallel intersection-free QEM simplification (Algorithm 1;
// SPEC.md:473-574), device resident.  Per iteration (bulk synchronous,
// SPEC.md:563):
//
//   incidence  vertex -> alive faces CSR by counting sort; every list sorted by face id
//   edges      per vertex a: sorted unique neighbours b > a  -> lexicographic edge ids (P5)
//   cost       Eq. 1 per valid edge (FP64, fmad off): merged quadric, adjugate placement with
//              the 1-norm condition fallback to {mid, a, b}, edge length, skinny ring cost;
//              key = f32 bits << 32 | id
//   propagate  64-bit atomicMin edge keys -> vertices (REDG.MIN.64), face key = min of its
//              vertices, then faces -> vertices; an edge is marked iff both endpoints' face
//              minima equal its key (== every face of its 1-ring holds it; Gautron et al.)
//   link       link condition (mesh.cpp:301-358) per marked edge on the pre-batch mesh
//   trim       marked edges in key order; keep while the batch would not undershoot (P9)
//   collapse   b -> a in b's faces, shared faces deleted, x placed, K_a += K_b (mesh.cpp:363-395)
//   undo       grid broad phase over the faces owned by applied collapses, probed by every alive
//              face, exact narrow phase; owners of intersecting faces revert from the pre-batch
//              snapshot and are flagged invalid; repeat until clean
//   flags      invalid list (sorted (a<<32|b) keys), kept one iteration, accumulated across
//              zero-collapse iterations up to `tolerance`
// The host reads a handful of counters per iteration (edge count, marked count, collapse and
// undo results) to size the next launches and to drive the termination rule.
#include <cub/cub.cuh>

#include <algorithm>

#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace pcu {
namespace {

// Vertices with at most kLocalDeg incident faces keep their per-thread sets in registers/local
// memory; larger valences (unbounded, as the reference's std::set-based code) work in global
// scratch regions aligned with the CSR incidence (2 slots per incidence entry + 1 per vertex), which
// no other thread touches: marked edges have disjoint 1-rings, so their endpoints are distinct.
constexpr int kLocalDeg = 32;
static_assert(kLocalDeg <= 32, "link_condition_warp holds one incident face per lane");
constexpr double k4Sqrt3 = 6.928203230275509;

struct Counters {
  unsigned long long edges, marked, link_fail, newinv, query, removed, applied, err, cap, undone, restored, nan;
};

__device__ __forceinline__ D3 P3(const double* X, int v) { return D3{X[3 * v], X[3 * v + 1], X[3 * v + 2]}; }
__device__ __forceinline__ bool has(const int32_t* t, int v) { return t[0] == v || t[1] == v || t[2] == v; }

// ------------------------------------------------------------------------- incidence
__global__ void k_deg(const int32_t* __restrict__ F, const uint8_t* __restrict__ falive, int64_t nf,
                      uint32_t* __restrict__ deg) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf || !falive[f]) return;
  atomicAdd(&deg[F[3 * f]], 1u);
  atomicAdd(&deg[F[3 * f + 1]], 1u);
  atomicAdd(&deg[F[3 * f + 2]], 1u);
}

__global__ void k_fill(const int32_t* __restrict__ F, const uint8_t* __restrict__ falive, int64_t nf,
                       const uint32_t* __restrict__ off, uint32_t* __restrict__ cur, int32_t* __restrict__ inc) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf || !falive[f]) return;
  for (int k = 0; k < 3; ++k) {
    const int v = F[3 * f + k];
    inc[off[v] + atomicAdd(&cur[v], 1u)] = static_cast<int32_t>(f);
  }
}

// one vertex's incident faces in ascending id (the pinned gather / traversal order)
__device__ __forceinline__ void sort_list(int32_t* L, int n) {
  for (int i = 1; i < n; ++i) {
    const int32_t x = L[i];
    int j = i - 1;
    while (j >= 0 && L[j] > x) {
      L[j + 1] = L[j];
      --j;
    }
    L[j + 1] = x;
  }
}

__global__ void k_sort_lists(const uint32_t* __restrict__ off, const uint32_t* __restrict__ deg, int64_t nv,
                             int32_t* __restrict__ inc) {
  const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (v >= nv) return;
  sort_list(inc + off[v], static_cast<int>(deg[v]));
}

// quadrics gathered in ascending face id
__device__ void face_quadric(const double* X, const int32_t* t, double* o) {
  const D3 p0 = P3(X, t[0]), p1 = P3(X, t[1]), p2 = P3(X, t[2]);
  const D3 n = cross(sub(p1, p0), sub(p2, p0));
  const double len = sqrt(sqn(n));
  if (!(len > 0.0)) {
    for (int k = 0; k < 10; ++k) o[k] = 0.0;
    return;
  }
  const double a = n.x / len, b = n.y / len, c = n.z / len;
  const double d = -((a * p0.x + b * p0.y) + c * p0.z);
  const double w = 0.5 * len;
  o[0] = w * (a * a); o[1] = w * (a * b); o[2] = w * (a * c); o[3] = w * (a * d);
  o[4] = w * (b * b); o[5] = w * (b * c); o[6] = w * (b * d);
  o[7] = w * (c * c); o[8] = w * (c * d); o[9] = w * (d * d);
}

__global__ void k_quadrics(const double* __restrict__ X, const int32_t* __restrict__ F, const uint32_t* __restrict__ off,
                           const uint32_t* __restrict__ deg, const int32_t* __restrict__ inc, int64_t nv,
                           double* __restrict__ Q) {
  const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (v >= nv) return;
  double q[10];
  for (int k = 0; k < 10; ++k) q[k] = 0.0;
  for (uint32_t i = 0; i < deg[v]; ++i) {
    double fq[10];
    face_quadric(X, F + 3 * inc[off[v] + i], fq);
    for (int k = 0; k < 10; ++k) q[k] = q[k] + fq[k];
  }
  for (int k = 0; k < 10; ++k) Q[10 * v + k] = q[k];
}

// ----------------------------------------------------------------------------- edges
// neighbours b > a of vertex a, sorted unique; returns the count.  nb/mult hold >= 2 deg(a) slots.
// mult[i] = number of alive faces holding edge (a, nb[i]).
template <class I, class M>
__device__ int upper_neighbours(int a, const int32_t* __restrict__ F, const uint32_t* __restrict__ off,
                                const uint32_t* __restrict__ deg, const int32_t* __restrict__ inc, I* nb, M* mult) {
  const int d = static_cast<int>(deg[a]);
  int n = 0;
  for (int i = 0; i < d; ++i) {
    const int32_t* t = F + 3 * inc[off[a] + i];
    for (int k = 0; k < 3; ++k)
      if (t[k] > a) nb[n++] = t[k];
  }
  for (int i = 1; i < n; ++i) {
    const int32_t x = nb[i];
    int j = i - 1;
    while (j >= 0 && nb[j] > x) {
      nb[j + 1] = nb[j];
      --j;
    }
    nb[j + 1] = x;
  }
  int u = 0;
  for (int i = 0; i < n;) {
    int j = i;
    while (j < n && nb[j] == nb[i]) ++j;
    nb[u] = nb[i];
    mult[u] = static_cast<uint8_t>(min(j - i, 255));
    ++u;
    i = j;
  }
  return u;
}

// per vertex a: its upper neighbours b > a (ascending) with the face count of edge ab; the
// sorted list is parked in the CSR-aligned scratch (2 slots per incident face) for k_edge_fill
// (each vertex's thread first sorts its own incidence list: k_fill appends in atomic order, and
// every later kernel of the iteration reads the lists in ascending face id)
__global__ void k_edge_count(const int32_t* __restrict__ F, const uint32_t* __restrict__ off,
                             const uint32_t* __restrict__ deg, int32_t* __restrict__ inc, int64_t nv,
                             uint32_t* __restrict__ ecount, int32_t* __restrict__ snb, uint8_t* __restrict__ smult,
                             Counters* cnt) {
  const int64_t a = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (a >= nv) return;
  sort_list(inc + off[a], static_cast<int>(deg[a]));
  const int64_t s0 = 2 * static_cast<int64_t>(off[a]);
  const int d = static_cast<int>(deg[a]);
  int u = 0;
  int bad = 0;
  if (d <= kLocalDeg) {
    int32_t nb[2 * kLocalDeg];
    uint8_t mult[2 * kLocalDeg];
    u = d ? upper_neighbours(static_cast<int>(a), F, off, deg, inc, nb, mult) : 0;
    for (int i = 0; i < u; ++i) {
      bad |= (mult[i] != 1 && mult[i] != 2);
      snb[s0 + i] = nb[i];
      smult[s0 + i] = mult[i];
    }
  } else {  // high valence: sort and deduplicate in the vertex's own CSR-aligned scratch slots
    u = upper_neighbours(static_cast<int>(a), F, off, deg, inc, snb + s0, smult + s0);
    for (int i = 0; i < u; ++i) bad |= (smult[s0 + i] != 1 && smult[s0 + i] != 2);
  }
  if (bad) atomicAdd(&cnt->err, 1ull);  // non-manifold edge: input must come from stage 1
  ecount[a] = static_cast<uint32_t>(u);
}

__global__ void k_edge_fill(const uint32_t* __restrict__ off, const uint32_t* __restrict__ ecount, int64_t nv,
                            const uint32_t* __restrict__ eoff, const int32_t* __restrict__ snb,
                            const uint8_t* __restrict__ smult, int32_t* __restrict__ ea, int32_t* __restrict__ eb,
                            uint8_t* __restrict__ enf, unsigned long long* __restrict__ total) {
  const int64_t a = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (a >= nv) return;
  const int u = static_cast<int>(ecount[a]);
  if (a == nv - 1) *total = static_cast<unsigned long long>(eoff[a]) + static_cast<unsigned>(u);  // edge count
  const int64_t s0 = 2 * static_cast<int64_t>(off[a]);
  const uint32_t e0 = eoff[a];
  for (int i = 0; i < u; ++i) {
    ea[e0 + i] = static_cast<int32_t>(a);
    eb[e0 + i] = snb[s0 + i];
    enf[e0 + i] = smult[s0 + i];
  }
}

// invalid (a, b) pairs live in an open-addressing hash set (linear probing,
// empty = ~0): one insert pass per iteration instead of a sort, one probe per edge instead of a
// binary search.  Membership is all that is read, so the result does not depend on the layout.
__device__ __forceinline__ uint64_t inv_hash(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  return k ^ (k >> 33);
}

__global__ void k_inv_insert(const uint64_t* __restrict__ keys, int64_t n, unsigned long long* __restrict__ tab,
                             uint64_t mask) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i];
  if (k == ~0ull) return;  // a pair dropped by compact_state
  for (uint64_t h = inv_hash(k) & mask;; h = (h + 1) & mask) {
    const unsigned long long prev = atomicCAS(&tab[h], ~0ull, k);
    if (prev == ~0ull || prev == k) return;
  }
}

__global__ void k_mark_invalid(const int32_t* __restrict__ ea, const int32_t* __restrict__ eb,
                               const unsigned long long* __restrict__ d_ne, const uint64_t* __restrict__ tab,
                               uint64_t mask, int64_t ninv, uint8_t* __restrict__ valid) {
  const int64_t ne = static_cast<int64_t>(*d_ne);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = (static_cast<uint64_t>(ea[e]) << 32) | static_cast<uint32_t>(eb[e]);
    bool hit = false;
    if (ninv > 0)
      for (uint64_t h = inv_hash(key) & mask;; h = (h + 1) & mask) {
        const uint64_t t = tab[h];
        if (t == key) {
          hit = true;
          break;
        }
        if (t == ~0ull) break;
      }
    valid[e] = hit ? 0 : 1;
  }
}

// ------------------------------------------------------------------------------ cost
__device__ double qeval(const double* q, D3 p) {
  const double x = p.x, y = p.y, z = p.z;
  double r = q[0] * x * x;
  r = r + 2.0 * q[1] * x * y;
  r = r + 2.0 * q[2] * x * z;
  r = r + 2.0 * q[3] * x;
  r = r + q[4] * y * y;
  r = r + 2.0 * q[5] * y * z;
  r = r + 2.0 * q[6] * y;
  r = r + q[7] * z * z;
  r = r + 2.0 * q[8] * z;
  r = r + q[9];
  return r < 0.0 ? 0.0 : r;
}

__device__ double ring_skinny(const double* X, const int32_t* F, const int32_t* ia, int na, const int32_t* ib, int nb,
                              int a, int b, D3 x) {
  // faces of ring(a) U ring(b) in ascending id order (the pinned summation order); the next
  // face's index triple is fetched one step ahead so its load overlaps the current face's math
  int i = 0, j = 0;
  auto next = [&]() -> int {
    if (i < na || j < nb) {
      if (j == nb || (i < na && ia[i] < ib[j])) return ia[i++];
      if (i == na || ib[j] < ia[i]) return ib[j++];
      ++j;
      return ia[i++];
    }
    return -1;
  };
  double cs = 0.0;
  int f = next();
  int t0 = 0, t1 = 0, t2 = 0;
  if (f >= 0) {
    t0 = F[3 * f];
    t1 = F[3 * f + 1];
    t2 = F[3 * f + 2];
  }
  while (f >= 0) {
    const int fn = next();
    int u0 = 0, u1 = 0, u2 = 0;
    if (fn >= 0) {
      u0 = F[3 * fn];
      u1 = F[3 * fn + 1];
      u2 = F[3 * fn + 2];
    }
    const bool ha = t0 == a || t1 == a || t2 == a, hb = t0 == b || t1 == b || t2 == b;
    if (!(ha && hb)) {
      const int tt[3] = {t0, t1, t2};
      D3 P[3];
      for (int k = 0; k < 3; ++k) P[k] = (tt[k] == a || tt[k] == b) ? x : P3(X, tt[k]);
      const D3 n = cross(sub(P[1], P[0]), sub(P[2], P[0]));
      const double area = 0.5 * sqrt(sqn(n));
      const double l01 = sqn(sub(P[1], P[0])), l12 = sqn(sub(P[2], P[1])), l20 = sqn(sub(P[0], P[2]));
      const double den = (l01 + l12) + l20;
      const double c = den > 0.0 ? (k4Sqrt3 * area) / den : 0.0;
      cs = cs + (1.0 - c);
    }
    f = fn;
    t0 = u0;
    t1 = u1;
    t2 = u2;
  }
  return cs;
}

// Eq. 1 for edge (a, b) under the merged quadric K_a + K_b: placement x (adjugate solve, or the
// cheapest of {mid, a, b} when det == 0 or the 1-norm condition exceeds 1e8, P8) and its cost
__device__ __forceinline__ double edge_cost_eval(const double* __restrict__ X, const int32_t* __restrict__ F,
                                                 const double* __restrict__ Q, const uint32_t* __restrict__ off,
                                                 const uint32_t* __restrict__ deg, const int32_t* __restrict__ inc,
                                                 int a, int b, double we, double ws, D3& x) {
  double q[10];
  for (int k = 0; k < 10; ++k) q[k] = Q[10 * a + k] + Q[10 * b + k];
  const D3 pa = P3(X, a), pb = P3(X, b);
  const double l = sqrt(sqn(sub(pa, pb)));
  const double m00 = q[0], m01 = q[1], m02 = q[2], m10 = q[1], m11 = q[4], m12 = q[5], m20 = q[2], m21 = q[5],
               m22 = q[7];
  const double det = m00 * (m11 * m22 - m12 * m21) - m01 * (m10 * m22 - m12 * m20) + m02 * (m10 * m21 - m11 * m20);
  bool ok = det != 0.0;
  x = D3{0.0, 0.0, 0.0};
  if (ok) {
    const double rdet = 1.0 / det;  // adjugate * (1/det)
    const double i00 = (m11 * m22 - m12 * m21) * rdet, i01 = (m02 * m21 - m01 * m22) * rdet,
                 i02 = (m01 * m12 - m02 * m11) * rdet, i10 = (m12 * m20 - m10 * m22) * rdet,
                 i11 = (m00 * m22 - m02 * m20) * rdet, i12 = (m02 * m10 - m00 * m12) * rdet,
                 i20 = (m10 * m21 - m11 * m20) * rdet, i21 = (m01 * m20 - m00 * m21) * rdet,
                 i22 = (m00 * m11 - m01 * m10) * rdet;
    const double nA = fmax(fmax((fabs(m00) + fabs(m10)) + fabs(m20), (fabs(m01) + fabs(m11)) + fabs(m21)),
                           (fabs(m02) + fabs(m12)) + fabs(m22));
    const double nI = fmax(fmax((fabs(i00) + fabs(i10)) + fabs(i20), (fabs(i01) + fabs(i11)) + fabs(i21)),
                           (fabs(i02) + fabs(i12)) + fabs(i22));
    const double cond = nA * nI;
    if (!(cond <= 1e8)) {
      ok = false;
    } else {
      const double b0 = q[3], b1 = q[6], b2 = q[8];
      x = D3{-((i00 * b0 + i01 * b1) + i02 * b2), -((i10 * b0 + i11 * b1) + i12 * b2),
             -((i20 * b0 + i21 * b1) + i22 * b2)};
    }
  }
  const int32_t* ia = inc + off[a];
  const int32_t* ib = inc + off[b];
  const int na = static_cast<int>(deg[a]), nb = static_cast<int>(deg[b]);
  double cost;
  if (ok) {
    cost = (qeval(q, x) + we * l) + ws * ring_skinny(X, F, ia, na, ib, nb, a, b, x);
  } else {
    const D3 c0 = D3{(pa.x + pb.x) * 0.5, (pa.y + pb.y) * 0.5, (pa.z + pb.z) * 0.5};
    x = c0;
    cost = (qeval(q, c0) + we * l) + ws * ring_skinny(X, F, ia, na, ib, nb, a, b, c0);
    const double ca = (qeval(q, pa) + we * l) + ws * ring_skinny(X, F, ia, na, ib, nb, a, b, pa);
    if (ca < cost) {
      cost = ca;
      x = pa;
    }
    const double cb = (qeval(q, pb) + we * l) + ws * ring_skinny(X, F, ia, na, ib, nb, a, b, pb);
    if (cb < cost) {
      cost = cb;
      x = pb;
    }
  }
  return cost;
}

// pack_cost: f32 bits of max(cost, 0) << 32 | id
__device__ __forceinline__ uint64_t pack_key(double cost, uint64_t id) {
  const float cf = __double2float_rn(cost < 0.0 ? 0.0 : cost);
  return (static_cast<uint64_t>(__float_as_uint(cf)) << 32) | id;
}

#ifndef PCU_COST_MINB
#define PCU_COST_MINB 8
#endif
__global__ void __launch_bounds__(128, PCU_COST_MINB) k_cost(const double* __restrict__ X, const int32_t* __restrict__ F, const double* __restrict__ Q,
                       const uint32_t* __restrict__ off, const uint32_t* __restrict__ deg,
                       const int32_t* __restrict__ inc, const int32_t* __restrict__ ea, const int32_t* __restrict__ eb,
                       const uint8_t* __restrict__ valid, const unsigned long long* __restrict__ d_ne, double we,
                       double ws, uint64_t* __restrict__ key, double* __restrict__ place, Counters* cnt) {
  const int64_t ne = static_cast<int64_t>(*d_ne);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!valid[e]) {
      key[e] = ~0ull;
      continue;
    }
    D3 x;
    const double cost = edge_cost_eval(X, F, Q, off, deg, inc, ea[e], eb[e], we, ws, x);
    if (cost != cost) {
      atomicAdd(&cnt->nan, 1ull);
      key[e] = ~0ull;
      continue;
    }
    key[e] = pack_key(cost, static_cast<uint64_t>(e));
    place[3 * e] = x.x;
    place[3 * e + 1] = x.y;
    place[3 * e + 2] = x.z;
  }
}

// standalone edge_cost for explicit edges (granular C-ABI)
__global__ void k_edge_cost_raw(const double* __restrict__ X, const int32_t* __restrict__ F, const double* __restrict__ Q,
                                const uint32_t* __restrict__ off, const uint32_t* __restrict__ deg,
                                const int32_t* __restrict__ inc, const int32_t* __restrict__ edges, int64_t n, double we,
                                double ws, double* __restrict__ cost, double* __restrict__ place) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  D3 x;
  cost[i] = edge_cost_eval(X, F, Q, off, deg, inc, edges[2 * i], edges[2 * i + 1], we, ws, x);
  place[3 * i] = x.x;
  place[3 * i + 1] = x.y;
  place[3 * i + 2] = x.z;
}

__global__ void k_pack_cost(const double* __restrict__ cost, const uint32_t* __restrict__ ids, int64_t n,
                            uint64_t* __restrict__ keys, unsigned long long* __restrict__ nan) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double c = cost[i];
  if (c != c) {
    atomicAdd(nan, 1ull);
    keys[i] = ~0ull;
    return;
  }
  keys[i] = pack_key(c, ids[i]);
}

// --------------------------------------------------------------------- propagation
__global__ void k_prop_edges(const int32_t* __restrict__ ea, const int32_t* __restrict__ eb,
                             const uint64_t* __restrict__ key, const uint8_t* __restrict__ valid,
                             const unsigned long long* __restrict__ d_ne, unsigned long long* __restrict__ vmin) {
  const int64_t ne = static_cast<int64_t>(*d_ne);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!valid[e]) continue;
    atomicMin(&vmin[ea[e]], static_cast<unsigned long long>(key[e]));
    atomicMin(&vmin[eb[e]], static_cast<unsigned long long>(key[e]));
  }
}

__global__ void k_prop_faces(const int32_t* __restrict__ F, const uint8_t* __restrict__ falive, int64_t nf,
                             const unsigned long long* __restrict__ vmin, unsigned long long* __restrict__ vfmin) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf || !falive[f]) return;
  const int v0 = F[3 * f], v1 = F[3 * f + 1], v2 = F[3 * f + 2];
  unsigned long long k = vmin[v0];
  k = vmin[v1] < k ? vmin[v1] : k;
  k = vmin[v2] < k ? vmin[v2] : k;
  atomicMin(&vfmin[v0], k);
  atomicMin(&vfmin[v1], k);
  atomicMin(&vfmin[v2], k);
}

__global__ void k_mark(const int32_t* __restrict__ ea, const int32_t* __restrict__ eb, const uint64_t* __restrict__ key,
                       const uint8_t* __restrict__ valid, const unsigned long long* __restrict__ d_ne,
                       const unsigned long long* __restrict__ vfmin, uint64_t* __restrict__ marked, Counters* cnt) {
  const int64_t ne = static_cast<int64_t>(*d_ne);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!valid[e]) continue;
    const uint64_t k = key[e];
    if (k == vfmin[ea[e]] && k == vfmin[eb[e]]) marked[agg_inc(&cnt->marked)] = k;
  }
}

// ---------------------------------------------------------------------- link condition
// restatement of mesh.cpp:301-358 on the CSR incidence (-2 = the virtual boundary vertex)
__device__ int faces_of_edge(int a, int b, const int32_t* F, const uint32_t* off, const uint32_t* deg,
                             const int32_t* inc) {
  int c = 0;
  for (uint32_t i = 0; i < deg[a]; ++i) c += has(F + 3 * inc[off[a] + i], b);
  return c;
}

// sorted unique link vertex set of v (+ -2 if boundary); returns size.  One pass over the
// incident faces builds the multiset of their other vertices (a vertex counted once per face);
// after sorting, v is a boundary vertex (mesh.cpp:298-356: some ring vertex lies in exactly one
// incident face) iff some value occurs once — the same verdict without the O(deg^2) rescans.
template <class I>
__device__ int link_set(int v, const int32_t* F, const uint32_t* off, const uint32_t* deg, const int32_t* inc, I* out) {
  int n = 0;
  const int d = static_cast<int>(deg[v]);
  const int32_t* L = inc + off[v];
  for (int i = 0; i < d; ++i) {
    const int32_t* t = F + 3 * L[i];
    const int32_t t0 = t[0], t1 = t[1], t2 = t[2];
    if (t0 != v) out[n++] = t0;
    if (t1 != v && t1 != t0) out[n++] = t1;
    if (t2 != v && t2 != t0 && t2 != t1) out[n++] = t2;
  }
  for (int i = 1; i < n; ++i) {
    const int32_t x = out[i];
    int j = i - 1;
    while (j >= 0 && out[j] > x) {
      out[j + 1] = out[j];
      --j;
    }
    out[j + 1] = x;
  }
  bool boundary = false;
  int u = 0;
  for (int i = 0; i < n;) {
    int k = i + 1;
    while (k < n && out[k] == out[i]) ++k;
    boundary |= (k - i) == 1;
    out[u++] = out[i];
    i = k;
  }
  if (boundary) {  // -2 sorts first
    for (int i = u; i > 0; --i) out[i] = out[i - 1];
    out[0] = -2;
    ++u;
  }
  return u;
}

// la / lb: >= 2 deg + 1 slots each (link sets of a and b); common = la ∩ lb is written in place
// over la (its write position never passes the read position)
template <class I>
__device__ bool link_condition(int a, int b, const int32_t* F, const uint32_t* off, const uint32_t* deg,
                               const int32_t* inc, I* la, I* lb) {
  const int na = link_set(a, F, off, deg, inc, la);
  const int nb = link_set(b, F, off, deg, inc, lb);
  I* common = la;
  int nc = 0;
  for (int i = 0, j = 0; i < na && j < nb;) {
    if (la[i] < lb[j]) ++i;
    else if (lb[j] < la[i]) ++j;
    else {
      common[nc++] = la[i];
      ++i;
      ++j;
    }
  }
  // link(ab): opposite vertices of faces(a,b) (+ -2 if boundary edge).  A manifold edge has at
  // most two faces (k_edge_count rejects anything else before the first batch); more than 6
  // opposite vertices cannot equal a link set here, so the edge fails the condition.
  int32_t lab[8];
  int nl = 0, nfe = 0;
  for (uint32_t i = 0; i < deg[a]; ++i) {
    const int32_t* t = F + 3 * inc[off[a] + i];
    if (!has(t, b)) continue;
    ++nfe;
    for (int k = 0; k < 3; ++k)
      if (t[k] != a && t[k] != b) {
        if (nl == 7) return false;
        lab[nl++] = t[k];
      }
  }
  if (nfe == 1) lab[nl++] = -2;
  for (int i = 1; i < nl; ++i) {
    const int32_t x = lab[i];
    int j = i - 1;
    while (j >= 0 && lab[j] > x) {
      lab[j + 1] = lab[j];
      --j;
    }
    lab[j + 1] = x;
  }
  int ul = 0;
  for (int i = 0; i < nl; ++i)
    if (ul == 0 || lab[ul - 1] != lab[i]) lab[ul++] = lab[i];
  if (ul != nc) return false;
  for (int i = 0; i < nc; ++i)
    if (lab[i] != common[i]) return false;
  const bool has_vb = nc > 0 && common[0] == -2;
  for (int i = 0; i < nc; ++i) {
    const int x = common[i];
    if (x == -2) continue;
    for (int j = 0; j < nc; ++j) {
      const int y = common[j];
      if (y == -2 || y <= x) continue;
      bool in_la = false, in_lb = false;
      for (uint32_t k = 0; k < deg[x]; ++k) {
        const int32_t* t = F + 3 * inc[off[x] + k];
        if (!has(t, y)) continue;
        if (has(t, a)) in_la = true;
        if (has(t, b)) in_lb = true;
      }
      if (in_la && in_lb) return false;
    }
    if (has_vb && faces_of_edge(a, x, F, off, deg, inc) == 1 && faces_of_edge(b, x, F, off, deg, inc) == 1)
      return false;
  }
  return true;
}

// The same verdict with one warp per edge, for vertices of at most 32 incident faces: lane i holds
// the i-th incident face of a and of b, and the sets of link_condition are counted with shuffles
// instead of sorted per thread.  With valid faces every incident face contributes exactly its two
// other vertices, and the checks reduce to (link_condition, step by step):
//   * boundary(v): some ring vertex of v lies in exactly one incident face;
//   * link(ab) = the opposite vertices of the faces holding a and b (+ -2 if exactly one face);
//     every opposite vertex is in link(a) ∩ link(b), so link(a) ∩ link(b) = link(ab) iff their
//     sizes agree and -2 is in both or neither (8+ faces on ab: false, as link_condition);
//   * then for each pair x < y of common vertices, no faces {x, y, a} and {x, y, b} both; and
//     with -2 common, no x on exactly one face with a and exactly one face with b.
__device__ bool link_condition_warp(int a, int b, const int32_t* __restrict__ F, const uint32_t* __restrict__ off,
                                    const uint32_t* __restrict__ deg, const int32_t* __restrict__ inc, int lane) {
  constexpr unsigned kAll = 0xffffffffu;
  const int da = static_cast<int>(deg[a]), db = static_cast<int>(deg[b]);
  int ua = -1, wa = -1, ub = -1, wb = -1, opp = -1;
  bool hb = false;
  if (lane < da) {
    const int32_t* t = F + 3 * inc[off[a] + lane];
    const int t0 = t[0], t1 = t[1], t2 = t[2];
    ua = t0 == a ? t1 : t0;
    wa = (t0 == a || t1 == a) ? t2 : t1;
    hb = ua == b || wa == b;
    if (hb) opp = ua == b ? wa : ua;
  }
  if (lane < db) {
    const int32_t* t = F + 3 * inc[off[b] + lane];
    const int t0 = t[0], t1 = t[1], t2 = t[2];
    ub = t0 == b ? t1 : t0;
    wb = (t0 == b || t1 == b) ? t2 : t1;
  }
  int cau = 0, caw = 0, cbu = 0, cbw = 0;  // multiplicities in the own link multiset
  bool ibu = false, ibw = false;           // a's ring vertices found in b's ring
  bool fu = true, fw = wa != ua;           // first occurrence among a's ring entries
  bool fo = hb;                            // first occurrence among the opposite vertices
  const int n = max(da, db);
  for (int j = 0; j < n; ++j) {
    const int xu = __shfl_sync(kAll, ua, j), xw = __shfl_sync(kAll, wa, j);
    const int yu = __shfl_sync(kAll, ub, j), yw = __shfl_sync(kAll, wb, j);
    const int xo = __shfl_sync(kAll, opp, j);
    cau += (xu == ua) + (xw == ua);
    caw += (xu == wa) + (xw == wa);
    cbu += (yu == ub) + (yw == ub);
    cbw += (yu == wb) + (yw == wb);
    ibu |= yu == ua || yw == ua;
    ibw |= yu == wa || yw == wa;
    if (j < lane) {
      fu &= xu != ua && xw != ua;
      fw &= xu != wa && xw != wa;
      fo &= xo != opp;
    }
  }
  const bool va = lane < da, vb = lane < db;
  const bool bnd_a = __any_sync(kAll, va && (cau == 1 || caw == 1));
  const bool bnd_b = __any_sync(kAll, vb && (cbu == 1 || cbw == 1));
  const int nfe = __popc(__ballot_sync(kAll, hb));
  if (nfe >= 8) return false;
  const int ncommon = __popc(__ballot_sync(kAll, va && fu && ibu)) + __popc(__ballot_sync(kAll, va && fw && ibw)) +
                      ((bnd_a && bnd_b) ? 1 : 0);
  const unsigned om = __ballot_sync(kAll, fo);  // lanes holding the distinct opposite vertices
  const int nlab = __popc(om) + (nfe == 1 ? 1 : 0);
  if (nfe == 1 && !(bnd_a && bnd_b)) return false;
  if (nlab != ncommon) return false;
  const bool has_vb = bnd_a && bnd_b;
  for (unsigned m = om; m;) {
    const int jx = __ffs(m) - 1;
    m &= m - 1;
    const int x = __shfl_sync(kAll, opp, jx);
    for (unsigned m2 = om; m2;) {
      const int jy = __ffs(m2) - 1;
      m2 &= m2 - 1;
      const int y = __shfl_sync(kAll, opp, jy);
      if (y <= x) continue;
      const bool in_la = __any_sync(kAll, va && ((ua == x && wa == y) || (ua == y && wa == x)));
      const bool in_lb = __any_sync(kAll, vb && ((ub == x && wb == y) || (ub == y && wb == x)));
      if (in_la && in_lb) return false;
    }
    if (has_vb) {
      const int fa = __popc(__ballot_sync(kAll, va && (ua == x || wa == x)));
      const int fb = __popc(__ballot_sync(kAll, vb && (ub == x || wb == x)));
      if (fa == 1 && fb == 1) return false;
    }
  }
  return true;
}

// marked[w] -> pass flag, removal count; failures appended to the invalid list.  One warp per
// marked edge; a vertex with more than 32 incident faces takes the per-thread path (lane 0) with
// its CSR-aligned global scratch (marked edges never share a vertex).
__global__ void k_link_warp(const uint64_t* __restrict__ marked, int64_t nm_host,
                            const unsigned long long* __restrict__ nm_dev, const int32_t* __restrict__ ea,
                            const int32_t* __restrict__ eb, const uint8_t* __restrict__ enf,
                            const int32_t* __restrict__ F, const uint32_t* __restrict__ off,
                            const uint32_t* __restrict__ deg, const int32_t* __restrict__ inc,
                            uint32_t* __restrict__ rem, uint64_t* __restrict__ newinv, Counters* cnt,
                            int32_t* __restrict__ lscr) {
  const int lane = threadIdx.x & 31;
  const int64_t nm = nm_dev ? static_cast<int64_t>(*nm_dev) : nm_host;  // (device count: no host read)
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < nm; w += nw) {
    const uint32_t e = static_cast<uint32_t>(marked[w]);
    const int a = ea[e], b = eb[e];
    bool ok;
    if (deg[a] <= 32 && deg[b] <= 32) {
      ok = link_condition_warp(a, b, F, off, deg, inc, lane);
    } else {
      ok = false;
      if (lane == 0)
        ok = link_condition(a, b, F, off, deg, inc, lscr + 2 * static_cast<int64_t>(off[a]) + a,
                            lscr + 2 * static_cast<int64_t>(off[b]) + b);
      ok = __shfl_sync(0xffffffffu, ok, 0);
    }
    if (lane != 0) continue;
    if (ok) {
      rem[w] = enf[e];
    } else {
      rem[w] = 0;
      atomicAdd(&cnt->link_fail, 1ull);
      newinv[atomicAdd(&cnt->newinv, 1ull)] = (static_cast<uint64_t>(a) << 32) | static_cast<uint32_t>(b);
    }
  }
}

// ----------------------------------------------------------------------------- collapse
struct Batch {
  int32_t* ca;      // kept vertex
  int32_t* cb;      // removed vertex
  uint8_t* applied;
  double* oldx;     // 3 per collapse
  double* oldq;     // 10 per collapse
  uint32_t* nrem;   // faces removed
};

__device__ __forceinline__ void collapse_one(int64_t i, const uint64_t* __restrict__ marked,
                                             const uint32_t* __restrict__ rem, const uint32_t* __restrict__ remoff,
                                             int64_t alive_faces, int64_t target, const int32_t* __restrict__ ea,
                                             const int32_t* __restrict__ eb, const double* __restrict__ place,
                                             const uint32_t* __restrict__ off, const uint32_t* __restrict__ deg,
                                             const int32_t* __restrict__ inc, double* __restrict__ X,
                                             int32_t* __restrict__ F, uint8_t* __restrict__ falive,
                                             uint8_t* __restrict__ valive, double* __restrict__ Q,
                                             int32_t* __restrict__ owner, int32_t* __restrict__ qfaces, Batch B,
                                             Counters* cnt) {
  B.applied[i] = 0;
  if (rem[i] == 0) return;                                                          // failed the link condition
  if (remoff && !(alive_faces - static_cast<int64_t>(remoff[i]) > target)) return;  // overshoot trim (P9)
  const uint32_t e = static_cast<uint32_t>(marked[i]);
  const int a = ea[e], b = eb[e];
  B.ca[i] = a;
  B.cb[i] = b;
  B.nrem[i] = rem[i];
  for (int k = 0; k < 3; ++k) B.oldx[3 * i + k] = X[3 * a + k];
  for (int k = 0; k < 10; ++k) B.oldq[10 * i + k] = Q[10 * a + k];
  for (uint32_t j = 0; j < deg[b]; ++j) {
    const int f = inc[off[b] + j];
    int32_t* t = F + 3 * f;
    if (has(t, a)) {
      falive[f] = 0;
    } else {
      for (int k = 0; k < 3; ++k)
        if (t[k] == b) t[k] = a;
    }
  }
  for (int k = 0; k < 3; ++k) X[3 * a + k] = place[3 * e + k];
  for (int k = 0; k < 10; ++k) Q[10 * a + k] = Q[10 * a + k] + Q[10 * b + k];
  valive[b] = 0;
  B.applied[i] = 1;
  agg_add(&cnt->applied, 1ull);
  agg_add(&cnt->removed, static_cast<unsigned long long>(rem[i]));
  // owned faces: alive faces of a and of b after the collapse
  for (uint32_t j = 0; j < deg[a]; ++j) {
    const int f = inc[off[a] + j];
    if (falive[f]) {
      owner[f] = static_cast<int32_t>(i);
      qfaces[agg_inc(&cnt->query)] = f;
    }
  }
  for (uint32_t j = 0; j < deg[b]; ++j) {
    const int f = inc[off[b] + j];
    if (falive[f]) {
      owner[f] = static_cast<int32_t>(i);
      qfaces[agg_inc(&cnt->query)] = f;
    }
  }
}

__global__ void k_collapse(const uint64_t* __restrict__ marked, int64_t nm, const uint32_t* __restrict__ rem,
                           const uint32_t* __restrict__ remoff, int64_t alive_faces, int64_t target,
                           const int32_t* __restrict__ ea, const int32_t* __restrict__ eb,
                           const double* __restrict__ place, const uint32_t* __restrict__ off,
                           const uint32_t* __restrict__ deg, const int32_t* __restrict__ inc, double* __restrict__ X,
                           int32_t* __restrict__ F, uint8_t* __restrict__ falive, uint8_t* __restrict__ valive,
                           double* __restrict__ Q, int32_t* __restrict__ owner, int32_t* __restrict__ qfaces,
                           Batch B, Counters* cnt, const unsigned long long* __restrict__ nm_dev) {
  // remoff == nullptr: no overshoot trim can fire this iteration; nm_dev: the marked count stays
  // on the device (grid-stride over it)
  const int64_t n = nm_dev ? static_cast<int64_t>(*nm_dev) : nm;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    collapse_one(i, marked, rem, remoff, alive_faces, target, ea, eb, place, off, deg, inc, X, F, falive, valive, Q,
                 owner, qfaces, B, cnt);
}

// keep query faces whose owner is still applied
__global__ void k_requery(const int32_t* __restrict__ qin, int64_t n, const int32_t* __restrict__ owner,
                          const uint8_t* __restrict__ applied, int32_t* __restrict__ qout, Counters* cnt) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int f = qin[i];
  const int o = owner[f];
  if (o >= 0 && applied[o]) qout[agg_inc(&cnt->query)] = f;
}

__global__ void k_revert(int64_t nm, const uint8_t* __restrict__ revert, const uint32_t* __restrict__ off,
                         const uint32_t* __restrict__ deg, const int32_t* __restrict__ inc,
                         const int32_t* __restrict__ Fprev, double* __restrict__ X, int32_t* __restrict__ F,
                         uint8_t* __restrict__ falive, uint8_t* __restrict__ valive, double* __restrict__ Q,
                         int32_t* __restrict__ owner, Batch B, uint64_t* __restrict__ newinv, Counters* cnt,
                         int32_t* __restrict__ restored) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nm || !revert[i] || !B.applied[i]) return;
  const int a = B.ca[i], b = B.cb[i];
  // restored faces = the pre-batch ring(a) ∪ ring(b) (listed for the next undo round)
  for (uint32_t j = 0; j < deg[a]; ++j) {
    const int f = inc[off[a] + j];
    if (owner[f] == i) owner[f] = -1;
    if (!has(Fprev + 3 * f, b)) restored[agg_inc(&cnt->restored)] = f;
  }
  for (uint32_t j = 0; j < deg[b]; ++j) {
    const int f = inc[off[b] + j];
    if (owner[f] == i) owner[f] = -1;
    falive[f] = 1;
    for (int k = 0; k < 3; ++k) F[3 * f + k] = Fprev[3 * f + k];
    restored[agg_inc(&cnt->restored)] = f;
  }
  for (int k = 0; k < 3; ++k) X[3 * a + k] = B.oldx[3 * i + k];
  for (int k = 0; k < 10; ++k) Q[10 * a + k] = B.oldq[10 * i + k];
  valive[b] = 1;
  B.applied[i] = 0;
  atomicAdd(&cnt->applied, ~0ull);  // -1
  atomicAdd(&cnt->undone, 1ull);
  atomicAdd(&cnt->removed, static_cast<unsigned long long>(-static_cast<long long>(B.nrem[i])));
  newinv[atomicAdd(&cnt->newinv, 1ull)] = (static_cast<uint64_t>(a) << 32) | static_cast<uint32_t>(b);
}

// ------------------------------------------------------------------------------ compaction
__global__ void k_used(const int32_t* __restrict__ F, const uint8_t* __restrict__ falive, int64_t nf,
                       uint32_t* __restrict__ used) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf || !falive[f]) return;
  for (int k = 0; k < 3; ++k) used[F[3 * f + k]] = 1u;
}
__global__ void k_vkeep(const uint8_t* __restrict__ valive, int64_t nv, uint32_t* __restrict__ used) {
  const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (v < nv) used[v] = (used[v] && valive[v]) ? 1u : 0u;
}
__global__ void k_fkeep(const uint8_t* __restrict__ falive, int64_t nf, uint32_t* __restrict__ fk) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f < nf) fk[f] = falive[f] ? 1u : 0u;
}
__global__ void k_compact(const double* __restrict__ X, const int32_t* __restrict__ F, int64_t nv, int64_t nf,
                          const uint32_t* __restrict__ vkeep, const uint32_t* __restrict__ vmap,
                          const uint32_t* __restrict__ fkeep, const uint32_t* __restrict__ fmap,
                          double* __restrict__ Xo, int32_t* __restrict__ Fo) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < nv && vkeep[i])
    for (int k = 0; k < 3; ++k) Xo[3 * vmap[i] + k] = X[3 * i + k];
  if (i < nf && fkeep[i])
    for (int k = 0; k < 3; ++k) Fo[3 * fmap[i] + k] = static_cast<int32_t>(vmap[F[3 * i + k]]);
}

// Mid-run compaction: drop dead faces/vertices, renumbering both order-preservingly. Edge ids
// (lexicographic ranks over alive edges), incidence order, collapse direction (a < b) and the
// invalid-pair order are all invariant under a monotone renumbering, so results are unchanged.
__global__ void k_compact_state(const double* __restrict__ X, const double* __restrict__ Q,
                                const int32_t* __restrict__ F, int64_t nv, int64_t nf,
                                const uint32_t* __restrict__ vkeep, const uint32_t* __restrict__ vmap,
                                const uint32_t* __restrict__ fkeep, const uint32_t* __restrict__ fmap,
                                double* __restrict__ Xo, double* __restrict__ Qo, int32_t* __restrict__ Fo) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < nv && vkeep[i]) {
    const uint32_t j = vmap[i];
    for (int k = 0; k < 3; ++k) Xo[3 * j + k] = X[3 * i + k];
    for (int k = 0; k < 10; ++k) Qo[10 * j + k] = Q[10 * i + k];
  }
  if (i < nf && fkeep[i])
    for (int k = 0; k < 3; ++k) Fo[3 * fmap[i] + k] = static_cast<int32_t>(vmap[F[3 * i + k]]);
}
__global__ void k_u8_to_u32(const uint8_t* __restrict__ a, int64_t n, uint32_t* __restrict__ o) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) o[i] = a[i] ? 1u : 0u;
}
__global__ void k_inv_remap(uint64_t* __restrict__ inv, int64_t n, const uint32_t* __restrict__ vkeep,
                            const uint32_t* __restrict__ vmap) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint32_t a = static_cast<uint32_t>(inv[i] >> 32), b = static_cast<uint32_t>(inv[i]);
  inv[i] = (vkeep[a] && vkeep[b]) ? (static_cast<uint64_t>(vmap[a]) << 32) | vmap[b] : ~0ull;
}

}  // namespace

// --------------------------------------------------------- standalone SPEC operations (C-ABI)
namespace {
// link_condition_holds per query edge (mesh.cpp:301-358); -1 = not an edge of the mesh (the
// reference throws std::invalid_argument, mesh.cpp:302).  High-valence queries get private
// global scratch at lofs[i] (query edges may share vertices, unlike a marked batch).
__global__ void k_link_sizes(const int32_t* __restrict__ edges, int64_t n, const uint32_t* __restrict__ deg,
                             uint32_t* __restrict__ sz) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint32_t da = deg[edges[2 * i]], db = deg[edges[2 * i + 1]];
  sz[i] = (da <= kLocalDeg && db <= kLocalDeg) ? 0u : 2 * da + 2 * db + 2;
}
// one warp per queried edge: vertices of at most 32 faces take link_condition_warp (the batch's
// check), larger ones the per-thread link_condition in lane 0 with per-edge scratch
__global__ void k_link_pairs(const int32_t* __restrict__ edges, int64_t n, const int32_t* __restrict__ F,
                             const uint32_t* __restrict__ off, const uint32_t* __restrict__ deg,
                             const int32_t* __restrict__ inc, const uint32_t* __restrict__ lofs,
                             int32_t* __restrict__ lscr, int32_t* __restrict__ out) {
  const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;  // warp-uniform
  const int a = min(edges[2 * i], edges[2 * i + 1]), b = max(edges[2 * i], edges[2 * i + 1]);
  if (a == b || faces_of_edge(a, b, F, off, deg, inc) == 0) {
    if (lane == 0) out[i] = -1;
    return;
  }
  bool ok = false;
  if (deg[a] <= kLocalDeg && deg[b] <= kLocalDeg) {
    ok = link_condition_warp(a, b, F, off, deg, inc, lane);
  } else if (lane == 0) {
    int32_t* base = lscr + lofs[i];
    ok = link_condition(a, b, F, off, deg, inc, base, base + 2 * deg[a] + 1);
  }
  if (lane == 0) out[i] = ok ? 1 : 0;
}

struct StaticAdj {  // vertex -> face CSR of a whole mesh (every face alive), lists ascending
  DevBuf<uint8_t> alive;
  DevBuf<uint32_t> deg, off, cur;
  DevBuf<int32_t> inc;
  StaticAdj(Ctx& ctx, const int32_t* F, int64_t nv, int64_t nf) {
    cudaStream_t st = ctx.stream;
    alive.alloc(nf ? nf : 1, st);
    deg.alloc(nv ? nv : 1, st);
    off.alloc(nv ? nv : 1, st);
    cur.alloc(nv ? nv : 1, st);
    inc.alloc(3 * nf + 1, st);
    if (nf) PCU_CUDA(cudaMemsetAsync(alive.get(), 1, nf, st));
    PCU_CUDA(cudaMemsetAsync(deg.get(), 0, nv * sizeof(uint32_t), st));
    PCU_CUDA(cudaMemsetAsync(cur.get(), 0, nv * sizeof(uint32_t), st));
    if (nf) PCU_LAUNCH(ctx, k_deg, grid_for(nf, 256), 256, 0, F, alive.get(), nf, deg.get());
    exclusive_scan_u32(ctx, deg.get(), off.get(), nv);
    if (nf) PCU_LAUNCH(ctx, k_fill, grid_for(nf, 256), 256, 0, F, alive.get(), nf, off.get(), cur.get(), inc.get());
    PCU_LAUNCH(ctx, k_sort_lists, grid_for(nv, 256), 256, 0, off.get(), deg.get(), nv, inc.get());
  }
};
}  // namespace

void quadrics_of(Ctx& ctx, const double* X, const int32_t* F, int64_t nv, int64_t nf, double* dQ) {
  if (nv == 0) return;
  StaticAdj A(ctx, F, nv, nf);
  PCU_LAUNCH(ctx, k_quadrics, grid_for(nv, 128), 128, 0, X, F, A.off.get(), A.deg.get(), A.inc.get(), nv, dQ);
}

void edge_cost_of(Ctx& ctx, const double* X, const int32_t* F, int64_t nv, int64_t nf, const int32_t* d_edges,
                  int64_t n, double we, double ws, double* d_cost, double* d_place) {
  if (n == 0) return;
  StaticAdj A(ctx, F, nv, nf);
  DevBuf<double> Q(10 * (nv ? nv : 1), ctx.stream);
  PCU_LAUNCH(ctx, k_quadrics, grid_for(nv, 128), 128, 0, X, F, A.off.get(), A.deg.get(), A.inc.get(), nv, Q.get());
  PCU_LAUNCH(ctx, k_edge_cost_raw, grid_for(n, 128), 128, 0, X, F, Q.get(), A.off.get(), A.deg.get(), A.inc.get(),
             d_edges, n, we, ws, d_cost, d_place);
}

int64_t pack_cost_of(Ctx& ctx, const double* d_cost, const uint32_t* d_ids, int64_t n, uint64_t* d_keys) {
  if (n == 0) return 0;
  DevBuf<unsigned long long> nan(1, ctx.stream);
  nan.memset(0, ctx.stream);
  PCU_LAUNCH(ctx, k_pack_cost, grid_for(n, 256), 256, 0, d_cost, d_ids, n, d_keys, nan.get());
  return static_cast<int64_t>(read_scalar(ctx, nan.get()));
}

void link_condition_of(Ctx& ctx, const int32_t* F, int64_t nv, int64_t nf, const int32_t* d_edges, int64_t n,
                       int32_t* d_out) {
  if (n == 0) return;
  StaticAdj A(ctx, F, nv, nf);
  DevBuf<uint32_t> sz(n, ctx.stream), lofs(n, ctx.stream);
  PCU_LAUNCH(ctx, k_link_sizes, grid_for(n, 256), 256, 0, d_edges, n, A.deg.get(), sz.get());
  exclusive_scan_u32(ctx, sz.get(), lofs.get(), n);
  const int64_t tot = static_cast<int64_t>(read_scalar(ctx, lofs.get() + n - 1)) + read_scalar(ctx, sz.get() + n - 1);
  DevBuf<int32_t> lscr(tot ? tot : 1, ctx.stream);
  PCU_LAUNCH(ctx, k_link_pairs, grid_for(32 * n, 256), 256, 0, d_edges, n, F, A.off.get(), A.deg.get(), A.inc.get(),
             lofs.get(), lscr.get(), d_out);
}

// ---------------------------------------------------------------- stepwise driver (Algorithm 1)
// One QEM run as a state object whose methods are the SPEC operations of one iteration, in order:
//   prepare()             quadrics are kept; CSR incidence, lexicographic edges, invalid flags,
//                         edge_cost + pack_cost for every valid edge
//   propagate_and_mark()  per-face min keys, independent edges
//   collapse_batch()      link condition, overshoot trim, parallel collapse
//   undo_loop()           detect on batch-modified faces, revert owners, repeat
//   end_iteration()       invalid-flag retention and the stall counter
// simplify_run() drives it to the target (simplify_to); the C-ABI exposes the
// same steps one by one (pamopt_cu_qem_*), so the granular operations ARE the pipeline code.
struct QemState {
  Ctx& ctx;
  cudaStream_t st;
  DevBuf<double>& V;
  DevBuf<int32_t>& Fb;
  int64_t& nv;
  int64_t& nf;
  int64_t target;
  SimplifyParams P;
  SimplifyStats& S;
  double* X = nullptr;
  int32_t* F = nullptr;
  DevBuf<uint8_t> falive, valive;
  DevBuf<double> Q;
  DevBuf<uint32_t> deg, off, cur, ecount, eoff;
  int64_t ecap;
  DevBuf<int32_t> rlist, inc, ea, eb, owner, qf, qf2, Fprev, snb, lscr;
  DevBuf<uint8_t> enf, valid, revert, smult;
  DevBuf<uint64_t> key, marked, marked_sorted;
  const uint64_t* mlist = nullptr;  // this iteration's marked list (marked_sorted or marked)
  bool deferred = false;            // marked count read after the batch (see propagate_and_mark)
  bool key_order = false;           // stepwise API: always sort the marked list
  const bool undo_stats = std::getenv("PAMOPT_UNDO_STATS") != nullptr;
  DevBuf<double> place;
  DevBuf<unsigned long long> vmin, vfmin;
  DevBuf<uint32_t> rem, remoff;
  DevBuf<Counters> cnt;
  DevBuf<uint64_t> inv, newinv;
  int64_t ninv = 0;
  DevBuf<uint64_t> inv_tab;  // hash set of the ninv invalid pairs (k_inv_insert)
  uint64_t inv_mask = 0;

  void build_inv_table() {
    if (ninv == 0) return;
    uint64_t cap = 1024;
    while (cap < 2 * static_cast<uint64_t>(ninv)) cap <<= 1;
    inv_tab.ensure(cap, st);
    inv_mask = cap - 1;
    PCU_CUDA(cudaMemsetAsync(inv_tab.get(), 0xFF, cap * 8, st));
    PCU_LAUNCH(ctx, k_inv_insert, grid_for(ninv, 256), 256, 0, inv.get(), ninv,
               reinterpret_cast<unsigned long long*>(inv_tab.get()), inv_mask);
  }
  DevBuf<int32_t> bca, bcb;
  DevBuf<uint8_t> bapplied;
  DevBuf<double> boldx, boldq;
  DevBuf<uint32_t> bnrem;
  Batch B;
  IsectScratch* isc = nullptr;
  size_t sort_tmp_bytes = 0;
  DevBuf<uint8_t> sort_tmp;
  int64_t alive_faces = 0, alive_verts = 0;
  int retain = 0, zero_run = 0;
  int64_t ne_hint = 0;
  std::vector<uint8_t> ds_host;
  void* hpin = nullptr;  // pinned: Counters, then the detection scalars
  unsigned gs_grid = 0;
  // per-iteration results
  int64_t ne = 0, nm = 0, succ = 0, nnew = 0, nq = 0;
  int rounds = 0;
  Counters hc{};  // counters read at the collapse-batch synchronisation
  int phase = 0;  // 0 idle, 1 prepared, 2 marked, 3 collapsed, 4 undone

  QemState(Ctx& c, DevBuf<double>& V_, DevBuf<int32_t>& F_, int64_t& nv_, int64_t& nf_, int64_t target_,
           const SimplifyParams& P_, SimplifyStats& S_)
      : ctx(c), st(c.stream), V(V_), Fb(F_), nv(nv_), nf(nf_), target(target_), P(P_), S(S_) {
    X = V.get();
    F = Fb.get();
    falive.alloc(nf ? nf : 1, st);
    valive.alloc(nv ? nv : 1, st);
    if (nf) PCU_CUDA(cudaMemsetAsync(falive.get(), 1, nf, st));
    if (nv) PCU_CUDA(cudaMemsetAsync(valive.get(), 1, nv, st));
    Q.alloc(10 * (nv ? nv : 1), st);
    for (DevBuf<uint32_t>* b : {&deg, &off, &cur, &ecount, &eoff}) b->alloc(nv ? nv : 1, st);
    ecap = 3 * nf + 16;
    rlist.alloc(3 * nf + 16, st);
    inc.alloc(3 * nf + 16, st);
    ea.alloc(ecap, st);
    eb.alloc(ecap, st);
    owner.alloc(nf + 16, st);
    qf.alloc(3 * nf + 16, st);
    qf2.alloc(3 * nf + 16, st);
    Fprev.alloc(3 * nf + 16, st);
    snb.alloc(6 * nf + 16, st);  // upper-neighbour scratch, 2 slots per incidence entry
    lscr.alloc(6 * nf + nv + 16, st);  // high-valence link-set scratch (2 per incidence + 1 per vertex)
    enf.alloc(ecap, st);
    valid.alloc(ecap, st);
    revert.alloc(ecap, st);
    smult.alloc(6 * nf + 16, st);
    key.alloc(ecap, st);
    marked.alloc(ecap, st);
    marked_sorted.alloc(ecap, st);
    place.alloc(3 * ecap, st);
    vmin.alloc(nv ? nv : 1, st);
    vfmin.alloc(nv ? nv : 1, st);
    rem.alloc(ecap, st);
    remoff.alloc(ecap, st);
    cnt.alloc(1, st);
    inv.alloc(16, st);
    newinv.alloc(ecap, st);
    bca.alloc(ecap, st);
    bcb.alloc(ecap, st);
    bapplied.alloc(ecap, st);
    boldx.alloc(3 * ecap, st);
    boldq.alloc(10 * ecap, st);
    bnrem.alloc(ecap, st);
    B = Batch{bca.get(), bcb.get(), bapplied.get(), boldx.get(), boldq.get(), bnrem.get()};
    isc = isect_scratch_create();
    alive_faces = nf;
    alive_verts = nv;
    ne_hint = 3 * nf / 2 + 16;
    ds_host.resize(detect_scalars_size());
    // pinned landing zone for the per-sync counter reads (a pageable D2H copy stages through the
    // driver and costs several us more per synchronisation)
    PCU_CUDA(cudaMallocHost(&hpin, sizeof(Counters) + ds_host.size()));
    gs_grid = static_cast<unsigned>(ctx.num_sms * 16);
    ctx.prof.reset(st);
    if (nf == 0 || nv == 0) return;
    fill_multi(ctx, {{deg.get(), nv * sizeof(uint32_t), 0}, {cur.get(), nv * sizeof(uint32_t), 0}});
    build_incidence();
    boxes_init(ctx, *isc, X, F, nf, falive.get());
    PCU_LAUNCH(ctx, k_quadrics, grid_for(nv, 128), 128, 0, X, F, off.get(), deg.get(), inc.get(), nv, Q.get());
  }
  ~QemState() {
    isect_scratch_destroy(isc);
    if (hpin) cudaFreeHost(hpin);
  }
  QemState(const QemState&) = delete;
  QemState& operator=(const QemState&) = delete;

  bool done() const { return nf == 0 || !(alive_faces > target && zero_run < P.stall); }

  // (deg and cur must be zero on entry: the constructor and prepare() reset them).  prepare()
  // leaves the per-vertex sort to k_edge_count, its next kernel.
  void build_incidence(bool sort_lists = true) {
    PCU_LAUNCH(ctx, k_deg, grid_for(nf, 256), 256, 0, F, falive.get(), nf, deg.get());
    exclusive_scan_u32(ctx, deg.get(), off.get(), nv);
    PCU_LAUNCH(ctx, k_fill, grid_for(nf, 256), 256, 0, F, falive.get(), nf, off.get(), cur.get(), inc.get());
    if (sort_lists) PCU_LAUNCH(ctx, k_sort_lists, grid_for(nv, 256), 256, 0, off.get(), deg.get(), nv, inc.get());
  }

  // Host synchronisations per iteration: one after marking, one after the collapse batch, one
  // per undo round (counters + detection scalars fetched together).
  Counters sync_counters(bool with_detect) {
    uint8_t* hc = static_cast<uint8_t*>(hpin);
    PCU_CUDA(cudaMemcpyAsync(hc, cnt.get(), sizeof(Counters), cudaMemcpyDeviceToHost, st));
    if (with_detect)
      PCU_CUDA(cudaMemcpyAsync(hc + sizeof(Counters), detect_scalars_ptr(*isc), ds_host.size(),
                               cudaMemcpyDeviceToHost, st));
    PCU_CUDA(cudaStreamSynchronize(st));
    Counters h;
    std::memcpy(&h, hc, sizeof(Counters));
    if (with_detect) std::memcpy(ds_host.data(), hc + sizeof(Counters), ds_host.size());
    return h;
  }

  // shrink the working set once a sizeable fraction of it is dead (one host sync per compaction).
  // Edge ids (lexicographic ranks over alive edges), incidence order, collapse direction (a < b)
  // and the invalid-pair order are all invariant under a monotone renumbering.
  void compact_state() {
    DevBuf<uint32_t> vk(nv, st), vmap(nv, st), fk(nf, st), fmap(nf, st);
    PCU_LAUNCH(ctx, k_u8_to_u32, grid_for(nv, 256), 256, 0, valive.get(), nv, vk.get());
    PCU_LAUNCH(ctx, k_u8_to_u32, grid_for(nf, 256), 256, 0, falive.get(), nf, fk.get());
    exclusive_scan_u32(ctx, vk.get(), vmap.get(), nv);
    exclusive_scan_u32(ctx, fk.get(), fmap.get(), nf);
    const int64_t nv2 = static_cast<int64_t>(read_scalar(ctx, vmap.get() + nv - 1)) + read_scalar(ctx, vk.get() + nv - 1);
    const int64_t nf2 = static_cast<int64_t>(read_scalar(ctx, fmap.get() + nf - 1)) + read_scalar(ctx, fk.get() + nf - 1);
    DevBuf<double> Xo(3 * (nv2 ? nv2 : 1), st), Qo(10 * (nv2 ? nv2 : 1), st);
    DevBuf<int32_t> Fo(3 * (nf2 ? nf2 : 1), st);
    PCU_LAUNCH(ctx, k_compact_state, grid_for(std::max(nv, nf), 256), 256, 0, X, Q.get(), F, nv, nf, vk.get(),
               vmap.get(), fk.get(), fmap.get(), Xo.get(), Qo.get(), Fo.get());
    if (ninv) {
      PCU_LAUNCH(ctx, k_inv_remap, grid_for(ninv, 256), 256, 0, inv.get(), ninv, vk.get(), vmap.get());
      build_inv_table();  // dropped pairs (~0) are not inserted
    }
    V = std::move(Xo);
    Q = std::move(Qo);
    Fb = std::move(Fo);
    X = V.get();
    F = Fb.get();
    nv = nv2;
    nf = nf2;
    PCU_CUDA(cudaMemsetAsync(falive.get(), 1, nf, st));
    PCU_CUDA(cudaMemsetAsync(valive.get(), 1, nv, st));
    boxes_init(ctx, *isc, X, F, nf, falive.get());
  }

  // edges, invalid flags, edge_cost + pack_cost
  void prepare() {
    PCU_REQUIRE(phase == 0, PAMOPT_CU_EINVAL, "qem: prepare() out of order");
    S.iterations++;
    ctx.prof.mark(st, "misc");
    if (alive_faces * 5 < nf * 3 && nf > 4096) compact_state();
    ctx.prof.mark(st, "compact_state");
    // this iteration's resets in one launch: the incidence counters, the counters block, the
    // per-vertex minima propagate_and_mark() fills and the face owners collapse_batch() sets
    const uint64_t nvb = S.iterations > 1 ? nv * sizeof(uint32_t) : 0;
    fill_multi(ctx, {{deg.get(), nvb, 0}, {cur.get(), nvb, 0}, {cnt.get(), sizeof(Counters), 0},
                     {vmin.get(), static_cast<uint64_t>(nv) * 8, 0xFF}, {vfmin.get(), static_cast<uint64_t>(nv) * 8, 0xFF},
                     {owner.get(), static_cast<uint64_t>(nf) * 4, 0xFF}});
    if (S.iterations > 1) build_incidence(false);
    ctx.prof.mark(st, "incidence");
    unsigned long long* d_ne = &cnt.get()->edges;
    // edges (device-side count; kernels below stride over it)
    PCU_LAUNCH(ctx, k_edge_count, grid_for(nv, 128), 128, 0, F, off.get(), deg.get(), inc.get(), nv, ecount.get(),
               snb.get(), smult.get(), cnt.get());
    exclusive_scan_u32(ctx, ecount.get(), eoff.get(), nv);
    PCU_LAUNCH(ctx, k_edge_fill, grid_for(nv, 128), 128, 0, off.get(), ecount.get(), nv, eoff.get(), snb.get(),
               smult.get(), ea.get(), eb.get(), enf.get(), d_ne);
    ctx.prof.mark(st, "edges");
    const unsigned eg = std::min<unsigned>(grid_for(ne_hint, 128), gs_grid);
    PCU_LAUNCH(ctx, k_mark_invalid, eg, 128, 0, ea.get(), eb.get(), d_ne, inv_tab.get(), inv_mask, ninv,
               valid.get());
    PCU_LAUNCH(ctx, k_cost, eg, 128, 0, X, F, Q.get(), off.get(), deg.get(), inc.get(), ea.get(), eb.get(), valid.get(),
               d_ne, P.we, P.ws, key.get(), place.get(), cnt.get());
    ctx.prof.mark(st, "cost");
    phase = 1;
  }

  // per-face min keys and the independent set; one host sync
  void propagate_and_mark() {
    PCU_REQUIRE(phase == 1, PAMOPT_CU_EINVAL, "qem: propagate_and_mark() out of order");
    unsigned long long* d_ne = &cnt.get()->edges;
    const unsigned eg = std::min<unsigned>(grid_for(ne_hint, 128), gs_grid);
    // (vmin / vfmin were reset to ~0 by prepare())
    PCU_LAUNCH(ctx, k_prop_edges, eg, 256, 0, ea.get(), eb.get(), key.get(), valid.get(), d_ne, vmin.get());
    PCU_LAUNCH(ctx, k_prop_faces, grid_for(nf, 256), 256, 0, F, falive.get(), nf, vmin.get(), vfmin.get());
    PCU_LAUNCH(ctx, k_mark, eg, 256, 0, ea.get(), eb.get(), key.get(), valid.get(), d_ne, vfmin.get(), marked.get(),
               cnt.get());
    succ = 0;
    rounds = 0;
    nnew = 0;
    nq = 0;
    // Deferred mode (the hot loop after iteration 1): marked edges share no vertex, so at most
    // alive_verts / 2 of them each remove at most 2 faces; when even that cannot reach the
    // target, no overshoot trim can fire, the marked order does not matter, and the link check
    // and the collapse run over the device-side count.  The counters are read once, after the
    // batch (sync 2), instead of here.
    deferred = !key_order && S.iterations > 1 && alive_faces - alive_verts > target;
    if (deferred) {
      mlist = marked.get();
      ctx.prof.mark(st, "propagate+mark");
      phase = 2;
      return;
    }
    Counters h = sync_counters(false);  // ---- sync 1
    account_marking(h);
    if (S.iterations == 1)
      PCU_REQUIRE(h.err == 0, PAMOPT_CU_EINVAL, "simplify_to: non-manifold input (an edge has >2 faces); run stage 1");
    ctx.prof.mark(st, "propagate+mark");
    mlist = marked_sorted.get();
    // Marked keys in ascending order fix the overshoot trim (P9), which applies the cheapest
    // collapses first.  Marked edges have disjoint face neighbourhoods, so when no trim can fire
    // (every collapse removes at most 2 faces) the batch's result does not depend on the order and
    // the hot loop uses k_mark's list as is; the stepwise API keeps key order for its views.
    // (h.err counts edges with more than 2 faces; with none, every collapse removes <= 2 faces)
    const bool any_order = !key_order && h.err == 0 && alive_faces - 2 * nm > target;
    if (nm > 0 && any_order) mlist = marked.get();
    if (nm > 0 && !any_order) {
      if (!small_sort_u64(ctx, marked.get(), marked_sorted.get(), nm)) {
        size_t need = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, need, marked.get(), marked_sorted.get(), static_cast<int>(nm), 0, 64,
                                       st);
        if (need > sort_tmp_bytes) {
          sort_tmp.alloc(need, st);
          sort_tmp_bytes = need;
        }
        cudaEvent_t sev = ctx.prof.kt ? ctx.prof.kbegin(st) : nullptr;
        cub::DeviceRadixSort::SortKeys(sort_tmp.get(), sort_tmp_bytes, marked.get(), marked_sorted.get(),
                                       static_cast<int>(nm), 0, 64, st);
        if (sev) ctx.prof.kend("cub_sort_marked", sev, st);
      }
    }
    phase = 2;
  }

  // counters of the marking step (read at sync 1, or at sync 2 in deferred mode)
  void account_marking(const Counters& h) {
    ne = static_cast<int64_t>(h.edges);
    ne_hint = ne;
    nm = static_cast<int64_t>(h.marked);
    S.face_iterations += alive_faces;
    S.alg_bytes += 28 * alive_faces + 92 * alive_verts + 8 * ne;
    PCU_REQUIRE(h.nan == 0, PAMOPT_CU_ENUMERIC, "simplify_to: NaN edge cost");
  }

  // link condition on the pre-batch mesh, overshoot trim, parallel collapse
  void collapse_batch() {
    PCU_REQUIRE(phase == 2, PAMOPT_CU_EINVAL, "qem: collapse_batch() out of order");
    phase = 3;
    if (!deferred && nm == 0) return;
    const unsigned long long* nm_dev = deferred ? &cnt.get()->marked : nullptr;
    {
      // the pre-batch face copy (the undo loop's restore source) runs on the aux stream while the
      // link condition is evaluated (both only read F)
      AuxFork fork(ctx);
      PCU_CUDA(cudaMemcpyAsync(Fprev.get(), F, 3 * nf * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx.stream));
      fork.to_main();
      const unsigned lg = deferred ? gs_grid : grid_for(32 * nm, 256);
      PCU_LAUNCH(ctx, k_link_warp, lg, 256, 0, mlist, nm, nm_dev, ea.get(), eb.get(), enf.get(), F, off.get(),
                 deg.get(), inc.get(), rem.get(), newinv.get(), cnt.get(), lscr.get());
      if (!deferred) exclusive_scan_u32(ctx, rem.get(), remoff.get(), nm);
    }
    ctx.prof.mark(st, "sort+link");
    const unsigned cg = deferred ? gs_grid : grid_for(nm, 128);
    PCU_LAUNCH(ctx, k_collapse, cg, 128, 0, mlist, nm, rem.get(), deferred ? nullptr : remoff.get(), alive_faces,
               target, ea.get(), eb.get(), place.get(), off.get(), deg.get(), inc.get(), X, F, falive.get(),
               valive.get(), Q.get(), owner.get(), qf.get(), B, cnt.get(), nm_dev);
    hc = sync_counters(false);  // ---- sync 2
    if (deferred) {
      account_marking(hc);
      PCU_REQUIRE(hc.err == 0, PAMOPT_CU_EINVAL, "simplify_to: non-manifold edge during simplification");
    }
    ctx.prof.mark(st, "collapse");
    nq = static_cast<int64_t>(hc.query);
    // (the moved / renamed faces get their boxes in the first undo round: they are its build set)
  }

  // detect -> revert owners -> repeat until clean
  void undo_loop() {
    PCU_REQUIRE(phase == 3, PAMOPT_CU_EINVAL, "qem: undo_loop() out of order");
    phase = 4;
    if (nm == 0) return;
    int32_t* qa = qf.get();
    int32_t* qb = qf2.get();
    bool first_round = true;
    int64_t nrest = 0;
    int64_t nqr = nq;
    Counters h = hc;
    while (nqr > 0) {
      // the round's resets ride in the detection's fill launch (the query counter was read at the
      // last synchronisation; k_revert does not use it)
      const std::initializer_list<FillRange> resets = {{revert.get(), static_cast<uint64_t>(nm), 0},
                                                       {&cnt.get()->restored, 8, 0},
                                                       {&cnt.get()->query, 8, 0}};
      if (first_round)
        undo_detect_async(ctx, *isc, X, F, nf, falive.get(), qa, nqr, owner.get(), revert.get(), resets);
      else
        undo_detect_restored_async(ctx, *isc, X, F, nf, falive.get(), rlist.get(), nrest, qa, nqr, owner.get(),
                                   revert.get(), resets);
      PCU_LAUNCH(ctx, k_revert, grid_for(nm, 128), 128, 0, nm, revert.get(), off.get(), deg.get(), inc.get(),
                 Fprev.get(), X, F, falive.get(), valive.get(), Q.get(), owner.get(), B, newinv.get(), cnt.get(),
                 rlist.get());
      // rebuild the query list from still-applied collapses
      PCU_LAUNCH(ctx, k_requery, grid_for(nqr, 256), 256, 0, qa, nqr, owner.get(), B.applied, qb, cnt.get());
      h = sync_counters(true);  // ---- sync per round
      unsigned long long found = 0, ncand = 0;
      int redo = 0;
      unsigned long long ncls[3];
      detect_read(ds_host.data(), &found, &redo, &ncand, ncls);
      if (undo_stats)  // PAMOPT_UNDO_STATS=1: one line per detection round (diagnostics)
        std::fprintf(stderr, "undo it=%lld round=%d alive=%lld queries=%lld restored=%lld cand=%llu cls=%llu/%llu/%llu found=%llu\n",
                     static_cast<long long>(S.iterations), rounds, static_cast<long long>(alive_faces),
                     static_cast<long long>(nqr), static_cast<long long>(nrest), ncand, ncls[0], ncls[1], ncls[2], found);
      ctx.prof.mark(st, "undo_round");
      if (redo) {  // candidate buffer overflow: nothing was flagged or reverted; grow and repeat
        detect_grow(*isc, ncand);
        continue;
      }
      if (found == 0) break;
      ++rounds;
      first_round = false;
      nqr = static_cast<int64_t>(h.query);
      nrest = static_cast<int64_t>(h.restored);
      std::swap(qa, qb);
    }
    // restored faces get their boxes in the next round (its build set); after the last round the
    // faces restored by it still need them
    if (nqr == 0 && nrest > 0) boxes_update(ctx, *isc, X, F, rlist.get(), nrest, falive.get());
    succ = static_cast<int64_t>(h.applied);
    alive_faces -= static_cast<int64_t>(h.removed);
    nnew = static_cast<int64_t>(h.newinv);
    S.link_failures += static_cast<int64_t>(h.link_fail);
    S.undone += static_cast<int64_t>(h.undone);
  }

  // statistics and the invalid-flag update (SPEC.md:559 stall counter)
  void end_iteration() {
    PCU_REQUIRE(phase == 4, PAMOPT_CU_EINVAL, "qem: end_iteration() out of order");
    S.undo_hist[std::min(rounds, 7)]++;
    S.max_undo_rounds = std::max<int64_t>(S.max_undo_rounds, rounds);
    S.collapses += succ;
    alive_verts -= succ;
    S.per_iter.push_back(succ);
    bool keep_old;  // (duplicates are harmless for the binary search)
    if (succ > 0) {
      keep_old = false;
      retain = 0;
      zero_run = 0;
    } else {
      ++zero_run;
      ++retain;
      keep_old = retain < P.tolerance;
      if (!keep_old) retain = 0;
    }
    if (!keep_old) {  // the set restarts from this iteration's pairs: swap the buffers
      std::swap(inv, newinv);
      if (newinv.n < static_cast<size_t>(ecap)) newinv.alloc(ecap, st);
      ninv = nnew;
      build_inv_table();
    } else if (nnew) {  // the set grows: append, and insert the new pairs into the table
      if (inv.n < static_cast<size_t>(ninv + nnew)) {
        DevBuf<uint64_t> grown(2 * static_cast<size_t>(ninv + nnew), st);
        if (ninv) PCU_CUDA(cudaMemcpyAsync(grown.get(), inv.get(), ninv * 8, cudaMemcpyDeviceToDevice, st));
        inv = std::move(grown);
      }
      PCU_CUDA(cudaMemcpyAsync(inv.get() + ninv, newinv.get(), nnew * 8, cudaMemcpyDeviceToDevice, st));
      const bool fresh = ninv == 0;
      ninv += nnew;
      if (fresh || 2 * static_cast<uint64_t>(ninv) > inv_mask + 1)
        build_inv_table();
      else
        PCU_LAUNCH(ctx, k_inv_insert, grid_for(nnew, 256), 256, 0, newinv.get(), nnew,
                   reinterpret_cast<unsigned long long*>(inv_tab.get()), inv_mask);
    }
    ctx.prof.mark(st, "invalid_update");
    phase = 0;
  }

  void iterate() {
    prepare();
    propagate_and_mark();
    collapse_batch();
    undo_loop();
    end_iteration();
  }

  // compaction (mesh.cpp:278-292): alive vertices used by alive faces, order preserving
  void finish() {
    if (nf == 0 || nv == 0) return;
    DevBuf<uint32_t> vk(nv, st), vmap(nv, st), fk(nf, st), fmap(nf, st);
    vk.memset(0, st);
    PCU_LAUNCH(ctx, k_used, grid_for(nf, 256), 256, 0, F, falive.get(), nf, vk.get());
    PCU_LAUNCH(ctx, k_vkeep, grid_for(nv, 256), 256, 0, valive.get(), nv, vk.get());
    PCU_LAUNCH(ctx, k_fkeep, grid_for(nf, 256), 256, 0, falive.get(), nf, fk.get());
    exclusive_scan_u32(ctx, vk.get(), vmap.get(), nv);
    exclusive_scan_u32(ctx, fk.get(), fmap.get(), nf);
    const int64_t nv2 = static_cast<int64_t>(read_scalar(ctx, vmap.get() + nv - 1)) + read_scalar(ctx, vk.get() + nv - 1);
    const int64_t nf2 = static_cast<int64_t>(read_scalar(ctx, fmap.get() + nf - 1)) + read_scalar(ctx, fk.get() + nf - 1);
    DevBuf<double> Vo(3 * (nv2 ? nv2 : 1), st);
    DevBuf<int32_t> Fo(3 * (nf2 ? nf2 : 1), st);
    PCU_LAUNCH(ctx, k_compact, grid_for(std::max(nv, nf), 256), 256, 0, X, F, nv, nf, vk.get(), vmap.get(), fk.get(),
               fmap.get(), Vo.get(), Fo.get());
    V = std::move(Vo);
    Fb = std::move(Fo);
    nv = nv2;
    nf = nf2;
    X = V.get();
    F = Fb.get();
    ctx.prof.mark(st, "compact");
    ctx.prof.dump("simplify");
  }
};

namespace {
__global__ void k_face_keys(const int32_t* __restrict__ F, const uint8_t* __restrict__ falive, int64_t nf,
                            const unsigned long long* __restrict__ vmin, uint64_t* __restrict__ out) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  if (!falive[f]) {
    out[f] = ~0ull;
    return;
  }
  unsigned long long k = vmin[F[3 * f]];
  k = vmin[F[3 * f + 1]] < k ? vmin[F[3 * f + 1]] : k;
  k = vmin[F[3 * f + 2]] < k ? vmin[F[3 * f + 2]] : k;
  out[f] = k;
}
}  // namespace

QemState* qem_create(Ctx& ctx, DevBuf<double>& V, DevBuf<int32_t>& F, int64_t& nv, int64_t& nf, int64_t target,
                     const SimplifyParams& P, SimplifyStats& S) {
  PCU_REQUIRE(target >= 0, PAMOPT_CU_EINVAL, "simplify_to: negative target");
  auto* q = new QemState(ctx, V, F, nv, nf, target, P, S);
  q->key_order = true;
  return q;
}
void qem_destroy(QemState* q) { delete q; }
bool qem_done(const QemState* q) { return q->done(); }
void qem_prepare(QemState* q) { q->prepare(); }
void qem_propagate_and_mark(QemState* q) { q->propagate_and_mark(); }
void qem_collapse_batch(QemState* q) { q->collapse_batch(); }
void qem_undo_loop(QemState* q) { q->undo_loop(); }
void qem_end_iteration(QemState* q) { q->end_iteration(); }
void qem_finish(QemState* q) { q->finish(); }
int qem_phase(const QemState* q) { return q->phase; }

QemView qem_view(QemState* q) {
  QemView v;
  v.nv = q->nv;
  v.nf = q->nf;
  v.ne = q->phase >= 2 ? q->ne : static_cast<int64_t>(read_scalar(q->ctx, &q->cnt.get()->edges));
  v.nm = q->nm;
  v.alive_faces = q->alive_faces;
  v.X = q->X;
  v.F = q->F;
  v.falive = q->falive.get();
  v.valive = q->valive.get();
  v.Q = q->Q.get();
  v.ea = q->ea.get();
  v.eb = q->eb.get();
  v.key = q->key.get();
  v.place = q->place.get();
  v.valid = q->valid.get();
  v.marked_sorted = q->mlist;
  v.rem = q->rem.get();
  v.applied = q->B.applied;
  v.rounds = q->rounds;
  v.succ = q->succ;
  return v;
}

void qem_face_keys(QemState* q, uint64_t* d_out) {
  PCU_REQUIRE(q->phase >= 2, PAMOPT_CU_EINVAL, "qem: face keys exist after propagate_and_mark()");
  PCU_LAUNCH(q->ctx, k_face_keys, grid_for(q->nf, 256), 256, 0, q->F, q->falive.get(), q->nf, q->vmin.get(), d_out);
}

void simplify_run(Ctx& ctx, DevBuf<double>& V, DevBuf<int32_t>& Fb, int64_t& nv, int64_t& nf, int64_t target,
                  const SimplifyParams& P, SimplifyStats& S) {
  PCU_REQUIRE(target >= 0, PAMOPT_CU_EINVAL, "simplify_to: negative target");
  if (nf <= target || nf == 0) return;
  QemState q(ctx, V, Fb, nv, nf, target, P, S);
  while (!q.done()) q.iterate();
  q.finish();
}

}  // namespace pcu

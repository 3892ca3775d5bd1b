// metrics.cu — certification and quality metrics beside the hot path:
//   * analyze_topology (mesh.cpp:113-150): sorted (edge key, face) entries give the edge
//     incidence runs; a thread per vertex runs the single-fan test (mesh.cpp:65-109) over its
//     CSR incidence slice with global scratch, so any valence works.
//   * nearest_primitive (lbvh.cpp:192-237): a Karras LBVH over 30-bit Morton codes, f32 boxes
//     rounded outward, one thread per query with a nearest-first stack; pruning is conservative
//     (bound shrunk by 1e-12 relative) so the exact argmin — ties to the lower face id — is never
//     cut.  Distances use the pinned ptri_sq, so results equal the reference bit for bit.
//   * the pinned area-weighted sampler (integer weights, order-free prefix sums), Chamfer,
//     Hausdorff and the minimum internal angle (SPEC quality_metrics).
#include <cub/cub.cuh>

#include <string>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace pcu {
namespace {

__device__ __forceinline__ D3 ldv(const double* V, int64_t i) { return D3{V[3 * i], V[3 * i + 1], V[3 * i + 2]}; }

__device__ __forceinline__ uint64_t ekey(int32_t u, int32_t v) {
  const uint32_t a = static_cast<uint32_t>(min(u, v)), b = static_cast<uint32_t>(max(u, v));
  return (static_cast<uint64_t>(a) << 32) | b;
}

// ------------------------------------------------------------------------ topology
__global__ void k_topo_entries(const int32_t* __restrict__ F, int64_t nf, uint64_t* __restrict__ ekeys,
                               int32_t* __restrict__ efaces, uint64_t* __restrict__ vkeys,
                               uint32_t* __restrict__ vdeg) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  const int32_t t[3] = {F[3 * f], F[3 * f + 1], F[3 * f + 2]};
  for (int k = 0; k < 3; ++k) {
    ekeys[3 * f + k] = ekey(t[k], t[(k + 1) % 3]);
    efaces[3 * f + k] = static_cast<int32_t>(f);
    const bool dup = (k >= 1 && t[k] == t[0]) || (k == 2 && t[k] == t[1]);
    vkeys[3 * f + k] = dup ? ~0ull : (static_cast<uint64_t>(t[k]) << 32) | static_cast<uint32_t>(f);
    if (!dup) atomicAdd(&vdeg[t[k]], 1u);
  }
}

__global__ void k_run_heads(const uint64_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ head) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

__global__ void k_run_starts(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ head,
                             const uint32_t* __restrict__ hpos, int64_t n, int64_t* __restrict__ start,
                             uint64_t* __restrict__ ukeys) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n && head[i]) {
    start[hpos[i]] = i;
    ukeys[hpos[i]] = keys[i];
  }
}

__global__ void k_run_stats(const int64_t* __restrict__ start, int64_t ne, uint32_t* __restrict__ nmflag,
                            unsigned long long* __restrict__ boundary) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= ne) return;
  const int64_t c = start[e + 1] - start[e];
  nmflag[e] = (c != 1 && c != 2) ? 1u : 0u;
  if (c == 1) agg_inc(boundary);
}

__device__ __forceinline__ int64_t lower_u64(const uint64_t* a, int64_t n, uint64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// single-fan test per vertex (mesh.cpp:65-109): neighbours across 2-face edges at v, <= 2
// distinct per incident face, and one connected component.  Scratch is indexed by the
// vertex's CSR slots, so nothing is capped.
__global__ void k_fan(const int32_t* __restrict__ F, int64_t nv, const uint32_t* __restrict__ off,
                      const uint32_t* __restrict__ deg, const int32_t* __restrict__ inc,
                      const uint64_t* __restrict__ ukeys, const int64_t* __restrict__ start, int64_t ne,
                      const int32_t* __restrict__ efaces, int32_t* __restrict__ nb2, uint8_t* __restrict__ vis,
                      int32_t* __restrict__ stk, uint32_t* __restrict__ bad, unsigned long long* __restrict__ used) {
  const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (v >= nv) return;
  const int m = static_cast<int>(deg[v]);
  bad[v] = 0;
  if (m == 0) return;
  agg_inc(used);
  const int64_t base = off[v];
  const int32_t* L = inc + base;
  for (int i = 0; i < m; ++i) {
    const int32_t f = L[i];
    int cnt = 0, n0 = -1, n1 = -1;
    for (int k = 0; k < 3; ++k) {
      const int32_t a = F[3 * static_cast<int64_t>(f) + k], b = F[3 * static_cast<int64_t>(f) + (k + 1) % 3];
      if (a != v && b != v) continue;
      const int64_t e = lower_u64(ukeys, ne, ekey(a, b));
      if (start[e + 1] - start[e] != 2) continue;
      for (int64_t j = start[e]; j < start[e] + 2; ++j) {
        const int32_t g = efaces[j];
        if (g == f) continue;
        int lo = 0, hi = m;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (L[mid] < g) lo = mid + 1;
          else hi = mid;
        }
        if (lo == n0 || lo == n1) continue;
        if (cnt == 0) n0 = lo;
        else if (cnt == 1) n1 = lo;
        ++cnt;
      }
    }
    if (cnt > 2) {
      bad[v] = 1;
      return;
    }
    nb2[2 * (base + i)] = n0;
    nb2[2 * (base + i) + 1] = n1;
    vis[base + i] = 0;
  }
  int top = 0, seen = 1;
  stk[base + top++] = 0;
  vis[base] = 1;
  while (top > 0) {
    const int i = stk[base + --top];
    for (int q = 0; q < 2; ++q) {
      const int j = nb2[2 * (base + i) + q];
      if (j >= 0 && !vis[base + j]) {
        vis[base + j] = 1;
        ++seen;
        stk[base + top++] = j;
      }
    }
  }
  if (seen != m) bad[v] = 1;
}

template <class T>
__global__ void k_compact_flagged(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, int64_t n,
                                  const T* __restrict__ src, T* __restrict__ dst) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n && flag[i]) dst[pos[i]] = src ? src[i] : static_cast<T>(i);
}

__global__ void k_low32(const uint64_t* __restrict__ k, int64_t n, int32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = static_cast<int32_t>(k[i] & 0xffffffffu);
}

// --------------------------------------------------------------------------- LBVH
struct BNode {
  float lo[3], hi[3];
  int32_t left, right;  // >= 0 internal node, < 0: leaf ~k (sorted position k)
};

__device__ __forceinline__ float fdown(double x) { return __double2float_rd(x); }
__device__ __forceinline__ float fup(double x) { return __double2float_ru(x); }

__global__ void k_face_bounds(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t nf,
                              float* __restrict__ fb, unsigned int* __restrict__ scene) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  const D3 a = ldv(V, F[3 * f]), b = ldv(V, F[3 * f + 1]), c = ldv(V, F[3 * f + 2]);
  const double lo[3] = {fmin(fmin(a.x, b.x), c.x), fmin(fmin(a.y, b.y), c.y), fmin(fmin(a.z, b.z), c.z)};
  const double hi[3] = {fmax(fmax(a.x, b.x), c.x), fmax(fmax(a.y, b.y), c.y), fmax(fmax(a.z, b.z), c.z)};
  for (int k = 0; k < 3; ++k) {
    fb[6 * f + k] = fdown(lo[k]);
    fb[6 * f + 3 + k] = fup(hi[k]);
    // scene centroid bounds via order-preserving float keys
    const float cm = static_cast<float>(0.5 * (lo[k] + hi[k]));
    const unsigned int u = __float_as_uint(cm);
    const unsigned int key = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    atomicMin(&scene[k], key);
    atomicMax(&scene[3 + k], key);
  }
}

__device__ __forceinline__ float unkey(unsigned int key) {
  return __uint_as_float((key & 0x80000000u) ? (key & 0x7fffffffu) : ~key);
}

__device__ __forceinline__ uint32_t spread10(uint32_t x) {
  x &= 0x3ffu;
  x = (x | (x << 16)) & 0x030000FFu;
  x = (x | (x << 8)) & 0x0300F00Fu;
  x = (x | (x << 4)) & 0x030C30C3u;
  x = (x | (x << 2)) & 0x09249249u;
  return x;
}

__global__ void k_morton(const float* __restrict__ fb, int64_t nf, const unsigned int* __restrict__ scene,
                         uint64_t* __restrict__ keys) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  uint32_t q[3];
  for (int k = 0; k < 3; ++k) {
    const float lo = unkey(scene[k]), hi = unkey(scene[3 + k]);
    const float c = 0.5f * (fb[6 * f + k] + fb[6 * f + 3 + k]);
    const float ext = hi - lo;
    float t = ext > 0.f ? (c - lo) / ext : 0.f;
    t = fminf(fmaxf(t, 0.f), 1.f);
    q[k] = static_cast<uint32_t>(fminf(t * 1024.f, 1023.f));
  }
  const uint32_t code = (spread10(q[0]) << 2) | (spread10(q[1]) << 1) | spread10(q[2]);
  keys[f] = (static_cast<uint64_t>(code) << 32) | static_cast<uint32_t>(f);
}

__device__ __forceinline__ int delta(const uint64_t* k, int64_t n, int64_t i, int64_t j) {
  if (j < 0 || j >= n) return -1;
  return __clzll(static_cast<long long>(k[i] ^ k[j]));  // keys unique (face id in the low bits)
}

// Karras 2012: internal node i covers a key range; children are internal nodes or leaves
__global__ void k_karras(const uint64_t* __restrict__ k, int64_t n, BNode* __restrict__ nodes,
                         int32_t* __restrict__ parent) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n - 1) return;
  const int d = (delta(k, n, i, i + 1) - delta(k, n, i, i - 1)) >= 0 ? 1 : -1;
  const int dmin = delta(k, n, i, i - d);
  int64_t lmax = 2;
  while (delta(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
  int64_t l = 0;
  for (int64_t t = lmax >> 1; t >= 1; t >>= 1)
    if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
  const int64_t j = i + l * d;
  const int dnode = delta(k, n, i, j);
  int64_t s = 0;
  int64_t t = l;
  do {
    t = (t + 1) >> 1;
    if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
  } while (t > 1);
  const int64_t gamma = i + s * d + min(d, 0);
  const int64_t lo = min(i, j), hi = max(i, j);
  const int32_t left = (lo == gamma) ? ~static_cast<int32_t>(gamma) : static_cast<int32_t>(gamma);
  const int32_t right = (hi == gamma + 1) ? ~static_cast<int32_t>(gamma + 1) : static_cast<int32_t>(gamma + 1);
  nodes[i].left = left;
  nodes[i].right = right;
  // parent links: internal nodes at [0, n-1), leaves at [n-1, 2n-1)
  parent[left >= 0 ? left : (n - 1) + ~left] = static_cast<int32_t>(i);
  parent[right >= 0 ? right : (n - 1) + ~right] = static_cast<int32_t>(i);
}

__global__ void k_refit(const uint64_t* __restrict__ k, int64_t n, const float* __restrict__ fb,
                        BNode* __restrict__ nodes, const int32_t* __restrict__ parent,
                        unsigned int* __restrict__ flags) {
  const int64_t leaf = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (leaf >= n) return;
  int32_t p = parent[(n - 1) + leaf];
  while (p >= 0) {
    __threadfence();
    if (atomicAdd(&flags[p], 1u) == 0) return;  // the sibling subtree is not finished yet
    __threadfence();
    float lo[3], hi[3];
    for (int c = 0; c < 2; ++c) {
      const int32_t ch = c == 0 ? nodes[p].left : nodes[p].right;
      const float* b;
      float tmp[6];
      if (ch < 0) {
        const int64_t face = static_cast<int64_t>(k[~ch] & 0xffffffffu);
        b = fb + 6 * face;
      } else {
        volatile const BNode* q = nodes + ch;
        for (int a = 0; a < 3; ++a) {
          tmp[a] = q->lo[a];
          tmp[3 + a] = q->hi[a];
        }
        b = tmp;
      }
      for (int a = 0; a < 3; ++a) {
        lo[a] = c == 0 ? b[a] : fminf(lo[a], b[a]);
        hi[a] = c == 0 ? b[3 + a] : fmaxf(hi[a], b[3 + a]);
      }
    }
    volatile BNode* w = nodes + p;
    for (int a = 0; a < 3; ++a) {
      w->lo[a] = lo[a];
      w->hi[a] = hi[a];
    }
    p = parent[p];
  }
}

__device__ __forceinline__ double box_sq(const float* lo, const float* hi, D3 p) {
  const double dx = fmax(fmax(static_cast<double>(lo[0]) - p.x, 0.0), p.x - static_cast<double>(hi[0]));
  const double dy = fmax(fmax(static_cast<double>(lo[1]) - p.y, 0.0), p.y - static_cast<double>(hi[1]));
  const double dz = fmax(fmax(static_cast<double>(lo[2]) - p.z, 0.0), p.z - static_cast<double>(hi[2]));
  return (dx * dx + dy * dy) + dz * dz;
}

// point–triangle squared distance with the closest point (distance.cpp:26-79)
__device__ double ptri_closest(D3 p, D3 a, D3 b, D3 c, D3& q) {
  const D3 n = cross(sub(b, a), sub(c, a));
  const double nn = sqn(n);
  double best = __longlong_as_double(0x7ff0000000000000ll);
  q = a;
  if (nn > 0.0) {
    const D3 ap = sub(p, a);
    const double dist_n = dot(ap, n);
    const double s = dist_n / nn;
    const D3 proj = D3{p.x - s * n.x, p.y - s * n.y, p.z - s * n.z};
    const D3 v0 = sub(b, a), v1 = sub(c, a), v2 = sub(proj, a);
    const double d00 = sqn(v0), d01 = dot(v0, v1), d11 = sqn(v1);
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
  const D3 E[3][2] = {{a, b}, {b, c}, {c, a}};
  for (int k = 0; k < 3; ++k) {
    const D3 u = E[k][0], ab = sub(E[k][1], E[k][0]);
    const double denom = sqn(ab);
    double t = denom > 0.0 ? dot(sub(p, u), ab) / denom : 0.0;
    t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);
    const D3 s = axpy(u, t, ab);
    const double d2 = sqn(sub(p, s));
    if (d2 < best) {
      best = d2;
      q = s;
    }
  }
  return best;
}

constexpr int kStack = 128;
constexpr double kShrink = 1.0 - 1e-12;  // conservative pruning margin over FP64 rounding

// One thread per query: depth-first, nearer child first, entries carry their box bound.  Leaves
// are stack entries too (encoded ~sorted position).  The global min over (d2, face id) is
// unique, so the visit order only affects speed.
__global__ void __launch_bounds__(128) k_nearest(const double* __restrict__ V, const int32_t* __restrict__ F,
                                                 int64_t nf, const BNode* __restrict__ nodes,
                                                 const uint64_t* __restrict__ keys, const float* __restrict__ fb,
                                                 const double* __restrict__ pts, int64_t n, int32_t* __restrict__ face,
                                                 double* __restrict__ d2out, double* __restrict__ closest,
                                                 unsigned long long* __restrict__ overflow) {
  const int64_t qi = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (qi >= n) return;
  const D3 p = ldv(pts, qi);
  double best = __longlong_as_double(0x7ff0000000000000ll);
  int32_t bf = -1;
  int32_t stack[kStack];
  double sb[kStack];
  int top = 0;
  auto bound_of = [&](int32_t e) {
    if (e < 0) {
      const int64_t f = static_cast<int64_t>(keys[~e] & 0xffffffffu);
      return box_sq(fb + 6 * f, fb + 6 * f + 3, p);
    }
    return box_sq(nodes[e].lo, nodes[e].hi, p);
  };
  const int32_t root = nf == 1 ? ~0 : 0;
  stack[top] = root;
  sb[top++] = bound_of(root);
  while (top > 0) {
    --top;
    const int32_t e = stack[top];
    if (sb[top] * kShrink > best) continue;
    if (e < 0) {
      const int32_t f = static_cast<int32_t>(keys[~e] & 0xffffffffu);
      const int64_t f3 = 3 * static_cast<int64_t>(f);
      const double d2 = ptri_sq(p, ldv(V, F[f3]), ldv(V, F[f3 + 1]), ldv(V, F[f3 + 2]));
      if (d2 < best || (d2 == best && f < bf)) {
        best = d2;
        bf = f;
      }
      continue;
    }
    const int32_t ch[2] = {nodes[e].left, nodes[e].right};
    const double db[2] = {bound_of(ch[0]), bound_of(ch[1])};
    const int near = db[0] <= db[1] ? 0 : 1;
    for (int s = 0; s < 2; ++s) {
      const int c = s == 0 ? 1 - near : near;  // farther first, nearer on top
      if (db[c] * kShrink > best) continue;
      if (top == kStack) {
        atomicAdd(overflow, 1ull);
        continue;
      }
      stack[top] = ch[c];
      sb[top++] = db[c];
    }
  }
  face[qi] = bf;
  d2out[qi] = best;
  if (closest) {
    D3 q = D3{0.0, 0.0, 0.0};
    if (bf >= 0) {
      const int64_t f3 = 3 * static_cast<int64_t>(bf);
      ptri_closest(p, ldv(V, F[f3]), ldv(V, F[f3 + 1]), ldv(V, F[f3 + 2]), q);
    }
    closest[3 * qi] = q.x;
    closest[3 * qi + 1] = q.y;
    closest[3 * qi + 2] = q.z;
  }
}

// ------------------------------------------------------------------------- sampling
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t hash_k(uint64_t seed, uint64_t k) {
  return mix64(seed + (k + 1) * 0x9E3779B97F4A7C15ull);
}
__device__ __forceinline__ double unit53(uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }

__global__ void k_areas(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t nf,
                        double* __restrict__ area, unsigned long long* __restrict__ amax_bits) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  const D3 a = ldv(V, F[3 * f]), b = ldv(V, F[3 * f + 1]), c = ldv(V, F[3 * f + 2]);
  const double A = 0.5 * sqrt(sqn(cross(sub(b, a), sub(c, a))));
  area[f] = A;
  atomicMax(amax_bits, static_cast<unsigned long long>(__double_as_longlong(A)));  // A >= 0: bits order
}

__global__ void k_weights(const double* __restrict__ area, int64_t nf, const unsigned long long* __restrict__ amax_bits,
                          uint64_t* __restrict__ w) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  const double amax = __longlong_as_double(static_cast<long long>(*amax_bits));
  w[f] = static_cast<uint64_t>(floor(area[f] / amax * 4294967296.0));
}

__global__ void k_sample(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t nf,
                         const uint64_t* __restrict__ cum, int64_t n, uint64_t seed, double* __restrict__ pts,
                         int32_t* __restrict__ fid) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint64_t W = cum[nf - 1];
  const uint64_t h0 = hash_k(seed, 3 * i), h1 = hash_k(seed, 3 * i + 1), h2 = hash_k(seed, 3 * i + 2);
  const uint64_t t = __umul64hi(h0, W);
  int64_t lo = 0, hi = nf;  // first f with cum[f] > t
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cum[mid] > t) hi = mid;
    else lo = mid + 1;
  }
  const int64_t f = lo;
  const double u1 = unit53(h1), u2 = unit53(h2);
  const double s = sqrt(u1);
  const double wa = 1.0 - s, wb = s * (1.0 - u2), wc = s * u2;
  const D3 a = ldv(V, F[3 * f]), b = ldv(V, F[3 * f + 1]), c = ldv(V, F[3 * f + 2]);
  pts[3 * i] = (a.x * wa + b.x * wb) + c.x * wc;
  pts[3 * i + 1] = (a.y * wa + b.y * wb) + c.y * wc;
  pts[3 * i + 2] = (a.z * wa + b.z * wb) + c.z * wc;
  if (fid) fid[i] = static_cast<int32_t>(f);
}

__global__ void k_corner_cos(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t nf,
                             unsigned long long* __restrict__ maxkey) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  const D3 p[3] = {ldv(V, F[3 * f]), ldv(V, F[3 * f + 1]), ldv(V, F[3 * f + 2])};
  double m = -1.0;
  if (!(sqn(cross(sub(p[1], p[0]), sub(p[2], p[0]))) > 0.0)) {
    m = 1.0;
  } else {
    for (int k = 0; k < 3; ++k) {
      const D3 u = sub(p[(k + 1) % 3], p[k]), w = sub(p[(k + 2) % 3], p[k]);
      double c = dot(u, w) / sqrt(sqn(u) * sqn(w));
      c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
      m = fmax(m, c);
    }
  }
  // order-preserving key of a double in [-1, 1]
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(m));
  const unsigned long long key = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
  atomicMax(maxkey, key);
}

__global__ void k_d2_stats(const double* __restrict__ d2, int64_t n, double* __restrict__ sum_out,
                           unsigned long long* __restrict__ max_bits) {
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  double s = 0.0, mx = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    s += d2[i];
    mx = fmax(mx, d2[i]);
  }
  const double bs = BR(tmp).Sum(s);
  if (threadIdx.x == 0) sum_out[blockIdx.x] = bs;
  atomicMax(max_bits, static_cast<unsigned long long>(__double_as_longlong(mx)));
}

}  // namespace

// ================================================================================= host
void analyze_topology(Ctx& ctx, const int32_t* dF, int64_t nf, int64_t nv, TopologyResult& out) {
  cudaStream_t st = ctx.stream;
  out = TopologyResult();
  if (nf == 0) {
    out.manifold = out.watertight = 1;
    return;
  }
  const int64_t ne3 = 3 * nf;
  DevBuf<uint64_t> ekeys(ne3, st), vkeys(ne3, st), ekeys2(ne3, st), vkeys2(ne3, st);
  DevBuf<int32_t> efaces(ne3, st), efaces2(ne3, st);
  DevBuf<uint32_t> vdeg(nv ? nv : 1, st), voff(nv ? nv : 1, st);
  PCU_CUDA(cudaMemsetAsync(vdeg.get(), 0, (nv ? nv : 1) * 4, st));
  PCU_LAUNCH(ctx, k_topo_entries, grid_for(nf, 256), 256, 0, dF, nf, ekeys.get(), efaces.get(), vkeys.get(),
             vdeg.get());
  {
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, ekeys.get(), ekeys2.get(), efaces.get(), efaces2.get(),
                                    static_cast<int>(ne3), 0, 64, st);
    DevBuf<uint8_t> tmp(need, st);
    PCU_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), need, ekeys.get(), ekeys2.get(), efaces.get(), efaces2.get(),
                                             static_cast<int>(ne3), 0, 64, st));
    ++ctx.launches;
  }
  sort_pairs_u64(ctx, vkeys.get(), ne3);  // (v, f) ascending; duplicates (~0) last
  // edge runs
  DevBuf<uint32_t> head(ne3, st), hpos(ne3, st);
  PCU_LAUNCH(ctx, k_run_heads, grid_for(ne3, 256), 256, 0, ekeys2.get(), ne3, head.get());
  exclusive_scan_u32(ctx, head.get(), hpos.get(), ne3);
  const int64_t ne = static_cast<int64_t>(read_scalar(ctx, hpos.get() + ne3 - 1)) + read_scalar(ctx, head.get() + ne3 - 1);
  DevBuf<int64_t> start(ne + 1, st);
  DevBuf<uint64_t> ukeys(ne, st);
  PCU_LAUNCH(ctx, k_run_starts, grid_for(ne3, 256), 256, 0, ekeys2.get(), head.get(), hpos.get(), ne3, start.get(),
             ukeys.get());
  PCU_CUDA(cudaMemcpyAsync(start.get() + ne, &ne3, 8, cudaMemcpyHostToDevice, st));
  DevBuf<uint32_t> nmflag(ne, st), nmpos(ne, st);
  DevBuf<unsigned long long> ctr(2, st);
  PCU_CUDA(cudaMemsetAsync(ctr.get(), 0, 16, st));
  PCU_LAUNCH(ctx, k_run_stats, grid_for(ne, 256), 256, 0, start.get(), ne, nmflag.get(), ctr.get());
  exclusive_scan_u32(ctx, nmflag.get(), nmpos.get(), ne);
  const int64_t n_nme = static_cast<int64_t>(read_scalar(ctx, nmpos.get() + ne - 1)) + read_scalar(ctx, nmflag.get() + ne - 1);
  DevBuf<uint64_t> nme(n_nme ? n_nme : 1, st);
  PCU_LAUNCH(ctx, k_compact_flagged<uint64_t>, grid_for(ne, 256), 256, 0, nmflag.get(), nmpos.get(), ne, ukeys.get(),
             nme.get());
  // vertex incidence CSR (sorted (v, f) keys)
  exclusive_scan_u32(ctx, vdeg.get(), voff.get(), nv);
  DevBuf<int32_t> inc(ne3, st);
  PCU_LAUNCH(ctx, k_low32, grid_for(ne3, 256), 256, 0, vkeys.get(), ne3, inc.get());
  DevBuf<int32_t> nb2(2 * ne3, st), stk(ne3, st);
  DevBuf<uint8_t> vis(ne3, st);
  DevBuf<uint32_t> bad(nv, st), badpos(nv, st);
  PCU_LAUNCH(ctx, k_fan, grid_for(nv, 128), 128, 0, dF, nv, voff.get(), vdeg.get(), inc.get(), ukeys.get(),
             start.get(), ne, efaces2.get(), nb2.get(), vis.get(), stk.get(), bad.get(), ctr.get() + 1);
  exclusive_scan_u32(ctx, bad.get(), badpos.get(), nv);
  const int64_t n_nmv = static_cast<int64_t>(read_scalar(ctx, badpos.get() + nv - 1)) + read_scalar(ctx, bad.get() + nv - 1);
  DevBuf<int32_t> nmv(n_nmv ? n_nmv : 1, st);
  PCU_LAUNCH(ctx, k_compact_flagged<int32_t>, grid_for(nv, 256), 256, 0, bad.get(), badpos.get(), nv,
             static_cast<const int32_t*>(nullptr), nmv.get());
  unsigned long long hc[2];
  PCU_CUDA(cudaMemcpyAsync(hc, ctr.get(), 16, cudaMemcpyDeviceToHost, st));
  out.nm_edges.resize(n_nme);
  out.nm_verts.resize(n_nmv);
  if (n_nme) PCU_CUDA(cudaMemcpyAsync(out.nm_edges.data(), nme.get(), n_nme * 8, cudaMemcpyDeviceToHost, st));
  if (n_nmv) PCU_CUDA(cudaMemcpyAsync(out.nm_verts.data(), nmv.get(), n_nmv * 4, cudaMemcpyDeviceToHost, st));
  PCU_CUDA(cudaStreamSynchronize(st));
  out.boundary = static_cast<int64_t>(hc[0]);
  out.manifold = (n_nme == 0 && n_nmv == 0) ? 1 : 0;
  out.watertight = (out.manifold && out.boundary == 0) ? 1 : 0;
  out.euler = static_cast<int64_t>(hc[1]) - ne + nf;
}

struct Lbvh {
  DevBuf<uint64_t> keys;
  DevBuf<BNode> nodes;
  DevBuf<float> fb;  // per-face f32 boxes, rounded outward
  int64_t nf = 0;
};

static void lbvh_build(Ctx& ctx, const double* dV, const int32_t* dF, int64_t nf, Lbvh& B) {
  cudaStream_t st = ctx.stream;
  B.nf = nf;
  B.fb.alloc(6 * nf, st);
  float* fb = B.fb.get();
  DevBuf<unsigned int> scene(6, st);
  const unsigned int init[6] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0u, 0u, 0u};
  PCU_CUDA(cudaMemcpyAsync(scene.get(), init, sizeof(init), cudaMemcpyHostToDevice, st));
  PCU_LAUNCH(ctx, k_face_bounds, grid_for(nf, 256), 256, 0, dV, dF, nf, fb, scene.get());
  B.keys.alloc(nf, st);
  PCU_LAUNCH(ctx, k_morton, grid_for(nf, 256), 256, 0, fb, nf, scene.get(), B.keys.get());
  sort_pairs_u64(ctx, B.keys.get(), nf);
  B.nodes.alloc(nf > 1 ? nf - 1 : 1, st);
  if (nf > 1) {
    DevBuf<int32_t> parent(2 * nf - 1, st);
    DevBuf<unsigned int> flags(nf - 1, st);
    PCU_CUDA(cudaMemsetAsync(parent.get(), 0xFF, 4, st));  // root has no parent
    PCU_CUDA(cudaMemsetAsync(flags.get(), 0, (nf - 1) * 4, st));
    PCU_LAUNCH(ctx, k_karras, grid_for(nf - 1, 256), 256, 0, B.keys.get(), nf, B.nodes.get(), parent.get());
    PCU_LAUNCH(ctx, k_refit, grid_for(nf, 256), 256, 0, B.keys.get(), nf, fb, B.nodes.get(), parent.get(),
               flags.get());
  }
}

void nearest_primitive(Ctx& ctx, const double* dV, const int32_t* dF, int64_t nf, const double* d_pts, int64_t n,
                       int32_t* d_face, double* d_d2, double* d_closest) {
  if (n == 0) return;
  PCU_REQUIRE(nf > 0, PAMOPT_CU_EINVAL, "nearest_primitive: empty mesh");
  Lbvh B;
  lbvh_build(ctx, dV, dF, nf, B);
  DevBuf<unsigned long long> ovf(1, ctx.stream);
  PCU_CUDA(cudaMemsetAsync(ovf.get(), 0, 8, ctx.stream));
  PCU_LAUNCH(ctx, k_nearest, grid_for(n, 128), 128, 0, dV, dF, nf, B.nodes.get(), B.keys.get(), B.fb.get(), d_pts, n,
             d_face, d_d2, d_closest, ovf.get());
  PCU_REQUIRE(read_scalar(ctx, ovf.get()) == 0, PAMOPT_CU_ECUDA, "nearest_primitive: traversal stack overflow");
}

bool sample_points(Ctx& ctx, const double* dV, const int32_t* dF, int64_t nf, int64_t n, uint64_t seed,
                   double* d_pts, int32_t* d_fid, double* total_area) {
  cudaStream_t st = ctx.stream;
  if (nf == 0) return false;
  DevBuf<double> area(nf, st);
  DevBuf<unsigned long long> amax(1, st);
  PCU_CUDA(cudaMemsetAsync(amax.get(), 0, 8, st));
  PCU_LAUNCH(ctx, k_areas, grid_for(nf, 256), 256, 0, dV, dF, nf, area.get(), amax.get());
  const unsigned long long ab = read_scalar(ctx, amax.get());
  double am;
  std::memcpy(&am, &ab, 8);
  if (!(am > 0.0)) return false;
  DevBuf<uint64_t> w(nf, st), cum(nf, st);
  PCU_LAUNCH(ctx, k_weights, grid_for(nf, 256), 256, 0, area.get(), nf, amax.get(), w.get());
  {
    size_t need = 0;
    cub::DeviceScan::InclusiveSum(nullptr, need, w.get(), cum.get(), nf, st);
    DevBuf<uint8_t> tmp(need, st);
    PCU_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), need, w.get(), cum.get(), nf, st));
    ++ctx.launches;
  }
  if (total_area) {
    DevBuf<double> s(1, st);
    size_t need = 0;
    cub::DeviceReduce::Sum(nullptr, need, area.get(), s.get(), nf, st);
    DevBuf<uint8_t> tmp(need, st);
    PCU_CUDA(cub::DeviceReduce::Sum(tmp.get(), need, area.get(), s.get(), nf, st));
    ++ctx.launches;
    *total_area = read_scalar(ctx, s.get());
  }
  if (n > 0) PCU_LAUNCH(ctx, k_sample, grid_for(n, 128), 128, 0, dV, dF, nf, cum.get(), n, seed, d_pts, d_fid);
  return true;
}

// directed sampled distances a -> b: (sum of d^2, max d^2, area of a)
void directed_d2(Ctx& ctx, const double* Va, const int32_t* Fa, int64_t nfa, const double* Vb, const int32_t* Fb,
                 int64_t nfb, int64_t n, uint64_t seed, double& sum_d2, double& max_d2, double& area_a) {
  cudaStream_t st = ctx.stream;
  DevBuf<double> pts(3 * n, st), d2(n, st);
  DevBuf<int32_t> face(n, st);
  PCU_REQUIRE(sample_points(ctx, Va, Fa, nfa, n, seed, pts.get(), nullptr, &area_a), PAMOPT_CU_EINVAL,
              "metrics: zero-area mesh");
  PCU_REQUIRE(nfb > 0, PAMOPT_CU_EINVAL, "metrics: empty mesh");
  nearest_primitive(ctx, Vb, Fb, nfb, pts.get(), n, face.get(), d2.get(), nullptr);
  const unsigned blocks = std::min<unsigned>(grid_for(n, 256), 592);
  DevBuf<double> part(blocks, st);
  DevBuf<unsigned long long> mx(1, st);
  PCU_CUDA(cudaMemsetAsync(mx.get(), 0, 8, st));
  PCU_LAUNCH(ctx, k_d2_stats, blocks, 256, 0, d2.get(), n, part.get(), mx.get());
  std::vector<double> hp(blocks);
  unsigned long long hm = 0;
  PCU_CUDA(cudaMemcpyAsync(hp.data(), part.get(), blocks * 8, cudaMemcpyDeviceToHost, st));
  PCU_CUDA(cudaMemcpyAsync(&hm, mx.get(), 8, cudaMemcpyDeviceToHost, st));
  PCU_CUDA(cudaStreamSynchronize(st));
  sum_d2 = 0.0;
  for (double x : hp) sum_d2 += x;
  std::memcpy(&max_d2, &hm, 8);
}

// IndexedMesh::validate (mesh.cpp:31-43): the first face (lowest id) that references a vertex
// outside [0, nv) or repeats an index.  key = f << 2 | reason (1 = out of range, 2 = repeated),
// reduced with one 64-bit atomicMin, so the reported face is the reference's first offender.
__global__ void k_validate(const int32_t* __restrict__ F, int64_t nf, int64_t nv, unsigned long long* __restrict__ key) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  const int32_t a = F[3 * f], b = F[3 * f + 1], c = F[3 * f + 2];
  const bool range = a < 0 || a >= nv || b < 0 || b >= nv || c < 0 || c >= nv;
  const bool rep = a == b || b == c || a == c;
  if (range || rep) atomicMin(key, (static_cast<unsigned long long>(f) << 2) | (range ? 1ull : 2ull));
}

void validate_mesh(Ctx& ctx, const int32_t* dF, int64_t nf, int64_t nv) {
  if (nf <= 0) return;
  DevBuf<unsigned long long> k(1, ctx.stream);
  PCU_CUDA(cudaMemsetAsync(k.get(), 0xFF, 8, ctx.stream));
  PCU_LAUNCH(ctx, k_validate, grid_for(nf, 256), 256, 0, dF, nf, nv, k.get());
  const unsigned long long key = read_scalar(ctx, k.get());
  if (key == ~0ull) return;
  const int64_t f = static_cast<int64_t>(key >> 2);
  int32_t t[3];
  PCU_CUDA(cudaMemcpyAsync(t, dF + 3 * f, sizeof(t), cudaMemcpyDeviceToHost, ctx.stream));
  PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  std::string msg = "invalid mesh: face " + std::to_string(f);
  if ((key & 3) == 1) {
    int32_t bad = t[0];
    for (int i = 0; i < 3; ++i)
      if (t[i] < 0 || t[i] >= nv) {
        bad = t[i];
        break;
      }
    msg += " references vertex " + std::to_string(bad);
  } else {
    msg += " has repeated vertex indices";
  }
  throw Error(PAMOPT_CU_EINVAL, msg);
}

std::vector<int32_t> index_range(Ctx& ctx, const int32_t* d, int64_t n) {
  DevBuf<int32_t> mm(2, ctx.stream);
  size_t need = 0;
  cub::DeviceReduce::Min(nullptr, need, d, mm.get(), n, ctx.stream);
  size_t need2 = 0;
  cub::DeviceReduce::Max(nullptr, need2, d, mm.get() + 1, n, ctx.stream);
  DevBuf<uint8_t> tmp(std::max(need, need2), ctx.stream);
  PCU_CUDA(cub::DeviceReduce::Min(tmp.get(), need, d, mm.get(), n, ctx.stream));
  PCU_CUDA(cub::DeviceReduce::Max(tmp.get(), need2, d, mm.get() + 1, n, ctx.stream));
  ctx.launches += 2;
  std::vector<int32_t> h(2);
  PCU_CUDA(cudaMemcpyAsync(h.data(), mm.get(), 8, cudaMemcpyDeviceToHost, ctx.stream));
  PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  return h;
}

double max_corner_cos(Ctx& ctx, const double* dV, const int32_t* dF, int64_t nf) {
  DevBuf<unsigned long long> k(1, ctx.stream);
  PCU_CUDA(cudaMemsetAsync(k.get(), 0, 8, ctx.stream));
  PCU_LAUNCH(ctx, k_corner_cos, grid_for(nf, 256), 256, 0, dV, dF, nf, k.get());
  const unsigned long long key = read_scalar(ctx, k.get());
  const unsigned long long u = (key >> 63) ? (key & 0x7fffffffffffffffull) : ~key;
  double m;
  std::memcpy(&m, &u, 8);
  return m;
}

}  // namespace pcu

// udf.cu — stage 1a: narrow-band UDF over the voxel-grid hierarchy (SPEC.md:157-236,
// PAPER.md:55-74) and the fused UDF->SDF band subtraction.
//
// Device pipeline (all on the context stream, inputs resident in HBM):
//   1. prep      per triangle: vertices + AABB into a 128 B record (one coalesced load later)
//   2. level 0   per triangle: the r=8 cells of its conservative index box that pass the
//                pinned predicate -> (cell, tri) pairs, warp-aggregated append
//   3. refine    per surviving pair x 8 children, levels 16 .. r_b (r_b = max(8, R/8), the
//                "brick" level: one brick = bs^3 finest cells, bs = R/r_b <= 8)
//   4. bin       counting sort of brick-level pairs by brick; work items of <= 128 triangles
//   5. brick     one CTA per work item: every warp takes a triangle, descends the last
//                log2(bs) levels inside the brick with ballots (8 -> 64 -> 512 cell masks in
//                shared memory), dilates the finest mask to the (bs+1)^3 brick vertices and
//                evaluates each needed vertex ONCE per triangle; per-vertex minima live in
//                shared memory (64-bit atomicMin on the f64 bit pattern, order independent),
//                then merge into the per-brick global block
//   6. finalize  per lattice vertex: min over the <=8 bricks that hold it, sqrt, f32, and the
//                band subtraction s = (float)((double)u - eps); no candidate -> +INF / +1.0
// The pinned predicate: box_d2(c, aabb) <= (thr+1e-9)^2 && sqrt(ptri_sq(c,t))
// <= thr, thr = 3/R + 0.8660254037844386/r — FP64, no FMA contraction.
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace pcu {
namespace {

constexpr double kHalfSqrt3 = 0.8660254037844386;
constexpr int kChunk = 128;  // triangles per brick work item

struct __align__(16) TriD {  // loaded as sizeof/16 int4 words by k_brick
  double a[3], b[3], c[3], lo[3], hi[3];
  float ab[3], ac[3];  // local frame (b-a, c-a computed in FP64, rounded to FP32)
  float n[3];          // unit normal (FP32)
  float binv[3];       // inverse Gram matrix of (ab, ac): [g11, -g01, g00] / det
  float blo[3], bhi[3];  // AABB in the local frame (FP32)
  float L2;            // max squared edge length
  int wc;              // well conditioned: every corner angle has sin^2 >= 0.01
  float ie[3];         // FP32 1/|ab|^2, 1/|bc|^2, 1/|ca|^2 (0 for a zero-length edge; filter only)
};
static_assert(sizeof(TriD) % 16 == 0 && sizeof(TriD) / 16 <= 32, "TriD is copied by one warp in int4 words");

// FP32 point-triangle squared distance in the triangle's local frame (p relative to a).
// Used only as a certified filter for well-conditioned triangles (see survives / k_brick): its
// error is far below the 1e-4 * L^2 + 1e-3 * d^2 margin, so every decision it takes equals the
// FP64 decision; everything near a threshold is re-evaluated with the pinned FP64 routine.
// (Explicit FMAs and approximate reciprocals: the file is built with --fmad=false for the FP64
// parity arithmetic, but this filter only needs an error bound.)
__device__ __forceinline__ float fdot(float ax, float ay, float az, float bx, float by, float bz) {
  return __fmaf_rn(ax, bx, __fmaf_rn(ay, by, __fmul_rn(az, bz)));
}
__device__ __forceinline__ float fseg_sq(float px, float py, float pz, float ax, float ay, float az, float bx, float by,
                                         float bz, float inv_den) {
  const float ux = bx - ax, uy = by - ay, uz = bz - az;
  const float wx = px - ax, wy = py - ay, wz = pz - az;
  float t = fdot(wx, wy, wz, ux, uy, uz) * inv_den;  // inv_den = 0 for a zero-length edge
  t = fminf(fmaxf(t, 0.f), 1.f);
  const float qx = __fmaf_rn(-t, ux, wx), qy = __fmaf_rn(-t, uy, wy), qz = __fmaf_rn(-t, uz, wz);
  return fdot(qx, qy, qz, qx, qy, qz);
}
__device__ __forceinline__ float fptri_sq(const TriD& t, float px, float py, float pz) {
  const float bx = t.ab[0], by = t.ab[1], bz = t.ab[2], cx = t.ac[0], cy = t.ac[1], cz = t.ac[2];
  float best = __int_as_float(0x7f800000);
  // plane term with the precomputed unit normal: dn = p.n^, projection q = p - dn n^
  const float nx = t.n[0], ny = t.n[1], nz = t.n[2];
  const float dn = fdot(px, py, pz, nx, ny, nz);
  const float qx = __fmaf_rn(-dn, nx, px), qy = __fmaf_rn(-dn, ny, py), qz = __fmaf_rn(-dn, nz, pz);
  const float d20 = fdot(qx, qy, qz, bx, by, bz), d21 = fdot(qx, qy, qz, cx, cy, cz);
  const float v = __fmaf_rn(t.binv[0], d20, t.binv[1] * d21), w = __fmaf_rn(t.binv[1], d20, t.binv[2] * d21);
  if (v >= 0.f && w >= 0.f && v + w <= 1.f) best = dn * dn;
  best = fminf(best, fseg_sq(px, py, pz, 0.f, 0.f, 0.f, bx, by, bz, t.ie[0]));
  best = fminf(best, fseg_sq(px, py, pz, bx, by, bz, cx, cy, cz, t.ie[1]));
  best = fminf(best, fseg_sq(px, py, pz, cx, cy, cz, 0.f, 0.f, 0.f, t.ie[2]));
  return best;
}

// 0: fails, 1: survives, 2: undecided (needs survives_exact).  The box test is exact; the FP32
// decision is certified away from the threshold for well-conditioned triangles.
__device__ __forceinline__ int survives_fast(const TriD& t, double cx, double cy, double cz, double thr) {
  const double tb = thr + 1e-9;
  const double dx = fmax(fmax(t.lo[0] - cx, cx - t.hi[0]), 0.0);
  const double dy = fmax(fmax(t.lo[1] - cy, cy - t.hi[1]), 0.0);
  const double dz = fmax(fmax(t.lo[2] - cz, cz - t.hi[2]), 0.0);
  if ((dx * dx + dy * dy) + dz * dz > tb * tb) return 0;
  if (t.wc) {  // certified FP32 decision away from the threshold
    const float px = static_cast<float>(cx - t.a[0]), py = static_cast<float>(cy - t.a[1]),
                pz = static_cast<float>(cz - t.a[2]);
    const float d2 = fptri_sq(t, px, py, pz);
    const float L2 = fmaxf(t.L2, px * px + py * py + pz * pz);
    const float th2 = static_cast<float>(thr * thr);
    const float m = 1e-4f * L2 + 1e-3f * th2;
    if (d2 < th2 - m) return 1;
    if (d2 > th2 + m) return 0;
  }
  return 2;
}

// the pinned predicate itself: sqrt(ptri_sq) <= thr in FP64
__device__ __forceinline__ bool survives_exact(const TriD& t, double cx, double cy, double cz, double thr) {
  const double d2 = ptri_sq(D3{cx, cy, cz}, D3{t.a[0], t.a[1], t.a[2]}, D3{t.b[0], t.b[1], t.b[2]},
                            D3{t.c[0], t.c[1], t.c[2]});
  return sqrt(d2) <= thr;
}

__device__ __forceinline__ bool survives(const TriD& t, double cx, double cy, double cz, double thr) {
  const int s = survives_fast(t, cx, cy, cz, thr);
  return s == 2 ? survives_exact(t, cx, cy, cz, thr) : s == 1;
}

// 1/r for a power of two r, exactly (exponent bits): x * inv_pow2(r) == x / r bit for bit
__device__ __forceinline__ double inv_pow2(int r) {
  return __longlong_as_double(static_cast<long long>(1023 - (__ffs(r) - 1)) << 52);
}

// 3/R + (sqrt(3)/2)/r with R, r powers of two: the products by exact reciprocals equal the
// quotients bit for bit, and avoid two FP64 divisions per call
__device__ __forceinline__ double level_thr(int R, int r) {
  return 3.0 * inv_pow2(R) + kHalfSqrt3 * inv_pow2(r);
}

__global__ void k_prep(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t nf,
                       TriD* __restrict__ T) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nf) return;
  const int i0 = F[3 * i], i1 = F[3 * i + 1], i2 = F[3 * i + 2];
  TriD t;
  for (int k = 0; k < 3; ++k) {
    t.a[k] = V[3 * i0 + k];
    t.b[k] = V[3 * i1 + k];
    t.c[k] = V[3 * i2 + k];
    t.lo[k] = fmin(fmin(t.a[k], t.b[k]), t.c[k]);
    t.hi[k] = fmax(fmax(t.a[k], t.b[k]), t.c[k]);
  }
  const D3 A{t.a[0], t.a[1], t.a[2]}, B{t.b[0], t.b[1], t.b[2]}, C{t.c[0], t.c[1], t.c[2]};
  const D3 ab = sub(B, A), ac = sub(C, A), bc = sub(C, B);
  for (int k = 0; k < 3; ++k) {
    t.ab[k] = static_cast<float>(k == 0 ? ab.x : (k == 1 ? ab.y : ab.z));
    t.ac[k] = static_cast<float>(k == 0 ? ac.x : (k == 1 ? ac.y : ac.z));
  }
  const double lab = sqn(ab), lac = sqn(ac), lbc = sqn(bc);
  t.L2 = static_cast<float>(fmax(fmax(lab, lac), lbc));
  {
    const float fl[3] = {static_cast<float>(lab), static_cast<float>(lbc), static_cast<float>(lac)};
    for (int k = 0; k < 3; ++k) t.ie[k] = fl[k] > 0.f ? 1.0f / fl[k] : 0.f;
  }
  const D3 nv = cross(ab, ac);
  const double n2 = sqn(nv);
  {
    const double inv = n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0;
    t.n[0] = static_cast<float>(nv.x * inv);
    t.n[1] = static_cast<float>(nv.y * inv);
    t.n[2] = static_cast<float>(nv.z * inv);
    const double g00 = lab, g01 = dot(ab, ac), g11 = lac, gd = g00 * g11 - g01 * g01;
    const double gi = gd > 0.0 ? 1.0 / gd : 0.0;
    t.binv[0] = static_cast<float>(g11 * gi);
    t.binv[1] = static_cast<float>(-g01 * gi);
    t.binv[2] = static_cast<float>(g00 * gi);
    for (int k = 0; k < 3; ++k) {
      t.blo[k] = static_cast<float>(t.lo[k] - t.a[k]);
      t.bhi[k] = static_cast<float>(t.hi[k] - t.a[k]);
    }
  }
  // sin^2 of the three corner angles: |n|^2 / (|e1|^2 |e2|^2)
  const bool wc = lab > 0.0 && lac > 0.0 && lbc > 0.0 && n2 >= 0.01 * lab * lac && n2 >= 0.01 * lab * lbc &&
                  n2 >= 0.01 * lac * lbc;
  t.wc = wc ? 1 : 0;
  T[i] = t;
}

// warp-aggregated append of one 64-bit value per active lane with `keep`
__device__ __forceinline__ void append(bool keep, uint64_t val, uint64_t* out, unsigned long long* cnt,
                                       uint64_t cap) {
  const unsigned m = __ballot_sync(__activemask(), keep);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(cnt, static_cast<unsigned long long>(__popc(m)));
  base = __shfl_sync(__activemask(), base, leader);
  if (keep) {
    const uint64_t pos = base + __popc(m & ((1u << lane) - 1u));
    if (pos < cap) out[pos] = val;
  }
}

// slab pruning: a level-r cell z covers lattice planes [z*R/r, (z+1)*R/r]; cells that touch no
// plane of the slab [zp0, zp1] cannot change any slab sample and are not emitted
__device__ __forceinline__ bool in_slab(int zc, int R, int r, int zp0, int zp1) {
  const int s = R / r;
  return zc * s <= zp1 && (zc + 1) * s >= zp0;
}

__global__ void k_level0(const TriD* __restrict__ T, int64_t nf, int R, uint64_t* out,
                         unsigned long long* cnt, uint64_t cap, int zp0, int zp1) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool active = i < nf;
  TriD t;
  int lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
  const int r = 8;
  const double thr = level_thr(R, r);
  if (active) {
    t = T[i];
    const double tb = thr + 1e-9;
    for (int k = 0; k < 3; ++k) {
      lo[k] = max(0, static_cast<int>(floor((t.lo[k] - tb) * r - 0.5)) - 1);
      hi[k] = min(r - 1, static_cast<int>(ceil((t.hi[k] + tb) * r - 0.5)) + 1);
    }
  }
  const int nx = hi[0] - lo[0] + 1, ny = hi[1] - lo[1] + 1, nz = hi[2] - lo[2] + 1;
  const int n = active ? nx * ny * nz : 0;
  // every lane walks its own box; ballots need convergence -> loop to the warp max
  int nmax = n;
  for (int o = 16; o; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
  for (int j = 0; j < nmax; ++j) {
    bool keep = false;
    uint64_t val = 0;
    if (j < n) {
      const int x = lo[0] + j % nx, y = lo[1] + (j / nx) % ny, z = lo[2] + j / (nx * ny);
      const double ir = inv_pow2(r);
      keep = in_slab(z, R, r, zp0, zp1) && survives(t, (x + 0.5) * ir, (y + 0.5) * ir, (z + 0.5) * ir, thr);
      val = (static_cast<uint64_t>(x + r * (y + r * z)) << 32) | static_cast<uint64_t>(i);
    }
    append(keep, val, out, cnt, cap);
  }
}

__global__ void k_refine(const uint64_t* __restrict__ in, uint64_t n_in, const TriD* __restrict__ T,
                         int R, int r, uint64_t* out, unsigned long long* cnt, uint64_t cap, int zp0, int zp1) {
  const uint64_t gid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  bool keep = false;
  uint64_t val = 0;
  if (gid < n_in * 8) {
    const uint64_t pr = in[gid >> 3];
    const int ch = static_cast<int>(gid & 7);
    const uint32_t pc = static_cast<uint32_t>(pr >> 32), tri = static_cast<uint32_t>(pr);
    const int rp = r >> 1;
    const int px = pc % rp, py = (pc / rp) % rp, pz = pc / (rp * rp);
    const int x = 2 * px + (ch & 1), y = 2 * py + ((ch >> 1) & 1), z = 2 * pz + ((ch >> 2) & 1);
    const TriD t = T[tri];
    const double ir = inv_pow2(r);
    keep = in_slab(z, R, r, zp0, zp1) && survives(t, (x + 0.5) * ir, (y + 0.5) * ir, (z + 0.5) * ir, level_thr(R, r));
    val = (static_cast<uint64_t>(x + r * (y + r * z)) << 32) | tri;
  }
  append(keep, val, out, cnt, cap);
}

__global__ void k_brick_count(const uint64_t* __restrict__ pairs, uint64_t n, uint32_t* __restrict__ cnt) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) atomicAdd(&cnt[pairs[i] >> 32], 1u);
}

__global__ void k_brick_scatter(const uint64_t* __restrict__ pairs, uint64_t n, const uint32_t* __restrict__ off,
                                uint32_t* __restrict__ cursor, uint32_t* __restrict__ tris) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint32_t b = static_cast<uint32_t>(pairs[i] >> 32);
  const uint32_t pos = atomicAdd(&cursor[b], 1u);
  tris[off[b] + pos] = static_cast<uint32_t>(pairs[i]);
}

// per brick: compact id (or -1) and number of work items
__global__ void k_brick_items(const uint32_t* __restrict__ cnt, int64_t nb, uint32_t* __restrict__ nitems,
                              uint32_t* __restrict__ isactive) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nb) return;
  nitems[i] = (cnt[i] + kChunk - 1) / kChunk;
  isactive[i] = cnt[i] > 0 ? 1u : 0u;
}

struct Item {
  uint32_t brick;    // dense brick index
  uint32_t compact;  // active brick id
  uint32_t begin, end;
};

__global__ void k_make_items(const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ off,
                             const uint32_t* __restrict__ item_off, const uint32_t* __restrict__ act_off,
                             int64_t nb, Item* __restrict__ items, int32_t* __restrict__ bmap) {
  const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (b >= nb) return;
  const uint32_t c = cnt[b];
  bmap[b] = c ? static_cast<int32_t>(act_off[b]) : -1;
  if (!c) return;
  uint32_t k = item_off[b];
  for (uint32_t s = 0; s < c; s += kChunk, ++k)
    items[k] = Item{static_cast<uint32_t>(b), act_off[b], off[b] + s, off[b] + min(c, s + kChunk)};
}

// One CTA (8 warps) per work item.  bs = cells per brick edge (1..8), J = log2(bs).
// Divergence-free inner loops: every level first compacts its candidate cells (children of the
// previous level's survivors) into a shared-memory list; the finest survivors are dilated to
// brick vertices with bit-row operations (8-bit cell rows -> 9-bit vertex rows) and compacted,
// so all 32 lanes evaluate distances on useful work.  Vertex distances: a certified FP32
// evaluation first (well-conditioned triangles) skips every triangle that cannot lower the
// vertex's running minimum; the rest are evaluated with the pinned FP64 routine.
#ifndef PCU_BRICK_MINB
#define PCU_BRICK_MINB 3
#endif
__global__ void __launch_bounds__(256, PCU_BRICK_MINB) k_brick(const Item* __restrict__ items, const uint32_t* __restrict__ tris,
                                                  const TriD* __restrict__ T, int R, int rb, int bs, int J,
                                                  uint32_t* __restrict__ blocks) {
  __shared__ unsigned long long vmin[729];
  __shared__ uint32_t rows[8][16];        // finest-level survivor bit rows: byte (y + bs z) holds x bits
  __shared__ uint16_t list[8][2][512];    // ping-pong survivor lists (local cell index at level j)
  __shared__ uint16_t vlist[8][729];      // needed vertices, packed x | y<<4 | z<<8
  __shared__ uint16_t equeue[8][64];      // vertices queued for the FP64 evaluation
  __shared__ TriD tsh[8];
  __shared__ unsigned next_tri;  // dynamic triangle distribution among the warps (load balance)
  const Item it = items[blockIdx.x];
  if (threadIdx.x == 0) next_tri = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv1 = bs + 1, nvb = nv1 * nv1 * nv1;
  for (int v = threadIdx.x; v < nvb; v += blockDim.x) vmin[v] = ~0ull;
  __syncthreads();
  const int bx = it.brick % rb, by = (it.brick / rb) % rb, bz = it.brick / (rb * rb);
  const unsigned lt = (1u << lane) - 1u;
  for (;;) {
    unsigned kk = 0;
    if (lane == 0) kk = atomicAdd(&next_tri, 1u);
    kk = __shfl_sync(0xffffffffu, kk, 0);
    const uint32_t k = it.begin + kk;
    if (k >= it.end) break;
    {  // cooperative 16-byte copy of the triangle record
      constexpr int kW = static_cast<int>(sizeof(TriD) / 16);
      const int4* src = reinterpret_cast<const int4*>(T + tris[k]);
      if (lane < kW) reinterpret_cast<int4*>(&tsh[warp])[lane] = __ldg(src + lane);
    }
    __syncwarp();
    const TriD& t = tsh[warp];
    // level 0 inside the brick: the brick itself survived (the pair exists)
    int cur = 0, nsurv = 1;
    if (lane == 0) list[warp][0][0] = 0;
    __syncwarp();
    for (int j = 1; j <= J; ++j) {
      const int lp = j - 1;  // log2 of the parent side
      const int r = rb << j;
      const double thr = level_thr(R, r), ir = inv_pow2(r);
      const int ncand = nsurv * 8;
      int nout = 0;
      for (int base = 0; base < ncand; base += 32) {
        const int c = base + lane;
        bool keep = false;
        int cell = 0;
        if (c < ncand) {
          const int pc = list[warp][cur][c >> 3], ch = c & 7;
          const int px = pc & ((1 << lp) - 1), py = (pc >> lp) & ((1 << lp) - 1), pz = pc >> (2 * lp);
          const int x = 2 * px + (ch & 1), y = 2 * py + ((ch >> 1) & 1), z = 2 * pz + ((ch >> 2) & 1);
          cell = x | (y << j) | (z << (2 * j));
          const int gx = (bx << j) + x, gy = (by << j) + y, gz = (bz << j) + z;
          keep = survives(t, (gx + 0.5) * ir, (gy + 0.5) * ir, (gz + 0.5) * ir, thr);
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) list[warp][cur ^ 1][nout + __popc(m & lt)] = static_cast<uint16_t>(cell);
        nout += __popc(m);
      }
      __syncwarp();
      cur ^= 1;
      nsurv = nout;
      if (nsurv == 0) break;
    }
    if (nsurv == 0) {
      __syncwarp();
      continue;
    }
    // finest survivors -> 8-bit rows (row = y + bs*z) -> dilated 9-bit vertex rows -> list
    if (lane < 16) rows[warp][lane] = 0u;
    __syncwarp();
    for (int i = lane; i < nsurv; i += 32) {
      const int c = list[warp][cur][i];
      const int x = c & (bs - 1), row = c >> J;
      atomicOr(&rows[warp][row >> 2], (1u << x) << (8 * (row & 3)));
    }
    __syncwarp();
    const uint8_t* rb8 = reinterpret_cast<const uint8_t*>(rows[warp]);
    const int nrows = nv1 * nv1;
    int nneed = 0;
    for (int base = 0; base < nrows; base += 32) {
      const int vr = base + lane;
      uint32_t m = 0;
      if (vr < nrows) {
        const int vy = vr % nv1, vz = vr / nv1;
        for (int dz = 0; dz < 2; ++dz)
          for (int dy = 0; dy < 2; ++dy) {
            const int cy = vy - dy, cz = vz - dz;
            if (cy >= 0 && cz >= 0 && cy < bs && cz < bs) m |= rb8[cy + bs * cz];
          }
        m = m | (m << 1);
      }
      const int cnt = __popc(m);
      int incl = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int pos = nneed + incl - cnt;
      if (m) {
        const int vy = vr % nv1, vz = vr / nv1;
        while (m) {
          const int x = __ffs(m) - 1;
          m &= m - 1;
          vlist[warp][pos++] = static_cast<uint16_t>(x | (vy << 4) | (vz << 8));
        }
      }
      nneed += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    const D3 A{t.a[0], t.a[1], t.a[2]}, Bv{t.b[0], t.b[1], t.b[2]}, Cv{t.c[0], t.c[1], t.c[2]};
    const double iR = inv_pow2(R);
    // Pass over the needed vertices: the certified FP32 filter decides which vertices this
    // triangle may lower; those are queued (warp ballot) and evaluated in FP64 32 at a time, so
    // the expensive pinned routine always runs with a full warp.
    int qn = 0;
    auto eval = [&](int pk) {
      const int vx = pk & 15, vy = (pk >> 4) & 15, vz = pk >> 8;
      const int v = vx + nv1 * (vy + nv1 * vz);
      const D3 p{static_cast<double>(bx * bs + vx) * iR, static_cast<double>(by * bs + vy) * iR,
                 static_cast<double>(bz * bs + vz) * iR};
      const double d2 = ptri_sq(p, A, Bv, Cv);
      atomicMin(&vmin[v], static_cast<unsigned long long>(__double_as_longlong(d2)));
    };
    for (int base = 0; base < nneed; base += 32) {
      const int i = base + lane;
      bool need = false;
      int pk = 0;
      if (i < nneed) {
        pk = vlist[warp][i];
        need = true;
        if (t.wc) {
          const int vx = pk & 15, vy = (pk >> 4) & 15, vz = pk >> 8;
          const int v = vx + nv1 * (vy + nv1 * vz);
          const double px64 = static_cast<double>(bx * bs + vx) * iR, py64 = static_cast<double>(by * bs + vy) * iR,
                       pz64 = static_cast<double>(bz * bs + vz) * iR;
          // this triangle cannot lower the vertex's running minimum: skip the FP64 evaluation
          // (the minimum is order independent, so skipping never changes the result).  Cheap
          // lower bounds first (plane distance, box distance), then the FP32 distance.
          const double curm = __longlong_as_double(static_cast<long long>(vmin[v]));  // NaN while unset
          const float px = static_cast<float>(px64 - t.a[0]), py = static_cast<float>(py64 - t.a[1]),
                      pz = static_cast<float>(pz64 - t.a[2]);
          const float L2 = fmaxf(t.L2, fdot(px, py, pz, px, py, pz));
          const float skip = __fmaf_rn(1e-4f, L2, static_cast<float>(curm * (1.0 + 1e-3)));  // NaN: never skip
          const float dn = fdot(px, py, pz, t.n[0], t.n[1], t.n[2]);
          if (dn * dn > skip) {
            need = false;
          } else {
            const float ex = fmaxf(fmaxf(t.blo[0] - px, px - t.bhi[0]), 0.f),
                        ey = fmaxf(fmaxf(t.blo[1] - py, py - t.bhi[1]), 0.f),
                        ez = fmaxf(fmaxf(t.blo[2] - pz, pz - t.bhi[2]), 0.f);
            if (fdot(ex, ey, ez, ex, ey, ez) > skip || fptri_sq(t, px, py, pz) > skip) need = false;
          }
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, need);
      if (need) equeue[warp][qn + __popc(m & lt)] = static_cast<uint16_t>(pk);
      qn += __popc(m);
      __syncwarp();
      if (qn >= 32) {
        eval(equeue[warp][qn - 32 + lane]);
        qn -= 32;
        __syncwarp();
      }
    }
    if (lane < qn) eval(equeue[warp][lane]);
    __syncwarp();
  }
  __syncthreads();
  // merge into the brick's global block as the f32 UDF value: (float)sqrt(.) is monotone, so
  // the min over f32 bit patterns of (float)sqrt(d2) equals (float)sqrt(min d2) exactly
  uint32_t* blk = blocks + static_cast<uint64_t>(it.compact) * nvb;
  for (int v = threadIdx.x; v < nvb; v += blockDim.x)
    if (vmin[v] != ~0ull) {
      const float u = static_cast<float>(sqrt(__longlong_as_double(static_cast<long long>(vmin[v]))));
      atomicMin(&blk[v], __float_as_uint(u));
    }
}

// mode 0: UDF (+INF sentinel); mode 1: SDF (u - eps, sentinel +1.0).  One warp per lattice row
// (y, z): the brick candidates along y and z are computed once per row, then the warp walks the
// row 32 samples at a time (bs is a power of two: brick coordinates by shifts, no division per
// sample).  With `signs`, each step's ballot of (s < 0) is stored as one 32-bit word (bit x & 31
// of word x >> 5 of the row): the DMC classify passes read this 17 MB mask (C3) instead of the
// 540 MB lattice.
__global__ void __launch_bounds__(256) k_finalize(const uint32_t* __restrict__ blocks, const int32_t* __restrict__ bmap,
                                                  int R, int rb, int bs, int mode, double eps, float* __restrict__ out,
                                                  int z0, int z1, uint32_t* __restrict__ signs) {
  const int n1 = R + 1, W = (n1 + 31) >> 5, nv1 = bs + 1, lgbs = __ffs(bs) - 1;
  const int rows = n1 * (z1 - z0);
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int64_t bvol = static_cast<int64_t>(nv1) * nv1 * nv1;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows; row += nwarps) {
    const int zr = row / n1, y = row - zr * n1, z = z0 + zr;
    int bys[2], bzs[2], nby = 0, nbz = 0;
    if ((y >> lgbs) < rb) bys[nby++] = y >> lgbs;
    if ((y & (bs - 1)) == 0 && y > 0) bys[nby++] = (y >> lgbs) - 1;
    if ((z >> lgbs) < rb) bzs[nbz++] = z >> lgbs;
    if ((z & (bs - 1)) == 0 && z > 0) bzs[nbz++] = (z >> lgbs) - 1;
    if (!bmap) nbz = 0;
    float* orow = out + static_cast<int64_t>(row) * n1;
    for (int w = 0; w < W; ++w) {
      const int x = (w << 5) + lane;
      uint32_t best = 0xffffffffu;
      if (x < n1) {
        int bxs[2], nbx = 0;
        if ((x >> lgbs) < rb) bxs[nbx++] = x >> lgbs;
        if ((x & (bs - 1)) == 0 && x > 0) bxs[nbx++] = (x >> lgbs) - 1;
        for (int a = 0; a < nbz; ++a)
          for (int b = 0; b < nby; ++b) {
            const int* brow = bmap + rb * (bys[b] + rb * bzs[a]);
            const int ly = y - (bys[b] << lgbs), lz = z - (bzs[a] << lgbs);
            for (int c = 0; c < nbx; ++c) {
              const int cid = brow[bxs[c]];
              if (cid < 0) continue;
              const int lx = x - (bxs[c] << lgbs);
              const uint32_t val = blocks[cid * bvol + lx + nv1 * (ly + nv1 * lz)];
              best = val < best ? val : best;
            }
          }
      }
      float res;
      if (best == 0xffffffffu) {
        res = mode ? 1.0f : __int_as_float(0x7f800000);
      } else {
        const float u = __uint_as_float(best);
        res = mode ? static_cast<float>(static_cast<double>(u) - eps) : u;
      }
      if (x < n1) orow[x] = res;
      if (signs) {
        const unsigned m = __ballot_sync(0xffffffffu, x < n1 && res < 0.0f);
        if (lane == 0) signs[static_cast<int64_t>(row) * W + w] = m;
      }
    }
  }
}

__global__ void k_udf_to_sdf(float* g, int64_t n, double eps) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float u = g[i];
    g[i] = isinf(u) ? 1.0f : static_cast<float>(static_cast<double>(u) - eps);
  }
}

// debug: descend inside the brick to level jt and emit (cell at that level, tri)
__global__ void k_debug_pairs(const uint64_t* __restrict__ bpairs, uint64_t n, const TriD* __restrict__ T, int R,
                              int rb, int jt, uint64_t* out, unsigned long long* cnt, uint64_t cap) {
  const uint64_t gid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const int side = 1 << jt;
  const uint64_t per = static_cast<uint64_t>(side) * side * side;
  bool keep = false;
  uint64_t val = 0;
  if (gid < n * per) {
    const uint64_t pr = bpairs[gid / per];
    const int c = static_cast<int>(gid % per);
    const uint32_t b = static_cast<uint32_t>(pr >> 32), tri = static_cast<uint32_t>(pr);
    const int bx = b % rb, by = (b / rb) % rb, bz = b / (rb * rb);
    const int x = c % side, y = (c / side) % side, z = c / (side * side);
    const TriD t = T[tri];
    keep = true;
    for (int j = 1; j <= jt && keep; ++j) {
      const int sh = jt - j, r = rb << j;
      const int gx = bx * (1 << j) + (x >> sh), gy = by * (1 << j) + (y >> sh), gz = bz * (1 << j) + (z >> sh);
      const double ir = inv_pow2(r);
      keep = survives(t, (gx + 0.5) * ir, (gy + 0.5) * ir, (gz + 0.5) * ir, level_thr(R, r));
    }
    const int r = rb << jt;
    const uint64_t gx = bx * side + x, gy = by * side + y, gz = bz * side + z;
    val = ((gx + static_cast<uint64_t>(r) * (gy + static_cast<uint64_t>(r) * gz)) << 32) | tri;
  }
  append(keep, val, out, cnt, cap);
}

int ilog2(int x) {
  int l = 0;
  while ((1 << l) < x) ++l;
  return l;
}

}  // namespace

// Runs levels 8..r_b; returns the brick-level pairs (and the pairs of `keep_level` if >= 0).
static DevBuf<uint64_t> hierarchy_to_bricks(Ctx& ctx, const TriD* T, int64_t nf, int R, int rb,
                                            uint64_t& n_out, int keep_r, DevBuf<uint64_t>* kept,
                                            uint64_t* kept_n, int zp0 = 0, int zp1 = 1 << 30) {
  DevBuf<unsigned long long> cnt(1, ctx.stream);
  uint64_t cap = static_cast<uint64_t>(nf) * 16 + (1 << 16);
  DevBuf<uint64_t> cur;
  uint64_t n = 0;
  for (int r = 8; r <= rb; r <<= 1) {
    while (true) {
      DevBuf<uint64_t> out(cap, ctx.stream);
      cnt.memset(0, ctx.stream);
      if (r == 8) {
        PCU_LAUNCH(ctx, k_level0, grid_for(nf, 128), 128, 0, T, nf, R, out.get(), cnt.get(), cap, zp0, zp1);
      } else {
        PCU_LAUNCH(ctx, k_refine, grid_for(static_cast<int64_t>(n * 8), 256), 256, 0, cur.get(), n, T, R, r,
                   out.get(), cnt.get(), cap, zp0, zp1);
      }
      const uint64_t got = read_scalar(ctx, cnt.get());
      if (got > cap) {
        cap = got + got / 4 + 1024;
        continue;
      }
      cur = std::move(out);
      n = got;
      break;
    }
    if (r == keep_r && kept) {
      kept->alloc(n ? n : 1, ctx.stream);
      if (n) PCU_CUDA(cudaMemcpyAsync(kept->get(), cur.get(), n * 8, cudaMemcpyDeviceToDevice, ctx.stream));
      *kept_n = n;
    }
    cap = n * 8 + (1 << 16);
  }
  n_out = n;
  return cur;
}

void udf_run(Ctx& ctx, const double* dV, int64_t nv, const int32_t* dF, int64_t nf, int R, int mode, double eps,
             float* d_out, int z0, int z1, uint32_t* d_signs) {
  if (z1 < 0) z1 = R + 1;
  PCU_REQUIRE(z0 >= 0 && z0 < z1 && z1 <= R + 1, PAMOPT_CU_EINVAL, "compute_udf: bad slab plane range");
  (void)nv;
  PCU_REQUIRE(R >= 8 && (R & (R - 1)) == 0 && R <= 1024, PAMOPT_CU_EINVAL, "compute_udf: R must be a power of two in [8, 1024]");
  const int rb = R >= 64 ? R / 8 : 8;
  const int bs = R / rb, J = ilog2(bs);
  const int64_t n1 = R + 1;
  const int64_t nvert = n1 * n1 * n1;
  if (nf == 0) {
    PCU_LAUNCH(ctx, k_finalize, static_cast<unsigned>(ctx.num_sms * 8), 256, 0, nullptr, nullptr, R, rb, bs, mode, eps, d_out,
               z0, z1, d_signs);
    return;
  }
  DevBuf<TriD> T(nf, ctx.stream);
  PCU_LAUNCH(ctx, k_prep, grid_for(nf, 256), 256, 0, dV, dF, nf, T.get());
  uint64_t npairs = 0;
  DevBuf<uint64_t> bp = hierarchy_to_bricks(ctx, T.get(), nf, R, rb, npairs, -1, nullptr, nullptr, z0, z1 - 1);
  const int64_t nb = static_cast<int64_t>(rb) * rb * rb;
  DevBuf<uint32_t> bcnt(nb, ctx.stream), boff(nb, ctx.stream), bcur(nb, ctx.stream);
  DevBuf<uint32_t> nitems(nb, ctx.stream), item_off(nb, ctx.stream), isact(nb, ctx.stream), act_off(nb, ctx.stream);
  bcnt.memset(0, ctx.stream);
  bcur.memset(0, ctx.stream);
  DevBuf<uint32_t> tris(npairs ? npairs : 1, ctx.stream);
  if (npairs) {
    PCU_LAUNCH(ctx, k_brick_count, grid_for(static_cast<int64_t>(npairs), 256), 256, 0, bp.get(), npairs, bcnt.get());
  }
  exclusive_scan_u32(ctx, bcnt.get(), boff.get(), nb);
  if (npairs) {
    PCU_LAUNCH(ctx, k_brick_scatter, grid_for(static_cast<int64_t>(npairs), 256), 256, 0, bp.get(), npairs, boff.get(),
               bcur.get(), tris.get());
  }
  PCU_LAUNCH(ctx, k_brick_items, grid_for(nb, 256), 256, 0, bcnt.get(), nb, nitems.get(), isact.get());
  // totals: last offset + last count
  exclusive_scan_u32(ctx, nitems.get(), item_off.get(), nb);
  exclusive_scan_u32(ctx, isact.get(), act_off.get(), nb);
  uint32_t last_item_off = read_scalar(ctx, item_off.get() + nb - 1), last_nitems = read_scalar(ctx, nitems.get() + nb - 1);
  uint32_t last_act_off = read_scalar(ctx, act_off.get() + nb - 1), last_isact = read_scalar(ctx, isact.get() + nb - 1);
  const uint32_t n_items = last_item_off + last_nitems, n_active = last_act_off + last_isact;
  DevBuf<Item> items(n_items ? n_items : 1, ctx.stream);
  DevBuf<int32_t> bmap(nb, ctx.stream);
  PCU_LAUNCH(ctx, k_make_items, grid_for(nb, 256), 256, 0, bcnt.get(), boff.get(), item_off.get(), act_off.get(), nb,
             items.get(), bmap.get());
  const int nvb = (bs + 1) * (bs + 1) * (bs + 1);
  DevBuf<uint32_t> blocks(static_cast<size_t>(n_active ? n_active : 1) * nvb, ctx.stream);
  blocks.memset(0xFF, ctx.stream);
  if (n_items) {
    PCU_LAUNCH(ctx, k_brick, n_items, 256, 0, items.get(), tris.get(), T.get(), R, rb, bs, J, blocks.get());
  }
  PCU_LAUNCH(ctx, k_finalize, static_cast<unsigned>(ctx.num_sms * 16), 256, 0, blocks.get(), bmap.get(), R, rb, bs,
             mode, eps, d_out, z0, z1, d_signs);
  (void)nvert;
}

void udf_to_sdf_inplace(Ctx& ctx, float* g, int64_t n, double eps) {
  PCU_LAUNCH(ctx, k_udf_to_sdf, static_cast<unsigned>(ctx.num_sms * 16), 256, 0, g, n, eps);
}

std::vector<int64_t> hierarchy_pairs(Ctx& ctx, const double* dV, const int32_t* dF, int64_t nf, int R, int r) {
  PCU_REQUIRE(R >= 8 && (R & (R - 1)) == 0, PAMOPT_CU_EINVAL, "hierarchy_pairs: bad R");
  PCU_REQUIRE(r >= 8 && r <= R && (r & (r - 1)) == 0, PAMOPT_CU_EINVAL, "hierarchy_pairs: bad level");
  std::vector<int64_t> host;
  if (nf == 0) return host;
  const int rb = R >= 64 ? R / 8 : 8;
  DevBuf<TriD> T(nf, ctx.stream);
  PCU_LAUNCH(ctx, k_prep, grid_for(nf, 256), 256, 0, dV, dF, nf, T.get());
  uint64_t npairs = 0, nk = 0;
  DevBuf<uint64_t> kept;
  DevBuf<uint64_t> bp = hierarchy_to_bricks(ctx, T.get(), nf, R, rb, npairs, r <= rb ? r : -1, &kept, &nk);
  DevBuf<uint64_t> res;
  uint64_t nres = 0;
  if (r <= rb) {
    res = std::move(kept);
    nres = nk;
  } else {
    const int jt = ilog2(r / rb);
    const uint64_t per = 1ull << (3 * jt);
    DevBuf<unsigned long long> cnt(1, ctx.stream);
    uint64_t cap = npairs * per / 4 + 1024;
    while (true) {
      DevBuf<uint64_t> out(cap, ctx.stream);
      cnt.memset(0, ctx.stream);
      PCU_LAUNCH(ctx, k_debug_pairs, grid_for(static_cast<int64_t>(npairs * per), 256), 256, 0, bp.get(), npairs,
                 T.get(), R, rb, jt, out.get(), cnt.get(), cap);
      const uint64_t got = read_scalar(ctx, cnt.get());
      if (got > cap) {
        cap = got + 1024;
        continue;
      }
      res = std::move(out);
      nres = got;
      break;
    }
  }
  std::vector<uint64_t> raw(nres);
  if (nres) PCU_CUDA(cudaMemcpyAsync(raw.data(), res.get(), nres * 8, cudaMemcpyDeviceToHost, ctx.stream));
  PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  std::sort(raw.begin(), raw.end());
  host.resize(2 * nres);
  for (uint64_t i = 0; i < nres; ++i) {
    host[2 * i] = static_cast<int64_t>(raw[i] >> 32);
    host[2 * i + 1] = static_cast<int64_t>(raw[i] & 0xffffffffu);
  }
  return host;
}

}  // namespace pcu

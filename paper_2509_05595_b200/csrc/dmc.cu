// dmc.cu — stage 1b: Dual Marching Cubes with the paper's intersection corrections
// (PAPER.md:85-114,716-772), as count/write ("2-kernel gather") passes with
// deterministic prefix sums so the output order never depends on scheduling.
//
//   classify   dense scan of the R^3 cells, 2048 cells per CTA: per-CTA active counts, an
//              exclusive scan, then an ordered block-scan compaction -> active cells (x-fastest)
//   patches    per active cell: case, the C16/C19 flip mask (neighbour rule),
//              patch count -> scan -> patch vertices (sigmoid-smoothed crossings, centroid)
//   quads      per active cell and axis: the interior valid edge at its corner 0 -> quad from
//              the 4 cells' patches (dense cell -> active-id map), orientation, envelope
//              concavity split decision -> (faces, extra vertices) counts -> scan -> write
// The 256-entry patch table is generated on the host at load time (faces paired around
// positive corners on ambiguous faces; cycles of the pairing graph are patches) and placed in
// constant memory together with the doubly-covered-face masks and the flipped variants.
#include <cub/cub.cuh>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace pcu {
namespace {

struct PatchSet {
  uint8_t n;
  uint8_t dc;
  uint16_t mask[4];
  int8_t edge_patch[12];
};

__constant__ PatchSet c_base[256];
__constant__ PatchSet c_flip[256];  // resolution T on the (single) doubly-covered face

// ----------------------------------------------------------------- host table generation
// cube corner c = x | y<<1 | z<<2; edge e = 4*axis + sub (x: y+2z, y: x+2z, z: x+2y)
int h_edge_id(int axis, int lower_corner) {
  const int x = lower_corner & 1, y = (lower_corner >> 1) & 1, z = (lower_corner >> 2) & 1;
  return axis == 0 ? y + 2 * z : (axis == 1 ? 4 + x + 2 * z : 8 + x + 2 * y);
}

struct HFace {
  int corner[4];  // cyclic
  int edge[4];    // edge[i] between corner[i] and corner[i+1]
};

HFace h_face(int f) {
  const int axis = f >> 1, side = f & 1, b = (axis + 1) % 3, c = (axis + 2) % 3;
  static const int cyc[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
  HFace F;
  for (int i = 0; i < 4; ++i) F.corner[i] = (side << axis) | (cyc[i][0] << b) | (cyc[i][1] << c);
  for (int i = 0; i < 4; ++i) {
    const int p = F.corner[i], q = F.corner[(i + 1) & 3], d = p ^ q;
    F.edge[i] = h_edge_id(d == 1 ? 0 : (d == 2 ? 1 : 2), p & q);
  }
  return F;
}

PatchSet h_patches(int cs, int flip) {
  int nb[12][2], deg[12] = {0};
  auto join = [&](int a, int b) {
    nb[a][deg[a]++] = b;
    nb[b][deg[b]++] = a;
  };
  for (int f = 0; f < 6; ++f) {
    const HFace F = h_face(f);
    int sgn[4], crossing[4], nc = 0;
    for (int i = 0; i < 4; ++i) sgn[i] = (cs >> F.corner[i]) & 1;
    for (int i = 0; i < 4; ++i) nc += crossing[i] = sgn[i] != sgn[(i + 1) & 3];
    if (nc == 2) {
      int e[2], k = 0;
      for (int i = 0; i < 4; ++i)
        if (crossing[i]) e[k++] = F.edge[i];
      join(e[0], e[1]);
    } else if (nc == 4) {
      // pair the two edges around every corner of the connected sign: positive (S) or negative (T)
      const int around = (flip >> f) & 1;  // 1 -> around negative corners
      for (int i = 0; i < 4; ++i)
        if (sgn[i] == around) join(F.edge[(i + 3) & 3], F.edge[i]);
    }
  }
  PatchSet P{};
  for (int e = 0; e < 12; ++e) P.edge_patch[e] = -1;
  for (int e0 = 0; e0 < 12; ++e0) {
    if (!deg[e0] || P.edge_patch[e0] >= 0) continue;
    int prev = -1, cur = e0;
    uint16_t m = 0;
    do {
      m |= static_cast<uint16_t>(1u << cur);
      P.edge_patch[cur] = static_cast<int8_t>(P.n);
      const int nx = nb[cur][0] == prev ? nb[cur][1] : nb[cur][0];
      prev = cur;
      cur = nx;
    } while (cur != e0);
    P.mask[P.n++] = m;
  }
  return P;
}

int h_doubly_covered(int cs) {
  const PatchSet P = h_patches(cs, 0);
  int m = 0;
  for (int f = 0; f < 6; ++f) {
    const HFace F = h_face(f);
    int s[4];
    for (int i = 0; i < 4; ++i) s[i] = (cs >> F.corner[i]) & 1;
    const bool amb = s[0] == s[2] && s[1] == s[3] && s[0] != s[1];
    if (amb && P.edge_patch[F.edge[0]] == P.edge_patch[F.edge[1]] &&
        P.edge_patch[F.edge[0]] == P.edge_patch[F.edge[2]] && P.edge_patch[F.edge[0]] == P.edge_patch[F.edge[3]])
      m |= 1 << f;
  }
  return m;
}

struct HostTable {
  PatchSet base[256], flip[256];
  HostTable() {
    for (int cs = 0; cs < 256; ++cs) {
      base[cs] = h_patches(cs, 0);
      base[cs].dc = static_cast<uint8_t>(h_doubly_covered(cs));
      // every doubly-covered case has exactly one such face (checked at generation time)
      if (__builtin_popcount(base[cs].dc) > 1) throw Error(PAMOPT_CU_ECUDA, "dmc table: >1 doubly covered face");
      flip[cs] = base[cs].dc ? h_patches(cs, base[cs].dc) : base[cs];
      flip[cs].dc = base[cs].dc;
    }
  }
};

const HostTable& host_table() {
  static HostTable t;
  return t;
}

void upload_table(int device) {
  static std::mutex mu;
  static uint64_t done_mask = 0;
  std::lock_guard<std::mutex> lock(mu);
  if (device < 64 && ((done_mask >> device) & 1)) return;
  const HostTable& t = host_table();
  PCU_CUDA(cudaMemcpyToSymbol(c_base, t.base, sizeof(t.base)));
  PCU_CUDA(cudaMemcpyToSymbol(c_flip, t.flip, sizeof(t.flip)));
  if (device < 64) done_mask |= 1ull << device;
}

// ------------------------------------------------------------------------- device side
constexpr int kCellsPerBlock = 2048;

struct GridView {
  const float* s;
  int R;
  int64_t n1;
  int64_t zb;  // global z of the first resident lattice plane (0 for a whole grid)
  const uint32_t* sg = nullptr;  // sign mask of the resident planes: bit x&31 of word x>>5 per row
  int W = 0;                     // words per lattice row, ceil((R+1)/32)
  __device__ __forceinline__ float at(int64_t x, int64_t y, int64_t z) const {
    return s[x + n1 * (y + n1 * (z - zb))];
  }
  __device__ __forceinline__ int bit(int64_t x, int64_t row) const {
    return (sg[row * W + (x >> 5)] >> (x & 31)) & 1;
  }
  // 8-bit case, corner c = x | y<<1 | z<<2, bit set for a negative sample (sign(0) = +)
  __device__ __forceinline__ int case_of(int64_t x, int64_t y, int64_t z) const {
    const int64_t r = (z - zb) * n1 + y;
    return bit(x, r) | bit(x + 1, r) << 1 | bit(x, r + 1) << 2 | bit(x + 1, r + 1) << 3 | bit(x, r + n1) << 4 |
           bit(x + 1, r + n1) << 5 | bit(x, r + n1 + 1) << 6 | bit(x + 1, r + n1 + 1) << 7;
  }
};

// sign mask of resident planes (used when the SDF producer did not emit one): one warp per word
__global__ void k_pack_signs(const float* __restrict__ s, int64_t rows, int n1, int W, uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = rows * W;
  for (int64_t wi = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; wi < nw;
       wi += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t row = wi / W;
    const int x = (static_cast<int>(wi - row * W) << 5) + lane;
    const bool neg = x < n1 && s[row * n1 + x] < 0.0f;
    const unsigned m = __ballot_sync(0xffffffffu, neg);
    if (lane == 0) out[wi] = m;
  }
}

// R is a power of two: cell coordinates by shifts (no 64-bit division per cell)
__device__ __forceinline__ void cell_xyz(int64_t c, int R, int64_t& x, int64_t& y, int64_t& z) {
  const int lg = __ffs(R) - 1;
  x = c & (R - 1);
  y = (c >> lg) & (R - 1);
  z = c >> (2 * lg);
}

// Dense classify over the sign mask, 32 cells per lane: lane (row r, word w) loads the 4 rows'
// words w and w+1 (rows (y,z), (y+1,z), (y,z+1), (y+1,z+1); consecutive lanes read consecutive
// words of a row, so the loads coalesce) and forms the 8 corner masks of its 32 cells with funnel
// shifts.  A cell is active iff some corner is negative and not all are: active = OR & ~AND of
// the 8 masks — the whole dense pass is ~20 bit operations per 32 cells.  Lanes are ordered
// (row, word), rows (z, y), so per-block counts + a scan give the x-fastest compaction; the
// write pass assembles the 8-bit case only for the set bits.  All index math is 32-bit shifts.
struct SegCtx {
  int R, lg;     // cells per row, log2 R
  int lgw;       // log2 words per row (words of 32 cells; R < 32 -> 1 word)
  int nrows;     // rows of the classified layers: R * layers
  int z0;        // first cell layer
};

struct Corners {
  uint32_t m[8];  // m[c]: bit b = corner c of cell (32 w + b) is negative
  uint32_t valid;
};

__device__ __forceinline__ Corners corners_of(const GridView& g, const SegCtx& S, int lanei) {
  Corners K;
  const int row = lanei >> S.lgw, w = lanei & ((1 << S.lgw) - 1);
  const int y = row & (S.R - 1), z = S.z0 + (row >> S.lg);
  const uint32_t* p = g.sg + ((static_cast<int64_t>(z) - g.zb) * g.n1 + y) * g.W + w;
  const int64_t W = g.W, rW = g.n1 * g.W;
  const bool has1 = w + 1 < g.W;
  const uint32_t* q[4] = {p, p + W, p + rW, p + rW + W};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t lo = q[k][0], hi = has1 ? q[k][1] : 0u;
    K.m[2 * k] = lo;                             // corner (0, dy, dz): bit x
    K.m[2 * k + 1] = __funnelshift_r(lo, hi, 1);  // corner (1, dy, dz): bit x + 1
  }
  const int nvalid = min(32, S.R - (w << 5));
  K.valid = nvalid >= 32 ? 0xffffffffu : ((1u << nvalid) - 1u);
  return K;
}

__device__ __forceinline__ uint32_t active_mask(const Corners& K) {
  uint32_t o = 0u, a = 0xffffffffu;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    o |= K.m[c];
    a &= K.m[c];
  }
  return o & ~a & K.valid;
}

__global__ void __launch_bounds__(256) k_classify_count(GridView g, SegCtx S, int64_t nlanes,
                                                        uint32_t* __restrict__ bcount) {
  __shared__ uint32_t wsum[8];
  const int64_t li = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  uint32_t n = li < nlanes ? __popc(active_mask(corners_of(g, S, static_cast<int>(li)))) : 0u;
  for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < 8; ++i) t += wsum[i];
    bcount[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(256) k_classify_write(GridView g, SegCtx S, int64_t nlanes,
                                                        const uint32_t* __restrict__ boff,
                                                        uint32_t* __restrict__ cells, uint8_t* __restrict__ cases) {
  __shared__ uint32_t wsum[8];
  const int64_t li = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Corners K{};
  uint32_t act = 0u;
  if (li < nlanes) {
    K = corners_of(g, S, static_cast<int>(li));
    act = active_mask(K);
  }
  const uint32_t n = __popc(act);
  uint32_t incl = n;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  uint32_t run = boff[blockIdx.x] + incl - n;
  for (int i = 0; i < warp; ++i) run += wsum[i];
  if (!act) return;
  const int i = static_cast<int>(li);
  const int row = i >> S.lgw, w = i & ((1 << S.lgw) - 1);
  const uint32_t cbase = (static_cast<uint32_t>(row + S.R * S.z0) << S.lg) + (w << 5);  // (z*R + y)*R + 32w
  while (act) {
    const int b = __ffs(act) - 1;
    act &= act - 1;
    int cs = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) cs |= ((K.m[c] >> b) & 1u) << c;
    cells[run] = cbase + b;
    cases[run] = static_cast<uint8_t>(cs);
    ++run;
  }
}

__device__ __forceinline__ const PatchSet& patches_of(int cs, int flip) { return flip ? c_flip[cs] : c_base[cs]; }

__global__ void k_patch_count(GridView g, const uint32_t* __restrict__ cells, const uint8_t* __restrict__ cases,
                              int64_t na, uint8_t* __restrict__ flips, uint32_t* __restrict__ npatch,
                              uint32_t* __restrict__ cellmap, int64_t c0) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= na) return;
  const int cs = cases[i];
  int flip = 0;
  const int dc = c_base[cs].dc;
  if (dc) {
    int64_t xyz[3];
    cell_xyz(cells[i], g.R, xyz[0], xyz[1], xyz[2]);
    const int f = __ffs(dc) - 1, axis = f >> 1, side = f & 1;
    int64_t n[3] = {xyz[0], xyz[1], xyz[2]};
    n[axis] += side ? 1 : -1;
    if (n[axis] >= 0 && n[axis] < g.R) {
      const int ncs = g.case_of(n[0], n[1], n[2]);
      if ((c_base[ncs].dc >> (2 * axis + (1 - side))) & 1) flip = dc;
    }
  }
  flips[i] = static_cast<uint8_t>(flip);
  npatch[i] = patches_of(cs, flip).n;
  cellmap[cells[i] - c0] = static_cast<uint32_t>(i);
}

// x / R for the power-of-two R: the product by the exact reciprocal is the same double
__device__ __forceinline__ D3 gpoint(int64_t x, int64_t y, int64_t z, int R) {
  const double iR = __longlong_as_double(static_cast<long long>(1023 - (__ffs(R) - 1)) << 52);
  return D3{static_cast<double>(x) * iR, static_cast<double>(y) * iR, static_cast<double>(z) * iR};
}

__device__ __forceinline__ D3 crossing(D3 p0, D3 p1, float f0, float f1, double beta) {
  const double t = -static_cast<double>(f0) / (static_cast<double>(f1) - static_cast<double>(f0));
  const double ts = sigmoid_t(t, beta);
  return D3{p0.x + ts * (p1.x - p0.x), p0.y + ts * (p1.y - p0.y), p0.z + ts * (p1.z - p0.z)};
}

// edge e of the cell: lower corner and axis
__device__ __forceinline__ void edge_corners(int e, int& c0, int& axis) {
  axis = e >> 2;
  const int sub = e & 3, u = sub & 1, w = sub >> 1;
  c0 = axis == 0 ? ((u << 1) | (w << 2)) : (axis == 1 ? (u | (w << 2)) : (u | (w << 1)));
}

__global__ void k_patch_vertices(GridView g, const uint32_t* __restrict__ cells, const uint8_t* __restrict__ cases,
                                 const uint8_t* __restrict__ flips, const uint32_t* __restrict__ vbase, int64_t na,
                                 double beta, double* __restrict__ V) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= na) return;
  int64_t x, y, z;
  cell_xyz(cells[i], g.R, x, y, z);
  const PatchSet& P = patches_of(cases[i], flips[i]);
  for (int p = 0; p < P.n; ++p) {
    double sx = 0.0, sy = 0.0, sz = 0.0;
    int cnt = 0;
    for (int e = 0; e < 12; ++e) {
      if (!((P.mask[p] >> e) & 1)) continue;
      int c0, ax;
      edge_corners(e, c0, ax);
      const int c1 = c0 | (1 << ax);
      const int64_t x0 = x + (c0 & 1), y0 = y + ((c0 >> 1) & 1), z0 = z + ((c0 >> 2) & 1);
      const int64_t x1 = x + (c1 & 1), y1 = y + ((c1 >> 1) & 1), z1 = z + ((c1 >> 2) & 1);
      const D3 q = crossing(gpoint(x0, y0, z0, g.R), gpoint(x1, y1, z1, g.R), g.at(x0, y0, z0), g.at(x1, y1, z1), beta);
      sx = sx + q.x;
      sy = sy + q.y;
      sz = sz + q.z;
      ++cnt;
    }
    const int64_t vi = vbase[i] + p;
    V[3 * vi] = sx / cnt;
    V[3 * vi + 1] = sy / cnt;
    V[3 * vi + 2] = sz / cnt;
  }
}

struct QuadGeo {
  uint32_t q[4];
  D3 plo, phi;
  float f0, f1;
};

// Builds the quad of the axis-a valid edge at the corner 0 of active cell i (returns false if none)
__device__ __forceinline__ bool make_quad(GridView g, int64_t x, int64_t y, int64_t z, int a,
                                          const uint32_t* __restrict__ cellmap, const uint8_t* __restrict__ cases,
                                          const uint8_t* __restrict__ flips, const uint32_t* __restrict__ vbase,
                                          int64_t cbase, QuadGeo& Q) {
  const int64_t xyz[3] = {x, y, z};
  const int b = (a + 1) % 3, c = (a + 2) % 3;
  if (xyz[b] < 1 || xyz[c] < 1) return false;
  int64_t up[3] = {x, y, z};
  up[a] += 1;
  Q.f0 = g.at(x, y, z);
  Q.f1 = g.at(up[0], up[1], up[2]);
  if ((Q.f0 < 0.0f) == (Q.f1 < 0.0f)) return false;
  const int offs[4][2] = {{-1, -1}, {0, -1}, {0, 0}, {-1, 0}};
  for (int k = 0; k < 4; ++k) {
    int64_t cl[3] = {x, y, z};
    cl[b] += offs[k][0];
    cl[c] += offs[k][1];
    int c0 = 0;
    if (offs[k][0] == -1) c0 |= 1 << b;
    if (offs[k][1] == -1) c0 |= 1 << c;
    const int cx = c0 & 1, cy = (c0 >> 1) & 1, cz = (c0 >> 2) & 1;
    const int e = a == 0 ? cy + 2 * cz : (a == 1 ? 4 + cx + 2 * cz : 8 + cx + 2 * cy);
    const uint32_t j = cellmap[cl[0] + g.R * (cl[1] + static_cast<int64_t>(g.R) * cl[2]) - cbase];
    Q.q[k] = vbase[j] + patches_of(cases[j], flips[j]).edge_patch[e];
  }
  if (!(Q.f0 < 0.0f)) {  // lower endpoint positive: reverse so the normal points - -> +
    const uint32_t t = Q.q[1];
    Q.q[1] = Q.q[3];
    Q.q[3] = t;
  }
  Q.plo = gpoint(x, y, z, g.R);
  Q.phi = gpoint(up[0], up[1], up[2], g.R);
  return true;
}

__device__ __forceinline__ D3 ld3(const double* V, uint32_t i) { return D3{V[3 * i], V[3 * i + 1], V[3 * i + 2]}; }

// 1: diagonal 0-2, 2: diagonal 1-3, 3: four triangles around the edge crossing
__device__ __forceinline__ int split_code(const QuadGeo& Q, const double* __restrict__ V) {
  D3 P[4];
  for (int k = 0; k < 4; ++k) P[k] = ld3(V, Q.q[k]);
  const bool lower_neg = Q.f0 < 0.0f;
  const D3 vp = lower_neg ? Q.phi : Q.plo, vn = lower_neg ? Q.plo : Q.phi;
  bool conc[4];
  for (int k = 0; k < 4; ++k) {
    const D3 L = P[(k + 3) & 3], Rr = P[(k + 1) & 3];
    const double t1 = dot(sub(P[k], vp), cross(sub(L, vp), sub(Rr, vp)));
    const double t2 = dot(sub(P[k], vn), cross(sub(L, vn), sub(Rr, vn)));
    conc[k] = t1 < 0.0 || t2 > 0.0;
  }
  const bool d02 = conc[0] || conc[2], d13 = conc[1] || conc[3];
  if (d02 && !d13) return 1;
  if (d13 && !d02) return 2;
  if (d02 && d13) return 3;
  auto maxcos = [&](int i0, int i1, int i2) {
    const D3 T[3] = {P[i0], P[i1], P[i2]};
    double m = -2.0;
    for (int k = 0; k < 3; ++k) {
      const D3 u = sub(T[(k + 1) % 3], T[k]), w = sub(T[(k + 2) % 3], T[k]);
      const double cs = dot(u, w) / sqrt(sqn(u) * sqn(w));
      if (cs > m) m = cs;
    }
    return m;
  };
  const double m02 = fmax(maxcos(0, 1, 2), maxcos(0, 2, 3));
  const double m13 = fmax(maxcos(0, 1, 3), maxcos(1, 2, 3));
  return m02 <= m13 ? 1 : 2;
}

__global__ void k_quad_count(GridView g, const uint32_t* __restrict__ cells, const uint8_t* __restrict__ cases,
                             const uint8_t* __restrict__ flips, const uint32_t* __restrict__ vbase,
                             const uint32_t* __restrict__ cellmap, int64_t c0, int64_t own_z0, int64_t na,
                             const double* __restrict__ V, uint64_t* __restrict__ counts,
                             uint8_t* __restrict__ codes) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= na) return;
  int64_t x, y, z;
  cell_xyz(cells[i], g.R, x, y, z);
  uint32_t nfaces = 0, nextra = 0;
  uint8_t code = 0;
  for (int a = 0; a < 3 && z >= own_z0; ++a) {  // the layer below a slab only lends vertex ids
    QuadGeo Q;
    if (!make_quad(g, x, y, z, a, cellmap, cases, flips, vbase, c0, Q)) continue;
    const int sc = split_code(Q, V);
    code |= static_cast<uint8_t>(sc << (2 * a));
    nfaces += sc == 3 ? 4 : 2;
    nextra += sc == 3;
  }
  codes[i] = code;
  counts[i] = (static_cast<uint64_t>(nfaces) << 32) | nextra;
}

__global__ void k_quad_write(GridView g, const uint32_t* __restrict__ cells, const uint8_t* __restrict__ cases,
                             const uint8_t* __restrict__ flips, const uint32_t* __restrict__ vbase,
                             const uint32_t* __restrict__ cellmap, int64_t c0, int64_t na,
                             const uint8_t* __restrict__ codes, const uint64_t* __restrict__ offs, uint64_t nv_patch,
                             int64_t shift, double beta, double* __restrict__ V, int32_t* __restrict__ Fo) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= na || codes[i] == 0) return;
  int64_t x, y, z;
  cell_xyz(cells[i], g.R, x, y, z);
  uint64_t fo = offs[i] >> 32, eo = offs[i] & 0xffffffffu;
  for (int a = 0; a < 3; ++a) {
    const int sc = (codes[i] >> (2 * a)) & 3;
    if (!sc) continue;
    QuadGeo Q;
    make_quad(g, x, y, z, a, cellmap, cases, flips, vbase, c0, Q);
    for (int k = 0; k < 4; ++k) Q.q[k] -= static_cast<uint32_t>(shift);  // ids relative to the first own vertex
    const int32_t* q = reinterpret_cast<const int32_t*>(Q.q);
    int32_t* o = Fo + 3 * fo;
    if (sc == 1) {
      const int32_t t[6] = {(int32_t)q[0], (int32_t)q[1], (int32_t)q[2], (int32_t)q[0], (int32_t)q[2], (int32_t)q[3]};
      for (int k = 0; k < 6; ++k) o[k] = t[k];
      fo += 2;
    } else if (sc == 2) {
      const int32_t t[6] = {(int32_t)q[0], (int32_t)q[1], (int32_t)q[3], (int32_t)q[1], (int32_t)q[2], (int32_t)q[3]};
      for (int k = 0; k < 6; ++k) o[k] = t[k];
      fo += 2;
    } else {
      const uint64_t ve = nv_patch - shift + eo;
      const D3 p = crossing(Q.plo, Q.phi, Q.f0, Q.f1, beta);
      V[3 * ve] = p.x;
      V[3 * ve + 1] = p.y;
      V[3 * ve + 2] = p.z;
      const int32_t e = static_cast<int32_t>(ve);
      const int32_t t[12] = {(int32_t)q[0], (int32_t)q[1], e, (int32_t)q[1], (int32_t)q[2], e,
                             (int32_t)q[2], (int32_t)q[3], e, (int32_t)q[3], (int32_t)q[0], e};
      for (int k = 0; k < 12; ++k) o[k] = t[k];
      fo += 4;
      eo += 1;
    }
  }
}

// build_quads view: the quads in output order (cell, axis) with their valid
// edge (lower lattice vertex linear index * 3 + axis), endpoint samples and split decision
__global__ void k_quad_list(GridView g, const uint32_t* __restrict__ cells, const uint8_t* __restrict__ cases,
                            const uint8_t* __restrict__ flips, const uint32_t* __restrict__ vbase,
                            const uint32_t* __restrict__ cellmap, int64_t c0, int64_t na,
                            const uint8_t* __restrict__ codes, const uint32_t* __restrict__ qoff,
                            int32_t* __restrict__ quads, int64_t* __restrict__ qedge, float* __restrict__ qf,
                            uint8_t* __restrict__ qsplit) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= na || codes[i] == 0) return;
  int64_t x, y, z;
  cell_xyz(cells[i], g.R, x, y, z);
  uint32_t o = qoff[i];
  const int64_t n1 = g.R + 1;
  for (int a = 0; a < 3; ++a) {
    const int sc = (codes[i] >> (2 * a)) & 3;
    if (!sc) continue;
    QuadGeo Q;
    make_quad(g, x, y, z, a, cellmap, cases, flips, vbase, c0, Q);
    for (int k = 0; k < 4; ++k) quads[4 * o + k] = static_cast<int32_t>(Q.q[k]);
    qedge[o] = (x + n1 * (y + n1 * z)) * 3 + a;
    qf[2 * o] = Q.f0;
    qf[2 * o + 1] = Q.f1;
    qsplit[o] = static_cast<uint8_t>(sc);
    ++o;
  }
}

__global__ void k_quad_ncount(const uint8_t* __restrict__ codes, int64_t na, uint32_t* __restrict__ nq) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= na) return;
  const uint8_t c = codes[i];
  nq[i] = ((c & 3) != 0) + (((c >> 2) & 3) != 0) + (((c >> 4) & 3) != 0);
}

// triangulate_quads on explicit quads: edge = lower vertex * 3 + axis
__device__ __forceinline__ QuadGeo quad_from(const int32_t* quads, const int64_t* qedge, const float* qf, int64_t i,
                                             int R) {
  QuadGeo Q;
  for (int k = 0; k < 4; ++k) Q.q[k] = static_cast<uint32_t>(quads[4 * i + k]);
  const int64_t n1 = R + 1, lv = qedge[i] / 3;
  const int a = static_cast<int>(qedge[i] % 3);
  const int64_t x = lv % n1, y = (lv / n1) % n1, z = lv / (n1 * n1);
  int64_t up[3] = {x, y, z};
  up[a] += 1;
  Q.plo = gpoint(x, y, z, R);
  Q.phi = gpoint(up[0], up[1], up[2], R);
  Q.f0 = qf[2 * i];
  Q.f1 = qf[2 * i + 1];
  return Q;
}

__global__ void k_triq_count(const int32_t* __restrict__ quads, const int64_t* __restrict__ qedge,
                             const float* __restrict__ qf, int64_t nq, int R, const double* __restrict__ V,
                             uint8_t* __restrict__ code, uint64_t* __restrict__ counts) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nq) return;
  const QuadGeo Q = quad_from(quads, qedge, qf, i, R);
  const int sc = split_code(Q, V);
  code[i] = static_cast<uint8_t>(sc);
  counts[i] = (static_cast<uint64_t>(sc == 3 ? 4 : 2) << 32) | (sc == 3 ? 1u : 0u);
}

__global__ void k_triq_write(const int32_t* __restrict__ quads, const int64_t* __restrict__ qedge,
                             const float* __restrict__ qf, int64_t nq, int R, const uint8_t* __restrict__ code,
                             const uint64_t* __restrict__ offs, uint64_t nv_patch, double beta, double* __restrict__ V,
                             int32_t* __restrict__ Fo) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nq) return;
  const QuadGeo Q = quad_from(quads, qedge, qf, i, R);
  const int32_t* q = quads + 4 * i;
  int32_t* o = Fo + 3 * (offs[i] >> 32);
  const int sc = code[i];
  if (sc == 1) {
    const int32_t t[6] = {q[0], q[1], q[2], q[0], q[2], q[3]};
    for (int k = 0; k < 6; ++k) o[k] = t[k];
  } else if (sc == 2) {
    const int32_t t[6] = {q[0], q[1], q[3], q[1], q[2], q[3]};
    for (int k = 0; k < 6; ++k) o[k] = t[k];
  } else {
    const uint64_t ve = nv_patch + (offs[i] & 0xffffffffu);
    const D3 p = crossing(Q.plo, Q.phi, Q.f0, Q.f1, beta);
    V[3 * ve] = p.x;
    V[3 * ve + 1] = p.y;
    V[3 * ve + 2] = p.z;
    const int32_t e = static_cast<int32_t>(ve);
    const int32_t t[12] = {q[0], q[1], e, q[1], q[2], e, q[2], q[3], e, q[3], q[0], e};
    for (int k = 0; k < 12; ++k) o[k] = t[k];
  }
}

// interpolate_patch_vertex for explicit edges; bad[i] = equal signs
__global__ void k_interp(const double* __restrict__ p0, const double* __restrict__ p1, const float* __restrict__ f0,
                         const float* __restrict__ f1, int64_t n, double beta, double* __restrict__ out,
                         unsigned long long* __restrict__ bad) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  if ((f0[i] < 0.0f) == (f1[i] < 0.0f) || !isfinite(f0[i]) || !isfinite(f1[i])) {
    atomicAdd(bad, 1ull);
    out[3 * i] = out[3 * i + 1] = out[3 * i + 2] = 0.0;
    return;
  }
  const D3 q = crossing(D3{p0[3 * i], p0[3 * i + 1], p0[3 * i + 2]}, D3{p1[3 * i], p1[3 * i + 1], p1[3 * i + 2]}, f0[i],
                        f1[i], beta);
  out[3 * i] = q.x;
  out[3 * i + 1] = q.y;
  out[3 * i + 2] = q.z;
}

}  // namespace

void dmc_table_host(int32_t* out) {
  const HostTable& t = host_table();
  for (int cs = 0; cs < 256; ++cs) {
    out[6 * cs] = t.base[cs].n;
    for (int k = 0; k < 4; ++k) out[6 * cs + 1 + k] = t.base[cs].mask[k];
    out[6 * cs + 5] = t.base[cs].dc;
  }
}

namespace {
// first own patch vertex: vbase of the first active cell at or above the own layers
__global__ void k_own_split(const uint32_t* __restrict__ cells, const uint32_t* __restrict__ vbase, int64_t na,
                            uint64_t cthr, uint32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= na) return;
  if (cells[i] >= cthr && (i == 0 || cells[i - 1] < cthr)) *out = vbase[i];
}
}  // namespace

void dmc_extract_slab(Ctx& ctx, const float* d_planes, int R, int pz0, int pz1, int own_z0, int own_z1, double beta,
                      DmcResult& res, const uint32_t* d_signs) {
  upload_table(ctx.device);
  const int cz0 = own_z0 > 0 ? own_z0 - 1 : 0;  // the layer below lends its patch-vertex ids
  PCU_REQUIRE(R >= 2 && R <= 1024 && (R & (R - 1)) == 0, PAMOPT_CU_EINVAL, "dmc: R must be a power of two <= 1024");
  PCU_REQUIRE(own_z0 >= 0 && own_z0 < own_z1 && own_z1 <= R, PAMOPT_CU_EINVAL,
              "dmc slab: own cell layers must satisfy 0 <= z0 < z1 <= R");
  PCU_REQUIRE(pz0 <= std::max(own_z0 - 2, 0) && pz1 >= std::min(own_z1 + 2, R + 1) && pz0 >= 0 && pz1 <= R + 1,
              PAMOPT_CU_EINVAL, "dmc slab: resident planes must cover [z0-2, z1+2) clipped to the lattice");
  GridView g{d_planes, R, static_cast<int64_t>(R) + 1, pz0};
  g.W = (R + 1 + 31) / 32;
  DevBuf<uint32_t> packed;
  if (d_signs) {
    g.sg = d_signs;
  } else {  // one read of the resident planes; every dense pass below reads the mask instead
    const int64_t rows = static_cast<int64_t>(R + 1) * (pz1 - pz0);
    packed.alloc(rows * g.W, ctx.stream);
    PCU_LAUNCH(ctx, k_pack_signs, static_cast<unsigned>(ctx.num_sms * 16), 256, 0, d_planes, rows, R + 1, g.W,
               packed.get());
    g.sg = packed.get();
  }
  const int64_t rr = static_cast<int64_t>(R) * R;
  const int64_t c0 = rr * cz0;
  const int64_t ncell = rr * (own_z1 - cz0);
  SegCtx S;
  S.R = R;
  S.lg = __builtin_ctz(static_cast<unsigned>(R));
  S.lgw = R >= 32 ? S.lg - 5 : 0;
  S.z0 = cz0;
  S.nrows = R * (own_z1 - cz0);
  const int64_t nlanes = static_cast<int64_t>(S.nrows) << S.lgw;
  const int64_t nblk = (nlanes + 255) / 256;
  DevBuf<uint32_t> bcount(nblk, ctx.stream), boff(nblk, ctx.stream);
  PCU_LAUNCH(ctx, k_classify_count, static_cast<unsigned>(nblk), 256, 0, g, S, nlanes, bcount.get());
  exclusive_scan_u32(ctx, bcount.get(), boff.get(), nblk);
  const uint32_t na = read_scalar(ctx, boff.get() + nblk - 1) + read_scalar(ctx, bcount.get() + nblk - 1);
  res.cells.alloc(na ? na : 1, ctx.stream);
  res.cases.alloc(na ? na : 1, ctx.stream);
  res.flips.alloc(na ? na : 1, ctx.stream);
  res.n_active = na;
  PCU_LAUNCH(ctx, k_classify_write, static_cast<unsigned>(nblk), 256, 0, g, S, nlanes, boff.get(), res.cells.get(),
             res.cases.get());
  res.nvp_own = res.n_extra = 0;
  if (na == 0) {
    res.nv = res.nf = 0;
    res.V.alloc(1, ctx.stream);
    res.F.alloc(1, ctx.stream);
    return;
  }
  DevBuf<uint32_t> npatch(na, ctx.stream), vbase(na, ctx.stream);
  DevBuf<uint32_t> cellmap(ncell, ctx.stream);  // only active entries are written / read
  PCU_LAUNCH(ctx, k_patch_count, grid_for(na, 256), 256, 0, g, res.cells.get(), res.cases.get(), na, res.flips.get(),
             npatch.get(), cellmap.get(), c0);
  exclusive_scan_u32(ctx, npatch.get(), vbase.get(), na);
  const uint64_t nv_patch = static_cast<uint64_t>(read_scalar(ctx, vbase.get() + na - 1)) + read_scalar(ctx, npatch.get() + na - 1);
  uint64_t shift = 0;
  if (own_z0 > cz0) {
    DevBuf<uint32_t> split(1, ctx.stream);
    const uint32_t init = static_cast<uint32_t>(nv_patch);
    PCU_CUDA(cudaMemcpyAsync(split.get(), &init, 4, cudaMemcpyHostToDevice, ctx.stream));
    PCU_LAUNCH(ctx, k_own_split, grid_for(na, 256), 256, 0, res.cells.get(), vbase.get(), na,
               static_cast<uint64_t>(rr * own_z0), split.get());
    shift = read_scalar(ctx, split.get());
  }
  DevBuf<uint64_t> counts(na, ctx.stream), offs(na, ctx.stream);
  DevBuf<uint8_t> codes(na, ctx.stream);
  // patch vertices first (the quad pass reads them); extra vertices appended after
  DevBuf<double> Vp(3 * nv_patch, ctx.stream);
  PCU_LAUNCH(ctx, k_patch_vertices, grid_for(na, 128), 128, 0, g, res.cells.get(), res.cases.get(), res.flips.get(),
             vbase.get(), na, beta, Vp.get());
  PCU_LAUNCH(ctx, k_quad_count, grid_for(na, 128), 128, 0, g, res.cells.get(), res.cases.get(), res.flips.get(),
             vbase.get(), cellmap.get(), c0, static_cast<int64_t>(own_z0), na, Vp.get(), counts.get(), codes.get());
  exclusive_scan_u64(ctx, counts.get(), offs.get(), na);
  const uint64_t last = read_scalar(ctx, offs.get() + na - 1) + read_scalar(ctx, counts.get() + na - 1);
  const uint64_t nf = last >> 32, nextra = last & 0xffffffffu;
  res.nvp_own = nv_patch - shift;
  res.n_extra = nextra;
  res.nv = res.nvp_own + nextra;
  res.nf = nf;
  res.n_quads = 0;
  res.V.alloc(3 * (res.nv ? res.nv : 1), ctx.stream);
  res.F.alloc(3 * (nf ? nf : 1), ctx.stream);
  if (res.nvp_own)
    PCU_CUDA(cudaMemcpyAsync(res.V.get(), Vp.get() + 3 * shift, 3 * res.nvp_own * sizeof(double),
                             cudaMemcpyDeviceToDevice, ctx.stream));
  PCU_LAUNCH(ctx, k_quad_write, grid_for(na, 128), 128, 0, g, res.cells.get(), res.cases.get(), res.flips.get(),
             vbase.get(), cellmap.get(), c0, na, codes.get(), offs.get(), nv_patch, static_cast<int64_t>(shift), beta,
             res.V.get(), res.F.get());
  if (res.want_stages && shift == 0) {  // build_patches / build_quads views (whole grid)
    res.vbase = std::move(vbase);
    res.nv_patch = nv_patch;
    DevBuf<uint32_t> nq(na, ctx.stream), qoff(na, ctx.stream);
    PCU_LAUNCH(ctx, k_quad_ncount, grid_for(na, 256), 256, 0, codes.get(), na, nq.get());
    exclusive_scan_u32(ctx, nq.get(), qoff.get(), na);
    res.n_quads = static_cast<uint64_t>(read_scalar(ctx, qoff.get() + na - 1)) + read_scalar(ctx, nq.get() + na - 1);
    const uint64_t m = res.n_quads ? res.n_quads : 1;
    res.quads.alloc(4 * m, ctx.stream);
    res.qedge.alloc(m, ctx.stream);
    res.qf.alloc(2 * m, ctx.stream);
    res.qsplit.alloc(m, ctx.stream);
    PCU_LAUNCH(ctx, k_quad_list, grid_for(na, 128), 128, 0, g, res.cells.get(), res.cases.get(), res.flips.get(),
               res.vbase.get(), cellmap.get(), c0, na, codes.get(), qoff.get(), res.quads.get(), res.qedge.get(),
               res.qf.get(), res.qsplit.get());
  }
}

void triangulate_quads(Ctx& ctx, const double* d_patch_v, int64_t nv_patch, const int32_t* d_quads,
                       const int64_t* d_qedge, const float* d_qf, int64_t nq, int R, double beta, DevBuf<double>& V,
                       DevBuf<int32_t>& F, int64_t& nv, int64_t& nf) {
  upload_table(ctx.device);
  if (nq == 0) {
    nv = nv_patch;
    nf = 0;
    V.alloc(3 * (nv ? nv : 1), ctx.stream);
    if (nv) PCU_CUDA(cudaMemcpyAsync(V.get(), d_patch_v, 3 * nv * 8, cudaMemcpyDeviceToDevice, ctx.stream));
    F.alloc(1, ctx.stream);
    return;
  }
  DevBuf<uint8_t> code(nq, ctx.stream);
  DevBuf<uint64_t> counts(nq, ctx.stream), offs(nq, ctx.stream);
  PCU_LAUNCH(ctx, k_triq_count, grid_for(nq, 128), 128, 0, d_quads, d_qedge, d_qf, nq, R, d_patch_v, code.get(),
             counts.get());
  exclusive_scan_u64(ctx, counts.get(), offs.get(), nq);
  const uint64_t last = read_scalar(ctx, offs.get() + nq - 1) + read_scalar(ctx, counts.get() + nq - 1);
  nf = static_cast<int64_t>(last >> 32);
  nv = nv_patch + static_cast<int64_t>(last & 0xffffffffu);
  V.alloc(3 * (nv ? nv : 1), ctx.stream);
  F.alloc(3 * (nf ? nf : 1), ctx.stream);
  if (nv_patch) PCU_CUDA(cudaMemcpyAsync(V.get(), d_patch_v, 3 * nv_patch * 8, cudaMemcpyDeviceToDevice, ctx.stream));
  PCU_LAUNCH(ctx, k_triq_write, grid_for(nq, 128), 128, 0, d_quads, d_qedge, d_qf, nq, R, code.get(), offs.get(),
             static_cast<uint64_t>(nv_patch), beta, V.get(), F.get());
}

int64_t interpolate_patch_vertex(Ctx& ctx, const double* d_p0, const double* d_p1, const float* d_f0, const float* d_f1,
                                 int64_t n, double beta, double* d_out) {
  if (n == 0) return 0;
  DevBuf<unsigned long long> bad(1, ctx.stream);
  bad.memset(0, ctx.stream);
  PCU_LAUNCH(ctx, k_interp, grid_for(n, 256), 256, 0, d_p0, d_p1, d_f0, d_f1, n, beta, d_out, bad.get());
  return static_cast<int64_t>(read_scalar(ctx, bad.get()));
}

namespace {
__global__ void k_rebase(int32_t* __restrict__ F, int64_t n, int64_t patch_base, int64_t nvp_own, int64_t extra_base) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int64_t v = F[i];
  F[i] = static_cast<int32_t>(v < nvp_own ? patch_base + v : extra_base + (v - nvp_own));
}
}  // namespace

void mesh_rebase(Ctx& ctx, int32_t* dF, int64_t nidx, int64_t patch_base, int64_t nvp_own, int64_t extra_base) {
  if (nidx <= 0) return;
  PCU_LAUNCH(ctx, k_rebase, grid_for(nidx, 256), 256, 0, dF, nidx, patch_base, nvp_own, extra_base);
}

void dmc_extract(Ctx& ctx, const float* d_sdf, int R, double beta, DmcResult& res, const uint32_t* d_signs) {
  PCU_REQUIRE(R >= 2 && R <= 1024, PAMOPT_CU_EINVAL, "extract: R must be <= 1024 (32-bit cell ids)");
  dmc_extract_slab(ctx, d_sdf, R, 0, R + 1, 0, R, beta, res, d_signs);
}

}  // namespace pcu

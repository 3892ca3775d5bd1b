// ingest.cu — the on-disk format boundary, on the GPU:
//   * binary STL (mesh_io.cpp:309-366): the 50-byte facet records are decoded in parallel and
//     the corners welded by exact coordinate equality with the reference's numbering (vertices
//     in first-occurrence order, mesh_io.cpp:291-301): a stable radix sort of the (x, y, z)
//     float bit patterns groups equal corners, each group's first occurrence gets the next id in
//     corner order.  A corner with a NaN coordinate never equals anything (NaN != NaN), so it is
//     always a vertex of its own; -0.0 and +0.0 are told apart by their bits (the reference's
//     hash does the same, up to an unspecified bucket collision).
//   * binary little-endian PLY (mesh_io.cpp:135-255) with a fixed-size face record (a list of
//     exactly 3 indices per face — what the reference's own writer emits, mesh_io.cpp:256-266);
//     the header is parsed on the host, the body decoded in parallel.
//   * add_polygon's degenerate-face drop (mesh_io.cpp:32-42) and load_mesh's checks (index range,
//     empty mesh; mesh_io.cpp:381-384) follow.
//   * normalize_unit_cube (mesh_io.cpp:393-408): order-free min/max bounds, then the reference's
//     scale/translation arithmetic per component (bit-exact without FMA contraction).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace pcu {
namespace {

__device__ __forceinline__ uint32_t ld_u32_unaligned(const uint8_t* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
         (static_cast<uint32_t>(p[3]) << 24);
}
__device__ __forceinline__ uint64_t ld_u64_unaligned(const uint8_t* p) {
  return static_cast<uint64_t>(ld_u32_unaligned(p)) | (static_cast<uint64_t>(ld_u32_unaligned(p + 4)) << 32);
}

// corner c of facet i: record at 84 + 50 i; normal (12 B), then 3 x (3 x float32)
__global__ void k_stl_corners(const uint8_t* __restrict__ body, int64_t nc, uint32_t* __restrict__ kx,
                              uint64_t* __restrict__ kyz, uint32_t* __restrict__ idx, uint8_t* __restrict__ nan) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= nc) return;
  const uint8_t* p = body + 84 + 50 * (c / 3) + 12 + 12 * (c % 3);
  const uint32_t x = ld_u32_unaligned(p), y = ld_u32_unaligned(p + 4), z = ld_u32_unaligned(p + 8);
  kx[c] = x;
  kyz[c] = (static_cast<uint64_t>(y) << 32) | z;
  idx[c] = static_cast<uint32_t>(c);
  auto isnan32 = [](uint32_t b) { return (b & 0x7f800000u) == 0x7f800000u && (b & 0x007fffffu); };
  nan[c] = (isnan32(x) || isnan32(y) || isnan32(z)) ? 1 : 0;
}

// sorted order: group heads (a NaN corner is always its own group)
__global__ void k_weld_heads(const uint32_t* __restrict__ kx, const uint64_t* __restrict__ kyz,
                             const uint32_t* __restrict__ idx, const uint8_t* __restrict__ nan, int64_t n,
                             uint32_t* __restrict__ head) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  head[j] = (j == 0 || kx[j] != kx[j - 1] || kyz[j] != kyz[j - 1] || nan[idx[j]] || nan[idx[j - 1]]) ? 1u : 0u;
}

// representative (first occurrence) of every corner: the group's first element in sorted order
// (the sort is stable, so it has the smallest corner index)
__global__ void k_weld_rep(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ head,
                           const uint32_t* __restrict__ gid, int64_t n, uint32_t* __restrict__ gfirst) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j < n && head[j]) gfirst[gid[j]] = idx[j];
}
// gid = exclusive scan of the heads: element j belongs to group gid[j] + head[j] - 1
__global__ void k_weld_first(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ head,
                             const uint32_t* __restrict__ gid, const uint32_t* __restrict__ gfirst, int64_t n,
                             uint32_t* __restrict__ rep, uint32_t* __restrict__ isfirst) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const uint32_t c = idx[j], r = gfirst[gid[j] + head[j] - 1];
  rep[c] = r;
  isfirst[c] = (r == c) ? 1u : 0u;
}

__global__ void k_weld_emit(const uint8_t* __restrict__ body, const uint32_t* __restrict__ rep,
                            const uint32_t* __restrict__ isfirst, const uint32_t* __restrict__ vpos, int64_t nc,
                            double* __restrict__ V, int32_t* __restrict__ corner_vid) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= nc) return;
  const uint32_t vid = vpos[rep[c]];
  corner_vid[c] = static_cast<int32_t>(vid);
  if (isfirst[c]) {
    const uint8_t* p = body + 84 + 50 * (c / 3) + 12 + 12 * (c % 3);
    for (int k = 0; k < 3; ++k) V[3 * static_cast<int64_t>(vid) + k] = static_cast<double>(__uint_as_float(ld_u32_unaligned(p + 4 * k)));
  }
}

__global__ void k_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ perm, int64_t n,
                             uint32_t* __restrict__ dst) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j < n) dst[j] = src[perm[j]];
}
__global__ void k_gather_u64(const uint64_t* __restrict__ src, const uint32_t* __restrict__ perm, int64_t n,
                             uint64_t* __restrict__ dst) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j < n) dst[j] = src[perm[j]];
}

// add_polygon for triangles: keep faces without repeated indices
__global__ void k_keep_faces(const int32_t* __restrict__ tri, int64_t nf, uint32_t* __restrict__ keep) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= nf) return;
  const int32_t a = tri[3 * f], b = tri[3 * f + 1], c = tri[3 * f + 2];
  keep[f] = (a != b && b != c && a != c) ? 1u : 0u;
}
__global__ void k_compact_faces(const int32_t* __restrict__ tri, const uint32_t* __restrict__ keep,
                                const uint32_t* __restrict__ pos, int64_t nf, int32_t* __restrict__ out) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f < nf && keep[f])
    for (int k = 0; k < 3; ++k) out[3 * static_cast<int64_t>(pos[f]) + k] = tri[3 * f + k];
}

// ---------------------------------------------------------------------------- PLY
struct PlyLayout {
  int64_t vbase, vstride, nvert;  // vertex records
  int xo, yo, zo, xt, yt, zt;     // byte offsets and types (0 float, 1 double, 2 int32, ...)
  int64_t fbase, fstride, nface;  // face records (fixed size)
  int co, ct, io, it;             // list count offset/type, first index offset/type
};

__device__ __forceinline__ double ply_scalar(const uint8_t* p, int t) {
  switch (t) {
    case 0: return static_cast<double>(__uint_as_float(ld_u32_unaligned(p)));
    case 1: return __longlong_as_double(static_cast<long long>(ld_u64_unaligned(p)));
    case 2: return static_cast<double>(static_cast<int32_t>(ld_u32_unaligned(p)));
    case 3: return static_cast<double>(ld_u32_unaligned(p));
    case 4: return static_cast<double>(static_cast<int8_t>(p[0]));
    case 5: return static_cast<double>(p[0]);
    case 6: return static_cast<double>(static_cast<int16_t>(p[0] | (p[1] << 8)));
    default: return static_cast<double>(static_cast<uint16_t>(p[0] | (p[1] << 8)));
  }
}

__global__ void k_ply_vertices(const uint8_t* __restrict__ body, PlyLayout L, double* __restrict__ V) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= L.nvert) return;
  const uint8_t* r = body + L.vbase + L.vstride * i;
  V[3 * i] = ply_scalar(r + L.xo, L.xt);
  V[3 * i + 1] = ply_scalar(r + L.yo, L.yt);
  V[3 * i + 2] = ply_scalar(r + L.zo, L.zt);
}

__global__ void k_ply_faces(const uint8_t* __restrict__ body, PlyLayout L, int32_t* __restrict__ tri,
                            unsigned long long* __restrict__ bad) {
  const int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (f >= L.nface) return;
  const uint8_t* r = body + L.fbase + L.fstride * f;
  const double cnt = ply_scalar(r + L.co, L.ct);
  if (cnt != 3.0) atomicOr(bad, 1ull);  // not the fixed-size triangle layout
  const int isz = (L.it == 1) ? 8 : (L.it >= 6 ? 2 : (L.it >= 4 ? 1 : 4));
  for (int k = 0; k < 3; ++k) {
    const double v = ply_scalar(r + L.io + isz * k, L.it);
    if (!(v >= 0.0 && v < static_cast<double>(L.nvert))) atomicOr(bad, 2ull);  // index out of range
    tri[3 * f + k] = static_cast<int32_t>(v);
  }
}

// ------------------------------------------------------------------------ normalize
__global__ void k_bounds(const double* __restrict__ V, int64_t nv, unsigned long long* __restrict__ keys) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nv) return;
  for (int k = 0; k < 3; ++k) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(V[3 * i + k]));
    const unsigned long long key = (u >> 63) ? ~u : (u | 0x8000000000000000ull);  // order-preserving
    atomicMin(&keys[k], key);
    atomicMax(&keys[3 + k], key);
  }
}
__global__ void k_apply_transform(double* __restrict__ V, int64_t nv, double scale, double tx, double ty, double tz) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nv) return;
  V[3 * i] = V[3 * i] * scale + tx;
  V[3 * i + 1] = V[3 * i + 1] * scale + ty;
  V[3 * i + 2] = V[3 * i + 2] * scale + tz;
}

// NormalizationTransform::invert (mesh_io.hpp:35): (p - translation) / scale, per component
__global__ void k_invert_transform(double* __restrict__ V, int64_t nv, double scale, double tx, double ty, double tz) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nv) return;
  V[3 * i] = (V[3 * i] - tx) / scale;
  V[3 * i + 1] = (V[3 * i + 1] - ty) / scale;
  V[3 * i + 2] = (V[3 * i + 2] - tz) / scale;
}

double unkey(unsigned long long key) {
  const unsigned long long u = (key >> 63) ? (key & 0x7fffffffffffffffull) : ~key;
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}

// stable key/value radix sort (CUB) of n items
template <class K>
void sort_pairs_stable(Ctx& ctx, K* k, K* k2, uint32_t* v, uint32_t* v2, int64_t n) {
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, k, k2, v, v2, static_cast<int>(n), 0, static_cast<int>(8 * sizeof(K)),
                                  ctx.stream);
  DevBuf<uint8_t> tmp(need ? need : 1, ctx.stream);
  PCU_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), need, k, k2, v, v2, static_cast<int>(n), 0,
                                           static_cast<int>(8 * sizeof(K)), ctx.stream));
  ++ctx.launches;
}

// triangles (with possible repeats) -> the kept faces
void finish_faces(Ctx& ctx, DevBuf<int32_t>& tri, int64_t nf, IngestResult& out) {
  DevBuf<uint32_t> keep(nf ? nf : 1, ctx.stream), pos(nf ? nf : 1, ctx.stream);
  int64_t nk = 0;
  if (nf) {
    PCU_LAUNCH(ctx, k_keep_faces, grid_for(nf, 256), 256, 0, tri.get(), nf, keep.get());
    exclusive_scan_u32(ctx, keep.get(), pos.get(), nf);
    nk = static_cast<int64_t>(read_scalar(ctx, pos.get() + nf - 1)) + read_scalar(ctx, keep.get() + nf - 1);
  }
  out.F.alloc(3 * (nk ? nk : 1), ctx.stream);
  if (nk) PCU_LAUNCH(ctx, k_compact_faces, grid_for(nf, 256), 256, 0, tri.get(), keep.get(), pos.get(), nf, out.F.get());
  out.nf = nk;
  out.degenerate_dropped = nf - nk;
}

}  // namespace

void load_stl_binary(Ctx& ctx, const uint8_t* d_bytes, int64_t nbytes, uint32_t count, IngestResult& out) {
  cudaStream_t st = ctx.stream;
  PCU_REQUIRE(nbytes >= 84 + 50 * static_cast<int64_t>(count), PAMOPT_CU_EINVAL,
              "load_stl: truncated binary stl (fewer than 84 + 50 * count bytes)");
  const int64_t nc = 3 * static_cast<int64_t>(count);
  out = IngestResult();
  if (nc == 0) {
    out.V.alloc(1, st);
    out.F.alloc(1, st);
    return;
  }
  DevBuf<uint32_t> kx(nc, st), kx2(nc, st), idx(nc, st), idx2(nc, st);
  DevBuf<uint64_t> kyz(nc, st), kyz2(nc, st);
  DevBuf<uint8_t> nan(nc, st);
  PCU_LAUNCH(ctx, k_stl_corners, grid_for(nc, 256), 256, 0, d_bytes, nc, kx.get(), kyz.get(), idx.get(), nan.get());
  // LSD: stable by (y, z), then stable by x  ->  sorted by (x, y, z), ties in corner order
  sort_pairs_stable<uint64_t>(ctx, kyz.get(), kyz2.get(), idx.get(), idx2.get(), nc);
  {  // gather x in the new order
    DevBuf<uint32_t> xs(nc, st);
    PCU_LAUNCH(ctx, k_gather_u32, grid_for(nc, 256), 256, 0, kx.get(), idx2.get(), nc, xs.get());
    sort_pairs_stable<uint32_t>(ctx, xs.get(), kx2.get(), idx2.get(), idx.get(), nc);
  }
  // after the second sort: kx2 = sorted x, idx = corner ids in (x, y, z) order; rebuild y/z keys
  PCU_LAUNCH(ctx, k_gather_u64, grid_for(nc, 256), 256, 0, kyz.get(), idx.get(), nc, kyz2.get());
  DevBuf<uint32_t> head(nc, st), gid(nc, st);
  PCU_LAUNCH(ctx, k_weld_heads, grid_for(nc, 256), 256, 0, kx2.get(), kyz2.get(), idx.get(), nan.get(), nc, head.get());
  exclusive_scan_u32(ctx, head.get(), gid.get(), nc);
  const int64_t ng = static_cast<int64_t>(read_scalar(ctx, gid.get() + nc - 1)) + read_scalar(ctx, head.get() + nc - 1);
  DevBuf<uint32_t> gfirst(ng, st), rep(nc, st), isfirst(nc, st), vpos(nc, st);
  PCU_LAUNCH(ctx, k_weld_rep, grid_for(nc, 256), 256, 0, idx.get(), head.get(), gid.get(), nc, gfirst.get());
  PCU_LAUNCH(ctx, k_weld_first, grid_for(nc, 256), 256, 0, idx.get(), head.get(), gid.get(), gfirst.get(), nc,
             rep.get(), isfirst.get());
  exclusive_scan_u32(ctx, isfirst.get(), vpos.get(), nc);
  out.nv = ng;
  out.V.alloc(3 * ng, st);
  DevBuf<int32_t> tri(nc, st);
  PCU_LAUNCH(ctx, k_weld_emit, grid_for(nc, 256), 256, 0, d_bytes, rep.get(), isfirst.get(), vpos.get(), nc,
             out.V.get(), tri.get());
  out.welded = nc - ng;
  finish_faces(ctx, tri, count, out);
}

bool load_ply_binary(Ctx& ctx, const uint8_t* d_bytes, const PlyBinaryLayout& H, IngestResult& out) {
  cudaStream_t st = ctx.stream;
  out = IngestResult();
  PlyLayout L{};
  L.vbase = H.vbase;
  L.vstride = H.vstride;
  L.nvert = H.nvert;
  L.xo = H.off[0];
  L.yo = H.off[1];
  L.zo = H.off[2];
  L.xt = H.type[0];
  L.yt = H.type[1];
  L.zt = H.type[2];
  L.fbase = H.fbase;
  L.fstride = H.fstride;
  L.nface = H.nface;
  L.co = H.count_off;
  L.ct = H.count_type;
  L.io = H.index_off;
  L.it = H.index_type;
  out.nv = H.nvert;
  out.V.alloc(3 * (H.nvert ? H.nvert : 1), st);
  if (H.nvert) PCU_LAUNCH(ctx, k_ply_vertices, grid_for(H.nvert, 256), 256, 0, d_bytes, L, out.V.get());
  DevBuf<int32_t> tri(3 * (H.nface ? H.nface : 1), st);
  DevBuf<unsigned long long> bad(1, st);
  PCU_CUDA(cudaMemsetAsync(bad.get(), 0, 8, st));
  if (H.nface) PCU_LAUNCH(ctx, k_ply_faces, grid_for(H.nface, 256), 256, 0, d_bytes, L, tri.get(), bad.get());
  const unsigned long long b = read_scalar(ctx, bad.get());
  if (b & 1ull) return false;  // a face list is not a triangle: variable records (host decoder)
  PCU_REQUIRE(!(b & 2ull), PAMOPT_CU_EIO, "load_ply: face index out of range");
  finish_faces(ctx, tri, H.nface, out);
  return true;
}

void normalize_unit_cube(Ctx& ctx, double* dV, int64_t nv, double padding, double* scale_translation) {
  PCU_REQUIRE(nv > 0, PAMOPT_CU_EINVAL, "normalize_unit_cube: empty mesh");
  PCU_REQUIRE(padding >= 0 && padding < 0.5, PAMOPT_CU_EINVAL, "normalize_unit_cube: padding must be in [0, 0.5)");
  DevBuf<unsigned long long> keys(6, ctx.stream);
  const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
  PCU_CUDA(cudaMemcpyAsync(keys.get(), init, sizeof(init), cudaMemcpyHostToDevice, ctx.stream));
  PCU_LAUNCH(ctx, k_bounds, grid_for(nv, 256), 256, 0, dV, nv, keys.get());
  unsigned long long h[6];
  PCU_CUDA(cudaMemcpyAsync(h, keys.get(), sizeof(h), cudaMemcpyDeviceToHost, ctx.stream));
  PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  double lo[3], hi[3], ext[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = unkey(h[k]);
    hi[k] = unkey(h[3 + k]);
    ext[k] = hi[k] - lo[k];
  }
  const double longest = std::max(std::max(ext[0], ext[1]), ext[2]);
  PCU_REQUIRE(longest > 0, PAMOPT_CU_EINVAL, "normalize_unit_cube: all vertices coincide");
  const double scale = (1.0 - 2.0 * padding) / longest;
  double t[3];
  for (int k = 0; k < 3; ++k) {
    const double center = 0.5 * (lo[k] + hi[k]);
    t[k] = 0.5 - center * scale;
  }
  PCU_LAUNCH(ctx, k_apply_transform, grid_for(nv, 256), 256, 0, dV, nv, scale, t[0], t[1], t[2]);
  if (scale_translation) {
    scale_translation[0] = scale;
    for (int k = 0; k < 3; ++k) scale_translation[1 + k] = t[k];
  }
}

void denormalize(Ctx& ctx, double* dV, int64_t nv, const double* st) {
  if (nv <= 0) return;
  PCU_REQUIRE(st[0] > 0.0, PAMOPT_CU_EINVAL, "denormalize: scale must be positive");
  PCU_LAUNCH(ctx, k_invert_transform, grid_for(nv, 256), 256, 0, dV, nv, st[0], st[1], st[2], st[3]);
}

}  // namespace pcu

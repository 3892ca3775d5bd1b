// capi.cu — the extern "C" boundary (include/pamopt_cu.h).  Translates C++ exceptions into
// status codes + a thread-local message, owns the device-resident handles, and hosts the
// CUB-backed scan/sort helpers shared by the modules.
#include <cub/cub.cuh>

#include <chrono>
#include <functional>
#include <cmath>
#include <limits>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <algorithm>
#include <vector>
#include <sstream>

#include "common.cuh"
#include "kernels.cuh"

#include <atomic>
#include <memory>
#include <mutex>

// Handles keep their context alive: pamopt_cu_ctx_destroy on a context that still owns meshes or
// grids only marks it; the last handle freed releases it (no use-after-free at teardown).  The
// refcount and the dead/released flags change under one mutex, so exactly one caller releases.
struct pamopt_cu_ctx_s {
  pcu::Ctx ctx;
  std::mutex mu;
  int refs = 0;
  bool dead = false, released = false;
};

static void ctx_release(pamopt_cu_ctx c) {
  pcu::DeviceGuard g(c->ctx.device);
  if (c->ctx.scratch) cudaFreeAsync(c->ctx.scratch, c->ctx.stream);
  cudaStreamSynchronize(c->ctx.stream);
  c->ctx.release_aux();
  if (c->ctx.pin) cudaFreeHost(c->ctx.pin);
  cudaStreamDestroy(c->ctx.stream);
  delete c;
}

static void ctx_ref(pamopt_cu_ctx c) {
  std::lock_guard<std::mutex> l(c->mu);
  ++c->refs;
}

static void ctx_unref(pamopt_cu_ctx c) {
  bool rel;
  {
    std::lock_guard<std::mutex> l(c->mu);
    rel = --c->refs == 0 && c->dead && !c->released;
    if (rel) c->released = true;
  }
  if (rel) ctx_release(c);
}

static void ctx_mark_dead(pamopt_cu_ctx c) {
  bool rel;
  {
    std::lock_guard<std::mutex> l(c->mu);
    c->dead = true;
    rel = c->refs == 0 && !c->released;
    if (rel) c->released = true;
  }
  if (rel) ctx_release(c);
}

struct pamopt_cu_mesh_s {
  pamopt_cu_ctx owner;
  pcu::DevBuf<double> V;
  pcu::DevBuf<int32_t> F;
  int64_t nv = 0, nf = 0;
};

struct pamopt_cu_grid_s {
  pamopt_cu_ctx owner;
  int32_t R = 0;
  int32_t z0 = 0, z1 = 0;  // lattice planes [z0, z1) held (a z-slab, or the whole grid)
  pcu::DevBuf<float> g;
  pcu::DevBuf<uint32_t> signs;  // DMC sign mask emitted with a whole-grid SDF (empty otherwise)
  pcu::DmcResult last;  // debug view of the last extract
};

namespace pcu {

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

template <class Fn>
static int guarded(Fn&& fn) {
  try {
    fn();
    return PAMOPT_CU_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PAMOPT_CU_ECUDA;
  }
}

// ------------------------------------------------------------------------- CUB helpers
static void* tmp_storage(Ctx& ctx, size_t bytes) {
  if (bytes > ctx.scratch_bytes) {
    if (ctx.scratch) cudaFreeAsync(ctx.scratch, ctx.stream);
    ctx.scratch_bytes = bytes + bytes / 2 + 4096;
    PCU_CUDA(cudaMallocAsync(&ctx.scratch, ctx.scratch_bytes, ctx.stream));
  }
  return ctx.scratch;
}

// Small scans (most of the QEM loop's late iterations): one CTA, 16 items per thread, replaces
// CUB's two-launch chain.  Integer sums, so the result equals CUB's bit for bit; each thread
// reads its items before the block barrier and writes only its own, so in == out is safe.
constexpr int kSmallScanItems = 16, kSmallScan = 1024 * kSmallScanItems;
__global__ void __launch_bounds__(1024) k_small_scan(const uint32_t* in, int n, uint32_t* out) {
  __shared__ uint32_t wsum[32];
  const int base = threadIdx.x * kSmallScanItems;
  uint32_t v[kSmallScanItems];
  uint32_t tot = 0;
#pragma unroll
  for (int k = 0; k < kSmallScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : 0u;
    tot += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = tot;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = wsum[lane], wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    wsum[lane] = wi - w;
  }
  __syncthreads();
  uint32_t run = wsum[warp] + incl - tot;
#pragma unroll
  for (int k = 0; k < kSmallScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

// Up to 4 small memsets in one launch (the QEM loop issues several per step; at small sizes each
// separate cudaMemsetAsync costs a launch).  Ranges are filled as 32-bit words with the byte
// value replicated, and a byte tail; ranges above 1 MB go to cudaMemsetAsync instead.
__global__ void k_fill_multi(FillRanges fr) {
  uint64_t total = 0;  // the flattened space: each range padded to whole words
  for (int r = 0; r < fr.n; ++r) total += (fr.r[r].bytes + 3) / 4 * 4;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i * 4 < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t off = i * 4;
    for (int r = 0; r < fr.n; ++r) {
      const FillRange& R = fr.r[r];
      const uint64_t words = (R.bytes + 3) / 4;
      if (off < words * 4) {
        uint8_t* p = static_cast<uint8_t*>(R.p) + off;
        const uint32_t v = 0x01010101u * R.byte;
        if (off + 4 <= R.bytes && (reinterpret_cast<uintptr_t>(p) & 3u) == 0) {
          *reinterpret_cast<uint32_t*>(p) = v;
        } else {
          for (uint64_t b = off; b < R.bytes && b < off + 4; ++b) static_cast<uint8_t*>(R.p)[b] = R.byte;
        }
        break;
      }
      off -= words * 4;
    }
  }
}

void fill_multi(Ctx& ctx, std::initializer_list<FillRange> ranges) { fill_multi(ctx, ranges.begin(), ranges.size()); }

void fill_multi(Ctx& ctx, const FillRange* ranges, size_t count) {
  FillRanges fr{};
  uint64_t total = 0;
  for (size_t i = 0; i < count; ++i) {
    const FillRange& r = ranges[i];
    if (!r.p || r.bytes == 0) continue;
    if (r.bytes > (1u << 20)) {  // large: the copy engine's memset runs at HBM rate
      PCU_CUDA(cudaMemsetAsync(r.p, r.byte, r.bytes, ctx.stream));
      continue;
    }
    PCU_REQUIRE(fr.n < kMaxFillRanges, PAMOPT_CU_EINVAL, "fill_multi: too many ranges");
    PCU_REQUIRE((reinterpret_cast<uintptr_t>(r.p) & 3u) == 0, PAMOPT_CU_EINVAL, "fill_multi: unaligned range");
    fr.r[fr.n++] = r;
    total += (r.bytes + 3) / 4;
  }
  if (fr.n == 0) return;
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, static_cast<uint64_t>(ctx.num_sms) * 16));
  PCU_LAUNCH(ctx, k_fill_multi, g, 256, 0, fr);
}

void exclusive_scan_u32(Ctx& ctx, const uint32_t* in, uint32_t* out, int64_t n) {
  if (n <= 0) return;
  if (n <= kSmallScan) {
    PCU_LAUNCH(ctx, k_small_scan, 1, 1024, 0, in, static_cast<int>(n), out);
    return;
  }
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, n, ctx.stream);
  void* t = tmp_storage(ctx, need);
  cudaEvent_t e = ctx.prof.kt ? ctx.prof.kbegin(ctx.stream) : nullptr;
  PCU_CUDA(cub::DeviceScan::ExclusiveSum(t, need, in, out, n, ctx.stream));
  if (e) ctx.prof.kend("cub_scan_u32", e, ctx.stream);
  ++ctx.launches;
}

void exclusive_scan_u64(Ctx& ctx, const uint64_t* in, uint64_t* out, int64_t n) {
  if (n <= 0) return;
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, n, ctx.stream);
  void* t = tmp_storage(ctx, need);
  PCU_CUDA(cub::DeviceScan::ExclusiveSum(t, need, in, out, n, ctx.stream));
  ++ctx.launches;
}

// Small sorts (the QEM loop's marked keys and invalid pairs late in a run): one CTA bitonic
// sort in shared memory replaces CUB's multi-kernel radix sort, whose fixed launch chain
// dominates at these sizes.  Keys are unique or ties are identical values, so the result equals
// any other correct ascending sort.
constexpr int kSmallSort = 4096;
__global__ void __launch_bounds__(1024) k_small_sort(const uint64_t* __restrict__ in, int n, uint64_t* __restrict__ out) {
  __shared__ uint64_t sh[kSmallSort];
  int N = 1;
  while (N < n) N <<= 1;
  for (int i = threadIdx.x; i < N; i += blockDim.x) sh[i] = i < n ? in[i] : ~0ull;
  __syncthreads();
  for (int k = 2; k <= N; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = sh[i], b = sh[ixj];
          if ((a > b) == ((i & k) == 0)) {
            sh[i] = b;
            sh[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = sh[i];
}

bool small_sort_u64(Ctx& ctx, const uint64_t* in, uint64_t* out, int64_t n) {
  if (n > kSmallSort) return false;
  if (n > 0) PCU_LAUNCH(ctx, k_small_sort, 1, 1024, 0, in, static_cast<int>(n), out);
  return true;
}

void sort_pairs_u64(Ctx& ctx, uint64_t* keys, int64_t n, int end_bit) {
  if (n <= 1) return;
  if (small_sort_u64(ctx, keys, keys, n)) return;
  DevBuf<uint64_t> alt(n, ctx.stream);
  cub::DoubleBuffer<uint64_t> db(keys, alt.get());
  size_t need = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, need, db, static_cast<int>(n), 0, end_bit, ctx.stream);
  void* t = tmp_storage(ctx, need);
  cudaEvent_t e = ctx.prof.kt ? ctx.prof.kbegin(ctx.stream) : nullptr;
  PCU_CUDA(cub::DeviceRadixSort::SortKeys(t, need, db, static_cast<int>(n), 0, end_bit, ctx.stream));
  if (e) ctx.prof.kend("cub_sort_pairs_u64", e, ctx.stream);
  ++ctx.launches;
  if (db.Current() != keys)
    PCU_CUDA(cudaMemcpyAsync(keys, db.Current(), n * 8, cudaMemcpyDeviceToDevice, ctx.stream));
}

}  // namespace pcu

using pcu::guarded;

static void check_ctx(pamopt_cu_ctx c) { PCU_REQUIRE(c != nullptr, PAMOPT_CU_EINVAL, "null context"); }

template <class T>
static void d2h(pcu::Ctx& ctx, T* dst, const T* src, int64_t n) {
  if (dst && n > 0) PCU_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, ctx.stream));
}

extern "C" {

const char* pamopt_cu_last_error(void) { return pcu::g_last_error.c_str(); }
const char* pamopt_cu_version(void) { return "pamopt_cu 0.1 (sm_100a)"; }

int pamopt_cu_ctx_create(int32_t device, pamopt_cu_ctx* out) {
  return guarded([&] {
    PCU_REQUIRE(out != nullptr, PAMOPT_CU_EINVAL, "null output");
    int n = 0;
    PCU_CUDA(cudaGetDeviceCount(&n));
    PCU_REQUIRE(device >= 0 && device < n, PAMOPT_CU_EINVAL, "no such CUDA device");
    auto* c = new pamopt_cu_ctx_s();
    c->ctx.device = device;
    const char* pe = std::getenv("PAMOPT_PROFILE");
    c->ctx.prof.on = pe && pe[0] == '1';
    c->ctx.prof.kt = c->ctx.prof.kt_print = pe && pe[0] == '2';
    pcu::DeviceGuard g(device);
    PCU_CUDA(cudaStreamCreateWithFlags(&c->ctx.stream, cudaStreamNonBlocking));
    PCU_CUDA(cudaDeviceGetAttribute(&c->ctx.num_sms, cudaDevAttrMultiProcessorCount, device));
    cudaMemPool_t pool;
    PCU_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = ~0ull;  // keep freed blocks cached in the pool
    PCU_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    *out = c;
  });
}

int pamopt_cu_ctx_destroy(pamopt_cu_ctx c) {
  return guarded([&] {
    if (!c) return;
    ctx_mark_dead(c);
  });
}

void* pamopt_cu_ctx_stream(pamopt_cu_ctx c) { return c ? static_cast<void*>(c->ctx.stream) : nullptr; }

int pamopt_cu_ctx_synchronize(pamopt_cu_ctx c) {
  return guarded([&] {
    check_ctx(c);
    PCU_CUDA(cudaStreamSynchronize(c->ctx.stream));
  });
}

int64_t pamopt_cu_ctx_launches(pamopt_cu_ctx c) { return c ? c->ctx.launches : 0; }

int pamopt_cu_ctx_profile(pamopt_cu_ctx c, int on) {
  return guarded([&] {
    check_ctx(c);
    pcu::DeviceGuard g(c->ctx.device);
    c->ctx.prof.kflush();
    c->ctx.prof.kms.clear();
    c->ctx.prof.kn.clear();
    c->ctx.prof.kt = on != 0;
  });
}

int64_t pamopt_cu_ctx_kernel_times(pamopt_cu_ctx c, char* buf, int64_t cap) {
  if (!c) return 0;
  pcu::DeviceGuard g(c->ctx.device);
  c->ctx.prof.kflush();
  std::string out;
  char line[256];
  for (auto& kv : c->ctx.prof.kms) {
    std::snprintf(line, sizeof(line), "%s\t%.6f\t%lld\n", kv.first.c_str(), kv.second,
                  static_cast<long long>(c->ctx.prof.kn[kv.first]));
    out += line;
  }
  if (buf && cap > 0) {
    const int64_t k = std::min<int64_t>(cap - 1, static_cast<int64_t>(out.size()));
    std::memcpy(buf, out.data(), k);
    buf[k] = 0;
  }
  return static_cast<int64_t>(out.size());
}

// ---------------------------------------------------------------------------- meshes
static int mesh_create(pamopt_cu_ctx c, const double* v, int64_t nv, const int32_t* f, int64_t nf,
                       cudaMemcpyKind kind, pamopt_cu_mesh* out) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(out && nv >= 0 && nf >= 0 && (nv == 0 || v) && (nf == 0 || f), PAMOPT_CU_EINVAL, "bad mesh arguments");
    pcu::DeviceGuard g(c->ctx.device);
    std::unique_ptr<pamopt_cu_mesh_s> m(new pamopt_cu_mesh_s());  // freed (with its buffers) on a throw
    m->nv = nv;
    m->nf = nf;
    m->V.alloc(3 * (nv ? nv : 1), c->ctx.stream);
    m->F.alloc(3 * (nf ? nf : 1), c->ctx.stream);
    if (nv) PCU_CUDA(cudaMemcpyAsync(m->V.get(), v, 3 * nv * sizeof(double), kind, c->ctx.stream));
    if (nf) PCU_CUDA(cudaMemcpyAsync(m->F.get(), f, 3 * nf * sizeof(int32_t), kind, c->ctx.stream));
    m->owner = c;
    ctx_ref(c);
    *out = m.release();
  });
}

int pamopt_cu_mesh_upload(pamopt_cu_ctx c, const double* v, int64_t nv, const int32_t* f, int64_t nf,
                          pamopt_cu_mesh* out) {
  return mesh_create(c, v, nv, f, nf, cudaMemcpyHostToDevice, out);
}

int pamopt_cu_mesh_from_device(pamopt_cu_ctx c, const double* v, int64_t nv, const int32_t* f, int64_t nf,
                               pamopt_cu_mesh* out) {
  return mesh_create(c, v, nv, f, nf, cudaMemcpyDeviceToDevice, out);
}

int pamopt_cu_mesh_size(pamopt_cu_mesh m, int64_t* nv, int64_t* nf) {
  return guarded([&] {
    PCU_REQUIRE(m != nullptr, PAMOPT_CU_EINVAL, "null mesh");
    if (nv) *nv = m->nv;
    if (nf) *nf = m->nf;
  });
}

int pamopt_cu_mesh_download(pamopt_cu_mesh m, double* v, int32_t* f) {
  return guarded([&] {
    PCU_REQUIRE(m != nullptr, PAMOPT_CU_EINVAL, "null mesh");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    if (v && m->nv) PCU_CUDA(cudaMemcpyAsync(v, m->V.get(), 3 * m->nv * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    if (f && m->nf) PCU_CUDA(cudaMemcpyAsync(f, m->F.get(), 3 * m->nf * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx.stream));
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

int pamopt_cu_mesh_copy_to_device(pamopt_cu_mesh m, double* v, int32_t* f) {
  return guarded([&] {
    PCU_REQUIRE(m != nullptr, PAMOPT_CU_EINVAL, "null mesh");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    if (v && m->nv)
      PCU_CUDA(cudaMemcpyAsync(v, m->V.get(), 3 * m->nv * sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
    if (f && m->nf)
      PCU_CUDA(cudaMemcpyAsync(f, m->F.get(), 3 * m->nf * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx.stream));
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

int pamopt_cu_mesh_free(pamopt_cu_mesh m) {
  return guarded([&] {
    if (!m) return;
    pamopt_cu_ctx c = m->owner;
    {
      pcu::DeviceGuard g(c->ctx.device);
      delete m;
    }
    ctx_unref(c);
  });
}

// ---------------------------------------------------------------------------- stage 1a
static void check_indices(pcu::Ctx& ctx, const pamopt_cu_mesh_s* m) {
  if (m->nf == 0) return;
  const std::vector<int32_t> mm = pcu::index_range(ctx, m->F.get(), 3 * m->nf);
  PCU_REQUIRE(mm[0] >= 0 && mm[1] < m->nv, PAMOPT_CU_EINVAL, "invalid mesh: face index out of range");
}

// IndexedMesh::validate (mesh.cpp:31-43, thrown as std::invalid_argument at mesh.cpp:186-187):
// every hot-path entry rejects out-of-range and repeated face indices before any kernel reads them
static void validate(pcu::Ctx& ctx, const pamopt_cu_mesh_s* m) { pcu::validate_mesh(ctx, m->F.get(), m->nf, m->nv); }

static void check_R(int32_t R) {
  PCU_REQUIRE(R >= 8 && R <= 1024 && (R & (R - 1)) == 0, PAMOPT_CU_EINVAL, "R must be a power of two in [8, 1024] (DMC cell ids are 32-bit)");
}

static int make_grid(pamopt_cu_ctx c, pamopt_cu_mesh m, int32_t R, int mode, double eps, pamopt_cu_grid* out,
                     int32_t z0 = 0, int32_t z1 = -1) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(m && out, PAMOPT_CU_EINVAL, "null argument");
    check_R(R);
    if (mode == 1) {
      const double lo = 0.8660254037844386 / R, hi = 3.0 / R - 0.8660254037844386 / R;
      PCU_REQUIRE(eps >= lo && eps <= hi, PAMOPT_CU_EINVAL, "udf_to_sdf: epsilon out of range");
    }
    pcu::DeviceGuard g(c->ctx.device);
    if (z1 < 0) z1 = R + 1;
    PCU_REQUIRE(z0 >= 0 && z0 < z1 && z1 <= R + 1, PAMOPT_CU_EINVAL, "bad slab plane range");
    PCU_REQUIRE(m->owner == c, PAMOPT_CU_EINVAL, "mesh belongs to another context");
    validate(c->ctx, m);
    auto* gr = new pamopt_cu_grid_s();
    gr->owner = c;
    ctx_ref(c);
    gr->R = R;
    gr->z0 = z0;
    gr->z1 = z1;
    const int64_t n1 = R + 1;
    try {
      gr->g.alloc(n1 * n1 * (z1 - z0), c->ctx.stream);
      uint32_t* sg = nullptr;
      if (mode == 1 && z0 == 0 && z1 == R + 1) {  // whole-grid SDF: emit the DMC sign mask too
        gr->signs.alloc(n1 * n1 * ((n1 + 31) / 32), c->ctx.stream);
        sg = gr->signs.get();
      }
      pcu::udf_run(c->ctx, m->V.get(), m->nv, m->F.get(), m->nf, R, mode, eps, gr->g.get(), z0, z1, sg);
    } catch (...) {
      delete gr;
      ctx_unref(c);
      throw;
    }
    *out = gr;
  });
}

int pamopt_cu_compute_udf(pamopt_cu_ctx c, pamopt_cu_mesh m, int32_t R, pamopt_cu_grid* out) {
  return make_grid(c, m, R, 0, 0.0, out);
}

int pamopt_cu_compute_sdf(pamopt_cu_ctx c, pamopt_cu_mesh m, int32_t R, double eps, pamopt_cu_grid* out) {
  return make_grid(c, m, R, 1, eps, out);
}

int pamopt_cu_compute_sdf_slab(pamopt_cu_ctx c, pamopt_cu_mesh m, int32_t R, double eps, int32_t z0, int32_t z1,
                               pamopt_cu_grid* out) {
  return make_grid(c, m, R, 1, eps, out, z0, z1);
}

int pamopt_cu_grid_slab(pamopt_cu_grid gr, int32_t* z0, int32_t* z1) {
  return guarded([&] {
    PCU_REQUIRE(gr != nullptr, PAMOPT_CU_EINVAL, "null grid");
    if (z0) *z0 = gr->z0;
    if (z1) *z1 = gr->z1;
  });
}

int pamopt_cu_grid_copy_to_device(pamopt_cu_grid gr, void* dst) {
  return guarded([&] {
    PCU_REQUIRE(gr && dst, PAMOPT_CU_EINVAL, "null argument");
    pcu::Ctx& ctx = gr->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    const int64_t n1 = gr->R + 1;
    PCU_CUDA(cudaMemcpyAsync(dst, gr->g.get(), n1 * n1 * (gr->z1 - gr->z0) * sizeof(float), cudaMemcpyDeviceToDevice,
                             ctx.stream));
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

int pamopt_cu_grid_from_device(pamopt_cu_ctx c, int32_t R, const float* src, pamopt_cu_grid* out) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(R >= 8 && R <= 1024 && (R & (R - 1)) == 0 && src && out, PAMOPT_CU_EINVAL, "bad arguments (R: power of two in [8, 1024])");
    pcu::DeviceGuard g(c->ctx.device);
    auto* gr = new pamopt_cu_grid_s();
    gr->owner = c;
    ctx_ref(c);
    gr->R = R;
    gr->z0 = 0;
    gr->z1 = R + 1;
    const int64_t n1 = R + 1;
    gr->g.alloc(n1 * n1 * n1, c->ctx.stream);
    PCU_CUDA(cudaMemcpyAsync(gr->g.get(), src, n1 * n1 * n1 * sizeof(float), cudaMemcpyDeviceToDevice, c->ctx.stream));
    *out = gr;
  });
}

static int grid_slab_make(pamopt_cu_ctx c, int32_t R, int32_t z0, int32_t z1, const float* src, cudaMemcpyKind kind,
                          pamopt_cu_grid* out) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(R >= 8 && R <= 1024 && (R & (R - 1)) == 0 && src && out, PAMOPT_CU_EINVAL, "bad arguments (R: power of two in [8, 1024])");
    PCU_REQUIRE(0 <= z0 && z0 < z1 && z1 <= R + 1, PAMOPT_CU_EINVAL, "slab planes must satisfy 0 <= z0 < z1 <= R+1");
    pcu::DeviceGuard g(c->ctx.device);
    auto* gr = new pamopt_cu_grid_s();
    gr->owner = c;
    ctx_ref(c);
    gr->R = R;
    gr->z0 = z0;
    gr->z1 = z1;
    const int64_t n = static_cast<int64_t>(R + 1) * (R + 1) * (z1 - z0);
    gr->g.alloc(n, c->ctx.stream);
    PCU_CUDA(cudaMemcpyAsync(gr->g.get(), src, n * sizeof(float), kind, c->ctx.stream));
    if (kind == cudaMemcpyHostToDevice) PCU_CUDA(cudaStreamSynchronize(c->ctx.stream));
    *out = gr;
  });
}

int pamopt_cu_grid_slab_from_device(pamopt_cu_ctx c, int32_t R, int32_t z0, int32_t z1, const float* src,
                                    pamopt_cu_grid* out) {
  return grid_slab_make(c, R, z0, z1, src, cudaMemcpyDeviceToDevice, out);
}

int pamopt_cu_grid_slab_upload(pamopt_cu_ctx c, int32_t R, int32_t z0, int32_t z1, const float* samples,
                               pamopt_cu_grid* out) {
  return grid_slab_make(c, R, z0, z1, samples, cudaMemcpyHostToDevice, out);
}

// ------------------------------------------------------------------------------ ingest
static pamopt_cu_mesh mesh_from_ingest(pamopt_cu_ctx c, pcu::IngestResult& r) {
  auto* m = new pamopt_cu_mesh_s();
  m->owner = c;
  ctx_ref(c);
  m->nv = r.nv;
  m->nf = r.nf;
  m->V = std::move(r.V);
  m->F = std::move(r.F);
  return m;
}

int pamopt_cu_load_stl(pamopt_cu_ctx c, const void* bytes, int64_t nbytes, pamopt_cu_mesh* out,
                       pamopt_cu_load_stats* stats) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(bytes && out && nbytes >= 0, PAMOPT_CU_EINVAL, "null argument");
    const char* b = static_cast<const char*>(bytes);
    pcu::DeviceGuard g(c->ctx.device);
    pcu::IngestResult r;
    // a binary file can also start with "solid": ASCII only if "facet" appears (mesh_io.cpp:316-320)
    const bool ascii = nbytes >= 5 && std::strncmp(b, "solid", 5) == 0 &&
                       std::string_view(b, static_cast<size_t>(nbytes)).find("facet") != std::string_view::npos;
    if (ascii) {
      pcu::load_stl_ascii(c->ctx, b, nbytes, r);
    } else {
      PCU_REQUIRE(nbytes >= 84, PAMOPT_CU_EIO, "load_stl: truncated binary stl header");
      uint32_t count = 0;
      std::memcpy(&count, b + 80, 4);
      PCU_REQUIRE(nbytes >= 84 + 50 * static_cast<int64_t>(count), PAMOPT_CU_EIO,
                  "load_stl: truncated binary stl (fewer than 84 + 50 * count bytes)");
      pcu::DevBuf<uint8_t> d(static_cast<size_t>(nbytes), c->ctx.stream);
      PCU_CUDA(cudaMemcpyAsync(d.get(), bytes, static_cast<size_t>(nbytes), cudaMemcpyHostToDevice, c->ctx.stream));
      pcu::load_stl_binary(c->ctx, d.get(), nbytes, count, r);
    }
    PCU_REQUIRE(r.nf > 0, PAMOPT_CU_EIO, "load_stl: empty mesh (no faces)");
    if (stats) *stats = pamopt_cu_load_stats{r.degenerate_dropped, 0, r.welded};
    *out = mesh_from_ingest(c, r);
  });
}

int pamopt_cu_load_obj(pamopt_cu_ctx c, const void* bytes, int64_t nbytes, pamopt_cu_mesh* out,
                       pamopt_cu_load_stats* stats) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(bytes && out && nbytes >= 0, PAMOPT_CU_EINVAL, "null argument");
    pcu::DeviceGuard g(c->ctx.device);
    pcu::IngestResult r;
    int64_t tri = 0;
    pcu::load_obj_text(c->ctx, static_cast<const char*>(bytes), nbytes, r, &tri);
    PCU_REQUIRE(r.nf > 0, PAMOPT_CU_EIO, "load_obj: empty mesh (no faces)");
    if (stats) *stats = pamopt_cu_load_stats{r.degenerate_dropped, tri, 0};
    *out = mesh_from_ingest(c, r);
  });
}

// PLY header (mesh_io.cpp:141-185) -> fixed-size body layout for the GPU decoder
static pcu::PlyBinaryLayout ply_layout(const char* b, int64_t n, int64_t& body) {
  auto type_of = [](const std::string& t, int& code) -> int {
    if (t == "float" || t == "float32") { code = 0; return 4; }
    if (t == "double" || t == "float64") { code = 1; return 8; }
    if (t == "int" || t == "int32") { code = 2; return 4; }
    if (t == "uint" || t == "uint32") { code = 3; return 4; }
    if (t == "char" || t == "int8") { code = 4; return 1; }
    if (t == "uchar" || t == "uint8") { code = 5; return 1; }
    if (t == "short" || t == "int16") { code = 6; return 2; }
    if (t == "ushort" || t == "uint16") { code = 7; return 2; }
    throw pcu::Error(PAMOPT_CU_EINVAL, "load_ply: unknown ply type " + t);
  };
  const std::string text(b, static_cast<size_t>(std::min<int64_t>(n, 1 << 16)));
  const size_t eh = text.find("end_header");
  PCU_REQUIRE(text.compare(0, 3, "ply") == 0 && eh != std::string::npos, PAMOPT_CU_EINVAL,
              "load_ply: missing ply magic or end_header");
  const size_t nl = text.find('\n', eh);
  PCU_REQUIRE(nl != std::string::npos, PAMOPT_CU_EINVAL, "load_ply: truncated header");
  body = static_cast<int64_t>(nl + 1);
  struct Prop { std::string name; int code = 0, size = 0; bool list = false; int ccode = 0, csize = 0; };
  struct Elem { std::string name; int64_t count = 0; std::vector<Prop> props; };
  std::vector<Elem> els;
  std::string format;
  size_t pos = text.find('\n') + 1;
  while (pos < eh) {
    size_t e = text.find('\n', pos);
    std::string line = text.substr(pos, e - pos);
    pos = e + 1;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::istringstream ss(line);
    std::string tag;
    ss >> tag;
    if (tag == "format") {
      ss >> format;
    } else if (tag == "element") {
      Elem el;
      ss >> el.name >> el.count;
      els.push_back(el);
    } else if (tag == "property") {
      PCU_REQUIRE(!els.empty(), PAMOPT_CU_EINVAL, "load_ply: property before element");
      Prop p;
      std::string t;
      ss >> t;
      if (t == "list") {
        std::string ct, it;
        ss >> ct >> it >> p.name;
        p.list = true;
        p.csize = type_of(ct, p.ccode);
        p.size = type_of(it, p.code);
      } else {
        p.size = type_of(t, p.code);
        ss >> p.name;
      }
      els.back().props.push_back(p);
    }
  }
  PCU_REQUIRE(format == "binary_little_endian", PAMOPT_CU_EINVAL,
              "load_ply: only binary_little_endian bodies are decoded on the GPU (ascii: host loader)");
  pcu::PlyBinaryLayout L;
  int64_t off = body;
  bool have_v = false, have_f = false;
  for (const Elem& el : els) {
    int64_t stride = 0;
    int list_props = 0;
    for (const Prop& p : el.props) {
      if (p.list) {
        ++list_props;
        stride += p.csize + 3 * p.size;  // fixed 3-entry lists (verified on the GPU)
      } else {
        stride += p.size;
      }
    }
    if (el.name == "vertex") {
      PCU_REQUIRE(list_props == 0, PAMOPT_CU_EINVAL, "load_ply: list property in the vertex element");
      int64_t o = 0;
      int found = 0;
      for (const Prop& p : el.props) {
        const int k = p.name == "x" ? 0 : (p.name == "y" ? 1 : (p.name == "z" ? 2 : -1));
        if (k >= 0) {
          L.off[k] = static_cast<int>(o);
          L.type[k] = p.code;
          found |= 1 << k;
        }
        o += p.size;
      }
      PCU_REQUIRE(found == 7, PAMOPT_CU_EINVAL, "load_ply: vertex element lacks x/y/z");
      L.vbase = off;
      L.vstride = stride;
      L.nvert = el.count;
      have_v = true;
    } else if (el.name == "face") {
      PCU_REQUIRE(have_v, PAMOPT_CU_EINVAL, "load_ply: face element before the vertex element");
      PCU_REQUIRE(list_props == 1, PAMOPT_CU_EINVAL, "load_ply: face element needs exactly one list property");
      int64_t o = 0;
      for (const Prop& p : el.props) {
        if (p.list) {
          L.count_off = static_cast<int>(o);
          L.count_type = p.ccode;
          L.index_off = static_cast<int>(o + p.csize);
          L.index_type = p.code;
          o += p.csize + 3 * p.size;
        } else {
          o += p.size;
        }
      }
      L.fbase = off;
      L.fstride = stride;
      L.nface = el.count;
      have_f = true;
    } else {
      PCU_REQUIRE(list_props == 0 || have_f, PAMOPT_CU_EINVAL,
                  "load_ply: variable-size element before the faces (host loader)");
    }
    if (list_props == 0 || el.name == "face") off += stride * el.count;
  }
  PCU_REQUIRE(have_v, PAMOPT_CU_EINVAL, "load_ply: no vertex element");
  PCU_REQUIRE(!have_f || L.fbase + L.fstride * L.nface <= n, PAMOPT_CU_EINVAL, "load_ply: truncated binary body");
  PCU_REQUIRE(L.vbase + L.vstride * L.nvert <= n, PAMOPT_CU_EINVAL, "load_ply: truncated binary body");
  return L;
}

int pamopt_cu_load_ply(pamopt_cu_ctx c, const void* bytes, int64_t nbytes, pamopt_cu_mesh* out,
                       pamopt_cu_load_stats* stats) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(bytes && out && nbytes > 0, PAMOPT_CU_EINVAL, "null argument");
    const char* b = static_cast<const char*>(bytes);
    pcu::DeviceGuard g(c->ctx.device);
    pcu::IngestResult r;
    int64_t tri = 0;
    // fixed-size binary records (the reference writer's layout): decoded on the GPU; ASCII bodies
    // and variable-length face lists: the host decoder, record by record as mesh_io.cpp:186-244
    bool fixed = false;
    pcu::PlyBinaryLayout L;
    int64_t body = 0;
    try {
      L = ply_layout(b, nbytes, body);
      fixed = true;
    } catch (const pcu::Error&) {
      fixed = false;
    }
    if (fixed) {
      pcu::DevBuf<uint8_t> d(static_cast<size_t>(nbytes), c->ctx.stream);
      PCU_CUDA(cudaMemcpyAsync(d.get(), bytes, static_cast<size_t>(nbytes), cudaMemcpyHostToDevice, c->ctx.stream));
      fixed = pcu::load_ply_binary(c->ctx, d.get(), L, r);  // false: a face list is not a triangle
    }
    if (!fixed) pcu::load_ply_host(c->ctx, b, nbytes, r, &tri);
    PCU_REQUIRE(r.nf > 0, PAMOPT_CU_EIO, "load_ply: empty mesh (no faces)");
    if (stats) *stats = pamopt_cu_load_stats{r.degenerate_dropped, tri, 0};
    *out = mesh_from_ingest(c, r);
  });
}

int pamopt_cu_normalize_unit_cube(pamopt_cu_mesh m, double padding, double* st) {
  return guarded([&] {
    PCU_REQUIRE(m != nullptr, PAMOPT_CU_EINVAL, "null mesh");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    pcu::normalize_unit_cube(ctx, m->V.get(), m->nv, padding, st);
  });
}

int pamopt_cu_denormalize(pamopt_cu_mesh m, const double* st) {
  return guarded([&] {
    PCU_REQUIRE(m && st, PAMOPT_CU_EINVAL, "null argument");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    pcu::denormalize(ctx, m->V.get(), m->nv, st);
  });
}

int pamopt_cu_udf_to_sdf(pamopt_cu_grid gr, double eps) {
  return guarded([&] {
    PCU_REQUIRE(gr != nullptr, PAMOPT_CU_EINVAL, "null grid");
    const int R = gr->R;
    const double lo = 0.8660254037844386 / R, hi = 3.0 / R - 0.8660254037844386 / R;
    PCU_REQUIRE(eps >= lo && eps <= hi, PAMOPT_CU_EINVAL, "udf_to_sdf: epsilon out of range");
    pcu::Ctx& ctx = gr->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    const int64_t n1 = R + 1;
    pcu::udf_to_sdf_inplace(ctx, gr->g.get(), n1 * n1 * (gr->z1 - gr->z0), eps);
    gr->signs.release();  // the samples changed: the DMC repacks its mask
  });
}

int pamopt_cu_grid_upload(pamopt_cu_ctx c, int32_t R, const float* samples, pamopt_cu_grid* out) {
  return guarded([&] {
    check_ctx(c);
    check_R(R);
    PCU_REQUIRE(samples && out, PAMOPT_CU_EINVAL, "null argument");
    pcu::DeviceGuard g(c->ctx.device);
    auto* gr = new pamopt_cu_grid_s();
    gr->owner = c;
    ctx_ref(c);
    gr->R = R;
    gr->z0 = 0;
    gr->z1 = R + 1;
    const int64_t n1 = R + 1;
    gr->g.alloc(n1 * n1 * n1, c->ctx.stream);
    PCU_CUDA(cudaMemcpyAsync(gr->g.get(), samples, n1 * n1 * n1 * sizeof(float), cudaMemcpyHostToDevice, c->ctx.stream));
    *out = gr;
  });
}

int pamopt_cu_grid_resolution(pamopt_cu_grid gr, int32_t* R) {
  return guarded([&] {
    PCU_REQUIRE(gr && R, PAMOPT_CU_EINVAL, "null argument");
    *R = gr->R;
  });
}

int pamopt_cu_grid_download(pamopt_cu_grid gr, float* samples) {
  return guarded([&] {
    PCU_REQUIRE(gr && samples, PAMOPT_CU_EINVAL, "null argument");
    pcu::Ctx& ctx = gr->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    const int64_t n1 = gr->R + 1;
    PCU_CUDA(cudaMemcpyAsync(samples, gr->g.get(), n1 * n1 * (gr->z1 - gr->z0) * sizeof(float), cudaMemcpyDeviceToHost,
                             ctx.stream));
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

int pamopt_cu_grid_free(pamopt_cu_grid gr) {
  return guarded([&] {
    if (!gr) return;
    pamopt_cu_ctx c = gr->owner;
    {
      pcu::DeviceGuard g(c->ctx.device);
      delete gr;
    }
    ctx_unref(c);
  });
}

int pamopt_cu_hierarchy_pairs(pamopt_cu_ctx c, pamopt_cu_mesh m, int32_t R, int32_t r, int64_t* pairs, int64_t cap,
                              int64_t* n) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(m && n, PAMOPT_CU_EINVAL, "null argument");
    pcu::DeviceGuard g(c->ctx.device);
    validate(c->ctx, m);
    const std::vector<int64_t> h = pcu::hierarchy_pairs(c->ctx, m->V.get(), m->F.get(), m->nf, R, r);
    *n = static_cast<int64_t>(h.size() / 2);
    if (pairs) std::memcpy(pairs, h.data(), std::min<int64_t>(cap, *n) * 2 * sizeof(int64_t));
  });
}

// ---------------------------------------------------------------------------- stage 1b
int pamopt_cu_dmc_extract(pamopt_cu_grid gr, double beta, pamopt_cu_mesh* out) {
  return guarded([&] {
    PCU_REQUIRE(gr && out, PAMOPT_CU_EINVAL, "null argument");
    PCU_REQUIRE(beta > 0.0, PAMOPT_CU_EINVAL, "beta must be positive");
    PCU_REQUIRE(gr->z0 == 0 && gr->z1 == gr->R + 1, PAMOPT_CU_EINVAL, "extract: the grid is a z-slab; assemble it first");
    pcu::Ctx& ctx = gr->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    gr->last = pcu::DmcResult();
    pcu::dmc_extract(ctx, gr->g.get(), gr->R, beta, gr->last, gr->signs.get());
    auto* m = new pamopt_cu_mesh_s();
    m->owner = gr->owner;
    ctx_ref(gr->owner);
    m->nv = static_cast<int64_t>(gr->last.nv);
    m->nf = static_cast<int64_t>(gr->last.nf);
    m->V = std::move(gr->last.V);
    m->F = std::move(gr->last.F);
    *out = m;
  });
}

int pamopt_cu_dmc_extract_slab(pamopt_cu_grid gr, int32_t own_z0, int32_t own_z1, double beta, pamopt_cu_mesh* out,
                               int64_t counts[2]) {
  return guarded([&] {
    PCU_REQUIRE(gr && out && counts, PAMOPT_CU_EINVAL, "null argument");
    PCU_REQUIRE(beta > 0.0, PAMOPT_CU_EINVAL, "beta must be positive");
    pcu::Ctx& ctx = gr->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    gr->last = pcu::DmcResult();
    pcu::dmc_extract_slab(ctx, gr->g.get(), gr->R, gr->z0, gr->z1, own_z0, own_z1, beta, gr->last);
    auto* m = new pamopt_cu_mesh_s();
    m->owner = gr->owner;
    ctx_ref(gr->owner);
    m->nv = static_cast<int64_t>(gr->last.nv);
    m->nf = static_cast<int64_t>(gr->last.nf);
    m->V = std::move(gr->last.V);
    m->F = std::move(gr->last.F);
    counts[0] = static_cast<int64_t>(gr->last.nvp_own);
    counts[1] = static_cast<int64_t>(gr->last.n_extra);
    *out = m;
  });
}

int pamopt_cu_extract_slab_nccl(pamopt_cu_ctx c, pamopt_cu_mesh m, int32_t R, double eps, double beta, int32_t rank,
                                int32_t world, void* comm, pamopt_cu_mesh* out, int64_t counts[3]) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(m && out && counts, PAMOPT_CU_EINVAL, "null argument");
    PCU_REQUIRE(m->owner == c, PAMOPT_CU_EINVAL, "mesh belongs to another context");
    check_R(R);
    const double lo = 0.8660254037844386 / R, hi = 3.0 / R - 0.8660254037844386 / R;
    PCU_REQUIRE(eps >= lo && eps <= hi, PAMOPT_CU_EINVAL, "udf_to_sdf: epsilon out of range");
    PCU_REQUIRE(beta > 0.0, PAMOPT_CU_EINVAL, "beta must be positive");
    pcu::Ctx& ctx = c->ctx;
    pcu::DeviceGuard g(ctx.device);
    validate(ctx, m);
    *out = nullptr;
    std::unique_ptr<pamopt_cu_mesh_s> r(new pamopt_cu_mesh_s());
    pcu::slab_extract_nccl(ctx, m->V.get(), m->nv, m->F.get(), m->nf, R, eps, beta, rank, world, comm, r->V, r->F, r->nv,
                           r->nf, counts);
    if (rank != 0) return;
    r->owner = c;
    ctx_ref(c);
    *out = r.release();
  });
}

int pamopt_cu_nccl_comm_init_all(int32_t ndev, const int32_t* devs, void** comms) {
  return guarded([&] {
    PCU_REQUIRE(ndev >= 1 && devs && comms, PAMOPT_CU_EINVAL, "bad arguments");
    pcu::nccl_comm_init_all(ndev, devs, comms);
  });
}

int pamopt_cu_nccl_comm_destroy(void* comm) {
  return guarded([&] { pcu::nccl_comm_destroy(comm); });
}

int pamopt_cu_mesh_rebase(pamopt_cu_mesh m, int64_t patch_base, int64_t nvp_own, int64_t extra_base) {
  return guarded([&] {
    PCU_REQUIRE(m != nullptr, PAMOPT_CU_EINVAL, "null mesh");
    PCU_REQUIRE(patch_base >= 0 && nvp_own >= 0 && extra_base >= 0 && extra_base < (int64_t(1) << 31),
                PAMOPT_CU_EINVAL, "rebase: bad offsets");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    pcu::mesh_rebase(ctx, m->F.get(), 3 * m->nf, patch_base, nvp_own, extra_base);
  });
}

// ------------------------------------------------------------ certification / metrics
static constexpr uint64_t kSeedB = 0x632BE59BD9B4E019ull;


int pamopt_cu_analyze_topology(pamopt_cu_mesh m, pamopt_cu_topology* out, int32_t* edges, int64_t cap_e,
                               int32_t* verts, int64_t cap_v) {
  return guarded([&] {
    PCU_REQUIRE(m && out, PAMOPT_CU_EINVAL, "null argument");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    check_indices(ctx, m);
    pcu::TopologyResult t;
    pcu::analyze_topology(ctx, m->F.get(), m->nf, m->nv, t);
    out->manifold = t.manifold;
    out->watertight = t.watertight;
    out->euler_characteristic = t.euler;
    out->boundary_edge_count = t.boundary;
    out->n_nonmanifold_edges = static_cast<int64_t>(t.nm_edges.size());
    out->n_nonmanifold_vertices = static_cast<int64_t>(t.nm_verts.size());
    if (edges)
      for (int64_t i = 0; i < std::min<int64_t>(cap_e, out->n_nonmanifold_edges); ++i) {
        edges[2 * i] = static_cast<int32_t>(t.nm_edges[i] >> 32);
        edges[2 * i + 1] = static_cast<int32_t>(t.nm_edges[i] & 0xffffffffu);
      }
    if (verts)
      for (int64_t i = 0; i < std::min<int64_t>(cap_v, out->n_nonmanifold_vertices); ++i) verts[i] = t.nm_verts[i];
  });
}

int pamopt_cu_nearest_primitive(pamopt_cu_mesh m, const double* pts, int64_t n, int32_t* face, double* dist,
                                double* closest) {
  return guarded([&] {
    PCU_REQUIRE(m && (n == 0 || pts) && n >= 0, PAMOPT_CU_EINVAL, "bad arguments");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    if (n == 0) return;
    if (m->nf == 0) {  // empty tree: primitive -1, distance +INF (lbvh.cpp:194-197)
      for (int64_t i = 0; i < n; ++i) {
        if (face) face[i] = -1;
        if (dist) dist[i] = std::numeric_limits<double>::infinity();
        if (closest) closest[3 * i] = closest[3 * i + 1] = closest[3 * i + 2] = 0.0;
      }
      return;
    }
    check_indices(ctx, m);
    pcu::DevBuf<double> dp(3 * n, ctx.stream), d2(n, ctx.stream), dc(3 * n, ctx.stream);
    pcu::DevBuf<int32_t> df(n, ctx.stream);
    PCU_CUDA(cudaMemcpyAsync(dp.get(), pts, 3 * n * sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
    pcu::nearest_primitive(ctx, m->V.get(), m->F.get(), m->nf, dp.get(), n, df.get(), d2.get(), dc.get());
    std::vector<double> h2(n);
    PCU_CUDA(cudaMemcpyAsync(h2.data(), d2.get(), n * 8, cudaMemcpyDeviceToHost, ctx.stream));
    if (face) PCU_CUDA(cudaMemcpyAsync(face, df.get(), n * 4, cudaMemcpyDeviceToHost, ctx.stream));
    if (closest) PCU_CUDA(cudaMemcpyAsync(closest, dc.get(), 3 * n * 8, cudaMemcpyDeviceToHost, ctx.stream));
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    if (dist)
      for (int64_t i = 0; i < n; ++i) dist[i] = std::sqrt(h2[i]);
  });
}

int pamopt_cu_sample_points(pamopt_cu_mesh m, int64_t n, uint64_t seed, double* pts, int32_t* faces,
                            double* total_area) {
  return guarded([&] {
    PCU_REQUIRE(m && n >= 0 && (n == 0 || pts), PAMOPT_CU_EINVAL, "bad arguments");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    check_indices(ctx, m);
    pcu::DevBuf<double> dp(3 * (n ? n : 1), ctx.stream);
    pcu::DevBuf<int32_t> df(n ? n : 1, ctx.stream);
    double area = 0.0;
    PCU_REQUIRE(pcu::sample_points(ctx, m->V.get(), m->F.get(), m->nf, n, seed, dp.get(), df.get(), &area),
                PAMOPT_CU_EINVAL, "sample_points: zero-area mesh");
    if (n) PCU_CUDA(cudaMemcpyAsync(pts, dp.get(), 3 * n * 8, cudaMemcpyDeviceToHost, ctx.stream));
    if (n && faces) PCU_CUDA(cudaMemcpyAsync(faces, df.get(), n * 4, cudaMemcpyDeviceToHost, ctx.stream));
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    if (total_area) *total_area = area;
  });
}

static void two_sided(pamopt_cu_mesh a, pamopt_cu_mesh b, int64_t n, uint64_t seed, double& cd, double& hd) {
  PCU_REQUIRE(a && b && n > 0, PAMOPT_CU_EINVAL, "bad arguments");
  PCU_REQUIRE(a->owner == b->owner, PAMOPT_CU_EINVAL, "metrics: meshes belong to different contexts");
  pcu::Ctx& ctx = a->owner->ctx;
  pcu::DeviceGuard g(ctx.device);
  check_indices(ctx, a);
  check_indices(ctx, b);
  double sa, ma, aa, sb, mb, ab;
  pcu::directed_d2(ctx, a->V.get(), a->F.get(), a->nf, b->V.get(), b->F.get(), b->nf, n, seed, sa, ma, aa);
  pcu::directed_d2(ctx, b->V.get(), b->F.get(), b->nf, a->V.get(), a->F.get(), a->nf, n, seed + kSeedB, sb, mb, ab);
  cd = aa / static_cast<double>(n) * sa + ab / static_cast<double>(n) * sb;
  hd = std::sqrt(std::max(ma, mb));
}

int pamopt_cu_chamfer(pamopt_cu_mesh a, pamopt_cu_mesh b, int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    PCU_REQUIRE(out, PAMOPT_CU_EINVAL, "null argument");
    double cd, hd;
    two_sided(a, b, n, seed, cd, hd);
    *out = cd;
  });
}

int pamopt_cu_hausdorff(pamopt_cu_mesh a, pamopt_cu_mesh b, int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    PCU_REQUIRE(out, PAMOPT_CU_EINVAL, "null argument");
    double cd, hd;
    two_sided(a, b, n, seed, cd, hd);
    *out = hd;
  });
}

int pamopt_cu_min_internal_angle(pamopt_cu_mesh m, double* deg) {
  return guarded([&] {
    PCU_REQUIRE(m && deg, PAMOPT_CU_EINVAL, "null argument");
    PCU_REQUIRE(m->nf > 0, PAMOPT_CU_EINVAL, "min_internal_angle: empty mesh");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    check_indices(ctx, m);
    const double c = pcu::max_corner_cos(ctx, m->V.get(), m->F.get(), m->nf);
    *deg = std::acos(c) * (180.0 / 3.14159265358979323846);
  });
}

static void make_report(pamopt_cu_mesh ref, pamopt_cu_mesh m, int64_t n, uint64_t seed, pamopt_cu_mesh_report* out) {
  pcu::Ctx& ctx = m->owner->ctx;
  pcu::DeviceGuard g(ctx.device);
  check_indices(ctx, m);
  *out = pamopt_cu_mesh_report{};
  out->n_faces = m->nf;
  out->n_vertices = m->nv;
  out->cd = out->hd = std::numeric_limits<double>::quiet_NaN();
  if (ref) two_sided(ref, m, n, seed, out->cd, out->hd);
  out->min_angle_deg = m->nf ? std::acos(pcu::max_corner_cos(ctx, m->V.get(), m->F.get(), m->nf)) *
                                   (180.0 / 3.14159265358979323846)
                             : 0.0;
  pcu::TopologyResult t;
  pcu::analyze_topology(ctx, m->F.get(), m->nf, m->nv, t);
  out->manifold = t.manifold;
  out->watertight = t.watertight;
  const std::vector<int32_t> pairs =
      m->nf >= 2 ? pcu::self_intersections(ctx, m->V.get(), m->nv, m->F.get(), m->nf, nullptr, nullptr)
                 : std::vector<int32_t>();
  out->intersection_free = pairs.empty() ? 1 : 0;
}

int pamopt_cu_report(pamopt_cu_mesh ref, pamopt_cu_mesh m, int64_t n, uint64_t seed, pamopt_cu_mesh_report* out) {
  return guarded([&] {
    PCU_REQUIRE(m && out, PAMOPT_CU_EINVAL, "null argument");
    make_report(ref, m, n, seed, out);
  });
}

// ------------------------------------------------------------------------------ stage 3
static pcu::ProjectParams to_pp(const pamopt_cu_project_params& p) {
  pcu::ProjectParams q;
  q.iterations = p.iterations;
  q.refresh = p.refresh;
  q.cg_max = p.cg_max;
  q.elas_power = p.elas_power;
  q.samples = p.samples;
  q.seed = p.seed;
  q.kdis = p.kdis;
  q.kelas = p.kelas;
  q.kbend = p.kbend;
  q.kbar = p.kbar;
  q.dhat = p.dhat;
  q.cg_tol = p.cg_tol;
  q.elas_tau = p.elas_tau;
  return q;
}

int pamopt_cu_project_defaults(pamopt_cu_project_params* out) {
  return guarded([&] {
    PCU_REQUIRE(out, PAMOPT_CU_EINVAL, "null argument");
    const pcu::ProjectParams d;
    *out = pamopt_cu_project_params{d.iterations, d.refresh, d.cg_max, d.elas_power, d.samples, d.seed, d.kdis,
                                    d.kelas, d.kbend, d.kbar, d.dhat, d.cg_tol, d.elas_tau};
  });
}

int pamopt_cu_safe_project(pamopt_cu_mesh ms, pamopt_cu_mesh mi, const pamopt_cu_project_params* params,
                           pamopt_cu_project_stats* stats) {
  return pamopt_cu_safe_project_traced(ms, mi, params, stats, nullptr);
}

int pamopt_cu_safe_project_traced(pamopt_cu_mesh ms, pamopt_cu_mesh mi, const pamopt_cu_project_params* params,
                                  pamopt_cu_project_stats* stats, const pamopt_cu_project_trace* trace) {
  return guarded([&] {
    PCU_REQUIRE(ms && mi, PAMOPT_CU_EINVAL, "null mesh");
    PCU_REQUIRE(ms->owner == mi->owner, PAMOPT_CU_EINVAL, "safe_project: meshes belong to different contexts");
    pamopt_cu_project_params p;
    if (params) p = *params;
    else pamopt_cu_project_defaults(&p);
    PCU_REQUIRE(p.iterations >= 0 && p.refresh >= 1 && p.samples >= 1 && p.dhat > 0.0 && p.cg_max >= 1,
                PAMOPT_CU_EINVAL, "safe_project: bad parameters");
    pcu::Ctx& ctx = ms->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    check_indices(ctx, ms);
    check_indices(ctx, mi);
    pcu::ProjectStats st;
    pcu::ProjectTrace tr;
    if (trace) {
      PCU_REQUIRE(trace->max_iters >= 0 && trace->contact_cap >= 0, PAMOPT_CU_EINVAL, "safe_project: bad trace sizes");
      tr = pcu::ProjectTrace{trace->max_iters, trace->contact_cap, trace->X,        trace->grad,
                             trace->dir,       trace->targets,     trace->m2s,      trace->contacts,
                             trace->n_contacts, trace->scalars,    trace->samples};
    }
    pcu::safe_project(ctx, ms->V.get(), ms->nv, ms->F.get(), ms->nf, mi->V.get(), mi->F.get(), mi->nf, to_pp(p), st,
                      trace ? &tr : nullptr);
    if (stats)
      *stats = pamopt_cu_project_stats{st.iterations, st.cg_iterations, st.refreshes, st.converged, st.energy0,
                                       st.energy, st.grad_norm, st.last_alpha};
  });
}

int pamopt_cu_project_term(pamopt_cu_ctx c, int32_t term, int32_t cls, const double* coords, int32_t nv,
                           const double* rest, const pamopt_cu_project_params* params, double* out) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(coords && rest && out && term >= 0 && term <= 5, PAMOPT_CU_EINVAL, "bad arguments");
    pamopt_cu_project_params p;
    if (params) p = *params;
    else pamopt_cu_project_defaults(&p);
    pcu::DeviceGuard g(c->ctx.device);
    pcu::project_term_probe(c->ctx, term, cls, coords, nv, rest, to_pp(p), out);
  });
}

int pamopt_cu_dmc_active_cells(pamopt_cu_grid gr, int64_t* cells, uint8_t* cases, uint8_t* flips, int64_t cap,
                               int64_t* n) {
  return guarded([&] {
    PCU_REQUIRE(gr && n, PAMOPT_CU_EINVAL, "null argument");
    pcu::Ctx& ctx = gr->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    const int64_t na = gr->last.n_active;
    *n = na;
    const int64_t k = std::min(cap, na);
    if (k <= 0) return;
    std::vector<uint32_t> c32(k);
    PCU_CUDA(cudaMemcpyAsync(c32.data(), gr->last.cells.get(), k * 4, cudaMemcpyDeviceToHost, ctx.stream));
    if (cases) PCU_CUDA(cudaMemcpyAsync(cases, gr->last.cases.get(), k, cudaMemcpyDeviceToHost, ctx.stream));
    if (flips) PCU_CUDA(cudaMemcpyAsync(flips, gr->last.flips.get(), k, cudaMemcpyDeviceToHost, ctx.stream));
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    if (cells)
      for (int64_t i = 0; i < k; ++i) cells[i] = c32[i];
  });
}

int pamopt_cu_dmc_table(int32_t* out) {
  return guarded([&] {
    PCU_REQUIRE(out != nullptr, PAMOPT_CU_EINVAL, "null argument");
    pcu::dmc_table_host(out);
  });
}

// ----------------------------------------------------------- stage 1b, granular operations
int pamopt_cu_dmc_stages(pamopt_cu_grid gr, double beta, int64_t counts[3]) {
  return guarded([&] {
    PCU_REQUIRE(gr && counts, PAMOPT_CU_EINVAL, "null argument");
    PCU_REQUIRE(beta > 0.0, PAMOPT_CU_EINVAL, "beta must be positive");
    PCU_REQUIRE(gr->z0 == 0 && gr->z1 == gr->R + 1, PAMOPT_CU_EINVAL, "dmc stages: the grid is a z-slab");
    pcu::Ctx& ctx = gr->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    gr->last = pcu::DmcResult();
    gr->last.want_stages = true;
    pcu::dmc_extract(ctx, gr->g.get(), gr->R, beta, gr->last);
    counts[0] = gr->last.n_active;
    counts[1] = static_cast<int64_t>(gr->last.nv_patch);
    counts[2] = static_cast<int64_t>(gr->last.n_quads);
  });
}

int pamopt_cu_dmc_build_patches(pamopt_cu_grid gr, double* vertices, int64_t* patch_first) {
  return guarded([&] {
    PCU_REQUIRE(gr != nullptr, PAMOPT_CU_EINVAL, "null grid");
    PCU_REQUIRE(gr->last.want_stages, PAMOPT_CU_EINVAL, "build_patches: call pamopt_cu_dmc_stages first");
    pcu::Ctx& ctx = gr->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    const pcu::DmcResult& r = gr->last;
    d2h(ctx, vertices, r.V.get(), 3 * static_cast<int64_t>(r.nv_patch));  // V starts with the patch vertices
    std::vector<uint32_t> vb(patch_first ? r.n_active : 0);
    if (patch_first) d2h(ctx, vb.data(), r.vbase.get(), r.n_active);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    for (size_t i = 0; i < vb.size(); ++i) patch_first[i] = vb[i];
  });
}

int pamopt_cu_dmc_build_quads(pamopt_cu_grid gr, int32_t* quads, int64_t* edges, float* samples, uint8_t* split) {
  return guarded([&] {
    PCU_REQUIRE(gr != nullptr, PAMOPT_CU_EINVAL, "null grid");
    PCU_REQUIRE(gr->last.want_stages, PAMOPT_CU_EINVAL, "build_quads: call pamopt_cu_dmc_stages first");
    pcu::Ctx& ctx = gr->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    const pcu::DmcResult& r = gr->last;
    const int64_t n = static_cast<int64_t>(r.n_quads);
    d2h(ctx, quads, r.quads.get(), 4 * n);
    d2h(ctx, edges, r.qedge.get(), n);
    d2h(ctx, samples, r.qf.get(), 2 * n);
    d2h(ctx, split, r.qsplit.get(), n);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

int pamopt_cu_triangulate_quads(pamopt_cu_ctx c, int32_t R, const double* pv, int64_t nv, const int32_t* quads,
                                const int64_t* edges, const float* samples, int64_t nq, double beta, pamopt_cu_mesh* out) {
  return guarded([&] {
    check_ctx(c);
    check_R(R);
    PCU_REQUIRE(out && nv >= 0 && nq >= 0 && (nv == 0 || pv) && (nq == 0 || (quads && edges && samples)),
                PAMOPT_CU_EINVAL, "bad arguments");
    PCU_REQUIRE(beta > 0.0, PAMOPT_CU_EINVAL, "beta must be positive");
    const int64_t n1 = static_cast<int64_t>(R) + 1;
    for (int64_t i = 0; i < nq; ++i) {
      for (int k = 0; k < 4; ++k)
        PCU_REQUIRE(quads[4 * i + k] >= 0 && quads[4 * i + k] < nv, PAMOPT_CU_EINVAL, "quad vertex out of range");
      const int64_t lv = edges[i] / 3, a = edges[i] % 3;
      const int64_t xyz[3] = {lv % n1, (lv / n1) % n1, lv / (n1 * n1)};
      PCU_REQUIRE(edges[i] >= 0 && xyz[2] < n1 && xyz[a] + 1 < n1, PAMOPT_CU_EINVAL, "quad edge outside the lattice");
    }
    pcu::Ctx& ctx = c->ctx;
    pcu::DeviceGuard g(ctx.device);
    pcu::DevBuf<double> dv(3 * (nv ? nv : 1), ctx.stream);
    pcu::DevBuf<int32_t> dq(4 * (nq ? nq : 1), ctx.stream);
    pcu::DevBuf<int64_t> de(nq ? nq : 1, ctx.stream);
    pcu::DevBuf<float> df(2 * (nq ? nq : 1), ctx.stream);
    if (nv) PCU_CUDA(cudaMemcpyAsync(dv.get(), pv, 3 * nv * 8, cudaMemcpyHostToDevice, ctx.stream));
    if (nq) {
      PCU_CUDA(cudaMemcpyAsync(dq.get(), quads, 4 * nq * 4, cudaMemcpyHostToDevice, ctx.stream));
      PCU_CUDA(cudaMemcpyAsync(de.get(), edges, nq * 8, cudaMemcpyHostToDevice, ctx.stream));
      PCU_CUDA(cudaMemcpyAsync(df.get(), samples, 2 * nq * 4, cudaMemcpyHostToDevice, ctx.stream));
    }
    std::unique_ptr<pamopt_cu_mesh_s> m(new pamopt_cu_mesh_s());
    pcu::triangulate_quads(ctx, dv.get(), nv, dq.get(), de.get(), df.get(), nq, R, beta, m->V, m->F, m->nv, m->nf);
    m->owner = c;
    ctx_ref(c);
    *out = m.release();
  });
}

int pamopt_cu_interpolate_patch_vertex(pamopt_cu_ctx c, const double* p0, const double* p1, const float* f0,
                                       const float* f1, int64_t n, double beta, double* out) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(n >= 0 && (n == 0 || (p0 && p1 && f0 && f1 && out)), PAMOPT_CU_EINVAL, "null argument");
    PCU_REQUIRE(beta > 0.0, PAMOPT_CU_EINVAL, "beta must be positive");
    if (n == 0) return;
    pcu::Ctx& ctx = c->ctx;
    pcu::DeviceGuard g(ctx.device);
    pcu::DevBuf<double> a(3 * n, ctx.stream), b(3 * n, ctx.stream), o(3 * n, ctx.stream);
    pcu::DevBuf<float> x(n, ctx.stream), y(n, ctx.stream);
    PCU_CUDA(cudaMemcpyAsync(a.get(), p0, 3 * n * 8, cudaMemcpyHostToDevice, ctx.stream));
    PCU_CUDA(cudaMemcpyAsync(b.get(), p1, 3 * n * 8, cudaMemcpyHostToDevice, ctx.stream));
    PCU_CUDA(cudaMemcpyAsync(x.get(), f0, n * 4, cudaMemcpyHostToDevice, ctx.stream));
    PCU_CUDA(cudaMemcpyAsync(y.get(), f1, n * 4, cudaMemcpyHostToDevice, ctx.stream));
    const int64_t bad = pcu::interpolate_patch_vertex(ctx, a.get(), b.get(), x.get(), y.get(), n, beta, o.get());
    d2h(ctx, out, o.get(), 3 * n);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    PCU_REQUIRE(bad == 0, PAMOPT_CU_EINVAL, "interpolate_patch_vertex: f0 and f1 must change sign");
  });
}

// -------------------------------------------------------------------------- tri_isect
int pamopt_cu_self_intersections(pamopt_cu_mesh m, int32_t* pairs, int64_t cap, int64_t* n) {
  return guarded([&] {
    PCU_REQUIRE(m && n, PAMOPT_CU_EINVAL, "null argument");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    check_indices(ctx, m);
    const std::vector<int32_t> h = pcu::self_intersections(ctx, m->V.get(), m->nv, m->F.get(), m->nf, nullptr, nullptr);
    *n = static_cast<int64_t>(h.size() / 2);
    if (pairs) std::memcpy(pairs, h.data(), std::min<int64_t>(cap, *n) * 2 * sizeof(int32_t));
  });
}

int pamopt_cu_tri_tri_pairs(pamopt_cu_mesh m, const int32_t* pairs, int64_t n, int32_t* out) {
  return guarded([&] {
    PCU_REQUIRE(m && (n == 0 || (pairs && out)), PAMOPT_CU_EINVAL, "null argument");
    if (n == 0) return;
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    for (int64_t i = 0; i < 2 * n; ++i)
      PCU_REQUIRE(pairs[i] >= 0 && pairs[i] < m->nf, PAMOPT_CU_EINVAL, "face index out of range");
    check_indices(ctx, m);
    pcu::DevBuf<int32_t> dp(2 * n, ctx.stream), dout(n, ctx.stream);
    PCU_CUDA(cudaMemcpyAsync(dp.get(), pairs, 2 * n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx.stream));
    pcu::tri_tri_pairs(ctx, m->V.get(), m->F.get(), dp.get(), n, dout.get());
    PCU_CUDA(cudaMemcpyAsync(out, dout.get(), n * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx.stream));
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

static void pairs_call(pamopt_cu_mesh m, const int32_t* pairs, int64_t n,
                       const std::function<void(pcu::Ctx&, const int32_t*)>& fn) {
  PCU_REQUIRE(m && n >= 0 && (n == 0 || pairs), PAMOPT_CU_EINVAL, "null argument");
  if (n == 0) return;
  pcu::Ctx& ctx = m->owner->ctx;
  pcu::DeviceGuard g(ctx.device);
  for (int64_t i = 0; i < 2 * n; ++i)
    PCU_REQUIRE(pairs[i] >= 0 && pairs[i] < m->nf, PAMOPT_CU_EINVAL, "face index out of range");
  check_indices(ctx, m);
  pcu::DevBuf<int32_t> dp(2 * n, ctx.stream);
  PCU_CUDA(cudaMemcpyAsync(dp.get(), pairs, 2 * n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx.stream));
  fn(ctx, dp.get());
  PCU_CUDA(cudaStreamSynchronize(ctx.stream));
}

int pamopt_cu_classify_pair(pamopt_cu_mesh m, const int32_t* pairs, int64_t n, int32_t* shared, int32_t* coplanar) {
  return guarded([&] {
    pairs_call(m, pairs, n, [&](pcu::Ctx& ctx, const int32_t* dp) {
      pcu::DevBuf<int32_t> s(n, ctx.stream), c(n, ctx.stream);
      pcu::classify_pairs(ctx, m->V.get(), m->F.get(), dp, n, s.get(), c.get());
      d2h(ctx, shared, s.get(), n);
      d2h(ctx, coplanar, c.get(), n);
      PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    });
  });
}

static int by_class(pamopt_cu_mesh m, const int32_t* pairs, int64_t n, int mode, int32_t* out) {
  return guarded([&] {
    PCU_REQUIRE(n == 0 || out, PAMOPT_CU_EINVAL, "null argument");
    pairs_call(m, pairs, n, [&](pcu::Ctx& ctx, const int32_t* dp) {
      pcu::DevBuf<int32_t> o(n, ctx.stream);
      pcu::verdict_by_class(ctx, m->V.get(), m->F.get(), dp, n, mode, o.get());
      d2h(ctx, out, o.get(), n);
      PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    });
    for (int64_t i = 0; i < n; ++i)
      PCU_REQUIRE(out[i] >= 0, PAMOPT_CU_EINVAL,
                  mode == 1 ? "intersect_3d: coplanar pair (use intersect_coplanar)"
                            : "intersect_coplanar: non-coplanar pair (use intersect_3d)");
  });
}

int pamopt_cu_intersect_3d(pamopt_cu_mesh m, const int32_t* pairs, int64_t n, int32_t* out) {
  return by_class(m, pairs, n, 1, out);
}

int pamopt_cu_intersect_coplanar(pamopt_cu_mesh m, const int32_t* pairs, int64_t n, int32_t* out) {
  return by_class(m, pairs, n, 2, out);
}

// ---------------------------------------------------------------------------- stage 2
static pcu::SimplifyParams to_params(const pamopt_cu_simplify_params* p) {
  pcu::SimplifyParams P;
  if (p) {
    P.we = p->w_e;
    P.ws = p->w_s;
    P.tolerance = p->tolerance;
    P.stall = p->stall_iterations > 0 ? p->stall_iterations : 10;
  }
  PCU_REQUIRE(P.we >= 0 && P.ws >= 0 && P.tolerance >= 1, PAMOPT_CU_EINVAL, "bad simplify parameters");
  return P;
}

static void to_stats(const pcu::SimplifyStats& S, pamopt_cu_simplify_stats* o) {
  if (!o) return;
  o->iterations = S.iterations;
  o->collapses = S.collapses;
  o->undone = S.undone;
  o->link_failures = S.link_failures;
  o->max_undo_rounds = S.max_undo_rounds;
  for (int k = 0; k < 8; ++k) o->undo_hist[k] = S.undo_hist[k];
  o->face_iterations = S.face_iterations;
  o->alg_bytes = S.alg_bytes;
}

int pamopt_cu_simplify(pamopt_cu_mesh m, int64_t target, const pamopt_cu_simplify_params* params,
                       pamopt_cu_simplify_stats* stats, int64_t* per_iter, int64_t per_iter_cap) {
  return guarded([&] {
    PCU_REQUIRE(m != nullptr, PAMOPT_CU_EINVAL, "null mesh");
    const pcu::SimplifyParams P = to_params(params);
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    validate(ctx, m);
    pcu::SimplifyStats S;
    pcu::simplify_run(ctx, m->V, m->F, m->nv, m->nf, target, P, S);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    to_stats(S, stats);
    if (per_iter)
      for (int64_t i = 0; i < std::min<int64_t>(per_iter_cap, static_cast<int64_t>(S.per_iter.size())); ++i)
        per_iter[i] = S.per_iter[i];
  });
}

// ----------------------------------------------------------- stage 2, granular operations

int pamopt_cu_quadrics(pamopt_cu_mesh m, double* out) {
  return guarded([&] {
    PCU_REQUIRE(m && out, PAMOPT_CU_EINVAL, "null argument");
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    validate(ctx, m);
    pcu::DevBuf<double> q(10 * (m->nv ? m->nv : 1), ctx.stream);
    pcu::quadrics_of(ctx, m->V.get(), m->F.get(), m->nv, m->nf, q.get());
    d2h(ctx, out, q.get(), 10 * m->nv);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

static void check_edges(const pamopt_cu_mesh_s* m, const int32_t* edges, int64_t n) {
  for (int64_t i = 0; i < 2 * n; ++i)
    PCU_REQUIRE(edges[i] >= 0 && edges[i] < m->nv, PAMOPT_CU_EINVAL, "edge vertex out of range");
}

int pamopt_cu_edge_cost(pamopt_cu_mesh m, const int32_t* edges, int64_t n, double we, double ws, double* cost,
                        double* place) {
  return guarded([&] {
    PCU_REQUIRE(m && n >= 0 && (n == 0 || (edges && cost)), PAMOPT_CU_EINVAL, "null argument");
    PCU_REQUIRE(we >= 0 && ws >= 0, PAMOPT_CU_EINVAL, "edge_cost: weights must be >= 0");
    check_edges(m, edges, n);
    if (n == 0) return;
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    validate(ctx, m);
    pcu::DevBuf<int32_t> de(2 * n, ctx.stream);
    pcu::DevBuf<double> dc(n, ctx.stream), dp(3 * n, ctx.stream);
    PCU_CUDA(cudaMemcpyAsync(de.get(), edges, 2 * n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx.stream));
    pcu::edge_cost_of(ctx, m->V.get(), m->F.get(), m->nv, m->nf, de.get(), n, we, ws, dc.get(), dp.get());
    d2h(ctx, cost, dc.get(), n);
    d2h(ctx, place, dp.get(), 3 * n);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

int pamopt_cu_pack_cost(pamopt_cu_ctx c, const double* cost, const uint32_t* ids, int64_t n, uint64_t* keys) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(n >= 0 && (n == 0 || (cost && ids && keys)), PAMOPT_CU_EINVAL, "null argument");
    if (n == 0) return;
    pcu::Ctx& ctx = c->ctx;
    pcu::DeviceGuard g(ctx.device);
    pcu::DevBuf<double> dc(n, ctx.stream);
    pcu::DevBuf<uint32_t> di(n, ctx.stream);
    pcu::DevBuf<uint64_t> dk(n, ctx.stream);
    PCU_CUDA(cudaMemcpyAsync(dc.get(), cost, n * 8, cudaMemcpyHostToDevice, ctx.stream));
    PCU_CUDA(cudaMemcpyAsync(di.get(), ids, n * 4, cudaMemcpyHostToDevice, ctx.stream));
    const int64_t nan = pcu::pack_cost_of(ctx, dc.get(), di.get(), n, dk.get());
    d2h(ctx, keys, dk.get(), n);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    PCU_REQUIRE(nan == 0, PAMOPT_CU_ENUMERIC, "pack_cost: NaN cost");
  });
}

int pamopt_cu_link_condition(pamopt_cu_mesh m, const int32_t* edges, int64_t n, int32_t* out) {
  return guarded([&] {
    PCU_REQUIRE(m && n >= 0 && (n == 0 || (edges && out)), PAMOPT_CU_EINVAL, "null argument");
    check_edges(m, edges, n);
    if (n == 0) return;
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    validate(ctx, m);
    pcu::DevBuf<int32_t> de(2 * n, ctx.stream), dout(n, ctx.stream);
    PCU_CUDA(cudaMemcpyAsync(de.get(), edges, 2 * n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx.stream));
    pcu::link_condition_of(ctx, m->F.get(), m->nv, m->nf, de.get(), n, dout.get());
    d2h(ctx, out, dout.get(), n);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    for (int64_t i = 0; i < n; ++i)
      PCU_REQUIRE(out[i] >= 0, PAMOPT_CU_EINVAL, "link_condition_holds: unknown edge");
  });
}

struct pamopt_cu_qem_s {
  pamopt_cu_mesh mesh = nullptr;
  pcu::SimplifyStats S;
  pcu::QemState* q = nullptr;
  ~pamopt_cu_qem_s() {
    if (q) pcu::qem_destroy(q);
  }
};

extern "C++" {
template <class Fn>
static int with_qem(pamopt_cu_qem q, Fn&& fn) {
  return guarded([&] {
    PCU_REQUIRE(q && q->q, PAMOPT_CU_EINVAL, "null qem state");
    pcu::Ctx& ctx = q->mesh->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    fn(ctx);
  });
}
}

int pamopt_cu_qem_create(pamopt_cu_mesh m, int64_t target, const pamopt_cu_simplify_params* params, pamopt_cu_qem* out) {
  return guarded([&] {
    PCU_REQUIRE(m && out, PAMOPT_CU_EINVAL, "null argument");
    const pcu::SimplifyParams P = to_params(params);
    pcu::Ctx& ctx = m->owner->ctx;
    pcu::DeviceGuard g(ctx.device);
    validate(ctx, m);
    std::unique_ptr<pamopt_cu_qem_s> s(new pamopt_cu_qem_s());
    s->mesh = m;
    s->q = pcu::qem_create(ctx, m->V, m->F, m->nv, m->nf, target, P, s->S);
    *out = s.release();
  });
}

int pamopt_cu_qem_done(pamopt_cu_qem q, int32_t* done) {
  return with_qem(q, [&](pcu::Ctx&) {
    PCU_REQUIRE(done, PAMOPT_CU_EINVAL, "null argument");
    *done = pcu::qem_done(q->q) ? 1 : 0;
  });
}

int pamopt_cu_qem_prepare(pamopt_cu_qem q, int64_t* n_edges) {
  return with_qem(q, [&](pcu::Ctx&) {
    PCU_REQUIRE(!pcu::qem_done(q->q), PAMOPT_CU_EINVAL, "qem: the run is finished");
    pcu::qem_prepare(q->q);
    if (n_edges) *n_edges = pcu::qem_view(q->q).ne;
  });
}

int pamopt_cu_qem_edges(pamopt_cu_qem q, int32_t* edges, uint64_t* keys, double* place, uint8_t* valid, int64_t cap) {
  return with_qem(q, [&](pcu::Ctx& ctx) {
    PCU_REQUIRE(pcu::qem_phase(q->q) >= 1, PAMOPT_CU_EINVAL, "qem: edges exist after prepare()");
    const pcu::QemView v = pcu::qem_view(q->q);
    const int64_t n = std::min(cap, v.ne);
    if (n <= 0) return;
    std::vector<int32_t> a(edges ? n : 0), b(edges ? n : 0);
    if (edges) {
      d2h(ctx, a.data(), v.ea, n);
      d2h(ctx, b.data(), v.eb, n);
    }
    d2h(ctx, keys, v.key, n);
    d2h(ctx, place, v.place, 3 * n);
    d2h(ctx, valid, v.valid, n);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    if (edges)
      for (int64_t i = 0; i < n; ++i) {
        edges[2 * i] = a[i];
        edges[2 * i + 1] = b[i];
      }
    if (keys && place) {  // invalid edges carry no placement
      for (int64_t i = 0; i < n; ++i)
        if (keys[i] == ~0ull) place[3 * i] = place[3 * i + 1] = place[3 * i + 2] = 0.0;
    }
  });
}

int pamopt_cu_qem_propagate_and_mark(pamopt_cu_qem q, int64_t* n_marked) {
  return with_qem(q, [&](pcu::Ctx&) {
    pcu::qem_propagate_and_mark(q->q);
    if (n_marked) *n_marked = pcu::qem_view(q->q).nm;
  });
}

int pamopt_cu_qem_marked(pamopt_cu_qem q, uint32_t* ids, int64_t cap, uint64_t* face_keys, int64_t cap_faces) {
  return with_qem(q, [&](pcu::Ctx& ctx) {
    PCU_REQUIRE(pcu::qem_phase(q->q) >= 2, PAMOPT_CU_EINVAL, "qem: marked edges exist after propagate_and_mark()");
    const pcu::QemView v = pcu::qem_view(q->q);
    const int64_t n = std::min(cap, v.nm);
    std::vector<uint64_t> k(ids && n > 0 ? n : 0);
    if (ids && n > 0) d2h(ctx, k.data(), v.marked_sorted, n);
    if (face_keys && cap_faces > 0 && v.nf > 0) {
      pcu::DevBuf<uint64_t> fk(v.nf, ctx.stream);
      pcu::qem_face_keys(q->q, fk.get());
      d2h(ctx, face_keys, fk.get(), std::min(cap_faces, v.nf));
      PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    for (int64_t i = 0; i < static_cast<int64_t>(k.size()); ++i) ids[i] = static_cast<uint32_t>(k[i]);
  });
}

int pamopt_cu_qem_collapse_batch(pamopt_cu_qem q, uint8_t* link_ok, int64_t cap) {
  return with_qem(q, [&](pcu::Ctx& ctx) {
    pcu::qem_collapse_batch(q->q);
    const pcu::QemView v = pcu::qem_view(q->q);
    const int64_t n = std::min(cap, v.nm);
    if (link_ok && n > 0) {
      std::vector<uint32_t> r(n);
      d2h(ctx, r.data(), v.rem, n);
      PCU_CUDA(cudaStreamSynchronize(ctx.stream));
      for (int64_t i = 0; i < n; ++i) link_ok[i] = r[i] ? 1 : 0;
    }
  });
}

int pamopt_cu_qem_undo_loop(pamopt_cu_qem q, int32_t* rounds, int64_t* n_applied, uint8_t* applied, int64_t cap) {
  return with_qem(q, [&](pcu::Ctx& ctx) {
    pcu::qem_undo_loop(q->q);
    const pcu::QemView v = pcu::qem_view(q->q);
    if (rounds) *rounds = v.rounds;
    if (n_applied) *n_applied = v.succ;
    const int64_t n = std::min(cap, v.nm);
    if (applied && n > 0) {
      d2h(ctx, applied, v.applied, n);
      PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    }
  });
}

int pamopt_cu_qem_end_iteration(pamopt_cu_qem q, int64_t* alive_faces) {
  return with_qem(q, [&](pcu::Ctx&) {
    pcu::qem_end_iteration(q->q);
    if (alive_faces) *alive_faces = pcu::qem_view(q->q).alive_faces;
  });
}

int pamopt_cu_qem_mesh(pamopt_cu_qem q, double* v, int32_t* f, uint8_t* falive, int64_t* nv, int64_t* nf) {
  return with_qem(q, [&](pcu::Ctx& ctx) {
    const pcu::QemView w = pcu::qem_view(q->q);
    if (nv) *nv = w.nv;
    if (nf) *nf = w.nf;
    d2h(ctx, v, w.X, 3 * w.nv);
    d2h(ctx, f, w.F, 3 * w.nf);
    d2h(ctx, falive, w.falive, w.nf);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  });
}

int pamopt_cu_qem_finish(pamopt_cu_qem q, pamopt_cu_simplify_stats* stats) {
  return with_qem(q, [&](pcu::Ctx& ctx) {
    PCU_REQUIRE(pcu::qem_phase(q->q) == 0, PAMOPT_CU_EINVAL, "qem: finish() inside an iteration");
    pcu::qem_finish(q->q);
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    to_stats(q->S, stats);
  });
}

int pamopt_cu_qem_destroy(pamopt_cu_qem q) {
  return guarded([&] {
    if (!q) return;
    pcu::DeviceGuard g(q->mesh->owner->ctx.device);
    delete q;
  });
}

// ------------------------------------------------------------------------- run_pipeline
int pamopt_cu_pipeline_defaults(pamopt_cu_pipeline_config* out) {
  return guarded([&] {
    PCU_REQUIRE(out, PAMOPT_CU_EINVAL, "null argument");
    *out = pamopt_cu_pipeline_config{};
    out->resolution = 0;
    out->run_projection = 0;
    out->target_faces = 0;
    out->target_ratio = 0.01;
    out->beta = 5.0;
    out->eps = 0.0;
    out->simplify = pamopt_cu_simplify_params{1e-3, 5e-3, 4, 10};
    out->report_samples = 16384;
    out->seed = 42;
  });
}

// SPEC.md:224 default resolution rule
static int32_t auto_resolution(int64_t target) { return target < 50 ? 64 : (target < 1000 ? 128 : 256); }

int pamopt_cu_run_pipeline(pamopt_cu_ctx c, pamopt_cu_mesh in, const pamopt_cu_pipeline_config* cfg_in,
                           pamopt_cu_mesh* out, pamopt_cu_pipeline_report* rep) {
  return guarded([&] {
    check_ctx(c);
    PCU_REQUIRE(in && out && rep, PAMOPT_CU_EINVAL, "null argument");
    PCU_REQUIRE(in->owner == c, PAMOPT_CU_EINVAL, "mesh belongs to another context");
    pamopt_cu_pipeline_config cfg;
    if (cfg_in) cfg = *cfg_in;
    else pamopt_cu_pipeline_defaults(&cfg);
    *out = nullptr;
    *rep = pamopt_cu_pipeline_report{};
    const int64_t target = cfg.target_faces > 0
                               ? cfg.target_faces
                               : std::max<int64_t>(4, static_cast<int64_t>(cfg.target_ratio * static_cast<double>(in->nf)));
    PCU_REQUIRE(target >= 4, PAMOPT_CU_EINVAL, "run_pipeline: target_faces must be >= 4 (SPEC.md:541)");
    const int32_t R = cfg.resolution > 0 ? cfg.resolution : auto_resolution(target);
    check_R(R);
    const double eps = cfg.eps > 0.0 ? cfg.eps : 0.9 / R;
    const double lo = 0.8660254037844386 / R, hi = 3.0 / R - 0.8660254037844386 / R;
    PCU_REQUIRE(eps >= lo && eps <= hi, PAMOPT_CU_EINVAL, "udf_to_sdf: epsilon out of range");
    PCU_REQUIRE(cfg.beta > 0.0 && cfg.report_samples > 0, PAMOPT_CU_EINVAL, "run_pipeline: bad config");
    const pcu::SimplifyParams P = to_params(&cfg.simplify);
    pcu::Ctx& ctx = c->ctx;
    pcu::DeviceGuard g(ctx.device);
    validate(ctx, in);
    rep->resolution = R;
    rep->target_faces = target;
    rep->faces_in = in->nf;
    auto now = [&]() {
      PCU_CUDA(cudaStreamSynchronize(ctx.stream));
      return std::chrono::steady_clock::now();
    };
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
      return static_cast<float>(std::chrono::duration<double, std::milli>(b - a).count());
    };
    auto new_mesh = [&]() {
      std::unique_ptr<pamopt_cu_mesh_s> m(new pamopt_cu_mesh_s());
      m->owner = c;
      ctx_ref(c);
      return m;
    };
    const auto t0 = now();
    // normalise a copy (padding 2 * band)
    auto norm = new_mesh();
    norm->nv = in->nv;
    norm->nf = in->nf;
    norm->V.alloc(3 * (in->nv ? in->nv : 1), ctx.stream);
    norm->F.alloc(3 * (in->nf ? in->nf : 1), ctx.stream);
    PCU_CUDA(cudaMemcpyAsync(norm->V.get(), in->V.get(), 3 * in->nv * 8, cudaMemcpyDeviceToDevice, ctx.stream));
    PCU_CUDA(cudaMemcpyAsync(norm->F.get(), in->F.get(), 3 * in->nf * 4, cudaMemcpyDeviceToDevice, ctx.stream));
    pcu::normalize_unit_cube(ctx, norm->V.get(), norm->nv, 6.0 / R, rep->scale_translation);
    // stage 1: UDF -> SDF -> DMC
    auto m = new_mesh();
    {
      const int64_t n1 = R + 1;
      pcu::DevBuf<float> sdf(n1 * n1 * n1, ctx.stream);
      pcu::DevBuf<uint32_t> signs(n1 * n1 * ((n1 + 31) / 32), ctx.stream);
      pcu::udf_run(ctx, norm->V.get(), norm->nv, norm->F.get(), norm->nf, R, 1, eps, sdf.get(), 0, -1, signs.get());
      pcu::DmcResult d;
      pcu::dmc_extract(ctx, sdf.get(), R, cfg.beta, d, signs.get());
      m->nv = static_cast<int64_t>(d.nv);
      m->nf = static_cast<int64_t>(d.nf);
      m->V = std::move(d.V);
      m->F = std::move(d.F);
    }
    const auto t1 = now();
    float cert_ms = 0.f;
    auto certify = [&](int stage, bool extra_ok, const char* what) {
      const auto a = now();
      make_report(norm.get(), m.get(), cfg.report_samples, cfg.seed, &rep->stage[stage - 1]);
      cert_ms += ms(a, now());
      const pamopt_cu_mesh_report& r = rep->stage[stage - 1];
      if (r.manifold && r.watertight && r.intersection_free && extra_ok) return;
      rep->failed_stage = stage;
      char msg[256];
      std::snprintf(msg, sizeof(msg),
                    "run_pipeline: stage %d certification failed (manifold=%d watertight=%d intersection_free=%d%s)",
                    stage, r.manifold, r.watertight, r.intersection_free, what);
      *out = m.release();
      throw pcu::Error(PAMOPT_CU_ECERT, msg);
    };
    certify(1, m->nf > 0, m->nf > 0 ? "" : " empty DMC surface");
    // stage 2: QEM to the target (the stall rule may stop above it)
    pcu::SimplifyStats S;
    pcu::simplify_run(ctx, m->V, m->F, m->nv, m->nf, target, P, S);
    to_stats(S, &rep->simplify);
    rep->stalled = m->nf > target ? 1 : 0;
    const auto t2 = now();
    const bool stall_ok = m->nf <= target ||
                          (S.per_iter.size() >= static_cast<size_t>(P.stall) &&
                           std::all_of(S.per_iter.end() - P.stall, S.per_iter.end(), [](int64_t x) { return x == 0; }));
    certify(2, stall_ok, stall_ok ? "" : " face target missed without a stall");
    // stage 3 (optional): safe projection toward the input, connectivity unchanged
    auto t3 = now();
    if (cfg.run_projection) {
      pamopt_cu_project_params pp;
      pamopt_cu_project_defaults(&pp);
      pcu::ProjectStats ps;
      pcu::safe_project(ctx, m->V.get(), m->nv, m->F.get(), m->nf, norm->V.get(), norm->F.get(), norm->nf, to_pp(pp),
                        ps);
      t3 = now();
      rep->projected = 1;
      certify(3, true, "");
    }
    rep->stage_ms[0] = ms(t0, t1);
    rep->stage_ms[1] = ms(t1, t2);
    rep->stage_ms[2] = cfg.run_projection ? ms(t2, t3) - 0.f : 0.f;
    rep->stage_ms[3] = cert_ms;
    // back to the input's coordinates (mesh_io.cpp:410-412)
    pcu::denormalize(ctx, m->V.get(), m->nv, rep->scale_translation);
    rep->total_ms = ms(t0, now());
    *out = m.release();
  });
}

// ---------------------------------------------------------------------------- pipeline
static void remesh_impl(pamopt_cu_ctx c, pamopt_cu_mesh in, int32_t R, double eps, double beta, int64_t target,
                        const pamopt_cu_simplify_params* params, pamopt_cu_mesh* out, pamopt_cu_simplify_stats* stats,
                        pamopt_cu_stage_times* times) {
  check_ctx(c);
  PCU_REQUIRE(in && out, PAMOPT_CU_EINVAL, "null argument");
  check_R(R);
  const double lo = 0.8660254037844386 / R, hi = 3.0 / R - 0.8660254037844386 / R;
  PCU_REQUIRE(eps >= lo && eps <= hi, PAMOPT_CU_EINVAL, "udf_to_sdf: epsilon out of range");
  const pcu::SimplifyParams P = to_params(params);
  PCU_REQUIRE(in->owner == c, PAMOPT_CU_EINVAL, "mesh belongs to another context");
  pcu::Ctx& ctx = c->ctx;
  pcu::DeviceGuard g(ctx.device);
  validate(ctx, in);
  struct Events {  // destroyed on every exit path, including a throw from a stage
    cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
    ~Events() {
      for (auto x : e)
        if (x) cudaEventDestroy(x);
    }
  } evs;
  cudaEvent_t* ev = evs.e;
  for (int i = 0; i < 4; ++i) PCU_CUDA(cudaEventCreate(&ev[i]));
  PCU_CUDA(cudaEventRecord(ev[0], ctx.stream));
  const int64_t n1 = R + 1;
  pcu::DevBuf<float> sdf(n1 * n1 * n1, ctx.stream);
  pcu::DevBuf<uint32_t> signs(n1 * n1 * ((n1 + 31) / 32), ctx.stream);
  pcu::udf_run(ctx, in->V.get(), in->nv, in->F.get(), in->nf, R, 1, eps, sdf.get(), 0, -1, signs.get());
  PCU_CUDA(cudaEventRecord(ev[1], ctx.stream));
  pcu::DmcResult d;
  pcu::dmc_extract(ctx, sdf.get(), R, beta, d, signs.get());
  sdf.release();
  signs.release();
  PCU_CUDA(cudaEventRecord(ev[2], ctx.stream));
  auto* m = new pamopt_cu_mesh_s();
  m->owner = c;
  ctx_ref(c);
  m->nv = static_cast<int64_t>(d.nv);
  m->nf = static_cast<int64_t>(d.nf);
  m->V = std::move(d.V);
  m->F = std::move(d.F);
  pcu::SimplifyStats S;
  try {
    pcu::simplify_run(ctx, m->V, m->F, m->nv, m->nf, target, P, S);
  } catch (...) {
    delete m;
    ctx_unref(c);
    throw;
  }
  PCU_CUDA(cudaEventRecord(ev[3], ctx.stream));
  PCU_CUDA(cudaEventSynchronize(ev[3]));
  if (times) {
    PCU_CUDA(cudaEventElapsedTime(&times->udf_ms, ev[0], ev[1]));
    PCU_CUDA(cudaEventElapsedTime(&times->dmc_ms, ev[1], ev[2]));
    PCU_CUDA(cudaEventElapsedTime(&times->simplify_ms, ev[2], ev[3]));
    PCU_CUDA(cudaEventElapsedTime(&times->total_ms, ev[0], ev[3]));
    times->dmc_faces = static_cast<int64_t>(d.nf);
    times->dmc_vertices = static_cast<int64_t>(d.nv);
  }
  to_stats(S, stats);
  *out = m;
}

int pamopt_cu_remesh(pamopt_cu_ctx c, pamopt_cu_mesh in, int32_t R, double eps, double beta, int64_t target,
                     const pamopt_cu_simplify_params* params, pamopt_cu_mesh* out, pamopt_cu_simplify_stats* stats,
                     pamopt_cu_stage_times* times) {
  return guarded([&] { remesh_impl(c, in, R, eps, beta, target, params, out, stats, times); });
}

int pamopt_cu_remesh_host(pamopt_cu_ctx c, const double* v, int64_t nv, const int32_t* f, int64_t nf, int32_t R,
                          double eps, double beta, int64_t target, const pamopt_cu_simplify_params* params,
                          int64_t* out_nv, int64_t* out_nf, pamopt_cu_simplify_stats* stats,
                          pamopt_cu_stage_times* times) {
  pamopt_cu_mesh in = nullptr;
  int rc = pamopt_cu_mesh_upload(c, v, nv, f, nf, &in);
  if (rc) return rc;
  rc = guarded([&] {
    pamopt_cu_mesh out = nullptr;
    remesh_impl(c, in, R, eps, beta, target, params, &out, stats, times);
    pcu::Ctx& ctx = c->ctx;
    ctx.host_v.resize(3 * out->nv);
    ctx.host_f.resize(3 * out->nf);
    if (out->nv) PCU_CUDA(cudaMemcpyAsync(ctx.host_v.data(), out->V.get(), 3 * out->nv * 8, cudaMemcpyDeviceToHost, ctx.stream));
    if (out->nf) PCU_CUDA(cudaMemcpyAsync(ctx.host_f.data(), out->F.get(), 3 * out->nf * 4, cudaMemcpyDeviceToHost, ctx.stream));
    PCU_CUDA(cudaStreamSynchronize(ctx.stream));
    if (out_nv) *out_nv = out->nv;
    if (out_nf) *out_nf = out->nf;
    pamopt_cu_mesh_free(out);
  });
  pamopt_cu_mesh_free(in);
  return rc;
}

int pamopt_cu_remesh_fetch(pamopt_cu_ctx c, double* v, int32_t* f) {
  return guarded([&] {
    check_ctx(c);
    if (v) std::memcpy(v, c->ctx.host_v.data(), c->ctx.host_v.size() * 8);
    if (f) std::memcpy(f, c->ctx.host_f.data(), c->ctx.host_f.size() * 4);
  });
}

}  // extern "C"

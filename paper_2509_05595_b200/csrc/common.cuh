// common.cuh — shared runtime + device arithmetic of the B200 remesh path.
//
// Everything here compiles with `--fmad=false` (see build.py): every decision-bearing FP64
// operation rounds exactly like the FP64 scalar code it mirrors, so integer outputs (candidate
// lists, MC cases, DMC topology, collapse sets) are bit-identical to the checker.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <cstring>
#include <initializer_list>
#include <vector>

#include "../../include/pamopt_cu.h"

namespace pcu {

// ------------------------------------------------------------------------------- errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PCU_CUDA(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      throw ::pcu::Error(_e == cudaErrorMemoryAllocation ? PAMOPT_CU_ENOMEM : PAMOPT_CU_ECUDA, \
                         std::string(#expr) + ": " + cudaGetErrorString(_e));            \
  } while (0)

#define PCU_REQUIRE(cond, code, msg) \
  do {                               \
    if (!(cond)) throw ::pcu::Error((code), (msg)); \
  } while (0)

void set_last_error(const std::string& m);

// ------------------------------------------------------------------------------ profiler
// PAMOPT_PROFILE=1: synchronise at phase marks and accumulate host wall time per phase
// (diagnostics only; never enabled in timed runs).
struct Prof {
  bool on = false;
  bool kt = false;        // per-kernel device time (events around every launch)
  bool kt_print = false;  // PAMOPT_PROFILE=2: print the tally at the end of each simplify
  struct Pending {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pend;
  std::map<std::string, double> kms;
  std::map<std::string, int64_t> kn;
  cudaEvent_t kbegin(cudaStream_t s) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    return e;
  }
  void kend(const char* name, cudaEvent_t a, cudaStream_t s) {
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, s);
    pend.push_back({name, a, b});
    if (pend.size() > 8192) kflush();
  }
  void kflush() {
    for (auto& p : pend) {
      cudaEventSynchronize(p.b);
      float ms_ = 0.f;
      cudaEventElapsedTime(&ms_, p.a, p.b);
      kms[p.name] += ms_;
      kn[p.name] += 1;
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    pend.clear();
  }
  std::map<std::string, double> ms;
  std::map<std::string, int64_t> n;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(cudaStream_t s, const char* name) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    ms[name] += std::chrono::duration<double, std::milli>(now - t).count();
    n[name] += 1;
    t = now;
  }
  void reset(cudaStream_t s) {
    if (!on) return;
    cudaStreamSynchronize(s);
    t = std::chrono::steady_clock::now();
  }
  void dump(const char* title) {
    if (kt && kt_print) {
      kflush();
      double tot = 0;
      for (auto& kv : kms) tot += kv.second;
      std::fprintf(stderr, "[pamopt kernels] %s device total %.2f ms\n", title, tot);
      for (auto& kv : kms)
        std::fprintf(stderr, "  %-34s %10.3f ms  %8lld launches\n", kv.first.c_str(), kv.second, (long long)kn[kv.first]);
      kms.clear();
      kn.clear();
    }
    if (!on) return;
    double tot = 0;
    for (auto& kv : ms) tot += kv.second;
    std::fprintf(stderr, "[pamopt profile] %s total %.2f ms\n", title, tot);
    for (auto& kv : ms)
      std::fprintf(stderr, "  %-22s %10.2f ms  %8lld calls\n", kv.first.c_str(), kv.second, (long long)n[kv.first]);
    ms.clear();
    n.clear();
  }
};

// ------------------------------------------------------------------------------ context
struct Ctx {
  Prof prof;
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  int num_sms = 148;
  // scratch reused across calls
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  // last remesh_host result
  std::vector<double> host_v;
  std::vector<int32_t> host_f;
  // a second stream for independent kernels of one step (fork / join through the two events),
  // created on first use
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // pinned landing zone for read_scalar (a pageable D2H copy stages through the driver)
  void* pin = nullptr;
  void* pinned_scratch() {
    if (!pin) PCU_CUDA(cudaMallocHost(&pin, 256));
    return pin;
  }
  cudaStream_t aux_stream() {
    if (!aux) {
      PCU_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
      PCU_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      PCU_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    return aux;
  }
  void release_aux() {
    if (!aux) return;
    cudaStreamSynchronize(aux);
    cudaEventDestroy(ev_fork);
    cudaEventDestroy(ev_join);
    cudaStreamDestroy(aux);
    aux = nullptr;
  }
};

// launches between construction and destruction go to the context's aux stream, which first
// waits for everything already queued on the main stream; the destructor makes the main stream
// wait for the aux work (fork / join)
struct AuxFork {
  Ctx& ctx;
  cudaStream_t main;
  explicit AuxFork(Ctx& c) : ctx(c), main(c.stream) {
    cudaStream_t a = ctx.aux_stream();
    PCU_CUDA(cudaEventRecord(ctx.ev_fork, main));
    PCU_CUDA(cudaStreamWaitEvent(a, ctx.ev_fork, 0));
    ctx.stream = a;
  }
  // back to the main stream for launches that run concurrently with the aux ones
  void to_main() { ctx.stream = main; }
  ~AuxFork() {
    ctx.stream = main;
    cudaEventRecord(ctx.ev_join, ctx.aux);
    cudaStreamWaitEvent(main, ctx.ev_join, 0);
  }
};

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

// stream-ordered device buffer
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) PCU_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), st));
  }
  // grow-only reallocation (contents not preserved)
  void ensure(size_t count, cudaStream_t st) {
    if (count > n || p == nullptr) alloc(count > 0 ? count : 1, st);
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  T* get() const { return p; }
  void memset(int v, cudaStream_t st) {
    if (n) PCU_CUDA(cudaMemsetAsync(p, v, n * sizeof(T), st));
  }
};

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 0x7fffffff) g = 0x7fffffff;
  return static_cast<unsigned>(g);
}

#define PCU_LAUNCH(ctx, kernel, grid, block, smem, ...)                       \
  do {                                                                        \
    cudaEvent_t pcu_ev_ = (ctx).prof.kt ? (ctx).prof.kbegin((ctx).stream) : nullptr; \
    kernel<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);           \
    if (pcu_ev_) (ctx).prof.kend(#kernel, pcu_ev_, (ctx).stream);              \
    ++(ctx).launches;                                                         \
    PCU_CUDA(cudaGetLastError());                                             \
  } while (0)

// ------------------------------------------------------------------- CUB-backed helpers
// exclusive scan of n elements (in -> out), returns nothing; out may alias in.
// several byte-value fills (memset semantics) in one launch; pointers 4-byte aligned
struct FillRange {
  void* p;
  uint64_t bytes;
  uint8_t byte;
};
constexpr int kMaxFillRanges = 8;
struct FillRanges {
  FillRange r[kMaxFillRanges];
  int n;
};
void fill_multi(Ctx& ctx, std::initializer_list<FillRange> ranges);
void fill_multi(Ctx& ctx, const FillRange* ranges, size_t count);
void exclusive_scan_u32(Ctx& ctx, const uint32_t* in, uint32_t* out, int64_t n);
void exclusive_scan_u64(Ctx& ctx, const uint64_t* in, uint64_t* out, int64_t n);
void sort_pairs_u64(Ctx& ctx, uint64_t* keys, int64_t n, int end_bit = 64);
// one-CTA sort for n <= 4096 (in may alias out); false (nothing launched) if n is larger
bool small_sort_u64(Ctx& ctx, const uint64_t* in, uint64_t* out, int64_t n);
template <class T>
T read_scalar(Ctx& ctx, const T* dptr) {
  static_assert(sizeof(T) <= 256, "read_scalar: value too large for the pinned scratch");
  T h;
  void* p = ctx.pinned_scratch();
  PCU_CUDA(cudaMemcpyAsync(p, dptr, sizeof(T), cudaMemcpyDeviceToHost, ctx.stream));
  PCU_CUDA(cudaStreamSynchronize(ctx.stream));
  std::memcpy(&h, p, sizeof(T));
  return h;
}

// ------------------------------------------------------------ aggregated counter bumps
// One atomic per group of converged lanes instead of one per lane: single-address counters
// (list appends) otherwise serialise in the L2 atomic unit.
__device__ __forceinline__ unsigned long long agg_inc(unsigned long long* ctr) {
  namespace cg = cooperative_groups;
  cg::coalesced_group g = cg::coalesced_threads();
  unsigned long long base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(ctr, static_cast<unsigned long long>(g.size()));
  return g.shfl(base, 0) + g.thread_rank();
}
__device__ __forceinline__ void agg_add(unsigned long long* ctr, unsigned long long v) {
  namespace cg = cooperative_groups;
  cg::coalesced_group g = cg::coalesced_threads();
  unsigned long long s = v;
  for (unsigned o = 1; o < g.size(); o <<= 1) {
    const unsigned long long t = g.shfl_down(s, o);
    if (g.thread_rank() + o < g.size()) s += t;
  }
  if (g.thread_rank() == 0) atomicAdd(ctr, s);
}
// same, for lanes that may target different counters (grouped by label)
__device__ __forceinline__ unsigned long long agg_inc_labeled(unsigned long long* ctr, unsigned label) {
  namespace cg = cooperative_groups;
  cg::coalesced_group g = cg::labeled_partition(cg::coalesced_threads(), label);
  unsigned long long base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(ctr, static_cast<unsigned long long>(g.size()));
  return g.shfl(base, 0) + g.thread_rank();
}

// --------------------------------------------------------------------- device geometry
struct D3 {
  double x, y, z;
};

__host__ __device__ __forceinline__ D3 d3(double x, double y, double z) { return D3{x, y, z}; }
__host__ __device__ __forceinline__ D3 sub(D3 a, D3 b) { return D3{a.x - b.x, a.y - b.y, a.z - b.z}; }
// (x0*y0 + x1*y1) + x2*y2 — the Eigen fixed-size redux order (oracle/eigen_shim)
__host__ __device__ __forceinline__ double dot(D3 a, D3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__host__ __device__ __forceinline__ double sqn(D3 a) { return dot(a, a); }
__host__ __device__ __forceinline__ D3 cross(D3 a, D3 b) {
  return D3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__host__ __device__ __forceinline__ D3 axpy(D3 a, double t, D3 d) {  // a + t*d
  return D3{a.x + t * d.x, a.y + t * d.y, a.z + t * d.z};
}

// point–segment squared distance (distance.cpp:10-21)
__device__ __forceinline__ double pseg_sq(D3 p, D3 a, D3 b) {
  const D3 ab = sub(b, a);
  const double denom = sqn(ab);
  double t = denom > 0.0 ? dot(sub(p, a), ab) / denom : 0.0;
  t = t < 0.0 ? 0.0 : (1.0 < t ? 1.0 : t);
  return sqn(sub(p, axpy(a, t, ab)));
}

// point–triangle squared distance (distance.cpp:26-79): face candidate then edges, strict '<'
__device__ __forceinline__ double ptri_sq(D3 p, D3 a, D3 b, D3 c) {
  const D3 n = cross(sub(b, a), sub(c, a));
  const double nn = sqn(n);
  double best = __longlong_as_double(0x7ff0000000000000ll);
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
      if (v >= 0.0 && w >= 0.0 && v + w <= 1.0) best = dist_n * dist_n / nn;
    }
  }
  const double e0 = pseg_sq(p, a, b);
  if (e0 < best) best = e0;
  const double e1 = pseg_sq(p, b, c);
  if (e1 < best) best = e1;
  const double e2 = pseg_sq(p, c, a);
  if (e2 < best) best = e2;
  return best;
}

// ------------------------------------------------------------- pinned exp and sigmoid
// exp(x) = p(r) * 2^k, k = floor(x log2e + 1/2), r = (x - k ln2_hi) - k ln2_lo,
// p = degree-13 Taylor polynomial (Horner), 2^k assembled from bits (two steps below
// 2^-1022).  The DMC sigmoid t' = 1/(1+exp(-beta(t-1/2))) is evaluated with
// this exact op sequence so patch vertices are reproducible bit for bit.
__device__ __forceinline__ double pow2i(int k) {
  return __longlong_as_double(static_cast<long long>(k + 1023) << 52);
}
__device__ __forceinline__ double det_exp(double x) {
  if (x != x) return x;
  if (x > 709.0) return __longlong_as_double(0x7ff0000000000000ll);
  if (x < -745.0) return 0.0;
  const double kd = floor(x * 1.4426950408889634 + 0.5);
  const int k = static_cast<int>(kd);
  const double r = (x - kd * 6.93147180369123816490e-01) - kd * 1.90821492927058770002e-10;
  double p = 1.6059043836821613e-10;
  p = p * r + 2.0876756987868100e-09;
  p = p * r + 2.5052108385441720e-08;
  p = p * r + 2.7557319223985888e-07;
  p = p * r + 2.7557319223985893e-06;
  p = p * r + 2.4801587301587302e-05;
  p = p * r + 1.9841269841269841e-04;
  p = p * r + 1.3888888888888889e-03;
  p = p * r + 8.3333333333333332e-03;
  p = p * r + 4.1666666666666664e-02;
  p = p * r + 1.6666666666666666e-01;
  p = p * r + 0.5;
  p = p * r + 1.0;
  p = p * r + 1.0;
  if (k >= -1022) return p * pow2i(k);
  return (p * pow2i(k + 600)) * pow2i(-600);
}
__device__ __forceinline__ double sigmoid_t(double t, double beta) {
  return 1.0 / (1.0 + det_exp(-beta * (t - 0.5)));
}

}  // namespace pcu

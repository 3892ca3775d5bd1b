// FFMA / DFMA issue-rate microbenchmark (the compute-pipe roofline denominators for the
// FP32 certificate filters and the FP64 decision arithmetic; MEASURED_PEAKS.json has bf16 only).
// Each thread runs 8 independent FMA chains (enough ILP to hide the pipe latency); the grid is
// 148 SMs x 8 blocks x 256 threads.  Prints one JSON line with TFLOP/s (2 flops per FMA).
#include <cstdio>
#include <cuda_runtime.h>

template <class T>
__global__ void k_fma(T* out, int iters, T a, T b) {
  T x[8];
  for (int k = 0; k < 8; ++k) x[k] = static_cast<T>(threadIdx.x + k);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  T s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == static_cast<T>(-1.2345)) out[0] = s;  // keep the chains alive
}

template <class T>
double run(int sms) {
  T* out;
  cudaMalloc(&out, sizeof(T));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  k_fma<T><<<blocks, threads>>>(out, 64, T(0.999), T(0.001));  // warm up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_fma<T><<<blocks, threads>>>(out, iters, T(0.999), T(0.001));
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double f32 = run<float>(sms), f64 = run<double>(sms);
  std::printf("{\"ffma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"sms\": %d, \"max_clock_mhz\": %.0f}\n", f32, f64, sms,
              clk / 1000.0);
  return 0;
}

// Measurement infrastructure (not on the hot path): the FP32-pipe and MUFU
// (XU) throughput of this GPU, measured with independent dependency chains,
// and the SM count / clock read from the device.  bench.py divides the
// raster kernels' algorithmic lane-ops by the measured FP32 lane-op rate
// ("verify both the FP32 and MUFU peaks with a
// microbenchmark ... use the measured values as denominators").
//
// Each thread runs kChains independent chains of kIters dependent
// operations; with 8 CTAs of 256 threads per SM every SMSP has 16 warps to
// hide the 4-cycle FMA / ~20-cycle MUFU latency, so the rate measured is the
// issue/pipe throughput.  Lane-ops: one FFMA = 1 per thread, one FFMA2 = 2.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sss.h"

namespace {

constexpr int kThreads = 256;
constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(kThreads) ffma_kernel(float* out, float a, float b) {
  float x[kChains];
  asm volatile("mov.b32 %0, %0;" : "+f"(a));  // register operands (the 3-register form real code uses)
  asm volatile("mov.b32 %0, %0;" : "+f"(b));
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __fmaf_rn(x[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678f) out[threadIdx.x] = s;  // keeps the chains alive
}

__global__ void __launch_bounds__(kThreads) ffma2_kernel(float* out, float a, float b) {
  float2 x[kChains];
  asm volatile("mov.b32 %0, %0;" : "+f"(a));
  asm volatile("mov.b32 %0, %0;" : "+f"(b));
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __ffma2_rn(x[c], A, B);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c].x + x[c].y;
  if (s == 12345.678f) out[threadIdx.x] = s;
}

template <int OP>  // 0 ex2, 1 lg2, 2 rcp (MUFU)
__global__ void __launch_bounds__(kThreads) mufu_kernel(float* out, float a) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = 0.5f + threadIdx.x * 1e-5f + c * 1e-3f;
  for (int i = 0; i < kIters / 4; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      float y;
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[c]));
      else if (OP == 1) asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[c]));
      else asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[c]));
      x[c] = y;  // stays in a range where every op is defined (ex2 of ~1, lg2 of ~2^.., rcp)
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678f) out[threadIdx.x] = s;
}

template <typename F>
double time_ms(F launch, int reps = 5) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();  // warm-up
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

}  // namespace

// out[0] = scalar FFMA lane-ops/s, out[1] = FFMA2 lane-ops/s (2 per lane),
// out[2] = MUFU ex2 ops/s, out[3] = lg2 ops/s, out[4] = rcp ops/s,
// out[5] = SM count, out[6] = SM clock (kHz, cudaDevAttrClockRate).
// Returns 0 on success.
extern "C" int sss_alu_peaks(double* out) {
  int dev = 0, sms = 0, clk = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* buf = nullptr;
  if (cudaMalloc(&buf, kThreads * sizeof(float)) != cudaSuccess) return 1;
  const int blocks = sms * 8;
  const double threads = (double)blocks * kThreads;
  const double ms_f = time_ms([&] { ffma_kernel<<<blocks, kThreads>>>(buf, 0.999f, 1e-3f); });
  const double ms_f2 = time_ms([&] { ffma2_kernel<<<blocks, kThreads>>>(buf, 0.999f, 1e-3f); });
  const double ms_e = time_ms([&] { mufu_kernel<0><<<blocks, kThreads>>>(buf, 0.f); });
  const double ms_l = time_ms([&] { mufu_kernel<1><<<blocks, kThreads>>>(buf, 0.f); });
  const double ms_r = time_ms([&] { mufu_kernel<2><<<blocks, kThreads>>>(buf, 0.f); });
  cudaFree(buf);
  if (cudaGetLastError() != cudaSuccess) return 1;
  const double fma_ops = threads * kChains * kIters;
  const double mufu_ops = threads * kChains * (kIters / 4);
  out[0] = fma_ops / (ms_f * 1e-3);
  out[1] = 2.0 * fma_ops / (ms_f2 * 1e-3);
  out[2] = mufu_ops / (ms_e * 1e-3);
  out[3] = mufu_ops / (ms_l * 1e-3);
  out[4] = mufu_ops / (ms_r * 1e-3);
  out[5] = sms;
  out[6] = clk;
  return 0;
}

// peak.cu -- measured FP64 / FP32 FMA-pipe peak of the local B200, the
// roofline denominator bench.py reports against (MEASURED_PEAKS.json has no
// FP64/FP32 entry). Sustained for ~`seconds` so the clock settles under the
// power cap like a long join does.
#include <chrono>
#include <string>

#include "../../include/tsdict_cuda.h"
#include "tsd_internal.h"

namespace {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// clk[0..1]: SM clock and global timer (ns) at the start and end of block 0
template <int CH>
__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b, unsigned long long* clk) {
  const bool rec = blockIdx.x == 0 && threadIdx.x == 0 && clk;
  if (rec) {
    clk[0] = clock64();
    clk[1] = gtimer();
  }
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __fma_rn(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
  if (rec) {
    clk[2] = clock64();
    clk[3] = gtimer();
  }
}

template <int CH>
__global__ void __launch_bounds__(256) k_ffma(float* out, int iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __fmaf_rn(x[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678f) out[0] = s;
}

}  // namespace

extern "C" int tsd_measure_peak_clock(int precision, double seconds, double* flops, double* sm_mhz) {
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return tsd::kCudaError;
  void* buf = nullptr;
  if (cudaMalloc(&buf, 128) != cudaSuccess) return tsd::kCudaError;
  unsigned long long* clk = reinterpret_cast<unsigned long long*>(static_cast<char*>(buf) + 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // 8 CTAs x 256 threads per SM (16 warps per scheduler) x 8 independent
  // chains: far more FMAs in flight than the pipe latency needs
  const int blocks = nsm * 8, threads = 256;
  const int CH = 8;
  auto launch = [&](int iters) {
    if (precision == 0)
      k_dfma<CH><<<blocks, threads>>>((double*)buf, iters, 0.999999, 1e-7, clk);
    else
      k_ffma<CH><<<blocks, threads>>>((float*)buf, iters, 0.999999f, 1e-7f);
  };
  int iters = 2000;
  launch(iters);
  cudaDeviceSynchronize();
  float ms = 0;
  // calibrate to ~50 ms per launch
  for (;;) {
    cudaEventRecord(e0);
    launch(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms > 40.0f || iters > (1 << 26)) break;
    iters *= 2;
  }
  const int reps = std::max(1, (int)(seconds * 1000.0 / ms));
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch(iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double fmas = (double)blocks * threads * CH * (double)iters * reps;
  *flops = 2.0 * fmas / (ms * 1e-3);
  if (sm_mhz) {  // the SM clock over the last launch (block 0), FP64 only
    unsigned long long h[4] = {0, 0, 0, 0};
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    *sm_mhz = (precision == 0 && h[3] > h[1]) ? (double)(h[2] - h[0]) / (double)(h[3] - h[1]) * 1e3 : 0.0;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? 0 : tsd::kCudaError;
}

extern "C" int tsd_measure_peak(int precision, double seconds, double* flops) {
  return tsd_measure_peak_clock(precision, seconds, flops, nullptr);
}

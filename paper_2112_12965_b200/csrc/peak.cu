// peak.cu -- measured FP64 / FP32 FMA-pipe peak of the local B200, the
// roofline denominator bench.py reports against (MEASURED_PEAKS.json has no
// FP64/FP32 entry). Sustained for ~`seconds` so the clock settles under the
// power cap like a long join does.
#include <chrono>
#include <string>

#include "../../include/tsdict_cuda.h"
#include "tsd_internal.h"

namespace {

template <int CH>
__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
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

extern "C" int tsd_measure_peak(int precision, double seconds, double* flops) {
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return tsd::kCudaError;
  void* buf = nullptr;
  if (cudaMalloc(&buf, 64) != cudaSuccess) return tsd::kCudaError;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = nsm * 4, threads = 256;
  const int CH = 8;
  auto launch = [&](int iters) {
    if (precision == 0)
      k_dfma<CH><<<blocks, threads>>>((double*)buf, iters, 0.999999, 1e-7);
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
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? 0 : tsd::kCudaError;
}

// Does an ALU / LSU instruction between DFMAs cost the FP64 pipe issue
// cycles on sm_100a? Per loop iteration: 16 independent DFMA + K extra
// instructions of one kind; reports DFMA warp-instructions per SMSP per
// clock (peak 0.5 if a DFMA occupies the FP64 pipe 2 cycles).
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_c[2];

template <int K, int KIND>
__global__ void __launch_bounds__(256) k_mix(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) x[c] = threadIdx.x * 1e-3 + c;
  unsigned y[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) y[c] = threadIdx.x + c;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      x[c] = __fma_rn(x[c], a, b);
      if (c < K) {
        if (KIND == 0) asm volatile("add.u32 %0, %0, 7;" : "+r"(y[c & 7]));               // ALU
        if (KIND == 1) asm volatile("{.reg .pred p; setp.ge.s32 p, %0, 99; selp.u32 %0, 1, %0, p;}" : "+r"(y[c & 7]));
        if (KIND == 2) asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;" : "+r"(y[c & 7])); // LSU
        if (KIND == 3) asm volatile("mul.lo.u32 %0, %0, 3;" : "+r"(y[c & 7]));             // FMA pipe (IMAD)
      }
    }
  }
  unsigned long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) s += x[c];
  unsigned ys = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) ys += y[c];
  if (s == 12345.678 || ys == 1234567u) out[0] = s + ys;
  if (blockIdx.x == 0 && threadIdx.x == 0) g_c[0] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 64);
  const int blocks = sms * 4, threads = 256, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * blocks * threads * 16.0 * iters / (ms * 1e-3) / 1e12;
    printf("%-24s %8.3f ms  %6.2f TFLOP/s DFMA  (%.3f of 37.2 nominal)\n", name, ms, tf, tf / 37.2);
  };
#define R(K, KIND, NAME) run(NAME, [&] { k_mix<K, KIND><<<blocks, threads>>>(d, iters, 0.999999, 1e-7); })
  R(0, 0, "dfma only");
  R(4, 0, "+4 iadd");
  R(8, 0, "+8 iadd");
  R(16, 0, "+16 iadd");
  R(8, 1, "+8 isetp/sel");
  R(16, 1, "+16 isetp/sel");
  R(4, 2, "+4 shfl");
  R(8, 2, "+8 shfl");
  R(8, 3, "+8 imad");
  R(16, 3, "+16 imad");
  return 0;
}

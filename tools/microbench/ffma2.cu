// FP32 / FP64 FMA-pipe rates on sm_100a for the operand forms the sweeps use:
// does a 3-register FFMA / FFMA2 / DFMA issue at the pipe's full rate, and
// what does the FP32 sweep step (8 pairs x 2 FFMA2 + 16 ISETP + vote) cost?
// Reports warp-instructions per SMSP per clock of the FMA-class instruction.
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ void opaque(u64& v) { asm volatile("" : "+l"(v)); }
__device__ __forceinline__ void opaquef(float& v) { asm volatile("" : "+f"(v)); }
__device__ __forceinline__ void opaqued(double& v) { asm volatile("" : "+d"(v)); }

__device__ __forceinline__ u64 pk(float a, float b) {
  return ((u64)__float_as_uint(b) << 32) | __float_as_uint(a);
}

// KIND 0: scalar FFMA, 3 registers (x = fma(y[c], d, x))       16 per iter
// KIND 1: scalar FFMA, immediate operand (x = fma(x, 0.999f, d)) 16 per iter
// KIND 2: FFMA2, 3 register pairs (Q = fma2(F[c], D, Q))        16 per iter
// KIND 3: the sweep pattern Q = fma2(G, E, fma2(F, D, Q)), 8 pairs: 16 per iter
// KIND 4: KIND 3 + 16 ISETP (or-chains) + vote + branch
// KIND 5: DFMA, 3 registers, the FP64 sweep pattern cov = fma(g, e, fma(f, d, cov)), 8 slots: 16 per iter
// KIND 6: DFMA with immediate-like constant operand (x = fma(x, a, b)) 16 per iter
template <int KIND>
__global__ void k_rate(float* out, int iters, float seed) {
  float fv[16];
  u64 F[8], G[8], Q[8];
  double df[8], dg[8], cv[8];
#pragma unroll
  for (int c = 0; c < 16; ++c) fv[c] = seed * (c + 1) + threadIdx.x * 1e-6f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    F[c] = pk(seed * c, seed + c);
    G[c] = pk(seed - c, seed * 0.5f * c);
    Q[c] = pk(threadIdx.x * 1e-6f, c * 1e-3f);
    df[c] = seed * c;
    dg[c] = seed + c;
    cv[c] = threadIdx.x * 1e-6 + c;
  }
  float dd = seed * 0.25f;
  u64 D = pk(seed * 1e-3f, seed * 2e-3f), E = pk(seed * 3e-3f, seed * 4e-3f);
  double de = seed * 1e-3, dh = seed * 2e-3;
  opaquef(dd);
  opaque(D);
  opaque(E);
  opaqued(de);
  opaqued(dh);
  int thr[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) thr[c] = 0x7f000000 + c;
  unsigned hits = 0;
  for (int i = 0; i < iters; ++i) {
    if (KIND == 0) {
#pragma unroll
      for (int c = 0; c < 16; ++c) fv[c] = __fmaf_rn(fv[(c + 1) & 15], dd, fv[c]);
    } else if (KIND == 1) {
#pragma unroll
      for (int c = 0; c < 16; ++c) fv[c] = __fmaf_rn(fv[c], 0.999f, dd);
    } else if (KIND == 2) {
#pragma unroll
      for (int c = 0; c < 8; ++c) Q[c] = fma2(F[c], D, Q[c]);
#pragma unroll
      for (int c = 0; c < 8; ++c) Q[c] = fma2(G[c], E, Q[c]);
    } else if (KIND == 3 || KIND == 4) {
#pragma unroll
      for (int c = 0; c < 8; ++c) Q[c] = fma2(G[c], E, fma2(F[c], D, Q[c]));
      if (KIND == 4) {
        bool p = false;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          p |= (int)(unsigned)Q[c] >= thr[c];
          p |= (int)(unsigned)(Q[c] >> 32) >= thr[c + 8];
        }
        if (__any_sync(0xffffffffu, p)) {
          ++hits;
#pragma unroll
          for (int c = 0; c < 8; ++c) Q[c] = 0;
        }
      }
    } else if (KIND == 5) {
#pragma unroll
      for (int c = 0; c < 8; ++c) cv[c] = __fma_rn(dg[c], de, __fma_rn(df[c], dh, cv[c]));
    } else if (KIND == 6) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        cv[c] = __fma_rn(cv[c], 0.999, de);
        df[c] = __fma_rn(df[c], 0.999, dh);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) s += fv[c];
#pragma unroll
  for (int c = 0; c < 8; ++c) s += __uint_as_float((unsigned)Q[c]) + (float)cv[c] + (float)df[c];
  if (s == 12345.678f || hits == 12345) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  auto run = [&](const char* name, int wps, auto launch) {
    const int blocks = sms * wps / 4;  // 128-thread blocks
    launch(blocks);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch(blocks);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_inst = (double)blocks * 4 * 16.0 * iters;  // 16 FMA-class per iteration per warp
    const double per_smsp_clk = warp_inst / (sms * 4.0) / (ms * 1e-3 * clk * 1e3);
    printf("%-44s warps/SM %2d: %8.3f ms  %.3f FMA-class warp-inst / SMSP / clk (at %d MHz)\n", name, wps, ms,
           per_smsp_clk, clk / 1000);
  };
#define R(KIND, NAME)                                                                             \
  for (int w : {16, 32})                                                                          \
    run(NAME, w, [&](int b) { k_rate<KIND><<<b, 128>>>(d, iters, 1.0001f); });
  R(0, "FFMA 3-reg");
  R(1, "FFMA imm");
  R(2, "FFMA2 3-reg pairs");
  R(3, "FFMA2 sweep pattern (2 chained per pair)");
  R(4, "FFMA2 sweep pattern + 16 ISETP + vote");
  R(5, "DFMA sweep pattern (3-reg)");
  R(6, "DFMA imm/const operand");
  return 0;
}

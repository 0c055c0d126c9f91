// Pipe-throughput microbenchmarks for the join kernel design (sm_100a).
// Measures DFMA, DMMA (m8n8k4 f64), DFMA+DMMA concurrency, FFMA, FFMA2, DSETP,
// and DFMA mixed with ALU ops. Prints one line per test: ops/s and derived
// per-SM-per-clock rates using a clock64/globaltimer sample.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_clk[2];

template <int CH>
__global__ void dfma_k(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  unsigned long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = t1 - t0; }
}

template <int CH>
__global__ void ffma_k(float* out, int iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678f) out[0] = s;
}

template <int CH>
__global__ void ffma2_k(float* out, int iters, float a, float b) {
  unsigned long long x[CH];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&av);
  unsigned long long B = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int c = 0; c < CH; ++c) { float2 t = make_float2(threadIdx.x * 1e-3f + c, c); x[c] = *reinterpret_cast<unsigned long long*>(&t); }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(A), "l"(B));
  }
  unsigned long long s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= x[c];
  if (s == 12345) out[0] = 1.f;
}

template <int CH>
__global__ void dmma_k(double* out, int iters) {
  double acc[CH][2];
  double av = threadIdx.x * 1e-3, bv = 0.999;
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c][0] = c; acc[c][1] = -c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

// DFMA chains plus DMMA in the same warp: per iteration CH DFMA + M DMMA
template <int CH, int M>
__global__ void mix_k(double* out, int iters, double a, double b) {
  double x[CH];
  double acc[M][2];
  double av = threadIdx.x * 1e-3, bv = 0.999;
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
#pragma unroll
  for (int c = 0; c < M; ++c) { acc[c][0] = c; acc[c][1] = -c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
#pragma unroll
    for (int c = 0; c < M; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
#pragma unroll
  for (int c = 0; c < M; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

// 3 DFMA + 1 setp.ge.or.s32 on the high word per chain step (the join cell shape)
template <int CH>
__global__ void cell_k(double* out, int iters, double a, double b, int thr) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  unsigned hit = 0;
  for (int i = 0; i < iters; ++i) {
    unsigned p = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      x[c] = fma(x[c], a, b);
      x[c] = fma(x[c], b, a);
      double s = fma(x[c], a, 1.0);
      int hi = __double2hiint(s);
      asm volatile("{.reg .pred q; setp.ne.u32 q, %0, 0; setp.ge.or.s32 q, %1, %2, q; selp.u32 %0, 1, 0, q;}" : "+r"(p) : "r"(hi), "r"(thr));
    }
    if (p) hit++;
  }
  double s = hit;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void dsetp_k(double* out, int iters, double a) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  unsigned cnt = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) cnt += (x[c] > a) ? 1u : 0u;
    a += 1e-30;
  }
  if (cnt == 1234567) out[0] = cnt;
}

int main() {
  int dev = 0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  int sms = pr.multiProcessorCount;
  printf("device %s SMs %d\n", pr.name, sms);
  double* d; float* f; CK(cudaMalloc(&d, 64)); CK(cudaMalloc(&f, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, double ops_per_launch, auto launch) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("%-28s %8.3f ms  %9.3f Tops/s  %s\n", name, best, ops_per_launch / (best * 1e-3) / 1e12, err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
  const int blocks = sms * 4, threads = 256;
  const double thr = double(blocks) * threads;
  int it = 20000;
  run("dfma ch8 (FMA ops)", thr * it * 8, [&] { dfma_k<8><<<blocks, threads>>>(d, it, 0.999, 1e-3); });
  run("dfma ch4 (FMA ops)", thr * it * 4, [&] { dfma_k<4><<<blocks, threads>>>(d, it, 0.999, 1e-3); });
  run("dfma ch8 2blk/SM", double(sms*2)*threads * it * 8, [&] { dfma_k<8><<<sms*2, threads>>>(d, it, 0.999, 1e-3); });
  run("ffma ch8 (FMA ops)", thr * it * 8, [&] { ffma_k<8><<<blocks, threads>>>(f, it, 0.999f, 1e-3f); });
  run("ffma2 ch8 (FMA ops)", thr * it * 16, [&] { ffma2_k<8><<<blocks, threads>>>(f, it, 0.999f, 1e-3f); });
  int itm = 4000;
  run("dmma ch4 (FMA ops)", thr / 32 * itm * 4 * 256, [&] { dmma_k<4><<<blocks, threads>>>(d, itm); });
  run("dmma ch8 (FMA ops)", thr / 32 * itm * 8 * 256, [&] { dmma_k<8><<<blocks, threads>>>(d, itm); });
  run("mix 8dfma+1dmma (FMA ops)", thr * it / 4 * 8 + thr / 32 * (it / 4) * 256, [&] { mix_k<8, 1><<<blocks, threads>>>(d, it / 4, 0.999, 1e-3); });
  run("mix 8dfma+2dmma (FMA ops)", thr * it / 4 * 8 + thr / 32 * (it / 4) * 512, [&] { mix_k<8, 2><<<blocks, threads>>>(d, it / 4, 0.999, 1e-3); });
  run("mix 16dfma+2dmma (FMA ops)", thr * it / 4 * 16 + thr / 32 * (it / 4) * 512, [&] { mix_k<16, 2><<<blocks, threads>>>(d, it / 4, 0.999, 1e-3); });
  run("cell 3dfma+isetp (cells)", thr * it / 4 * 8, [&] { cell_k<8><<<blocks, threads>>>(d, it / 4, 0.999, 1e-3, 0x7ff00000); });
  run("dsetp ch8 (setp ops)", thr * it * 8, [&] { dsetp_k<8><<<blocks, threads>>>(d, it, 0.5); });
  unsigned long long clk; CK(cudaMemcpyFromSymbol(&clk, g_clk, 8));
  // clock estimate: time one block-per-SM dfma run and compare clock64 delta
  cudaEventRecord(e0); dfma_k<8><<<sms, 256>>>(d, it, 0.999, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); CK(cudaMemcpyFromSymbol(&clk, g_clk, 8));
  printf("clock estimate: %llu cycles in <= %.3f ms -> >= %.0f MHz\n", clk, ms, clk / (ms * 1e3));
  return 0;
}

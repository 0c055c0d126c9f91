// Synthetic replica of one sweep step of k_join_f64 (R = 8 slots/lane) to
// find the inner-loop bottleneck. VAR bits: 1 = shuffle + lane-0 select,
// 2 = high-word test + predicate tree + vote + (never taken) branch,
// 4 = shared-memory loads/store of the step, 8 = deferred-vote style (vote of
// step k resolved after step k+1's DFMAs, via two register sets).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double shfl_up1(double v) {
  int lo = __double2loint(v), hi = __double2hiint(v);
  asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;\n" : "+r"(lo));
  asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;\n" : "+r"(hi));
  return __hiloint2double(hi, lo);
}
__device__ __forceinline__ bool vote_any(bool p) {
  unsigned r;
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n vote.sync.any.pred q, q, -1;\n selp.u32 %0, 1, 0, q;\n}\n"
               : "=r"(r) : "r"((unsigned)p));
  return r != 0;
}

template <int R, int VAR, int MINB>
__global__ void __launch_bounds__(64, MINB) k(double* out, int steps, int* hits) {
  __shared__ double sm[2][16][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double P[R], dfa[R], dga[R];
  int thr[R];
  for (int r = 0; r < R; ++r) {
    P[r] = lane * 0.01 + r;
    dfa[r] = 1e-3 * (r + 1) * (1.0 + 1e-9 * threadIdx.x);
    dga[r] = -1e-3 * (r + 2) * (1.0 + 1e-9 * blockIdx.x);
    thr[r] = 0x7fe00000;
  }
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) { sm[0][0][i] = 1e-4 * i; }
  __syncthreads();
  double dfb = 0.5, dgb = 0.25, e = 1.0;
  int cnt = 0;
  bool pend = false;
  double bKd[R];
  for (int r = 0; r < R; ++r) bKd[r] = 1e300 * (1.0 + 1e-9 * threadIdx.x);
  for (int s = 0; s < steps; s += R) {
    if (VAR & 64) {  // per-block threshold: thr = hi(bestK * min column norm of the block)
      const double nmin = sm[w][s & 7][lane & 7] + 1.0;
#pragma unroll
      for (int r = 0; r < R; ++r) thr[r] = __double2hiint((VAR & 128 ? sm[w][r][lane] : bKd[r]) * nmin);
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int ph = (R - u) & (R - 1);
      if (VAR & 4) {
        const double2 dd = *reinterpret_cast<const double2*>(&sm[w][u & 15][2 * (s & 15)]);
        dfb = dd.x; dgb = dd.y;
        e = sm[w][(u ^ 1) & 15][lane & 7];
        sm[w][u & 15][32 + (lane & 7)] = P[ph];
      }
      if (VAR & 1) {
        const double in = shfl_up1(P[ph]);
        P[ph] = lane == 0 ? e : in;
      }
      if (VAR & 16) {  // normalised recurrence: 3 FP64 ops per cell, one on the chain
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double& c = P[(r + ph) & (R - 1)];
          const double t = __fma_rn(dfa[r], dgb, dga[r] * dfb);
          c = __fma_rn(c, 0.999999, t);
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double& c = P[(r + ph) & (R - 1)];
          c = __fma_rn(dfa[r], dgb, c);
          c = __fma_rn(dga[r], dfb, c);
        }
      }
      if (VAR & 8) {  // deferred: resolve the previous step's vote after this step's math
        if (pend) {
          ++cnt;
#pragma unroll
          for (int r = 0; r < R; ++r) thr[r] += 1;
        }
        bool p[R];
#pragma unroll
        for (int r = 0; r < R; ++r) p[r] = __double2hiint(P[(r + ph) & (R - 1)]) >= thr[r];
#pragma unroll
        for (int ww = 1; ww < R; ww <<= 1)
#pragma unroll
          for (int r = 0; r + ww < R; r += 2 * ww) p[r] = p[r] | p[r + ww];
        pend = vote_any(p[0]);
      } else if (VAR & 2) {
        bool p[R];
#pragma unroll
        for (int r = 0; r < R; ++r) p[r] = __double2hiint(P[(r + ph) & (R - 1)]) >= thr[r];
#pragma unroll
        for (int ww = 1; ww < R; ww <<= 1)
#pragma unroll
          for (int r = 0; r + ww < R; r += 2 * ww) p[r] = p[r] | p[r + ww];
        if (vote_any(p[0])) {
          ++cnt;
          if (VAR & 32) {  // big inline body (like the exact update), never taken
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const double K = P[(r + ph) & (R - 1)] * dgb;
              if (K > (double)thr[r]) { thr[r] = __double2hiint(K) - 1; sm[w][r][lane] = K; }
              if (K < -(double)thr[r]) { thr[r] = __double2hiint(K) + 1; sm[w][r][lane + 32] = K; }
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) thr[r] += 1;
          }
        }
      }
    }
  }
  double acc = 0;
  for (int r = 0; r < R; ++r) acc += P[r];
  if (acc == 1234.5) out[0] = acc;
  if (cnt) atomicAdd(hits, cnt);
}

template <int R, int VAR, int MINB>
void run(const char* name, int blocks_per_sm) {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* out; int* hits;
  cudaMalloc(&out, 64); cudaMalloc(&hits, 4); cudaMemset(hits, 0, 4);
  const int steps = 1 << 14;
  const int grid = nsm * blocks_per_sm;
  k<R, VAR, MINB><<<grid, 64>>>(out, steps, hits);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<R, VAR, MINB><<<grid, 64>>>(out, steps, hits);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double cells = (double)grid * 64 * R * steps;
  int h; cudaMemcpy(&h, hits, 4, cudaMemcpyDeviceToHost);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k<R, VAR, MINB>);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<R, VAR, MINB>, 64, 0);
  printf("R=%2d regs=%3d occ=%d spill=%zu ", R, fa.numRegs, occ, fa.localSizeBytes);
  printf("%-34s warps/SM=%2d  %.3f Tcell/s  (%.1f%% of 17T DFMA/2)  hits=%d %s\n", name, 2 * blocks_per_sm,
         cells / ms / 1e9, cells / ms / 1e9 / 8.5 * 100, h, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<8, 7 | 64, 8>("R8 2-op +blockthr +shfl +test/vote +smem", 8);
  run<8, 13 | 64, 8>("R8 2-op +blockthr +shfl +DEFERRED +smem", 8);
  run<8, 7 | 64 | 128, 8>("R8 smem-bK", 8);
  run<16, 7 | 64 | 128, 6>("R16 smem-bK MINB6", 6);
  run<16, 7 | 64 | 128, 5>("R16 smem-bK MINB5", 5);
  run<16, 7 | 64 | 128, 4>("R16 smem-bK MINB4", 4);
  run<16, 7 | 64, 5>("R16 reg-bK MINB5", 5);
  run<16, 13 | 64 | 128, 5>("R16 smem-bK DEFERRED MINB5", 5);
  run<16, 13 | 64 | 128, 4>("R16 smem-bK DEFERRED MINB4", 4);
  run<16, 0, 6>("R16 dfma only", 6);
  return 0;
}

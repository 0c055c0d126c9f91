// Latency microbenchmarks (single warp, dependent chains): DFMA, DMUL, SHFL, FSEL+SHFL, VOTE+BRA loop.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* o, int n, double a, double b, long long* cyc) {
  double x = threadIdx.x; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); x = __fma_rn(x, a, b); }
  long long t1 = clock64(); o[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = (t1 - t0) / (4LL * n);
}
__global__ void k_dmul(double* o, int n, double a, long long* cyc) {
  double x = threadIdx.x + 1; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x * a; x = x * a; x = x * a; x = x * a; }
  long long t1 = clock64(); o[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = (t1 - t0) / (4LL * n);
}
__global__ void k_shfl(double* o, int n, long long* cyc) {
  int x = threadIdx.x; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __shfl_up_sync(~0u, x, 1) + 1; x = __shfl_up_sync(~0u, x, 1) + 1; }
  long long t1 = clock64(); o[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = (t1 - t0) / (2LL * n);
}
__global__ void k_vote(double* o, int n, double a, long long* cyc) {
  double x = threadIdx.x; int cnt = 0; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __fma_rn(x, a, 1e-9); if (__any_sync(~0u, __double2hiint(x) > 0x7fe00000)) { cnt++; x = 0; } }
  long long t1 = clock64(); o[threadIdx.x] = x + cnt; if (threadIdx.x == 0) *cyc = (t1 - t0) / n;
}
__global__ void k_lds(double* o, int n, long long* cyc) {
  __shared__ int s[1024]; for (int i = threadIdx.x; i < 1024; i += 32) s[i] = (i + 1) & 1023;
  __syncwarp(); int x = threadIdx.x; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = s[x]; x = s[x]; }
  long long t1 = clock64(); o[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = (t1 - t0) / (2LL * n);
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMallocManaged(&c, 8);
  const int n = 10000;
  k_dfma<<<1, 32>>>(o, n, 0.9999, 1e-7, c); cudaDeviceSynchronize(); k_dfma<<<1, 32>>>(o, n, 0.9999, 1e-7, c); cudaDeviceSynchronize(); printf("DFMA latency %lld cycles\n", *c);
  k_dmul<<<1, 32>>>(o, n, 0.9999, c); cudaDeviceSynchronize(); printf("DMUL latency %lld\n", *c);
  k_shfl<<<1, 32>>>(o, n, c); cudaDeviceSynchronize(); printf("SHFL+IADD latency %lld\n", *c);
  k_vote<<<1, 32>>>(o, n, 0.9999, c); cudaDeviceSynchronize(); printf("DFMA+VOTE+BRA loop %lld\n", *c);
  k_lds<<<1, 32>>>(o, n, c); cudaDeviceSynchronize(); printf("LDS latency %lld\n", *c);
  return 0;
}

// dprofile.cu -- distance profiles of one query window against every window
// of a series on sm_100a (reference profiles.hpp:164-260).
//
// distance_profile_naive (profiles.hpp:164-181) is znorm_distance
// (series.hpp:166-204) per window: Kahan sums of both windows, a two-pass
// variance and a Kahan covariance, the constancy threshold of the PAIR's
// largest magnitude. One thread per window evaluates exactly that sequence of
// IEEE operations with explicitly rounded adds and multiplies (no FMA
// contraction), so the values are bit-identical to the reference compiled
// without -march (CMakeLists.txt:3-10).
//
// distance_profile_mass (profiles.hpp:186-260) takes the series' window
// statistics and normalises sliding dot products. The reference forms the dot
// products with one FFT convolution (~1e-5 round-off near correlation 1,
// :252-257); here they are exact FP64 dot products of the centred query
// against the centred window (the 1 x n slice of the join, m FMAs per window,
// query staged in shared memory), with MASS's conventions kept: constant
// query -> 0 to constant windows and sqrt(2m) to the rest (:216-222),
// constant window -> sqrt(2m) (:243-246), the origin entry by znorm_distance
// (:252-257).
#include <cuda_runtime.h>

#include <cstdint>

#include "tsd_common.cuh"
#include "tsd_internal.h"

namespace tsd {
namespace {

constexpr int DB = 256;

struct KahanD {  // series.hpp:50-60, every operation rounded on its own
  double sum = 0.0, comp = 0.0;
  __device__ __forceinline__ void add(double x) {
    const double y = __dsub_rn(x, comp);
    const double t = __dadd_rn(sum, y);
    comp = __dsub_rn(__dsub_rn(t, sum), y);
    sum = t;
  }
};

__device__ __forceinline__ double constancy_threshold_d(double max_abs) {  // series.hpp:75-77
  return __dmul_rn(1e-8, max_abs > 1.0 ? max_abs : 1.0);
}

__device__ __forceinline__ double corr_to_dist_rn(double rho, double md) {  // series.hpp:153-161
  if (rho > 1.0) rho = 1.0;
  if (rho < -1.0) rho = -1.0;
  double d = __dsqrt_rn(__dmul_rn(__dmul_rn(2.0, md), __dsub_rn(1.0, rho)));
  const double dmax = __dmul_rn(2.0, __dsqrt_rn(md));
  if (d < 0.0) d = 0.0;
  if (d > dmax) d = dmax;
  return d;
}

// znorm_distance(q, w) with q's Kahan mean / variance and max |q| precomputed
// (they are the same sequence of operations for every window)
__device__ double znorm_window(const double* __restrict__ q, double mu_q, double va_q, double maxq,
                               const double* __restrict__ w, int m) {
  const double md = (double)m;
  double max_abs = maxq;
  KahanD sb;
  for (int i = 0; i < m; ++i) {
    const double b = w[i];
    sb.add(b);
    max_abs = fmax(max_abs, fabs(b));
  }
  const double mu_b = __ddiv_rn(sb.sum, md);
  KahanD vb, cv;
  for (int i = 0; i < m; ++i) {
    const double da = __dsub_rn(q[i], mu_q), db = __dsub_rn(w[i], mu_b);
    vb.add(__dmul_rn(db, db));
    cv.add(__dmul_rn(da, db));
  }
  const double sd_a = __dsqrt_rn(fmax(0.0, __ddiv_rn(va_q, md)));
  const double sd_b = __dsqrt_rn(fmax(0.0, __ddiv_rn(vb.sum, md)));
  const double eps = constancy_threshold_d(max_abs);
  const bool fa = sd_a < eps, fb = sd_b < eps;
  if (fa && fb) return 0.0;
  if (fa || fb) return __dsqrt_rn(__dmul_rn(2.0, md));
  const double rho = __ddiv_rn(cv.sum, __dmul_rn(md, __dmul_rn(sd_a, sd_b)));
  return corr_to_dist_rn(rho, md);
}

__global__ void __launch_bounds__(DB) k_dprof_naive(const double* __restrict__ x, int64_t cnt, int m,
                                                    const double* __restrict__ q, double mu_q, double va_q,
                                                    double maxq, double* __restrict__ out) {
  extern __shared__ double sq[];
  for (int t = threadIdx.x; t < m; t += DB) sq[t] = q[t];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * DB + threadIdx.x;
  if (i >= cnt) return;
  out[i] = znorm_window(sq, mu_q, va_q, maxq, x + i, m);
}

__global__ void __launch_bounds__(DB) k_dprof_mass(const double* __restrict__ x, int64_t cnt, int m,
                                                   const double* __restrict__ q, double mu_q, double va_q,
                                                   double maxq, double invn_q, int const_query,
                                                   const double* __restrict__ means, const double* __restrict__ invn,
                                                   const uint8_t* __restrict__ cmask, int64_t origin,
                                                   double* __restrict__ out) {
  extern __shared__ double sm[];
  double* sq = sm;       // raw query (origin entry)
  double* sc = sm + m;   // centred query
  for (int t = threadIdx.x; t < m; t += DB) {
    sq[t] = q[t];
    sc[t] = q[t] - mu_q;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * DB + threadIdx.x;
  if (i >= cnt) return;
  const double md = (double)m, far = sqrt(2.0 * md);
  double d;
  if (const_query) {
    d = cmask[i] ? 0.0 : far;  // profiles.hpp:216-222
  } else if (cmask[i]) {
    d = far;  // :243-246
  } else if (i == origin) {
    d = znorm_window(sq, mu_q, va_q, maxq, x + i, m);  // :252-257
  } else {
    const double c = means[i];
    double acc = 0.0;
    for (int t = 0; t < m; ++t) acc = __fma_rn(sc[t], x[i + t] - c, acc);
    d = corr_to_dist(acc * invn[i] * invn_q, md);  // :247-248
  }
  out[i] = d;
}

}  // namespace

int distance_profile_device(const double* d_x, int64_t n, const double* d_q, int m, const QueryMoments& qm,
                            const double* d_means, const double* d_invn, const uint8_t* d_cmask, int64_t origin,
                            double* d_out, cudaStream_t st) {
  const int64_t cnt = n - m + 1;
  const unsigned grid = (unsigned)((cnt + DB - 1) / DB);
  if (!d_means) {  // naive
    const size_t smem = sizeof(double) * (size_t)m;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_dprof_naive, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return kCudaError;
    k_dprof_naive<<<grid, DB, smem, st>>>(d_x, cnt, m, d_q, qm.mu, qm.var_sum, qm.max_abs, d_out);
  } else {
    const size_t smem = 2 * sizeof(double) * (size_t)m;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k_dprof_mass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return kCudaError;
    k_dprof_mass<<<grid, DB, smem, st>>>(d_x, cnt, m, d_q, qm.mu, qm.var_sum, qm.max_abs, qm.invn,
                                         qm.constant ? 1 : 0, d_means, d_invn, d_cmask, origin, d_out);
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kCudaError;
}

}  // namespace tsd

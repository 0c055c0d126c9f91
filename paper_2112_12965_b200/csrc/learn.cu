// learn.cu -- device kernels of the greedy dictionary-learning loop
// (learn_dictionary, dictionary.hpp:279-316).
//
// Per pick the reference (1) takes the argmin of the processed profile P - S
// over unmasked windows (first minimum wins), (2) masks the pick's
// neighbourhood, (3) computes the distance profile of the picked window by
// MASS (profiles.hpp:186-260) and folds it in, S = min(S, Sp), and (4) checks
// its stop rule. (1), (3) and the error-rule max run here; the select_state
// bookkeeping (context intervals, merge, stored samples) stays on the host
// (capi.cu), exactly as the reference keeps it.
//
// The distance profile is the 1 x n slice of the join: an exact FP64 direct
// dot product per window (m FMAs, no FFT), which removes MASS's ~1e-5 round-
// off near correlation 1 (profiles.hpp:252-257) while keeping its rules:
// constant query -> 0 to constant windows, sqrt(2m) otherwise; constant
// window -> sqrt(2m); the origin entry is the exact znorm_distance (computed
// on the host by the reference's algorithm and passed in).
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "tsd_common.cuh"
#include "tsd_internal.h"

namespace tsd {
namespace {

constexpr int LB = 256;  // threads per block of the reductions

struct ValIdx {
  double v;
  long long i;
};

__device__ __forceinline__ bool vi_less(double va, long long ia, double vb, long long ib) {
  return va < vb || (va == vb && ia < ib);
}

// lexicographic (value, index) minimum over unmasked windows of P - S
__global__ void __launch_bounds__(LB) k_argmin_partial(const double* __restrict__ P, const double* __restrict__ S,
                                                       const uint8_t* __restrict__ mask, int64_t cnt,
                                                       ValIdx* __restrict__ part) {
  double bv = 0.0;
  long long bi = -1;
  for (int64_t i = (int64_t)blockIdx.x * LB + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * LB) {
    if (mask[i]) continue;
    const double v = P[i] - S[i];
    if (bi < 0 || v < bv) {  // increasing i per thread: strict < keeps the first
      bv = v;
      bi = i;
    }
  }
  __shared__ ValIdx sh[LB];
  sh[threadIdx.x] = ValIdx{bv, bi};
  __syncthreads();
  for (int s = LB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const ValIdx o = sh[threadIdx.x + s];
      const ValIdx c = sh[threadIdx.x];
      if (o.i >= 0 && (c.i < 0 || vi_less(o.v, o.i, c.v, c.i))) sh[threadIdx.x] = o;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(LB) k_argmin_final(const ValIdx* __restrict__ part, int np, ValIdx* __restrict__ out) {
  ValIdx b{0.0, -1};
  for (int k = threadIdx.x; k < np; k += LB) {
    const ValIdx o = part[k];
    if (o.i >= 0 && (b.i < 0 || vi_less(o.v, o.i, b.v, b.i))) b = o;
  }
  __shared__ ValIdx sh[LB];
  sh[threadIdx.x] = b;
  __syncthreads();
  for (int s = LB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const ValIdx o = sh[threadIdx.x + s];
      const ValIdx c = sh[threadIdx.x];
      if (o.i >= 0 && (c.i < 0 || vi_less(o.v, o.i, c.v, c.i))) sh[threadIdx.x] = o;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// max over all of S (dictionary.hpp:306-307 scans every index)
__global__ void __launch_bounds__(LB) k_max_partial(const double* __restrict__ S, int64_t cnt, double* __restrict__ part) {
  double b = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * LB + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * LB) b = fmax(b, S[i]);
  __shared__ double sh[LB];
  sh[threadIdx.x] = b;
  __syncthreads();
  for (int s = LB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(LB) k_max_final(const double* __restrict__ part, int np, double* __restrict__ out) {
  double b = 0.0;
  for (int k = threadIdx.x; k < np; k += LB) b = fmax(b, part[k]);
  __shared__ double sh[LB];
  sh[threadIdx.x] = b;
  __syncthreads();
  for (int s = LB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// Sp[i] for every window i, folded into S (first pick: S = Sp).
// qc: the picked window minus its mean (m doubles).
__global__ void __launch_bounds__(LB) k_dprof_fold(const double* __restrict__ x, const double* __restrict__ mu,
                                                   const double* __restrict__ invn, const uint8_t* __restrict__ flag,
                                                   int64_t cnt, int m, const double* __restrict__ qc, double invn_q,
                                                   int const_query, int64_t origin, double origin_val, int first,
                                                   double* __restrict__ S) {
  extern __shared__ double sq[];
  for (int t = threadIdx.x; t < m; t += LB) sq[t] = qc[t];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * LB + threadIdx.x;
  if (i >= cnt) return;
  const double far = sqrt(2.0 * (double)m);
  const bool flat = (flag[i] & 2) != 0;
  double d;
  if (const_query) {
    d = flat ? 0.0 : far;  // profiles.hpp:216-222
  } else if (flat) {
    d = far;  // :243-246
  } else if (i == origin) {
    d = origin_val;  // :252-257
  } else {
    const double c = mu[i];
    double acc = 0.0;
    for (int t = 0; t < m; ++t) acc = __fma_rn(sq[t], x[i + t] - c, acc);
    d = corr_to_dist(acc * invn[i] * invn_q, m);  // :247-248
  }
  S[i] = first ? d : fmin(S[i], d);  // dictionary.hpp:298-303
}

// argmax over unsuppressed finite values, first maximum wins
// (find_discords' next_peak, dict_join.hpp:61-70)
__device__ __forceinline__ bool vi_more(double va, long long ia, double vb, long long ib) {
  return va > vb || (va == vb && ia < ib);
}

__global__ void __launch_bounds__(LB) k_argmax_partial(const double* __restrict__ vals, const uint8_t* __restrict__ sup,
                                                       int64_t cnt, ValIdx* __restrict__ part) {
  double bv = 0.0;
  long long bi = -1;
  for (int64_t i = (int64_t)blockIdx.x * LB + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * LB) {
    const double v = vals[i];
    if (sup[i] || !isfinite(v)) continue;
    if (bi < 0 || v > bv) {
      bv = v;
      bi = i;
    }
  }
  __shared__ ValIdx sh[LB];
  sh[threadIdx.x] = ValIdx{bv, bi};
  __syncthreads();
  for (int s = LB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const ValIdx o = sh[threadIdx.x + s];
      const ValIdx c = sh[threadIdx.x];
      if (o.i >= 0 && (c.i < 0 || vi_more(o.v, o.i, c.v, c.i))) sh[threadIdx.x] = o;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(LB) k_argmax_final(const ValIdx* __restrict__ part, int np, ValIdx* __restrict__ out) {
  ValIdx b{0.0, -1};
  for (int k = threadIdx.x; k < np; k += LB) {
    const ValIdx o = part[k];
    if (o.i >= 0 && (b.i < 0 || vi_more(o.v, o.i, b.v, b.i))) b = o;
  }
  __shared__ ValIdx sh[LB];
  sh[threadIdx.x] = b;
  __syncthreads();
  for (int s = LB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const ValIdx o = sh[threadIdx.x + s];
      const ValIdx c = sh[threadIdx.x];
      if (o.i >= 0 && (c.i < 0 || vi_more(o.v, o.i, c.v, c.i))) sh[threadIdx.x] = o;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

}  // namespace

int discord_peaks(const double* d_vals, int64_t cnt, int m, int64_t want, uint8_t* d_sup, void* d_scratch,
                  std::vector<int64_t>& at, std::vector<double>& score, cudaStream_t st) {
  const int np = (int)std::min<int64_t>(592, (cnt + LB - 1) / LB);
  ValIdx* part = reinterpret_cast<ValIdx*>(d_scratch);
  ValIdx* out = part + 592;
  const int64_t excl = m / 2;
  if (cudaMemsetAsync(d_sup, 0, cnt, st) != cudaSuccess) return kCudaError;
  at.clear();
  score.clear();
  while ((int64_t)at.size() < want) {
    k_argmax_partial<<<np, LB, 0, st>>>(d_vals, d_sup, cnt, part);
    k_argmax_final<<<1, LB, 0, st>>>(part, np, out);
    ValIdx h;
    if (cudaMemcpyAsync(&h, out, sizeof(ValIdx), cudaMemcpyDeviceToHost, st) != cudaSuccess) return kCudaError;
    if (cudaStreamSynchronize(st) != cudaSuccess) return kCudaError;
    if (h.i < 0) break;
    at.push_back(h.i);
    score.push_back(h.v);
      const int64_t lo = h.i >= excl ? h.i - excl : 0, hi = std::min<int64_t>(cnt, h.i + excl + 1);  // :80-84
    if (cudaMemsetAsync(d_sup + lo, 1, hi - lo, st) != cudaSuccess) return kCudaError;
  }
  return kOk;
}

int learn_argmin(const double* d_P, const double* d_S, const uint8_t* d_mask, int64_t cnt, void* d_scratch,
                 double* h_val, int64_t* h_idx, cudaStream_t st) {
  const int np = (int)std::min<int64_t>(592, (cnt + LB - 1) / LB);
  ValIdx* part = reinterpret_cast<ValIdx*>(d_scratch);
  ValIdx* out = part + 592;
  k_argmin_partial<<<np, LB, 0, st>>>(d_P, d_S, d_mask, cnt, part);
  k_argmin_final<<<1, LB, 0, st>>>(part, np, out);
  ValIdx h;
  if (cudaMemcpyAsync(&h, out, sizeof(ValIdx), cudaMemcpyDeviceToHost, st) != cudaSuccess) return kCudaError;
  if (cudaStreamSynchronize(st) != cudaSuccess) return kCudaError;
  *h_val = h.v;
  *h_idx = h.i;
  return kOk;
}

int learn_max(const double* d_S, int64_t cnt, void* d_scratch, double* h_max, cudaStream_t st) {
  const int np = (int)std::min<int64_t>(592, (cnt + LB - 1) / LB);
  double* part = reinterpret_cast<double*>(d_scratch);
  double* out = part + 592;
  k_max_partial<<<np, LB, 0, st>>>(d_S, cnt, part);
  k_max_final<<<1, LB, 0, st>>>(part, np, out);
  if (cudaMemcpyAsync(h_max, out, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess) return kCudaError;
  return cudaStreamSynchronize(st) == cudaSuccess ? kOk : kCudaError;
}

int learn_dprof_fold(const double* d_x, const WindowArrays& w, int m, const double* d_qc, double invn_q,
                     bool const_query, int64_t origin, double origin_val, bool first, double* d_S, cudaStream_t st) {
  const int64_t cnt = w.nwin;
  const size_t smem = sizeof(double) * (size_t)m;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(k_dprof_fold, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return kCudaError;
  k_dprof_fold<<<(unsigned)((cnt + LB - 1) / LB), LB, smem, st>>>(d_x, w.mu, w.invn, w.flag, cnt, m, d_qc, invn_q,
                                                                 const_query ? 1 : 0, origin, origin_val,
                                                                 first ? 1 : 0, d_S);
  return cudaGetLastError() == cudaSuccess ? kOk : kCudaError;
}

size_t learn_scratch_bytes() { return sizeof(ValIdx) * 600; }

}  // namespace tsd

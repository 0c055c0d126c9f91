// tsd_common.cuh -- shared device helpers for the tsdict B200 kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// TSD_CHECKED builds (tools/dev/abl_build.sh checked "-DTSD_CHECKED"): device
// bounds assertions on the global and shared buffers the kernels index, the
// stand-in for compute-sanitizer memcheck (closed on this GPU pool). A failed
// check prints its site and traps; release builds compile them out.
#ifdef TSD_CHECKED
#include <cstdio>
#define TSD_CHECK(cond)                                                                            \
  do {                                                                                             \
    if (!(cond)) {                                                                                 \
      printf("TSD_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__,  \
             (int)blockIdx.x, (int)threadIdx.x);                                                   \
      __trap();                                                                                    \
    }                                                                                              \
  } while (0)
#else
#define TSD_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace tsd {

// ---------------------------------------------------------------------------
// double-double arithmetic (error-free transforms), used by the window
// statistics so that window sums are formed without the prefix-magnitude
// cancellation the reference guards against (series.hpp:126-142).
// ---------------------------------------------------------------------------
struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = a + b;
  double e = b - (s - a);
  return {s, e};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  double p = a * b;
  double e = __fma_rn(a, b, -p);
  return {p, e};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div_d(dd a, double b) {
  double q1 = a.hi / b;
  dd p = two_prod(q1, b);
  dd r = dd_sub(a, p);
  double q2 = r.hi / b;
  p = two_prod(q2, b);
  r = dd_sub(r, p);
  double q3 = r.hi / b;
  dd q = quick_two_sum(q1, q2);
  return dd_add(q, dd{q3, 0.0});
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double shfl_up_d(double v, int delta) {
  return __shfl_up_sync(0xffffffffu, v, delta);
}

__device__ __forceinline__ int hi_word(double v) { return __double2hiint(v); }

// lexicographic (max corr, min index) -- reference profiles.hpp:70-77
__device__ __forceinline__ bool better(double c, int64_t j, double cur, int64_t cur_j) {
  return c > cur || (c == cur && j < cur_j);
}

__device__ __forceinline__ double clamp_corr(double c) {  // profiles.hpp:110-114
  return c > 1.0 ? 1.0 : (c < -1.0 ? -1.0 : c);
}

__device__ __forceinline__ double corr_to_dist(double rho, double md) {  // series.hpp:153-161
  if (rho > 1.0) rho = 1.0;
  if (rho < -1.0) rho = -1.0;
  double d = sqrt(2.0 * md * (1.0 - rho));
  const double dmax = 2.0 * sqrt(md);
  if (d < 0.0) d = 0.0;
  if (d > dmax) d = dmax;
  return d;
}

}  // namespace tsd

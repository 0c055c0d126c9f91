// stats.cu -- per-window statistics for the join (sm_100a).
//
// Replaces the reference compute_stats + make_diffs (series.hpp:83-150,
// profiles.hpp:89-99). The reference centres on a Kahan grand mean, takes
// compensated prefix sums and falls back to an exact per-window two-pass when
// the prefix magnitude threatens the std's ninth digit (series.hpp:126-142).
// Here the prefix sums of x and x^2 are carried in double-double precision
// (error-free transforms), so every window's first and second moment is
// formed to ~1e-30 relative and no fallback is needed; the flat threshold
// 1e-8*max(1, max|x|) (series.hpp:75-77) is evaluated per threshold group
// (one reference TimeSeries / 16384-window query block).
//
// Kernels:
//   k_group_max          max|x| per group + first series with a non-finite sample
//   k_window_stats_tile  (default) everything else, fused: per-tile prefixes in
//                        shared memory, all per-window arrays out
// and, for windows too long for a tile (or TSD_STATS_TILE=0), the global scans:
//   k_scan_partial  per-block double-double sums of x, x^2
//   k_scan_blocks   exclusive scan of the block sums (one CTA)
//   k_scan_apply    writes P1 = prefix(x), P2 = prefix(x^2) as double-double
//   k_window_stats  mean, std, invn, flat, df, dg per window
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "tsd_common.cuh"
#include "tsd_internal.h"

namespace tsd {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanPer = 16;  // samples per thread
constexpr int kScanBlock = kScanThreads * kScanPer;

__global__ void k_group_max(const double* __restrict__ x, const Group* __restrict__ groups, int ngroups, int m,
                            unsigned long long* __restrict__ gmax, int* __restrict__ bad_series, int gy0) {
  const int g = blockIdx.y + gy0;
  if (g >= ngroups) return;
  const Group G = groups[g];
  const int64_t s0 = G.wbeg, s1 = G.wend - 1 + m;  // sample range
  unsigned long long best = 0;
  bool bad = false;
  for (int64_t s = s0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < s1; s += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[s];
    if (!isfinite(v)) bad = true;
    const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v));
    best = b > best ? b : best;
  }
  // warp reduce
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
    best = ob > best ? ob : best;
  }
  if (bad) atomicMin(bad_series, G.series);
  if ((threadIdx.x & 31) == 0 && best) atomicMax(gmax + g, best);
}

__device__ __forceinline__ void load_pair(const double* __restrict__ x, int64_t i, int64_t n, dd& s1, dd& s2) {
  const double v = i < n ? x[i] : 0.0;
  s1 = {v, 0.0};
  s2 = two_prod(v, v);
}

struct dd2 {
  dd a, b;
};

__device__ __forceinline__ dd2 dd2_add(const dd2& p, const dd2& q) { return {dd_add(p.a, q.a), dd_add(p.b, q.b)}; }

__device__ __forceinline__ dd2 shfl_up_dd2(const dd2& v, int d) {
  dd2 r;
  r.a.hi = __shfl_up_sync(0xffffffffu, v.a.hi, d);
  r.a.lo = __shfl_up_sync(0xffffffffu, v.a.lo, d);
  r.b.hi = __shfl_up_sync(0xffffffffu, v.b.hi, d);
  r.b.lo = __shfl_up_sync(0xffffffffu, v.b.lo, d);
  return r;
}

// block-wide scan of one dd2 per thread; returns the EXCLUSIVE prefix (the
// sum over the lower threads), formed by shifting the inclusive scan one lane
// rather than as inclusive - own: a thread whose own sum dwarfs everything
// before it (a 1e60 excursion after 1e-6 data) would cancel the earlier
// prefix away. *total (thread 0's copy valid after the call) = block sum.
__device__ dd2 block_scan_excl(dd2 v, dd2* sh_warp, dd2* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    dd2 u = shfl_up_dd2(v, o);
    if (lane >= o) v = dd2_add(u, v);
  }
  if (lane == 31) sh_warp[wid] = v;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    dd2 w = lane < nw ? sh_warp[lane] : dd2{{0, 0}, {0, 0}};
    for (int o = 1; o < 32; o <<= 1) {
      dd2 u = shfl_up_dd2(w, o);
      if (lane >= o) w = dd2_add(u, w);
    }
    if (lane < nw) sh_warp[lane] = w;
  }
  __syncthreads();
  dd2 ex = shfl_up_dd2(v, 1);  // inclusive of the lane below, within the warp
  if (lane == 0) ex = dd2{{0, 0}, {0, 0}};
  if (wid > 0) ex = dd2_add(sh_warp[wid - 1], ex);
  if (total) *total = sh_warp[(blockDim.x >> 5) - 1];
  return ex;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_partial(const double* __restrict__ x, int64_t n,
                                                               dd2* __restrict__ block_sums) {
  __shared__ dd2 sh[32];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + (int64_t)threadIdx.x * kScanPer;
  dd2 acc{{0, 0}, {0, 0}};
#pragma unroll 4
  for (int k = 0; k < kScanPer; ++k) {
    dd a, b;
    load_pair(x, base + k, n, a, b);
    acc.a = dd_add(acc.a, a);
    acc.b = dd_add(acc.b, b);
  }
  dd2 tot;
  block_scan_excl(acc, sh, &tot);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

// exclusive scan of nblocks block sums in place, one CTA of 1024 threads
__global__ void __launch_bounds__(1024) k_scan_blocks(dd2* __restrict__ sums, int64_t nblocks) {
  __shared__ dd2 sh[32];
  const int64_t per = (nblocks + blockDim.x - 1) / blockDim.x;
  const int64_t b0 = (int64_t)threadIdx.x * per;
  dd2 acc{{0, 0}, {0, 0}};
  for (int64_t k = 0; k < per; ++k)
    if (b0 + k < nblocks) acc = dd2_add(acc, sums[b0 + k]);
  // exclusive prefix for this thread's range
  dd2 run = block_scan_excl(acc, sh, nullptr);
  __syncthreads();
  for (int64_t k = 0; k < per; ++k) {
    if (b0 + k < nblocks) {
      dd2 v = sums[b0 + k];
      sums[b0 + k] = run;
      run = dd2_add(run, v);
    }
  }
}

// P arrays hold n+1 entries: P[0] = 0, P[i+1] = sum_{t<=i}
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const double* __restrict__ x, int64_t n,
                                                             const dd2* __restrict__ block_excl,
                                                             double2* __restrict__ P1, double2* __restrict__ P2) {
  __shared__ dd2 sh[32];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + (int64_t)threadIdx.x * kScanPer;
  dd2 acc{{0, 0}, {0, 0}};
  for (int k = 0; k < kScanPer; ++k) {
    dd a, b;
    load_pair(x, base + k, n, a, b);
    acc.a = dd_add(acc.a, a);
    acc.b = dd_add(acc.b, b);
  }
  dd2 run = dd2_add(block_excl[blockIdx.x], block_scan_excl(acc, sh, nullptr));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    P1[0] = make_double2(0.0, 0.0);
    P2[0] = make_double2(0.0, 0.0);
  }
  for (int k = 0; k < kScanPer; ++k) {
    const int64_t i = base + k;
    if (i >= n) break;
    dd a, b;
    load_pair(x, i, n, a, b);
    run.a = dd_add(run.a, a);
    run.b = dd_add(run.b, b);
    P1[i + 1] = make_double2(run.a.hi, run.a.lo);
    P2[i + 1] = make_double2(run.b.hi, run.b.lo);
  }
}

// Window mean and variance from the double-double prefix sums. Their
// differences carry an absolute error of about 2^-100 x the prefix
// magnitude; when that threatens the variance's twelfth digit (a quiet
// window after a huge excursion somewhere earlier in the buffer) the window
// is redone in two compensated passes over its samples, as the reference
// does for its Kahan prefix sums (series.hpp:126-142).
__device__ __forceinline__ void window_moments(const double* __restrict__ x, const double2* __restrict__ P1,
                                               const double2* __restrict__ P2, int64_t p, int m, double& mean,
                                               double& var) {
  const double md = (double)m;
  const double2 a0 = P1[p], a1 = P1[p + m], b0 = P2[p], b1 = P2[p + m];
  const dd w1 = dd_sub(dd{a1.x, a1.y}, dd{a0.x, a0.y});
  const dd w2 = dd_sub(dd{b1.x, b1.y}, dd{b0.x, b0.y});
  const dd mu = dd_div_d(w1, md);
  const dd v = dd_div_d(dd_sub(w2, dd_mul(w1, mu)), md);
  mean = mu.hi + mu.lo;
  var = v.hi + v.lo;
  if (var < 0.0) var = 0.0;
  const double e2 = 0x1p-100 * (fabs(b1.x) + fabs(b0.x));                // error of w2
  const double e1 = 0x1p-100 * (fabs(a1.x) + fabs(a0.x));                // error of w1
  if (e2 > 1e-12 * md * var || e1 * e1 > 1e-24 * md * md * var) [[unlikely]] {
    dd s{0.0, 0.0};
    for (int t = 0; t < m; ++t) s = dd_add(s, dd{x[p + t], 0.0});
    const dd mu2 = dd_div_d(s, md);
    const double mc = mu2.hi + mu2.lo;
    dd q{0.0, 0.0};
    for (int t = 0; t < m; ++t) {
      const dd d = dd_sub(dd{x[p + t], 0.0}, mu2);
      q = dd_add(q, dd_mul(d, d));
    }
    const dd v2 = dd_div_d(q, md);
    mean = mc;
    var = v2.hi + v2.lo;
    if (var < 0.0) var = 0.0;
  }
}

// ---------------------------------------------------------------------------
// Fused tile form (the default while the tile's prefixes fit in shared memory):
// one CTA takes kTileWin consecutive windows, forms the double-double prefix
// sums of x and x^2 over JUST the samples those windows cover (tile + m
// samples, in shared memory) and writes every per-window array from them. No
// global prefix arrays and no scan kernels: the samples are read once per tile
// (plus the m - 1 halo) and 41 B per window go out -- the algorithmic bytes of
// against 8 + 2 x 32 B per sample written and read back by the
// three-kernel scan. Window sums are differences of LOCAL prefixes (at most
// kTileWin + m terms), so their absolute error is far below the global form's
// and the two-pass fallback of window_moments triggers even more rarely; the
// rounded means and variances are the same doubles (both forms carry ~1e-30).
// ---------------------------------------------------------------------------
constexpr int kTileThreads = 256;
constexpr int kTilePer = 8;
constexpr int kTileWin = kTileThreads * kTilePer;  // windows per CTA

__device__ __forceinline__ void tile_moments(const double* __restrict__ x, const double2* __restrict__ Q1,
                                             const double2* __restrict__ Q2, int64_t p, int loc, int m, double& mean,
                                             double& var) {
  const double md = (double)m;
  TSD_CHECK(loc >= 0 && Q1 + loc + m < Q2);  // inside the tile's first prefix array (Q2 follows it)
  const double2 a0 = Q1[loc], a1 = Q1[loc + m], b0 = Q2[loc], b1 = Q2[loc + m];
  const dd w1 = dd_sub(dd{a1.x, a1.y}, dd{a0.x, a0.y});
  const dd w2 = dd_sub(dd{b1.x, b1.y}, dd{b0.x, b0.y});
  const dd mu = dd_div_d(w1, md);
  const dd v = dd_div_d(dd_sub(w2, dd_mul(w1, mu)), md);
  mean = mu.hi + mu.lo;
  var = v.hi + v.lo;
  if (var < 0.0) var = 0.0;
  const double e2 = 0x1p-100 * (fabs(b1.x) + fabs(b0.x));
  const double e1 = 0x1p-100 * (fabs(a1.x) + fabs(a0.x));
  if (e2 > 1e-12 * md * var || e1 * e1 > 1e-24 * md * md * var) [[unlikely]] {
    // (the same two compensated passes as window_moments, series.hpp:126-142)
    dd s{0.0, 0.0};
    for (int t = 0; t < m; ++t) s = dd_add(s, dd{x[p + t], 0.0});
    const dd mu2 = dd_div_d(s, md);
    dd q{0.0, 0.0};
    for (int t = 0; t < m; ++t) {
      const dd d = dd_sub(dd{x[p + t], 0.0}, mu2);
      q = dd_add(q, dd_mul(d, d));
    }
    const dd v2 = dd_div_d(q, md);
    mean = mu2.hi + mu2.lo;
    var = v2.hi + v2.lo;
    if (var < 0.0) var = 0.0;
  }
}

__global__ void __launch_bounds__(kTileThreads)
    k_window_stats_tile(const double* __restrict__ x, int64_t n, int64_t nwin, int m,
                        const Group* __restrict__ groups, int ngroups, const unsigned long long* __restrict__ gmax,
                        double* __restrict__ mu, double* __restrict__ sdo, double* __restrict__ invn,
                        double* __restrict__ df, double* __restrict__ dg, uint8_t* __restrict__ flag) {
  extern __shared__ double2 tile_q[];
  __shared__ dd2 sh[32];
  const int64_t p0 = (int64_t)blockIdx.x * kTileWin;
  const int64_t sb = p0 > 0 ? p0 - 1 : 0;  // the window before the tile's first one feeds its dg
  const int64_t se = p0 + kTileWin + m - 1 < n ? p0 + kTileWin + m - 1 : n;
  const int len = (int)(se - sb);
  TSD_CHECK(len >= m && len <= kTileWin + m && se <= n);
  double2* Q1 = tile_q;            // Q1[k] = sum of x[sb .. sb + k), k = 0 .. len
  double2* Q2 = tile_q + len + 1;  // the same of x^2
  const int per = (len + kTileThreads - 1) / kTileThreads;
  const int k0 = threadIdx.x * per, k1 = k0 + per < len ? k0 + per : len;
  dd2 acc{{0, 0}, {0, 0}};
  for (int k = k0; k < k1; ++k) {
    const double v = x[sb + k];
    acc.a = dd_add(acc.a, dd{v, 0.0});
    acc.b = dd_add(acc.b, two_prod(v, v));
  }
  dd2 run = block_scan_excl(acc, sh, nullptr);
  if (threadIdx.x == 0) {
    Q1[0] = make_double2(0.0, 0.0);
    Q2[0] = make_double2(0.0, 0.0);
  }
  for (int k = k0; k < k1; ++k) {
    const double v = x[sb + k];
    run.a = dd_add(run.a, dd{v, 0.0});
    run.b = dd_add(run.b, two_prod(v, v));
    Q1[k + 1] = make_double2(run.a.hi, run.a.lo);
    Q2[k + 1] = make_double2(run.b.hi, run.b.lo);
  }
  __syncthreads();
  const double md = (double)m;
  // the group of the tile's first window; windows are visited in increasing
  // order, so the lookup only ever moves forward
  int g = -1;
  {
    int lo = 0, hi = ngroups - 1;
    const int64_t pf = p0 + threadIdx.x;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      if (groups[mid].wbeg <= pf) {
        g = mid;
        lo = mid + 1;
      } else {
        hi = mid - 1;
      }
    }
  }
  // phase 1: moments of the tile's windows (each once; the window before the
  // tile by thread 0), means parked in shared memory for the neighbours' dg
  double* smean = reinterpret_cast<double*>(tile_q + 2 * (len + 1));  // smean[i]: window p0 - 1 + i
  double mymean[kTilePer];
  if (threadIdx.x == 0 && p0 > 0) {
    double mean, var;
    tile_moments(x, Q1, Q2, p0 - 1, 0, m, mean, var);
    smean[0] = mean;
  }
#pragma unroll
  for (int k = 0; k < kTilePer; ++k) {
    const int64_t p = p0 + threadIdx.x + (int64_t)kTileThreads * k;
    mymean[k] = 0.0;
    if (p >= nwin) continue;
    while (g + 1 < ngroups && groups[g + 1].wbeg <= p) ++g;
    double mean, var;
    tile_moments(x, Q1, Q2, p, (int)(p - sb), m, mean, var);
    const double sd = sqrt(var);
    uint8_t f = 0;
    double iv = 0.0;
    if (g >= 0 && p < groups[g].wend) {
      const double mx = __longlong_as_double((long long)gmax[g]);
      const double eps = 1e-8 * (mx > 1.0 ? mx : 1.0);  // series.hpp:75-77
      const bool flat = sd < eps;                        // series.hpp:145
      f = flat ? 3 : 1;
      iv = flat ? 0.0 : 1.0 / (sd * sqrt(md));           // series.hpp:147
    }
    mu[p] = mean;
    if (sdo) sdo[p] = sd;
    invn[p] = iv;
    flag[p] = f;
    mymean[k] = mean;
    smean[threadIdx.x + kTileThreads * k + 1] = mean;
  }
  __syncthreads();
  // phase 2: make_diffs (profiles.hpp:89-99) on the concatenated buffer
#pragma unroll
  for (int k = 0; k < kTilePer; ++k) {
    const int64_t p = p0 + threadIdx.x + (int64_t)kTileThreads * k;
    if (p >= nwin) continue;
    double dfv = 0.0, dgv = 0.0;
    if (p > 0) {
      const double xin = x[p + m - 1], xout = x[p - 1];
      dfv = 0.5 * (xin - xout);
      dgv = (xin - mymean[k]) + (xout - smean[threadIdx.x + kTileThreads * k]);
    }
    df[p] = dfv;
    dg[p] = dgv;
  }
}

__global__ void k_window_stats(const double* __restrict__ x, const double2* __restrict__ P1,
                               const double2* __restrict__ P2, int64_t nwin, int m, const Group* __restrict__ groups,
                               int ngroups, const unsigned long long* __restrict__ gmax, double* __restrict__ mu,
                               double* __restrict__ sdo, double* __restrict__ invn, double* __restrict__ df,
                               double* __restrict__ dg, uint8_t* __restrict__ flag) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nwin) return;
  const double md = (double)m;
  double mean, var;
  window_moments(x, P1, P2, p, m, mean, var);
  const double sd = sqrt(var);
  // group lookup: last group with wbeg <= p
  int lo = 0, hi = ngroups - 1, g = -1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    if (groups[mid].wbeg <= p) {
      g = mid;
      lo = mid + 1;
    } else {
      hi = mid - 1;
    }
  }
  uint8_t f = 0;
  double iv = 0.0;
  if (g >= 0 && p < groups[g].wend) {
    const double mx = __longlong_as_double((long long)gmax[g]);
    const double eps = 1e-8 * (mx > 1.0 ? mx : 1.0);  // series.hpp:75-77
    const bool flat = sd < eps;                        // series.hpp:145
    f = flat ? 3 : 1;
    iv = flat ? 0.0 : 1.0 / (sd * sqrt(md));           // series.hpp:147
  }
  mu[p] = mean;
  if (sdo) sdo[p] = sd;
  invn[p] = iv;
  flag[p] = f;
  // make_diffs (profiles.hpp:89-99) on the concatenated buffer
  double dfv = 0.0, dgv = 0.0;
  if (p > 0) {
    double mean_prev, var_prev;
    window_moments(x, P1, P2, p - 1, m, mean_prev, var_prev);
    const double xin = x[p + m - 1], xout = x[p - 1];
    dfv = 0.5 * (xin - xout);
    dgv = (xin - mean) + (xout - mean_prev);
  }
  df[p] = dfv;
  dg[p] = dgv;
}

}  // namespace

#define CUDA_TRY(call)                                                        \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      if (err) *err = Error{kCudaError, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
      return kCudaError;                                                      \
    }                                                                         \
  } while (0)

static bool stats_tile_fits(int m, size_t* bytes) {
  // a tile's two prefix arrays and its window means in shared memory (m up to ~4000)
  const size_t b = 2 * sizeof(double2) * ((size_t)kTileWin + (size_t)m + 2) + sizeof(double) * (kTileWin + 2);
  if (bytes) *bytes = b;
  static const bool tile_off = getenv("TSD_STATS_TILE") && atoi(getenv("TSD_STATS_TILE")) == 0;
  return !tile_off && b <= (size_t)200 * 1024;
}

int window_stat_launches(int m) { return stats_tile_fits(m, nullptr) ? 2 : 5; }

int compute_windows(const double* d_x, int64_t n, int m, const std::vector<Group>& groups, int nseries,
                    WindowArrays& out, Arena& arena, cudaStream_t st, int* bad_series, Error* err,
                    const int** d_bad_out) {
  (void)nseries;
  const int64_t nwin = n - m + 1;
  const int ng = (int)groups.size();
  const int64_t nblk = (n + kScanBlock - 1) / kScanBlock;
  // scratch
  Group* d_groups = (Group*)arena.get(sizeof(Group) * ng);
  unsigned long long* d_gmax = (unsigned long long*)arena.get(sizeof(unsigned long long) * ng);
  int* d_bad = (int*)arena.get(sizeof(int) * 4);
  size_t tile_smem = 0;
  const bool tile = stats_tile_fits(m, &tile_smem);
  dd2* d_bs = tile ? nullptr : (dd2*)arena.get(sizeof(dd2) * nblk);
  double2* d_P1 = tile ? nullptr : (double2*)arena.get(sizeof(double2) * (n + 1));
  double2* d_P2 = tile ? nullptr : (double2*)arena.get(sizeof(double2) * (n + 1));
  out.nwin = nwin;
  out.mu = (double*)arena.get(sizeof(double) * nwin);
  out.sd = (double*)arena.get(sizeof(double) * nwin);
  out.invn = (double*)arena.get(sizeof(double) * nwin);
  out.df = (double*)arena.get(sizeof(double) * nwin);
  out.dg = (double*)arena.get(sizeof(double) * nwin);
  out.flag = (uint8_t*)arena.get(nwin + 16);
  if (!d_groups || !d_gmax || !d_bad || (!tile && (!d_bs || !d_P1 || !d_P2)) || !out.mu || !out.sd || !out.invn ||
      !out.df || !out.dg || !out.flag) {
    if (err) *err = Error{kCudaError, "device allocation failed for window statistics"};
    return kCudaError;
  }
  CUDA_TRY(cudaMemcpyAsync(d_groups, groups.data(), sizeof(Group) * ng, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(d_gmax, 0, sizeof(unsigned long long) * ng, st));
  const int big = 0x7fffffff;
  CUDA_TRY(cudaMemcpyAsync(d_bad, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  for (int gy0 = 0; gy0 < ng; gy0 += 65535) {
    const int gy = ng - gy0 < 65535 ? ng - gy0 : 65535;
    int64_t maxlen = 0;
    for (int g = gy0; g < gy0 + gy; ++g) maxlen = std::max<int64_t>(maxlen, groups[g].wend - 1 + m - groups[g].wbeg);
    int gx = (int)std::min<int64_t>((maxlen + 2047) / 2048, 64);
    if (gx < 1) gx = 1;
    k_group_max<<<dim3(gx, gy), 256, 0, st>>>(d_x, d_groups, ng, m, d_gmax, d_bad, gy0);
  }
  if (tile) {
    // (per device, so set on every call like the join kernels' -- a process may drive several GPUs)
    CUDA_TRY(cudaFuncSetAttribute(k_window_stats_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    k_window_stats_tile<<<(unsigned)((nwin + kTileWin - 1) / kTileWin), kTileThreads, tile_smem, st>>>(
        d_x, n, nwin, m, d_groups, ng, d_gmax, out.mu, out.sd, out.invn, out.df, out.dg, out.flag);
  } else {
    k_scan_partial<<<(unsigned)nblk, kScanThreads, 0, st>>>(d_x, n, d_bs);
    k_scan_blocks<<<1, 1024, 0, st>>>(d_bs, nblk);
    k_scan_apply<<<(unsigned)nblk, kScanThreads, 0, st>>>(d_x, n, d_bs, d_P1, d_P2);
    k_window_stats<<<(unsigned)((nwin + 255) / 256), 256, 0, st>>>(d_x, d_P1, d_P2, nwin, m, d_groups, ng, d_gmax,
                                                                    out.mu, out.sd, out.invn, out.df, out.dg,
                                                                    out.flag);
  }
  CUDA_TRY(cudaGetLastError());
  if (d_bad_out) {  // the caller reads the non-finite flag after its own synchronisation
    *d_bad_out = d_bad;
    *bad_series = -1;
    return kOk;
  }
  int bad = big;
  CUDA_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *bad_series = bad == big ? -1 : bad;
  return kOk;
}

static std::atomic<unsigned> g_arena_gen{1};  // bumped by every arena cudaMalloc / cudaFree

Arena::~Arena() {
  for (auto& b : blks) cudaFree(b.p);
  if (!blks.empty()) g_arena_gen.fetch_add(1);
}

bool device_free_bytes(size_t* free_bytes) {
  static thread_local unsigned gen = 0;
  static thread_local int dev_seen = -1;
  static thread_local size_t fr = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned g = g_arena_gen.load();
  if (g != gen || dev != dev_seen) {
    size_t tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return false;
    gen = g;
    dev_seen = dev;
  }
  *free_bytes = fr;
  return true;
}

void* Arena::get(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  if (bytes == 0) bytes = 256;
  while (cur < blks.size()) {
    Blk& b = blks[cur];
    if (b.used + bytes <= b.cap) {
      void* r = b.p + b.used;
      b.used += bytes;
      return r;
    }
    ++cur;
  }
  const size_t cap = bytes > (size_t(256) << 20) ? bytes : (size_t(256) << 20);
  void* p = nullptr;
  if (cudaMalloc(&p, cap) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  g_arena_gen.fetch_add(1);
  blks.push_back(Blk{(char*)p, cap, bytes});
  cur = blks.size() - 1;
  return p;
}

}  // namespace tsd

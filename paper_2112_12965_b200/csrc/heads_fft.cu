// heads_fft.cu -- left-edge "heads" of a dictionary join by FFT correlation.
//
// Every diagonal that enters segment s at its window 0 needs one m-term dot
// product (window_dot, profiles.hpp:101-108):
//   head(i, s) = cov(i, col0_s)
//              = sum_k (x[i+k] - c) * btil_s[k] - (mu_i - c) * e_s
// (btil_s = centred window 0 of segment s, e_s = sum btil_s, c any constant). Done directly that is m FMAs per
// (row, segment): for the headline config (m = 512, 1024-sample segments)
// as many FP64 operations as a third of the sweep itself. As a correlation
// of the query with btil_s it is O(log N) per output by FFT:
//   * the query is cut into blocks of Q rows (Q = multiple of the 256-row
//     band, Q <= N - m + 1), each block's N = 4096 samples transformed once;
//   * two segments share one complex inverse transform: with
//     z = btil_s + i btil_{s+1}, IFFT(X . Z[-f]) = corr(x, btil_s) +
//     i corr(x, btil_{s+1}) (x real), Z precomputed per dictionary;
//   * ~25 FP64 operations per head instead of 512 FMAs.
// Output: heads[s * hstride + i], read by k_join (join.cu) at the start of
// each (band, segment); the FP32 sweep scales them by its column scale.
//
// FFT: Stockham autosort, radix 16 x 3 passes, 256 threads, one 4096-point
// transform per CTA in padded shared memory (pad(i) = i + i/16 keeps the
// 16-byte accesses of every pass conflict-free). Thread j's last-pass values
// are outputs j + 256 r, which is also the input layout of the first pass --
// the forward transform's result stays in registers for all pairs.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "tsd_common.cuh"
#include "tsd_internal.h"

namespace tsd {
namespace {

constexpr int FFT_N = 4096;
constexpr int FFT_T = 256;  // threads per CTA = N / 16
constexpr int FFT_PAD = FFT_N + FFT_N / 16;

#define CUDA_TRY(x)                                                   \
  do {                                                                \
    cudaError_t e_ = (x);                                             \
    if (e_ != cudaSuccess) {                                          \
      if (err) *err = Error{kCudaError, cudaGetErrorString(e_)};      \
      return kCudaError;                                              \
    }                                                                 \
  } while (0)

__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -a.y * b.y), __fma_rn(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 rot(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// W16^e = exp(-+2 pi i e / 16) for the exponents a radix 4x4 split needs
template <bool INV>
__device__ __forceinline__ double2 w16(int e) {
  constexpr double C1 = 0.92387953251128673848, S1 = 0.38268343236508977173, H = 0.70710678118654752440;
  double c, s;  // exp(-2 pi i e / 16) = c - i s
  switch (e) {
    case 1: c = C1, s = S1; break;
    case 2: c = H, s = H; break;
    case 3: c = S1, s = C1; break;
    case 4: c = 0.0, s = 1.0; break;
    case 6: c = -H, s = H; break;
    case 9: c = -C1, s = -S1; break;
    default: c = 1.0, s = 0.0; break;
  }
  return make_double2(c, INV ? s : -s);
}

// 4-point DFT in place on a[o], a[o+d], a[o+2d], a[o+3d]
template <bool INV>
__device__ __forceinline__ void dft4(double2* a, int o, int d) {
  const double2 t0 = cadd(a[o], a[o + 2 * d]), t1 = csub(a[o], a[o + 2 * d]);
  const double2 t2 = cadd(a[o + d], a[o + 3 * d]), t3 = rot<INV>(csub(a[o + d], a[o + 3 * d]));
  a[o] = cadd(t0, t2);
  a[o + 2 * d] = csub(t0, t2);
  a[o + d] = cadd(t1, t3);
  a[o + 3 * d] = csub(t1, t3);
}

// 16-point DFT of v[0..15] (natural order in and out), n = 4 n1 + n2,
// k = k1 + 4 k2
template <bool INV>
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(v, n2, 4);  // over n1: v[n2 + 4 k1] = Y[n2][k1]
#pragma unroll
  for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
    for (int k1 = 1; k1 < 4; ++k1) v[n2 + 4 * k1] = cmul(v[n2 + 4 * k1], w16<INV>(n2 * k1));
  double2 t[16];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    // over n2: Y[n2][k1] at v[n2 + 4 k1] -> X[k1 + 4 k2]
    double2 a[4] = {v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]};
    dft4<INV>(a, 0, 1);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) t[k1 + 4 * k2] = a[k2];
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = t[k];
}

// One Stockham pass (radix 16) reading thread j's inputs j + 256 r from
// registers v. Ns = size of the sub-transforms already done (1, 16, 256).
// Pass Ns < 256 writes its outputs to shared memory; the caller syncs.
// twiddle exp(-2 pi i t / N) from the shared half table (t + N/2 -> negated)
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ stw, int t) {
  const double2 w = stw[t & (FFT_N / 2 - 1)];
  return (t & (FFT_N / 2)) ? make_double2(-w.x, -w.y) : w;
}

template <bool INV>
__device__ __forceinline__ void pass_compute(double2 (&v)[16], int j, int Ns, const double2* __restrict__ stw) {
  if (Ns > 1) {
    // w^r for r = 1..15 from four table entries (w, w^2, w^4, w^8; r k step < N)
    // and products of at most three of them
    const int t1 = (j & (Ns - 1)) * (FFT_N / (Ns * 16));
    double2 w[16];
    w[1] = twiddle(stw, t1);
    w[2] = twiddle(stw, 2 * t1);
    w[4] = twiddle(stw, 4 * t1);
    w[8] = twiddle(stw, 8 * t1);
    w[3] = cmul(w[1], w[2]);
    w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]);
    w[7] = cmul(w[3], w[4]);
    w[9] = cmul(w[1], w[8]);
    w[10] = cmul(w[2], w[8]);
    w[11] = cmul(w[3], w[8]);
    w[12] = cmul(w[4], w[8]);
    w[13] = cmul(w[5], w[8]);
    w[14] = cmul(w[6], w[8]);
    w[15] = cmul(w[7], w[8]);
#pragma unroll
    for (int r = 1; r < 16; ++r) {
      if (INV) w[r].y = -w[r].y;
      v[r] = cmul(v[r], w[r]);
    }
  }
  dft16<INV>(v);
}

// stage the half twiddle table (global, k_fft_twiddles) in shared memory
__device__ __forceinline__ void load_twiddles(double2* __restrict__ stw, const double2* __restrict__ tw) {
  for (int t = threadIdx.x; t < FFT_N / 2; t += blockDim.x) stw[t] = tw[t];
}

__device__ __forceinline__ void pass_store(double2* __restrict__ sm, const double2 (&v)[16], int j, int Ns) {
  const int idx = (j / Ns) * Ns * 16 + (j & (Ns - 1));
#pragma unroll
  for (int r = 0; r < 16; ++r) sm[pad16(idx + r * Ns)] = v[r];
}

__device__ __forceinline__ void pass_load(const double2* __restrict__ sm, double2 (&v)[16], int j) {
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = sm[pad16(j + 256 * r)];
}

// Full transform of v (thread j holds inputs j + 256 r) -> v (outputs j + 256 r)
template <bool INV>
__device__ __forceinline__ void fft4096(double2 (&v)[16], double2* sm, int j, const double2* __restrict__ stw) {
  pass_compute<INV>(v, j, 1, stw);
  __syncthreads();  // previous readers of sm are done
  pass_store(sm, v, j, 1);
  __syncthreads();
  pass_load(sm, v, j);
  pass_compute<INV>(v, j, 16, stw);
  __syncthreads();
  pass_store(sm, v, j, 16);
  __syncthreads();
  pass_load(sm, v, j);
  pass_compute<INV>(v, j, 256, stw);
}

__global__ void k_fft_twiddles(double2* tw) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < FFT_N) {
    double s, c;
    sincospi(2.0 * t / FFT_N, &s, &c);
    tw[t] = make_double2(c, -s);  // exp(-2 pi i t / N)
  }
}

// spec[p][f] = Z_p[(N - f) mod N], Z_p = FFT(btil_{2p} + i btil_{2p+1})
__global__ void __launch_bounds__(FFT_T, 1)
    k_pair_spectra(const double* __restrict__ btil, int nseg, int m, const double2* __restrict__ tw,
                   double2* __restrict__ spec) {
  extern __shared__ double2 fsm[];
  double2* stw = fsm + FFT_PAD;
  load_twiddles(stw, tw);
  const int p = blockIdx.x, j = threadIdx.x;
  const int s0 = 2 * p, s1 = 2 * p + 1;
  double2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int k = j + 256 * r;
    const double a = k < m ? btil[(int64_t)s0 * m + k] : 0.0;
    const double b = (k < m && s1 < nseg) ? btil[(int64_t)s1 * m + k] : 0.0;
    v[r] = make_double2(a, b);
  }
  fft4096<false>(v, fsm, j, stw);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int f = (FFT_N - (j + 256 * r)) & (FFT_N - 1);
    spec[(int64_t)p * FFT_N + f] = v[r];
  }
}

struct HeadsArgs {
  const double* x;  // query samples
  int64_t na;
  int64_t nrows;      // query windows
  int64_t hrows;      // rows to produce (bands * 256)
  int64_t hstride;    // heads row stride per segment
  const double* mua;  // window means
  const double2* spec;
  const double2* tw;
  const double* ebt;  // sum of btil per segment
  const SegDev* segs;
  const double* invn_b;   // column invn (seeds: K = head * invn_b, as the sweeps compute it)
  const uint8_t* flag_a;  // row flags (bit0 valid, bit1 flat)
  int nseg, npairs, m, Q;
  long long excl;  // self-join exclusion half-width (-1: AB join)
  int sym;         // symmetric self-join: a row's sweep evaluates only its upper-triangle heads
  double* heads;
  unsigned long long* seed;  // per row: order-preserving key of max_s head * kf (0 = none), or null
  int ppc;                   // pairs per CTA
  int64_t tri_rows;          // > 0: skip column blocks below each segment's first read column (see tsd_internal.h)
  long long tri_excl;
};

// A head (row i, column c) may seed row i only if row i's own sweep evaluates
// that very cell from the same head value: every admissible column (|i - c| >
// excl) in the AB / full self-join sweeps, only upper ones (c - i > excl) in
// the symmetric sweep (a lower cell is evaluated by the column side through the
// recurrence, whose rounding differs from the FFT head's).
struct HeadsArgs;
__device__ __forceinline__ bool seed_ok(const HeadsArgs& a, long long i, long long c);

// order-preserving map double -> u64 (key(a) < key(b) iff a < b; 0 below all)
__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ void cp16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(sdst)),
               "l"(gsrc));
}

// Shared memory: FFT work buffer (padded) | next pair spectrum (cp.async) |
// half twiddle table | per-row mean offsets. Thread j only ever touches
// spectrum / offset entries j + 256 r, so those need no barriers.
constexpr size_t HEADS_SMEM = sizeof(double2) * (FFT_PAD + FFT_N + FFT_N / 2) + sizeof(double) * FFT_N;

__device__ __forceinline__ bool seed_ok(const HeadsArgs& a, long long i, long long c) {
  if (a.excl < 0) return true;
  return c - i > a.excl || (!a.sym && i - c > a.excl);
}

__global__ void __launch_bounds__(FFT_T, 1) k_heads_fft(const HeadsArgs a) {
  extern __shared__ double2 fsm[];
  double2* zbuf = fsm + FFT_PAD;
  double2* stw = zbuf + FFT_N;
  double* dmu = reinterpret_cast<double*>(stw + FFT_N / 2);
  const int j = threadIdx.x;
  const int64_t blk0 = (int64_t)blockIdx.x * a.Q;
  const int p0 = blockIdx.y * a.ppc;
  int p1 = min(a.npairs, p0 + a.ppc);
  if (a.tri_rows > 0) {
    // pairs whose first read column lies past this block (first columns grow with s)
    while (p1 > p0 && ((((int64_t)(2 * (p1 - 1)) * a.tri_rows + a.tri_excl + 1) & ~int64_t(31)) >= blk0 + a.Q)) --p1;
    if (p1 == p0) return;
  }
  auto fetch = [&](int p) {
    const double2* sp = a.spec + (int64_t)p * FFT_N;
#pragma unroll
    for (int r = 0; r < 16; ++r) cp16(&zbuf[j + 256 * r], &sp[j + 256 * r]);
    asm volatile("cp.async.commit_group;\n" ::);
  };
  fetch(p0);
  load_twiddles(stw, a.tw);
  const double c = a.mua[blk0];  // centring constant of the block (any value is exact)
  double2 X[16];
  double mk[16];  // per-row running max of head * invn_b(col0)
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int64_t n = blk0 + j + 256 * r;
    X[r] = make_double2((n < a.na ? a.x[n] : c) - c, 0.0);
    dmu[j + 256 * r] = (n < a.nrows ? a.mua[n] : c) - c;
    mk[r] = -INFINITY;
  }
  __syncthreads();  // twiddles staged
  fft4096<false>(X, fsm, j, stw);
  const double invN = 1.0 / FFT_N;
  for (int p = p0; p < p1; ++p) {
    const int s0 = 2 * p, s1 = 2 * p + 1;
    const bool two = s1 < a.nseg;
    const int64_t c0 = a.seed ? a.segs[s0].col0 : 0, c1 = (two && a.seed) ? a.segs[s1].col0 : c0;
    const double e0 = a.ebt[s0], e1 = two ? a.ebt[s1] : 0.0;
    const double k0 = a.seed ? a.invn_b[c0] : 0.0, k1 = (two && a.seed) ? a.invn_b[c1] : 0.0;
    asm volatile("cp.async.wait_group 0;\n" ::);
    double2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = cmul(X[r], zbuf[j + 256 * r]);
    if (p + 1 < p1) fetch(p + 1);  // own entries only: no barrier needed
    fft4096<true>(v, fsm, j, stw);
    TSD_CHECK(s0 >= 0 && s0 < a.nseg && s1 >= 0 && s1 < a.nseg + 1);
    double* h0 = a.heads + (int64_t)s0 * a.hstride;
    double* h1 = a.heads + (int64_t)s1 * a.hstride;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int q = j + 256 * r;
      const int64_t i = blk0 + q;
      if (q < a.Q && i < a.hrows) {
        TSD_CHECK(i < a.hstride && (!two || s1 < a.nseg));
        const double d = dmu[q];
        const double g0 = v[r].x * invN - d * e0;
        h0[i] = g0;
        if (seed_ok(a, i, c0)) mk[r] = fmax(mk[r], g0 * k0);
        if (two) {
          const double g1 = v[r].y * invN - d * e1;
          h1[i] = g1;
          if (seed_ok(a, i, c1)) mk[r] = fmax(mk[r], g1 * k1);
        }
      }
    }
  }
  if (a.seed) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int q = j + 256 * r;
      const int64_t i = blk0 + q;
      if (q < a.Q && i < a.nrows && mk[r] > -INFINITY) atomicMax(&a.seed[i], order_key(mk[r]));
    }
  }
}

}  // namespace

// FFT round-off scales with the norm of the whole 4096-sample block, a
// window's covariance with its own: the ratio grows like sqrt(4096 / m) times
// the series' drift over a block. From m = 64 on the correlation error stays
// below ~4e-13 even on random walks; shorter windows take the direct m-term
// products, which are cheap exactly then.
int heads_fft_supported(int m) { return m >= 64 && m <= FFT_N - 512 + 1; }

int compute_heads_fft(const double* d_x, int64_t na, int64_t nrows, int64_t hrows, const double* d_mua,
                      const uint8_t* d_flag_a, const double* d_btil, const double* d_ebt, const double* d_invn_b,
                      const SegDev* d_segs, int nseg, int m, double* d_heads, int64_t hstride,
                      unsigned long long* d_seed, long long excl, int sym, Arena& arena, cudaStream_t st,
                      int* launches, Error* err, int64_t tri_rows, long long tri_excl) {
  const int npairs = (nseg + 1) / 2;
  double2* d_tw = (double2*)arena.get(sizeof(double2) * FFT_N);
  double2* d_spec = (double2*)arena.get(sizeof(double2) * FFT_N * (size_t)npairs);
  if (!d_tw || !d_spec) {
    if (err) *err = Error{kCudaError, "device allocation failed for the FFT heads"};
    return kCudaError;
  }
  const size_t smem = sizeof(double2) * (FFT_PAD + FFT_N / 2);
  const size_t smem_h = HEADS_SMEM;
  CUDA_TRY(cudaFuncSetAttribute(k_pair_spectra, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CUDA_TRY(cudaFuncSetAttribute(k_heads_fft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_h));
  k_fft_twiddles<<<FFT_N / 256, 256, 0, st>>>(d_tw);
  k_pair_spectra<<<npairs, FFT_T, smem, st>>>(d_btil, nseg, m, d_tw, d_spec);
  HeadsArgs a;
  a.x = d_x;
  a.na = na;
  a.nrows = nrows;
  a.hrows = hrows;
  a.hstride = hstride;
  a.mua = d_mua;
  a.spec = d_spec;
  a.tw = d_tw;
  a.ebt = d_ebt;
  a.segs = d_segs;
  a.invn_b = d_invn_b;
  a.flag_a = d_flag_a;
  a.nseg = nseg;
  a.npairs = npairs;
  a.m = m;
  a.Q = ((FFT_N - m + 1) / 256) * 256;
  a.heads = d_heads;
  a.seed = d_seed;
  a.excl = excl;
  a.sym = sym;
  a.tri_rows = tri_rows;
  a.tri_excl = tri_excl;
  const int64_t nblk = (hrows + a.Q - 1) / a.Q;
  {
    // up to 64 pairs per CTA (one forward transform per 64 inverse ones),
    // fewer while that would leave fewer than two CTAs per SM
    const char* e = getenv("TSD_HEADS_PPC");  // development override
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int ppc = 64;
    while (ppc > 1 && nblk * ((npairs + ppc - 1) / ppc) < 2 * nsm) ppc >>= 1;
    a.ppc = e ? std::max(1, atoi(e)) : ppc;
  }
  if (d_seed) CUDA_TRY(cudaMemsetAsync(d_seed, 0, sizeof(unsigned long long) * nrows, st));
  dim3 grid((unsigned)nblk, (unsigned)((npairs + a.ppc - 1) / a.ppc));
  k_heads_fft<<<grid, FFT_T, smem_h, st>>>(a);
  CUDA_TRY(cudaGetLastError());
  if (launches) *launches += 3;
  return kOk;
}

}  // namespace tsd

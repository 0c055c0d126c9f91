// join.cu -- z-normalised AB / dictionary join on sm_100a (FP64 path).
//
// Reference semantics: profiles.hpp:306-342 (ab_join) driven per segment by
// dictionary.hpp:149-193 (dict_min_profile). For every query window i and
// every valid dictionary window j (never straddling a segment boundary):
//   cov(i,j) = cov(i-1,j-1) + df_a[i]*dg_b[j] + dg_a[i]*df_b[j]   (profiles.hpp:330)
//   c = clamp(cov * invn_a[i] * invn_b[j])                         (:331-336)
//   row best: higher c wins, ties -> lower j                        (:70-77)
//
// B200 design:
//   * a warp owns a BAND of 256 consecutive query rows (8 per lane, "slots")
//     and sweeps the columns of every segment of its segment group. At step k
//     all lanes work on column k, so column data is a warp-uniform smem
//     broadcast and each slot's row data lives in registers for the whole
//     sweep. The diagonal recurrence moves one slot down per step (register
//     renaming, no moves) and crosses lanes with one shfl.up per step;
//   * lane 0's incoming diagonal comes from the bottom row of the band above
//     (edge buffer, staged through a 3-block smem ring with cp.async); lane 31
//     writes this band's bottom row back in place;
//   * diagonals entering a segment at its column 0 start from an exact head
//     (window_dot, profiles.hpp:101-108) computed as a register-blocked
//     sliding dot product; the first band of a task also computes the top
//     edge this way;
//   * per cell the FP64 pipe does 2 DFMA (update) + 1 DMUL (K = cov*invn_b);
//     the row test is one integer compare of K's high word against a
//     per-row threshold derived from the best K so far (conservative by one
//     high-word ulp). Only when some lane passes does the warp take the exact
//     slow path, which re-evaluates c exactly as the reference does and
//     applies the lexicographic rule. Row bests persist for the whole band
//     sweep, so after a short warm-up the slow path is rare.
#include <climits>
#include <cstdio>
#include <algorithm>

#include "tsd_common.cuh"
#include "tsd_internal.h"

namespace tsd {

namespace {

constexpr int R = 8;        // rows per lane
constexpr int H = 32 * R;   // rows per band
constexpr int WARPS = 4;    // warps per CTA
constexpr int T = 128;      // head staging chunk
__host__ __device__ constexpr int padidx(int i) { return i + (i >> 3); }
constexpr int SLIDE = padidx(H + T) + 8;

struct JoinArgs {
  const double* xa;
  int64_t na, nrows;
  const double* dfa;
  const double* dga;
  const double* invn_a;
  const double* mua;
  const uint8_t* flag_a;
  const double* xb;
  const double* mub;
  const double4* col;  // {df, dg, invn, 0} per concatenated column (padded by 64)
  const SegDev* segs;
  const int* seg_eoff;  // compact edge offset of each segment inside its group (even)
  const double* btil;   // [nseg][m] centred samples of each segment's window 0
  const double* ebt;    // [nseg] sum of btil
  int m;
  long long excl;
  int nbands, bands_per_task, ngroups, ntasks;
  const int* group_seg;  // [ngroups+1]
  int64_t ecap;          // per-warp edge capacity (doubles)
  double* edges;
  double* out_c;  // [ngroups][nrows]
  int64_t* out_j;
};

struct __align__(16) WarpSmem {
  double4 colbuf[2][32];
  double ering[96];
  double edummy[96];  // lanes 0..30 store here so lane 31's edge store needs no branch
  double scov[R][32];  // slow-path scratch: this step's covariances
  int sthr[R][32];     // slow-path scratch: thresholds
  double best_c[R][32];
  long long best_j[R][32];
  double ivan[R][32];
  double slide[SLIDE];
  double unif[T];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// out[r] = sum_{t<m} U[t] * (S[8*lane + r + t] - cS), U[t] = Ug[t] - cu.
// S samples at index >= s_avail read as cS (contribute 0). Returns sum U in *esum.
__device__ void sliding_dot(WarpSmem& sm, const double* __restrict__ Ug, double cu, const double* __restrict__ Sg,
                            int64_t s_avail, double cS, int m, int lane, double (&out)[R], double* esum) {
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = 0.0;
  double es = 0.0;
  const int base = R * lane;
  for (int t0 = 0; t0 < m; t0 += T) {
    const int tl = min(T, m - t0);
    __syncwarp();
    for (int q = lane; q < tl; q += 32) {
      const double u = Ug[t0 + q] - cu;
      sm.unif[q] = u;
      es += u;
    }
    for (int q = lane; q < H + tl; q += 32) {
      const int64_t gi = (int64_t)t0 + q;
      sm.slide[padidx(q)] = gi < s_avail ? Sg[gi] - cS : 0.0;
    }
    __syncwarp();
    double w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) w[r] = sm.slide[padidx(base + r)];
    int t = 0;
    for (; t + R <= tl; t += R) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const double uv = sm.unif[t + u];
#pragma unroll
        for (int r = 0; r < R; ++r) out[r] = __fma_rn(w[(r + u) & (R - 1)], uv, out[r]);
        w[u] = sm.slide[padidx(base + t + u + R)];
      }
    }
    // remainder (tl not a multiple of R): w[] holds S[base + t + (0..R-1)] in rotated order
    for (; t < tl; ++t) {
      const double uv = sm.unif[t];
#pragma unroll
      for (int r = 0; r < R; ++r) out[r] = __fma_rn(sm.slide[padidx(base + t + r)], uv, out[r]);
    }
  }
  if (esum) {
    for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
    *esum = es;
  }
}

struct SweepCtx {
  const double4* colg;  // global column data of this segment (col0 aligned)
  double* E;            // global edge array of this segment (j = 0 .. ncol-2)
  int ncol;
  int64_t colbase;  // concatenated column index of this segment's window 0
  long long row0;   // row of this lane's slot 0
  long long excl;   // self-join exclusion half-width, -1 for AB joins
  bool write_out;
};

// Slow path (taken by the whole warp when any lane's coarse test passed):
// exact reference evaluation and lexicographic update for every slot whose
// high-word test passed. Flat rows (invn_a == 0) follow profiles.hpp:332-336:
// c = 1 against a flat column, else clamp(cov*0*invn_b) = 0. The self-join
// exclusion zone |i - j| <= excl (profiles.hpp:273, :281-284) is rejected
// here. Kept out of line: it is rare after warm-up and would otherwise
// bloat every unrolled step.
__device__ __noinline__ void slow_all(WarpSmem& sm, int lane, double ivb, long long col, long long row0,
                                      long long excl) {
  for (int r = 0; r < R; ++r) {
    const double cov = sm.scov[r][lane];
    const double K = cov * ivb;
    const int thr = sm.sthr[r][lane];
    if (__double2hiint(K) < thr) continue;
    const long long row = row0 + r;
    if (excl >= 0 && (row - col <= excl && col - row <= excl)) continue;
    const double ia = sm.ivan[r][lane];
    double c;
    if (ia == 0.0) {
      c = ivb == 0.0 ? 1.0 : clamp_corr(cov * ia * ivb);
    } else {
      c = clamp_corr(cov * ia * ivb);  // profiles.hpp:331, :335
    }
    if (c > sm.best_c[r][lane]) {  // columns arrive in increasing order: ties never win
      sm.best_c[r][lane] = c;
      sm.best_j[r][lane] = col;
      int nt;
      if (ia == 0.0) {
        nt = c == 1.0 ? INT_MAX : INT_MIN;
      } else {
        const int h = __double2hiint(K);
        nt = h >= 0 ? h - 1 : INT_MIN;
      }
      sm.sthr[r][lane] = nt;
    }
  }
}

__device__ __forceinline__ double shfl_up1(double v) {
  int lo = __double2loint(v), hi = __double2hiint(v);
  asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;\n" : "+r"(lo));
  asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;\n" : "+r"(hi));
  return __hiloint2double(hi, lo);
}

__device__ __forceinline__ bool vote_any(bool p) {
  unsigned r;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n vote.sync.any.pred q, q, -1;\n selp.u32 %0, 1, 0, q;\n}\n"
      : "=r"(r)
      : "r"((unsigned)p));
  return r != 0;
}

template <bool FIRST, bool GUARD>
__device__ __forceinline__ void sweep_block(WarpSmem& sm, const SweepCtx& cx, int lane, int k0, double (&P)[R],
                                            const double (&dfa)[R], const double (&dga)[R], int (&thr)[R],
                                            const double (&head)[R]) {
  const int cslot = (k0 >> 5) & 1, ci = k0 & 31;
  const double* eprev = &sm.ering[(k0 + 95) % 96];  // E[k0-1]
  const double* ecur = &sm.ering[k0 % 96];          // E[k0 .. k0+6]
  // lane 31 stores into the ring, the others into a dummy copy of it
  double* sprev = (lane == 31 ? sm.ering : sm.edummy) + (k0 + 95) % 96;
  double* scur = (lane == 31 ? sm.ering : sm.edummy) + k0 % 96;
  const bool l0 = lane == 0;
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const int k = k0 + u;
    if (GUARD && k >= cx.ncol) break;
    const double2 dd = *reinterpret_cast<const double2*>(&sm.colbuf[cslot][ci + u]);
    const double dfb = dd.x, dgb = dd.y, ivb = sm.colbuf[cslot][ci + u].z;
    const int ph = (R - u) & (R - 1);  // physical register of slot 0 at this step
    if (FIRST && u == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) P[r] = head[r];
    } else {
      const double e = (u == 0) ? *eprev : ecur[u - 1];
      double in = shfl_up1(P[ph]);
      if (u == 0) *sprev = P[ph]; else scur[u - 1] = P[ph];
      P[ph] = l0 ? e : in;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double& c = P[(r + ph) & (R - 1)];
        c = __fma_rn(dfa[r], dgb, c);
        c = __fma_rn(dga[r], dfb, c);
      }
    }
    bool any = false;
#pragma unroll
    for (int r = 0; r < R; ++r) any |= __double2hiint(P[(r + ph) & (R - 1)] * ivb) >= thr[r];
    if (vote_any(any)) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        sm.scov[r][lane] = P[(r + ph) & (R - 1)];
        sm.sthr[r][lane] = thr[r];
      }
      slow_all(sm, lane, ivb, cx.colbase + k, cx.row0, cx.excl);
#pragma unroll
      for (int r = 0; r < R; ++r) thr[r] = sm.sthr[r][lane];
    }
  }
}

__device__ __forceinline__ void issue_chunk(WarpSmem& sm, const SweepCtx& cx, int lane, int c) {
  // column data for steps [32c, 32c+32): lane copies its column (32 B)
  const double4* src = cx.colg + 32 * c + lane;
  double4* dst = &sm.colbuf[c & 1][lane];
  cp16(dst, src);
  cp16(reinterpret_cast<char*>(dst) + 16, reinterpret_cast<const char*>(src) + 16);
  // edge block c: E[32c .. 32c+31] -> ring slot (c % 3)
  if (lane < 16) cp16(&sm.ering[(c % 3) * 32 + 2 * lane], cx.E + 32 * c + 2 * lane);
  cp_commit();
}

__device__ __forceinline__ void flush_block(WarpSmem& sm, const SweepCtx& cx, int lane, int b) {
  const int j = 32 * b + lane;
  if (j < cx.ncol - 1) cx.E[j] = sm.ering[(b % 3) * 32 + lane];
}

__device__ void sweep_segment(WarpSmem& sm, const SweepCtx& cx, int lane, const double (&dfa)[R],
                              const double (&dga)[R], int (&thr)[R], const double (&head)[R]) {
  double P[R];
  const int n = cx.ncol;
  const int nchunks = (n + 31) >> 5;
  __syncwarp();
  issue_chunk(sm, cx, lane, 0);
  if (nchunks > 1) issue_chunk(sm, cx, lane, 1); else cp_commit();
  cp_wait<1>();
  __syncwarp();
  int flushed = 0;  // blocks [0, flushed) written back
  // first 8-step block (contains k = 0)
  if (n <= R) {
    sweep_block<true, true>(sm, cx, lane, 0, P, dfa, dga, thr, head);
  } else {
    sweep_block<true, false>(sm, cx, lane, 0, P, dfa, dga, thr, head);
    int k0 = R;
    for (; k0 < n; k0 += R) {
      if ((k0 & 31) == 0) {
        const int c = k0 >> 5;  // chunk about to start
        __syncwarp();
        if (c >= 2 && cx.write_out) {
          flush_block(sm, cx, lane, c - 2);
          flushed = c - 1;
        }
        __syncwarp();
        if (c + 1 < nchunks) issue_chunk(sm, cx, lane, c + 1); else cp_commit();
        cp_wait<1>();
        __syncwarp();
      }
      if (k0 + R <= n)
        sweep_block<false, false>(sm, cx, lane, k0, P, dfa, dga, thr, head);
      else
        sweep_block<false, true>(sm, cx, lane, k0, P, dfa, dga, thr, head);
    }
  }
  cp_wait<0>();
  __syncwarp();
  if (cx.write_out) {
    const int last = (n - 2) >> 5;  // last edge block index holding j <= n-2
    for (int b = flushed; b <= last && n >= 2; ++b) flush_block(sm, cx, lane, b);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(32 * WARPS) k_join_f64(const JoinArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem* smem = reinterpret_cast<WarpSmem*>(smem_raw);
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  WarpSmem& sm = smem[wl];
  const int gw = blockIdx.x * WARPS + wl;
  const int nw = gridDim.x * WARPS;
  double* Ew = a.edges + (int64_t)gw * a.ecap;
  const int bpt = a.bands_per_task;

  for (int task = gw; task < a.ntasks; task += nw) {
    const int g = task % a.ngroups;
    const int b0 = (task / a.ngroups) * bpt;
    const int b1 = min(a.nbands, b0 + bpt);
    const int s_beg = a.group_seg[g], s_end = a.group_seg[g + 1];
    for (int b = b0; b < b1; ++b) {
      const int64_t i0 = (int64_t)b * H;
      double dfa[R], dga[R];
      int thr[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t i = i0 + R * lane + r;
        const bool in = i < a.nrows;
        const uint8_t f = in ? a.flag_a[i] : 0;
        dfa[r] = in ? a.dfa[i] : 0.0;
        dga[r] = in ? a.dga[i] : 0.0;
        sm.ivan[r][lane] = in ? a.invn_a[i] : 0.0;
        thr[r] = (f & 1) ? INT_MIN : INT_MAX;  // valid rows (flat rows: exact slow path)
        sm.best_c[r][lane] = -2.0;              // profiles.hpp:67
        sm.best_j[r][lane] = -1;
      }
      const double cA = a.mua[i0];
      for (int s = s_beg; s < s_end; ++s) {
        const SegDev sg = a.segs[s];
        SweepCtx cx;
        cx.colg = a.col + sg.col0;
        cx.E = Ew + a.seg_eoff[s];
        cx.ncol = sg.ncol;
        cx.colbase = sg.col0;
        cx.write_out = (b + 1 < b1);
        cx.row0 = i0 + R * lane;
        cx.excl = a.excl;
        if (b == b0 && sg.ncol >= 2) {
          // top edge of the task: E[j] = cov(re, j + delta), j = 0 .. ncol-2
          const int64_t re = i0 >= 1 ? i0 - 1 : 0;
          const int delta = i0 >= 1 ? 0 : 1;
          for (int q0 = delta; q0 < sg.ncol - 1 + delta; q0 += H) {
            double out[R];
            double eU;
            const double cS = a.mub[sg.col0 + q0];
            sliding_dot(sm, a.xa + re, a.mua[re], a.xb + sg.col0 + q0, (int64_t)sg.ncol + a.m - 1 - q0, cS, a.m,
                        lane, out, &eU);
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int q = q0 + R * lane + r;
              if (q < sg.ncol - 1 + delta) cx.E[q - delta] = out[r] - (a.mub[sg.col0 + q] - cS) * eU;
            }
          }
          __syncwarp();
          __threadfence_block();
        }
        // left edge: cov(i, col0) for the band's rows
        double head[R];
        {
          double out[R];
          sliding_dot(sm, a.btil + (int64_t)s * a.m, 0.0, a.xa + i0, a.na - i0, cA, a.m, lane, out, nullptr);
          const double e = a.ebt[s];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int64_t i = i0 + R * lane + r;
            const double mu = i < a.nrows ? a.mua[i] : cA;
            head[r] = out[r] - (mu - cA) * e;
          }
        }
        sweep_segment(sm, cx, lane, dfa, dga, thr, head);
      }
      // band results
      double* oc = a.out_c + (int64_t)g * a.nrows;
      int64_t* oj = a.out_j + (int64_t)g * a.nrows;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t i = i0 + R * lane + r;
        if (i < a.nrows) {
          oc[i] = sm.best_c[r][lane];
          oj[i] = sm.best_j[r][lane];
        }
      }
      __syncwarp();
    }
  }
}

// merge of per-group partials (lexicographic, group order = column order)
__global__ void k_merge_groups(double* __restrict__ c, int64_t* __restrict__ j, int64_t nrows, int ngroups) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double bc = c[i];
  int64_t bj = j[i];
  for (int g = 1; g < ngroups; ++g) {
    const double cc = c[(int64_t)g * nrows + i];
    const int64_t jj = j[(int64_t)g * nrows + i];
    if (jj >= 0 && (bj < 0 || better(cc, jj, bc, bj))) {
      bc = cc;
      bj = jj;
    }
  }
  c[i] = bc;
  j[i] = bj;
}

__global__ void k_pack_cols(const double* __restrict__ df, const double* __restrict__ dg,
                            const double* __restrict__ invn, int64_t n, double4* __restrict__ col) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n + 64) return;
  col[i] = i < n ? make_double4(df[i], dg[i], invn[i], 0.0) : make_double4(0, 0, 0, 0);
}

__global__ void k_btil(const double* __restrict__ xb, const double* __restrict__ mub, const SegDev* __restrict__ segs,
                       int m, double* __restrict__ btil, double* __restrict__ ebt) {
  const int s = blockIdx.x;
  const SegDev sg = segs[s];
  const double mu = mub[sg.col0];
  double acc = 0.0;
  for (int t = threadIdx.x; t < m; t += blockDim.x) {
    const double v = xb[sg.col0 + t] - mu;
    btil[(int64_t)s * m + t] = v;
    acc += v;
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sum += red[w];
    ebt[s] = sum;
  }
}

__global__ void k_epilogue(const double* __restrict__ bc, const int64_t* __restrict__ bj,
                           const uint8_t* __restrict__ flag, int64_t nrows, const SegDev* __restrict__ segs, int nseg,
                           int m, const int64_t* __restrict__ s_woff, const int64_t* __restrict__ s_ooff, int nser,
                           double* __restrict__ val, int64_t* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  if (!(flag[i] & 1)) return;
  int64_t o = i;
  if (nser > 1) {  // batched: row -> (series, window) -> packed output slot
    int lo = 0, hi = nser - 1, q = 0;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      if (s_woff[mid] <= i) {
        q = mid;
        lo = mid + 1;
      } else {
        hi = mid - 1;
      }
    }
    o = i - s_woff[q] + s_ooff[q];
  }
  const double c = bc[i];
  const int64_t j = bj[i];
  if (j < 0) {  // no admissible neighbour (profiles.hpp:149-151)
    val[o] = __longlong_as_double(0x7ff0000000000000LL);
    idx[o] = -1;
    return;
  }
  // concatenated column -> source coordinate (dictionary.hpp:183-188)
  int lo = 0, hi = nseg - 1, s = 0;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    if (segs[mid].col0 <= j) {
      s = mid;
      lo = mid + 1;
    } else {
      hi = mid - 1;
    }
  }
  val[o] = corr_to_dist(c, (double)m);
  idx[o] = segs[s].src0 + (j - segs[s].col0);
}

}  // namespace

#define CUDA_TRY(call)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      if (err) *err = Error{kCudaError, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
      return kCudaError;                                                                    \
    }                                                                                       \
  } while (0)

int run_join(const JoinInputs& in, double* d_best_c, int64_t* d_best_j, Arena& arena, cudaStream_t st, Error* err,
             int* launches) {
  if (in.precision != 0) {
    if (err) *err = Error{kInvalidArgument, "fp32 precision mode is not built in this version"};
    return kInvalidArgument;
  }
  const int m = in.m;
  const int nseg = (int)in.segs.size();
  const int64_t nrows = in.rows.nwin;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem_bytes = sizeof(WarpSmem) * WARPS;
  CUDA_TRY(cudaFuncSetAttribute(k_join_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_join_f64, 32 * WARPS, smem_bytes);
  if (occ < 1) occ = 1;
  const int nwarps = nsm * occ * WARPS;
  const int nbands = (int)((nrows + H - 1) / H);

  // segment groups: start with one group; split the dictionary while the
  // band count alone cannot fill the machine twice over
  int64_t total_cols = 0;
  for (const auto& s : in.segs) total_cols += s.ncol;
  int G = 1;
  while ((int64_t)nbands * G < 2LL * nwarps && G < nseg) G *= 2;
  if (G > nseg) G = nseg;
  std::vector<int> group_seg(G + 1, nseg);
  {
    int s = 0;
    int64_t acc = 0;
    group_seg[0] = 0;
    for (int g = 1; g < G; ++g) {
      const int64_t target = total_cols * g / G;
      while (s < nseg && acc + in.segs[s].ncol <= target) acc += in.segs[s++].ncol;
      if (s <= group_seg[g - 1]) s = std::min(nseg, group_seg[g - 1] + 1), acc = 0;
      group_seg[g] = s;
    }
    group_seg[G] = nseg;
  }
  std::vector<int> eoff(nseg);
  int64_t ecap = 0;
  for (int g = 0; g < G; ++g) {
    int64_t off = 0;
    for (int s = group_seg[g]; s < group_seg[g + 1]; ++s) {
      eoff[s] = (int)off;
      off += (in.segs[s].ncol + 1) & ~1;
    }
    ecap = std::max(ecap, off);
  }
  ecap = (ecap + 64 + 31) & ~int64_t(31);
  int bpt = (int)(((int64_t)nbands * G + nwarps - 1) / nwarps);
  if (bpt < 1) bpt = 1;
  const int nbr = (nbands + bpt - 1) / bpt;
  const int ntasks = nbr * G;
  const int grid = std::max(1, std::min(nsm * occ, (ntasks + WARPS - 1) / WARPS));
  const int used_warps = grid * WARPS;

  // device scratch
  SegDev* d_segs = (SegDev*)arena.get(sizeof(SegDev) * nseg);
  int* d_eoff = (int*)arena.get(sizeof(int) * nseg);
  int* d_gs = (int*)arena.get(sizeof(int) * (G + 1));
  double4* d_col = (double4*)arena.get(sizeof(double4) * (in.cols.nwin + 64));
  double* d_btil = (double*)arena.get(sizeof(double) * (int64_t)nseg * m);
  double* d_ebt = (double*)arena.get(sizeof(double) * nseg);
  double* d_edges = (double*)arena.get(sizeof(double) * ecap * used_warps);
  double* d_pc = G > 1 ? (double*)arena.get(sizeof(double) * nrows * G) : d_best_c;
  int64_t* d_pj = G > 1 ? (int64_t*)arena.get(sizeof(int64_t) * nrows * G) : d_best_j;
  if (!d_segs || !d_eoff || !d_gs || !d_col || !d_btil || !d_ebt || !d_edges || !d_pc || !d_pj) {
    if (err) *err = Error{kCudaError, "device allocation failed for the join"};
    return kCudaError;
  }
  CUDA_TRY(cudaMemcpyAsync(d_segs, in.segs.data(), sizeof(SegDev) * nseg, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_eoff, eoff.data(), sizeof(int) * nseg, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_gs, group_seg.data(), sizeof(int) * (G + 1), cudaMemcpyHostToDevice, st));
  int nl = 0;
  k_pack_cols<<<(unsigned)((in.cols.nwin + 64 + 255) / 256), 256, 0, st>>>(in.cols.df, in.cols.dg, in.cols.invn,
                                                                          in.cols.nwin, d_col);
  ++nl;
  k_btil<<<nseg, 128, 0, st>>>(in.xb, in.cols.mu, d_segs, m, d_btil, d_ebt);
  ++nl;
  JoinArgs a;
  a.xa = in.xa;
  a.na = in.na;
  a.nrows = nrows;
  a.dfa = in.rows.df;
  a.dga = in.rows.dg;
  a.invn_a = in.rows.invn;
  a.mua = in.rows.mu;
  a.flag_a = in.rows.flag;
  a.xb = in.xb;
  a.mub = in.cols.mu;
  a.col = d_col;
  a.segs = d_segs;
  a.seg_eoff = d_eoff;
  a.btil = d_btil;
  a.ebt = d_ebt;
  a.m = m;
  a.excl = in.excl;
  a.nbands = nbands;
  a.bands_per_task = bpt;
  a.ngroups = G;
  a.ntasks = ntasks;
  a.group_seg = d_gs;
  a.ecap = ecap;
  a.edges = d_edges;
  a.out_c = d_pc;
  a.out_j = d_pj;
  k_join_f64<<<grid, 32 * WARPS, smem_bytes, st>>>(a);
  ++nl;
  if (G > 1) {
    k_merge_groups<<<(unsigned)((nrows + 255) / 256), 256, 0, st>>>(d_pc, d_pj, nrows, G);
    ++nl;
    CUDA_TRY(cudaMemcpyAsync(d_best_c, d_pc, sizeof(double) * nrows, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d_best_j, d_pj, sizeof(int64_t) * nrows, cudaMemcpyDeviceToDevice, st));
  }
  CUDA_TRY(cudaGetLastError());
  if (launches) *launches += nl;
  return kOk;
}

int run_epilogue(const double* d_best_c, const int64_t* d_best_j, const uint8_t* d_row_flag, int64_t nrows,
                 const SegDev* d_segs, int nseg, int m, const int64_t* d_woff, const int64_t* d_ooff, int nser,
                 double* d_val, int64_t* d_idx, cudaStream_t st, Error* err) {
  k_epilogue<<<(unsigned)((nrows + 255) / 256), 256, 0, st>>>(d_best_c, d_best_j, d_row_flag, nrows, d_segs, nseg, m,
                                                               d_woff, d_ooff, nser, d_val, d_idx);
  CUDA_TRY(cudaGetLastError());
  return kOk;
}

}  // namespace tsd

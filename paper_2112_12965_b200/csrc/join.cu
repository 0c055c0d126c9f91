// join.cu -- z-normalised AB / dictionary / self join on sm_100a (FP64 path).
//
// Reference semantics: profiles.hpp:306-342 (ab_join) driven per segment by
// dictionary.hpp:149-193 (dict_min_profile), and profiles.hpp:266-301
// (self_join, exclusion zone as a parameter). For every query window i and
// every valid dictionary window j (never straddling a segment boundary):
//   cov(i,j) = cov(i-1,j-1) + df_a[i]*dg_b[j] + dg_a[i]*df_b[j]   (profiles.hpp:330)
//   c = clamp(cov * invn_a[i] * invn_b[j])                         (:331-336)
//   row best: higher c wins, ties -> lower j                        (:70-77)
//
// B200 design:
//   * a warp owns a BAND of 32*R consecutive query rows (R per lane,
//     "slots") and sweeps the columns of every segment of its segment group.
//     At step k all lanes work on column k, so column data is a warp-uniform
//     smem broadcast and each slot's row data lives in registers for the
//     whole sweep. The diagonal recurrence moves one slot down per step
//     (register renaming, no moves) and crosses lanes with one shfl.up;
//   * lane 0's incoming diagonal comes from the bottom row of the band above
//     (edge buffer, staged through a 3-block smem ring with cp.async); lane 31
//     writes this band's bottom row back in place;
//   * diagonals entering a segment at its column 0 start from an exact head
//     (window_dot, profiles.hpp:101-108) computed as a register-blocked
//     sliding dot product; the first band of a task computes the top edge
//     the same way;
//   * per cell the FP64 pipe does 2 DFMA (update) + 1 DMUL (K = cov*invn_b,
//     the row-constant invn_a factored out); the row test is ONE integer
//     compare of K's high word against a per-row threshold (high word of the
//     best K so far, minus one, so the test is conservative). Only when some
//     lane passes does the warp run the exact update (full-precision compare
//     of K, lowest column on ties since columns arrive in increasing order).
//     Flat rows (invn_a == 0) are resolved in the epilogue from the flat
//     column table (profiles.hpp:332-336 gives them c in {0, 1}).
#include <algorithm>
#include <chrono>
#include <queue>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "tsd_common.cuh"
#include "tsd_internal.h"

namespace tsd {

namespace {

#ifndef TSD_TB
#define TSD_TB 8
#endif
constexpr int TB = TSD_TB;  // threshold block (columns); nmin spans TB columns (k_pack_cols)
#ifndef TSD_WARPS
#define TSD_WARPS 2
#endif
constexpr int WARPS = TSD_WARPS;  // warps per CTA (independent; small CTAs give finer occupancy steps)
constexpr int T = 64;     // head / top-edge staging chunk (samples)
// Register budgets. The default kernels take __launch_bounds__(64, MINB): with
// MINB = 7 ptxas settles at 128 registers (a few bytes of call-site spills),
// so 8 two-warp CTAs fit per SM at run time. TSD_NREG* > 0 instead caps the
// registers with __maxnreg__ (the two qualifiers exclude each other): 144 ->
// 7 CTAs (14 warps) per SM.
#ifndef TSD_JOIN_MINB
#define TSD_JOIN_MINB 7
#endif
#ifndef TSD_JOIN_MINB32
#define TSD_JOIN_MINB32 7
#endif
#ifndef TSD_JOIN_MINB_SYM
#define TSD_JOIN_MINB_SYM 7
#endif
#ifndef TSD_NREG
#define TSD_NREG 0     // FP64 AB / full-matrix sweep
#endif
#ifndef TSD_NREG32
#define TSD_NREG32 0   // FP32 sweep
#endif
#ifndef TSD_NREG_WIDE
#define TSD_NREG_WIDE 0  // wide FP64 sweep (ablation build)
#endif
#ifndef TSD_NREG_SYM
#define TSD_NREG_SYM 0  // symmetric self-join sweep
#endif
#ifndef TSD_PRED_EDGE
#define TSD_PRED_EDGE 1  // lane 0's incoming diagonal by a predicated load over its shuffle result (no select)
#endif
#ifndef TSD_PIPE
#define TSD_PIPE 1  // the software-pipelined FP64 sweep (sweep_segment_p) for the AB / full-matrix joins
#endif

template <int R>
__host__ __device__ constexpr int padidx(int i) {
  return i + i / R;  // one pad double per R: lane-strided R-wide windows are bank-conflict free
}

template <int R>
struct Geo {
  static constexpr int H = 32 * R;  // rows per band
  static constexpr int SLIDE = padidx<R>(32 * R + T) + R;
};

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
  const double4* col;   // column data (k_pack_cols / k_pack_cols32), padded by 64
  double f32_sig, f32_siga;  // FP32 sweep: cov scale sigma_a * sigma_b, row-data scale sigma_a (powers of 2)
  const SegDev* segs;
  const int* seg_eoff;  // compact edge offset of each segment inside its group (even)
  const double* btil;   // [nseg][m] centred samples of each segment's window 0
  const double* ebt;    // [nseg] sum of btil
  int m;
  long long excl;  // self-join exclusion half-width (SELF kernels only)
  int nbands, bands_per_task, ngroups, ntasks;
  const int* group_seg;  // [ngroups+1]
  int64_t ecap;          // per-warp edge capacity (doubles)
  double* edges;
  double* hscr;   // per-warp head scratch [8][256]
  int dmma_heads; // heads on the FP64 tensor cores (else register-blocked sliding dot)
  const double* heads;  // precomputed final heads [seg][hstride] (heads_fft.cu), or null
  int64_t hstride;
  // per-row order key of the best known candidate, or null: seeded by the
  // heads (heads_fft.cu) and raised by every finished band (non-SYM)
  unsigned long long* seed;
  const double* tedge;  // top edges by FFT: tedge[r * tstride + c] = cov(top row of band range r, column c), or null
  int64_t tstride;
  double* out_c;  // [ngroups][nrows]
  int64_t* out_j;
  // symmetric self-join (SYM kernels): task queue and the column side
  const int4* tasks;             // {band0, band1, group, 0}, longest first
  int* task_next;                // dynamic task counter
  unsigned long long* ccand;     // [SYM_NC][ccols]: {order key of corr, row index} (16 B, 128-bit CAS)
  int64_t ccols;                 // columns per ccand copy
  double* cthr;                  // per column: kplus(best corr) * norm_b * (1 - 2^-40)
  // buffer extents for TSD_CHECKED builds
  int nseg_v;                    // virtual segments
  int64_t hrows_alloc;           // heads rows allocated per segment (hstride)
  int64_t tedge_rows;            // rows of the top-edge table
  int nwarps_alloc;              // warps with edge / head scratch
};

// W: the wide FP64 sweep (R = 16 rows per lane with FP64 bests)
template <int R, bool W = false>
struct __align__(16) WarpSmem {
  double4 colbuf[3][32];
  double ering[96];
  // SYM-only members (the symmetric sweep is the FP64 R = 8 kernel; the FP32
  // R = 16 layout keeps them as stubs to fit 8 CTAs per SM)
  static constexpr int NSYM = R == 8 ? 1 : 0;
  double cring[NSYM ? 96 : 1];   // SYM: column thresholds (cthr snapshot), same ring layout as ering
  double cminb[NSYM ? 24 : 1];   // SYM: weakest column threshold of each 4-column block of the ring
  double inva[NSYM ? R : 1][32];  // SYM: invn_a of each slot's row (column-side candidates)
  // SYM: column candidates found since the last chunk turn ({order key, row,
  // col}; at most 40 = the 8 steps after the last turn plus a segment's last
  // chunk, which has no turn), merged into ccand at the next turn or at the
  // segment end, one lane per entry. (Sizes matter: 8 two-warp CTAs per SM
  // leave 14080 B per warp.)
  unsigned long long cq_key[NSYM ? 40 : 1];
  unsigned cq_row[NSYM ? 40 : 1];
  int cq_col[NSYM ? 40 : 1];
  int cq_n;
  // best K = cov * invn_b per slot (row factor invn_a left out); +inf =
  // inactive row. The FP32 sweep (R = 16) keeps FP32 bests: float storage
  // fits its 16 rows per lane in 8 CTAs per SM
  std::conditional_t<R == 8 || W, double, float> bK[R][32];
  int bj[R][32];     // its concatenated column
  double slide[Geo<R>::SLIDE];
  double unif[T];
};

// 8 two-warp CTAs per SM: 233472 B of shared memory less 1 KiB reserved per CTA
static_assert(sizeof(WarpSmem<8>) <= 14080 && sizeof(WarpSmem<16>) <= 14080,
              "per-warp shared memory must fit 8 two-warp CTAs per SM");

#ifdef TSD_COUNT_EXACT
__device__ unsigned long long g_exact_count, g_step_count, g_exact_first, g_step_first, g_col_count, g_cas_count,
    g_true_steps, g_true_slots, g_rare_cycles, g_total_cycles;
#endif

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ double shfl_up1(double v) {
  int lo = __double2loint(v), hi = __double2hiint(v);
  asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;\n" : "+r"(lo));
  asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;\n" : "+r"(hi));
  return __hiloint2double(hi, lo);
}

// warp vote over R = 8 slot tests "hi(c~) >= thr": two independent 4-deep
// predicate chains joined by one OR (ptxas otherwise builds one 8-deep chain)
#ifndef TSD_VOTE1
#define TSD_VOTE1 1  // pipelined AB sweep: C4-shape kernel -1 %; the symmetric sweep keeps two chains (+5 % with one)
#endif
template <int R, bool CHAIN1 = false>
__device__ __forceinline__ bool vote_any8(const double (&P)[R], int ph, const int (&thr)[R]) {
  static_assert(R == 8, "vote_any8 is written for R = 8");
  unsigned r;
  if (CHAIN1) {  // one 8-deep predicate chain (no PLOP3 join): the pipelined sweep tests a column while
                 // the next one's DFMAs issue, so the longer chain stays off its critical path
    asm volatile(
        "{\n .reg .pred a;\n"
        " setp.ge.s32 a, %1, %9;\n setp.ge.or.s32 a, %2, %10, a;\n"
        " setp.ge.or.s32 a, %3, %11, a;\n setp.ge.or.s32 a, %4, %12, a;\n"
        " setp.ge.or.s32 a, %5, %13, a;\n setp.ge.or.s32 a, %6, %14, a;\n"
        " setp.ge.or.s32 a, %7, %15, a;\n setp.ge.or.s32 a, %8, %16, a;\n"
        " vote.sync.any.pred a, a, -1;\n selp.u32 %0, 1, 0, a;\n}\n"
        : "=r"(r)
        : "r"(__double2hiint(P[(0 + ph) & 7])), "r"(__double2hiint(P[(1 + ph) & 7])),
          "r"(__double2hiint(P[(2 + ph) & 7])), "r"(__double2hiint(P[(3 + ph) & 7])),
          "r"(__double2hiint(P[(4 + ph) & 7])), "r"(__double2hiint(P[(5 + ph) & 7])),
          "r"(__double2hiint(P[(6 + ph) & 7])), "r"(__double2hiint(P[(7 + ph) & 7])), "r"(thr[0]), "r"(thr[1]),
          "r"(thr[2]), "r"(thr[3]), "r"(thr[4]), "r"(thr[5]), "r"(thr[6]), "r"(thr[7]));
    return r != 0;
  }
  asm volatile(
      "{\n .reg .pred a, b;\n"
      " setp.ge.s32 a, %1, %9;\n setp.ge.s32 b, %5, %13;\n"
      " setp.ge.or.s32 a, %2, %10, a;\n setp.ge.or.s32 b, %6, %14, b;\n"
      " setp.ge.or.s32 a, %3, %11, a;\n setp.ge.or.s32 b, %7, %15, b;\n"
      " setp.ge.or.s32 a, %4, %12, a;\n setp.ge.or.s32 b, %8, %16, b;\n"
      " or.pred a, a, b;\n vote.sync.any.pred a, a, -1;\n selp.u32 %0, 1, 0, a;\n}\n"
      : "=r"(r)
      : "r"(__double2hiint(P[(0 + ph) & 7])), "r"(__double2hiint(P[(1 + ph) & 7])),
        "r"(__double2hiint(P[(2 + ph) & 7])), "r"(__double2hiint(P[(3 + ph) & 7])),
        "r"(__double2hiint(P[(4 + ph) & 7])), "r"(__double2hiint(P[(5 + ph) & 7])),
        "r"(__double2hiint(P[(6 + ph) & 7])), "r"(__double2hiint(P[(7 + ph) & 7])), "r"(thr[0]), "r"(thr[1]),
        "r"(thr[2]), "r"(thr[3]), "r"(thr[4]), "r"(thr[5]), "r"(thr[6]), "r"(thr[7]));
  return r != 0;
}


// out[r] = sum_{t<m} U[t] * (S[R*lane + r + t] - cS), U[t] = Ug[t] - cu.
// S samples at index >= s_avail read as cS (contribute 0). Returns sum U in *esum.
template <int R, bool W>
__device__ void sliding_dot(WarpSmem<R, W>& sm, const double* __restrict__ Ug, double cu, const double* __restrict__ Sg,
                            int64_t s_avail, double cS, int m, int lane, double (&out)[R], double* esum) {
  constexpr int H = Geo<R>::H;
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
      sm.slide[padidx<R>(q)] = gi < s_avail ? Sg[gi] - cS : 0.0;
    }
    __syncwarp();
    // padidx(base + t + j) = padidx(base + t) + j + j / R for t % R == 0
    const double* sp = &sm.slide[padidx<R>(base)];
    const double* up = sm.unif;
    double w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) w[r] = sp[r];
    int t = 0;
    for (; t + R <= tl; t += R, sp += R + 1, up += R) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const double uv = up[u];
#pragma unroll
        for (int r = 0; r < R; ++r) out[r] = __fma_rn(w[(r + u) & (R - 1)], uv, out[r]);
        w[u] = sp[u + R + 1];  // sample base + t + u + R
      }
    }
    for (; t < tl; ++t) {  // remainder
      const double uv = sm.unif[t];
#pragma unroll
      for (int r = 0; r < R; ++r) out[r] = __fma_rn(sm.slide[padidx<R>(base + t + r)], uv, out[r]);
    }
  }
  if (esum) {
    for (int o = 16; o > 0; o >>= 1) es += __shfl_xor_sync(0xffffffffu, es, o);
    *esum = es;
  }
}

// Left-edge heads of a band against a batch of up to 8 segments on the FP64
// tensor cores (mma.sync.m8n8k4.f64): H[i][s] = sum_k xt[i + k] * btil_s[k],
// a (256 x m) Toeplitz x (m x 8) product. The sweep is issue-bound, not
// FP64-pipe-bound (profiles/), and one DMMA does the work of 8 DFMA warp
// instructions. Output: hout[s * 256 + i] (per-warp global scratch), before
// the (mu_i - cS) * e_s correction and the column scale.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int R>
__device__ __noinline__ void heads_dmma(WarpSmem<R>& sm, const double* __restrict__ Sg, int64_t s_avail, double cS,
                                        const double* __restrict__ Bt, int nb, int m, int lane,
                                        double* __restrict__ hout) {
  static_assert(Geo<R>::H == 256, "heads_dmma tiles a 256-row band");
  static_assert(Geo<R>::SLIDE >= 96 + 8 * 33, "heads_dmma stages in sm.slide");
  const int g = lane >> 2, t = lane & 3;
  double* xs = sm.slide;       // 96 staged query samples: rows [64 grp, +64) x k [k0, +32)
  double* bs = sm.slide + 96;  // 8 segments x 32 k, row stride 33 (bank spread)
  for (int grp = 0; grp < 4; ++grp) {
    double c[8][2];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) c[mt][0] = c[mt][1] = 0.0;
    // register double buffer: chunk k0 + 32 is in flight while chunk k0 multiplies
    double xr[3], br[8];
    auto load = [&](int k0) {
      const int kl = min(32, m - k0);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int64_t gi = (int64_t)64 * grp + k0 + 32 * j + lane;
        xr[j] = gi < s_avail ? Sg[gi] : cS;
      }
#pragma unroll
      for (int sg = 0; sg < 8; ++sg) br[sg] = (sg < nb && lane < kl) ? Bt[(int64_t)sg * m + k0 + lane] : 0.0;
    };
    load(0);
    for (int k0 = 0; k0 < m; k0 += 32) {
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 3; ++j) xs[32 * j + lane] = xr[j] - cS;
#pragma unroll
      for (int sg = 0; sg < 8; ++sg) bs[sg * 33 + lane] = br[sg];
      __syncwarp();
      if (k0 + 32 < m) load(k0 + 32);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const double bv = bs[g * 33 + 4 * ks + t];  // B[k = t][n = g]
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) dmma884(c[mt][0], c[mt][1], xs[8 * mt + g + 4 * ks + t], bv);
      }
    }
    // C[row g][col 2t, 2t+1] of tile mt -> rows 64 grp + 8 mt + g, segments 2t, 2t+1
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const int row = 64 * grp + 8 * mt + g;
      hout[(2 * t) * 256 + row] = c[mt][0];
      hout[(2 * t + 1) * 256 + row] = c[mt][1];
    }
  }
  __syncwarp();
}

struct SweepCtx {
  const double4* colg;  // global column data of this segment (col0 aligned)
  double* E;            // global edge array of this segment (j = 0 .. ncol-2)
  int ncol;
  int colbase;     // concatenated column index of this segment's window 0
  long long row0;  // row of this lane's slot 0
  long long excl;  // self-join exclusion half-width
  bool write_out;
  bool first_seg;  // diagnostics only
  const double* cthr;  // SYM: column thresholds of this segment (col0 aligned)
  double namin;        // SYM: (smallest row norm among this lane's slots)
};

// chunk c of the segment: column data for steps [32c, 32c+32) -> colbuf[c%3],
// edge block c (E[32c .. 32c+31]) -> ring slot c%3
template <int R, bool W>
__device__ __forceinline__ void issue_chunk(WarpSmem<R, W>& sm, const SweepCtx& cx, int lane, int c) {
  const double4* src = cx.colg + 32 * c + lane;
  double4* dst = &sm.colbuf[c % 3][lane];
  cp16(dst, src);
  cp16(reinterpret_cast<char*>(dst) + 16, reinterpret_cast<const char*>(src) + 16);
  if (lane < 16) cp16(&sm.ering[(c % 3) * 32 + 2 * lane], cx.E + 32 * c + 2 * lane);
  else if (cx.cthr) cp16(&sm.cring[(c % 3) * 32 + 2 * (lane - 16)], cx.cthr + 32 * c + 2 * (lane - 16));
  cp_commit();
}

// SYM: once chunk c is resident, the weakest threshold of each of its eight
// 4-column blocks (one lane per block)
template <int R>
__device__ __forceinline__ void fold_cmin(WarpSmem<R>& sm, int lane, int c) {
  if (lane < 32 / TB) {
    const double* t = &sm.cring[(c % 3) * 32 + TB * lane];
    double v = t[0];
#pragma unroll
    for (int q = 1; q < TB; ++q) v = fmin(v, t[q]);
    sm.cminb[(c % 3) * (32 / TB) + lane] = v;
  }
  __syncwarp();
}

template <int R, bool W>
__device__ __forceinline__ void flush_block(WarpSmem<R, W>& sm, const SweepCtx& cx, int lane, int b) {
  const int j = 32 * b + lane;
  TSD_CHECK(b >= 0 && (b % 3) * 32 + lane < 96);
  if (j < cx.ncol - 1) cx.E[j] = sm.ering[(b % 3) * 32 + lane];
}

// ---------------------------------------------------------------------------
// Symmetric self-join, column side. The reference walks each admissible
// unordered pair once and updates both rows (profiles.hpp:287-297). A band
// here sweeps only columns j > i + excl (upper triangle); besides its own
// rows (row side, as in the AB join) every cell is a candidate for row j's
// profile -- the column side. Per step the warp tests all 8 x 32 cells of
// column j against one threshold: corr = cov * invn_a * invn_b > best_j
// implies cov > best_j * norm_b[j] * min(norm_a over the lane's rows), i.e.
// hi(cov) >= hi(cthr[j] * namin) with cthr[j] = kplus(best_j) * norm_b[j] *
// (1 - 2^-40) staged per chunk. A pass reduces the warp's best (corr, row)
// (max corr, lowest row) and merges it into ccand[j] with a 128-bit CAS.
__device__ __forceinline__ double kplus_d(double b) { return b > 0.0 ? b : -0.0; }
// 1/x for positive normal x without the division's divergent slow-path call
// (which would make the compiler guard every later shuffle and vote of the
// sweep with divergence checks): approximate reciprocal + two Newton steps,
// within an ulp or two -- used only inside thresholds that carry a 2^-40 slack
__device__ __forceinline__ double rcp_pos(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = __fma_rn(r, __fma_rn(-x, r, 1.0), r);
  return __fma_rn(r, __fma_rn(-x, r, 1.0), r);
}
// SYM column candidates are spread over SYM_NC copies (by task) so that the
// many bands sweeping the same columns at once do not serialise on one CAS
// target; the copies are merged per row after the join
constexpr int SYM_NC = 16;
__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

__device__ __forceinline__ void cas128(unsigned long long* p, unsigned long long clo, unsigned long long chi,
                                       unsigned long long nlo, unsigned long long nhi, unsigned long long& olo,
                                       unsigned long long& ohi) {
  asm volatile(
      "{\n .reg .b128 d, c, s;\n mov.b128 c, {%2, %3};\n mov.b128 s, {%4, %5};\n"
      " atom.global.cas.b128 d, [%6], c, s;\n mov.b128 {%0, %1}, d;\n}\n"
      : "=l"(olo), "=l"(ohi)
      : "l"(clo), "l"(chi), "l"(nlo), "l"(nhi), "l"(p)
      : "memory");
}

// vals: the lane's 8 slot covariances at column col (shared memory [8][32]);
// cm: slots that passed the column threshold. The warp's lexicographic best (max corr, lowest row) is found
// with three REDUX reductions on the order key and the row.
template <int R>
__device__ __noinline__ void col_update(WarpSmem<R>& sm, int lane, unsigned cm, int row0, int col, double invb,
                                        int excl, double* cthr) {
  // window indices fit 32 bits (the C ABI bounds n), which keeps this rarely
  // called function inside a few registers (no spills around the sweep)
  unsigned long long bk = 0;  // order key of the lane's best corr (0 = none)
  unsigned brow = 0xffffffffu;
  if (invb > 0.0) {
    // all slots at once (independent load -> multiply -> select chains, no
    // serial loop over the set bits); descending slots with >= keep the
    // lowest row on equal keys
#pragma unroll
    for (int r = R - 1; r >= 0; --r) {
      const int d = col - (row0 + r);
      const double ia = sm.inva[r][lane];  // 0 for inactive rows
      // the same rounding as the row side's clamp((cov * invn_b) * invn_a):
      // both rows of a pair see the bitwise-identical correlation, as in the
      // reference (one value updates both, profiles.hpp:289-296)
      const double c = clamp_corr(sm.slide[r * 32 + lane] * invb * ia);
      const unsigned long long k = order_key(c);
      const bool ok = ((cm >> r) & 1u) && ia > 0.0 && (d > excl || d < -excl);
      if (ok && k >= bk) {
        bk = k;
        brow = (unsigned)(row0 + r);
      }
    }
  }
  const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(bk >> 32));
  const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(bk >> 32) == hi ? (unsigned)bk : 0u);
  const unsigned long long wk = ((unsigned long long)hi << 32) | lo;
  const unsigned wrow = __reduce_min_sync(0xffffffffu, bk == wk ? brow : 0xffffffffu);
#ifdef TSD_COUNT_EXACT
  if (lane == 0) atomicAdd(&g_col_count, 1ull);
  if (lane == 0 && wk != 0) atomicAdd(&g_cas_count, 1ull);
#endif
  if (lane == 0 && wk != 0) {
    // raise the column threshold now (a real pair's value never exceeds the
    // row's final best; non-returning atomic) and queue the (corr, row)
    // candidate for the 128-bit merge at the next chunk turn
    const double t = kplus_d(key_value(wk)) * rcp_pos(invb) * (1.0 - 0x1p-40);
    atomicMax(reinterpret_cast<long long*>(cthr + col), __double_as_longlong(t));
    const int q = sm.cq_n;
    TSD_CHECK(q < 40);
    sm.cq_key[q] = wk;
    sm.cq_row[q] = wrow;
    sm.cq_col[q] = col;
    sm.cq_n = q + 1;
  }
}

// merge the queued column candidates: one lane per entry, all CAS latencies
// overlapped
template <int R>
__device__ __noinline__ void col_flush(WarpSmem<R>& sm, int lane, unsigned long long* ccand) {
  __syncwarp();
  // every loop runs a warp-uniform trip count (lane 0's count, votes): a
  // divergent exit from this call would make the compiler guard every
  // shuffle and vote of the sweep with divergence checks
  const int nq = __shfl_sync(0xffffffffu, sm.cq_n, 0);
  for (int base = 0; base < nq; base += 32) {
    const int e = base + lane;
    bool pend = e < nq;
    unsigned long long* p = ccand;
    unsigned long long nk = 0, ni = 0, ck = 0, ci = 0;
    if (pend) {
      TSD_CHECK(sm.cq_n <= 40 && sm.cq_col[e] >= 0);
      p = ccand + 2 * (long long)sm.cq_col[e];
      nk = sm.cq_key[e];
      ni = sm.cq_row[e];
      ck = p[0];  // may be torn: the CAS validates
      ci = p[1];
      pend = nk > ck || (nk == ck && ni < ci);
    }
    while (__any_sync(0xffffffffu, pend)) {
      if (pend) {
        unsigned long long ok, oi;
        cas128(p, ck, ci, nk, ni, ok, oi);
        if (ok == ck && oi == ci) {
          pend = false;
        } else {
          ck = ok;
          ci = oi;
          pend = nk > ck || (nk == ck && ni < ci);
        }
      }
    }
  }
  __syncwarp();
  if (lane == 0) sm.cq_n = 0;
  __syncwarp();
}

// SYM exact update, shared by every unrolled step (one copy of the code keeps
// the sweep loop inside the instruction cache). vals: the lane's 8 slot
// covariances in logical slot order (shared memory [8][32]). Row side as in
// sweep_block; column side via col_update. Returns the lane's mask of slots
// whose best changed (the caller refreshes their thresholds).
template <int R>
__device__ __noinline__ unsigned exact_update_sym(WarpSmem<R>& sm, int lane, int col, double invb, int tc, int row0,
                                                  int excl, double* cthr) {
  unsigned upd = 0, cm = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double v = sm.slide[r * 32 + lane];
    const double K = v * invb;
    const int d = row0 + r - col;
    if (K > sm.bK[r][lane] && (d > excl || d < -excl)) {  // profiles.hpp:70-77, :281-284
      sm.bK[r][lane] = K;
      sm.bj[r][lane] = col;
      upd |= 1u << r;
    }
    cm |= (__double2hiint(v) >= tc ? 1u : 0u) << r;
  }
  if (__any_sync(0xffffffffu, cm != 0)) col_update<R>(sm, lane, cm, row0, col, invb, excl, cthr);
  return upd;
}

// FP64 sweep: the unnormalised centred recurrence of the reference
// (profiles.hpp:330), 2 FMAs per cell,
//   cov(i, k) = cov(i-1, k-1) + df_a[i] dg_b[k] + dg_a[i] df_b[k],
// and a row test without a per-cell multiply: the candidate K = cov * invn_b
// (row factor invn_a left out) can beat bestK > 0 only if
//   cov > bestK / invn_b >= bestK * nmin(block),
// nmin = (1 - 2^-40) x the smallest window norm among the TB = 4 columns of
// the threshold block (k_pack_cols; the factor absorbs the roundings of the
// exact test). The threshold is compared on high words (integer pipe):
// thr = hi(bestK+ * nmin)
// with bestK+ = bestK if bestK > 0, else -0.0, whose product -0.0 has high
// word INT_MIN (passes everything). Inactive rows carry bestK = +inf
// (thr = hi(inf), never passed by a finite cov). A pass runs the exact update
// K = cov * invn_b > bestK against the real bestK in shared memory.
__device__ __forceinline__ double kplus(double bK) { return bK > 0.0 ? bK : -0.0; }

// Column data of one step (k_pack_cols: {df_b, dg_b, invn_b, nmin}), the
// incoming diagonal of lane 0 (edge ring) and of lanes 1..31 (shuffle)
struct StepIn {
  double dfb, dgb, e, in, nmin;  // nmin: loaded with the first column of a threshold block
};

__device__ __forceinline__ void prefetch(bool nm, const double4* cb, const double* ep, double v7, StepIn& d, bool l0) {
  if (nm) {  // constant after unrolling
    const double4 c = *cb;
    d.dfb = c.x;
    d.dgb = c.y;
    d.nmin = c.w;
  } else {
    const double2 c = *reinterpret_cast<const double2*>(cb);
    d.dfb = c.x;
    d.dgb = c.y;
  }
  d.in = shfl_up1(v7);
  // lane 0 overwrites its shuffle result with the band above's edge (a
  // predicated load instead of a per-step select on the ALU pipe)
  if (TSD_PRED_EDGE && l0) d.in = *ep;
  if (!TSD_PRED_EDGE) d.e = *ep;
}

template <int R>
struct SweepState {
  double P[R];    // slot registers: step k, slot r at P[(r - k) mod R]
  double bKp[R];  // kplus(bestK); bestK itself and its column live in sm.bK / sm.bj
  int thr[R];     // hi(bKp * nmin) of the current block
  StepIn nx;      // prefetched inputs of the next step
  bool dirty;     // (warp-uniform) a best changed: reload bKp at the next threshold block
};

// FP64 exact update of one step (AB / full-matrix self-join), shared by every
// unrolled step so the sweep loop stays small in the instruction cache: the
// lane's slot covariances staged in slot order (sm.slide[r * 32 + lane]),
// K = cov * invn_b against the best in sm.bK, strict > (columns arrive in
// increasing order, so ties keep the lower column, profiles.hpp:70-77; a flat
// column has invn_b = 0 -> K = 0, :332-336). Returns whether any best of the
// warp changed.
template <int R, bool SELF, bool W>
__device__ __noinline__ bool exact_update64(WarpSmem<R, W>& sm, int lane, int col, double invb, long long row0,
                                            long long excl) {
  bool any = false;
#ifdef TSD_COUNT_EXACT
  int nupd = 0;
#endif
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double K = sm.slide[r * 32 + lane] * invb;
    bool ok = K > sm.bK[r][lane];
    if (SELF) {
      const long long d = row0 + r - col;
      ok = ok && (d > excl || d < -excl);  // profiles.hpp:281-284
    }
    if (ok) {
      sm.bK[r][lane] = K;
      sm.bj[r][lane] = col;
      any = true;
    }
#ifdef TSD_COUNT_EXACT
    nupd += ok;
#endif
  }
#ifdef TSD_COUNT_EXACT
  {
    const unsigned anyu = __ballot_sync(0xffffffffu, nupd > 0);
    for (int o = 16; o; o >>= 1) nupd += __shfl_xor_sync(0xffffffffu, nupd, o);
    if (lane == 0 && anyu) atomicAdd(&g_true_steps, 1ull);
    if (lane == 0) atomicAdd(&g_true_slots, (unsigned long long)nupd);
  }
#endif
  return __any_sync(0xffffffffu, any);
}

// One block of R steps starting at k0 (k0 % R == 0, R | 32). FIRST: block 0,
// whose step 0 (heads, already in P) only needs its test. GUARD: steps may
// run past ncol. Ring/colbuf positions are resolved once per block: E[k0 ..
// k0+R-1] are contiguous, only E[k0-1] may sit in the previous ring block,
// and only step k0+R's column data in the next chunk.
template <int R, bool SELF, bool FIRST, bool GUARD, bool SYM>
__device__ __forceinline__ void sweep_block(WarpSmem<R>& sm, const SweepCtx& cx, int lane, int k0, int m96,
                                            SweepState<R>& S, const double (&dfa)[R], const double (&dga)[R],
                                            double* sbase, bool l0, const double* __restrict__ invn_a,
                                            long long nrows, unsigned long long* ccand, double* cthr) {
  // colbuf and the edge ring are both 96-entry rings indexed by column mod 96
  const int n = cx.ncol;
  const double4* cflat = &sm.colbuf[0][0];
  const double4* ccur = cflat + m96;
  const double4* cnext = cflat + (m96 + R == 96 ? 0 : m96 + R);
  const int ebase = m96;                                    // ring position of E[k0]
  double* const st_prev = sbase + (m96 == 0 ? 95 : m96 - 1);  // E[k0-1]
  double* const st_cur = sbase + ebase;
  double nmin = 0.0;
  int tcb = INT_MAX;  // SYM: column threshold of the current threshold block
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const int k = k0 + u;
    if (GUARD && k >= n) break;
    const int ph = (R - u) & (R - 1);  // physical register of slot 0 at this step
    if (u % TB == 0) {  // threshold block of TB columns (nmin prefetched with its first column)
      nmin = (FIRST && u == 0) ? ccur[0].w : S.nx.nmin;
      if (S.dirty) {  // bests raised by the shared exact update since the last block
#pragma unroll
        for (int r = 0; r < R; ++r) S.bKp[r] = kplus(sm.bK[r][lane]);
        S.dirty = false;
      }
#ifdef TSD_ABL_NOCOLFOLD
      if (false) {
#else
      if (SYM) {  // column side folded in: the block's weakest column threshold
#endif
        tcb = __double2hiint(sm.cminb[(ebase + u) / TB] * cx.namin);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) S.thr[r] = SYM ? min(__double2hiint(S.bKp[r] * nmin), tcb)
                                                  : __double2hiint(S.bKp[r] * nmin);
    }
    if (!(FIRST && u == 0)) {
      // fold in the incoming diagonal; lane 31 retires its bottom-row value (column k-1)
      (u == 0 ? st_prev : st_cur + u - 1)[0] = S.P[ph];
      S.P[ph] = TSD_PRED_EDGE ? S.nx.in : l0 ? S.nx.e : S.nx.in;
      const double dfb = S.nx.dfb, dgb = S.nx.dgb;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double& c = S.P[(r + ph) & (R - 1)];
        c = __fma_rn(dga[r], dfb, __fma_rn(dfa[r], dgb, c));  // profiles.hpp:330
      }
    }
    if (!GUARD || k + 1 < n)
      prefetch((u + 1) % TB == 0, u + 1 < R ? ccur + u + 1 : cnext, &sm.ering[ebase + u],
               S.P[(ph + R - 1) & (R - 1)], S.nx, l0);
#ifdef TSD_ABL_NOEXACT
    unsigned opaque0;  // 0, invisible to the compiler: the test stays, the exact update never runs
    asm volatile("mov.u32 %0, 0;" : "=r"(opaque0));
    if (vote_any8(S.P, ph, S.thr) && opaque0) [[unlikely]] {
#else
    if (vote_any8(S.P, ph, S.thr)) [[unlikely]] {
#endif
#ifdef TSD_COUNT_EXACT
      if (lane == 0) atomicAdd(&g_exact_count, 1ull);
      if (lane == 0 && cx.first_seg) atomicAdd(&g_exact_first, 1ull);
#endif
      // exact update: strict K > bestK (columns arrive in increasing order,
      // so ties keep the lower column, profiles.hpp:70-77); a flat column has
      // invn_b = 0 -> K = 0 (profiles.hpp:332-336)
      const double invb = ccur[u].z;
      const int col = cx.colbase + k;
      if constexpr (SYM) {
#pragma unroll
        for (int r = 0; r < R; ++r) sm.slide[r * 32 + lane] = S.P[(r + ph) & (R - 1)];
        __syncwarp();
        const int tc = __double2hiint(sm.cring[ebase + u] * cx.namin);  // this column's own threshold
        const unsigned upd =
            exact_update_sym<R>(sm, lane, col, invb, tc, (int)cx.row0, (int)cx.excl, cthr);
        // raised row bests: their thresholds are refreshed at the next
        // threshold block, as in the AB sweep
        S.dirty |= __any_sync(0xffffffffu, upd != 0);
      } else {
        // stage the slot values in slot order for the shared exact update;
        // the thresholds of raised bests are refreshed at the next threshold
        // block (stale ones only let more cells through to the exact test)
        // the high-word test passes whole 8-column threshold blocks at once;
        // the exact K against the register bests (possibly stale, so lower:
        // conservative) first, the shared update only if some slot may rise
        bool may = false;
#pragma unroll
        for (int r = 0; r < R; ++r) may |= S.P[(r + ph) & (R - 1)] * invb > S.bKp[r] || !(S.bKp[r] > 0.0);
        if (__any_sync(0xffffffffu, may)) {
#pragma unroll
          for (int r = 0; r < R; ++r) sm.slide[r * 32 + lane] = S.P[(r + ph) & (R - 1)];
          S.dirty |= exact_update64<R, SELF>(sm, lane, col, invb, cx.row0, cx.excl);
        }
      }
    }
  }
}

// Software-pipelined sweep of one segment. Per step: fold in the incoming
// diagonal, 2 DFMA per slot, prefetch the next step's column data / edge /
// shuffle, K = cov * invn_b, the high-word test of every slot against its
// threshold and one warp vote; the exact update runs only on a pass.
template <int R, bool SELF, bool SYM>
__device__ void sweep_segment(WarpSmem<R>& sm, const SweepCtx& cx, int lane, const double (&dfa)[R],
                              const double (&dga)[R], SweepState<R>& S, const double* __restrict__ invn_a,
                              long long nrows, unsigned long long* ccand, double* cthr) {
  static_assert(R == 8, "the sweep is written for R = 8 rows per lane");
  const int n = cx.ncol;
  const int nchunks = (n + 31) >> 5;
  // lane 31 stores the bottom row into the ring; lanes 0..30 into scratch
  // (sm.slide[256..351], unused while sweeping) so the store needs no branch
  double* const sbase = lane == 31 ? sm.ering : sm.slide + 256;
  const bool l0 = lane == 0;
  __syncwarp();
  issue_chunk(sm, cx, lane, 0);
  if (nchunks > 1) issue_chunk(sm, cx, lane, 1); else cp_commit();
  cp_wait<1>();
  __syncwarp();
  if (SYM) fold_cmin(sm, lane, 0);
  int flushed = 0;  // edge blocks [0, flushed) written back
  // blocks of R steps; every 32 / R blocks the next block opens chunk c:
  // make it resident, retire edge block c-2, start loading chunk c+1 (3-deep
  // rings keep the in-use slots intact)
  auto chunk_turn = [&](int c) {
    if (SYM && __any_sync(0xffffffffu, sm.cq_n != 0)) col_flush(sm, lane, ccand);
    __syncwarp();
    if (c >= 2 && cx.write_out) {
      flush_block(sm, cx, lane, c - 2);
      flushed = c - 1;
    }
    __syncwarp();
    if (c + 1 < nchunks) issue_chunk(sm, cx, lane, c + 1); else cp_commit();
#ifndef TSD_ABL_NOWAIT
    cp_wait<1>();
#endif
    __syncwarp();
    if (SYM) fold_cmin(sm, lane, c);
  };
  constexpr int BPC = 32 / R;  // blocks per chunk
  if (n <= R) {
    sweep_block<R, SELF, true, true, SYM>(sm, cx, lane, 0, 0, S, dfa, dga, sbase, l0, invn_a, nrows, ccand, cthr);
  } else {
    sweep_block<R, SELF, true, false, SYM>(sm, cx, lane, 0, 0, S, dfa, dga, sbase, l0, invn_a, nrows, ccand, cthr);
    // the turn happens before the LAST block of a chunk: that block's final
    // step prefetches the first column of the next chunk
    int k0 = R, m96 = R, bic = 1;  // column, column mod 96, block index inside the chunk
    for (; k0 + R <= n; k0 += R) {
      if (bic == BPC - 1 && k0 + R < n) chunk_turn((k0 + R) >> 5);
      sweep_block<R, SELF, false, false, SYM>(sm, cx, lane, k0, m96, S, dfa, dga, sbase, l0, invn_a, nrows, ccand,
                                             cthr);
      m96 = m96 + R == 96 ? 0 : m96 + R;
      bic = bic == BPC - 1 ? 0 : bic + 1;
    }
    if (k0 < n)
      sweep_block<R, SELF, false, true, SYM>(sm, cx, lane, k0, m96, S, dfa, dga, sbase, l0, invn_a, nrows, ccand,
                                             cthr);
  }
  cp_wait<0>();
  __syncwarp();
  if (SYM && __any_sync(0xffffffffu, sm.cq_n != 0)) col_flush(sm, lane, ccand);
#ifdef TSD_COUNT_EXACT
  if (lane == 0) atomicAdd(&g_step_count, (unsigned long long)n);
  if (lane == 0 && cx.first_seg) atomicAdd(&g_step_first, (unsigned long long)n);
#endif
  if (cx.write_out) {
    const int last = (n - 2) >> 5;  // last edge block holding j <= n-2
    for (int b = flushed; b <= last && n >= 2; ++b) flush_block(sm, cx, lane, b);
  }
  __syncwarp();
}

// ===========================================================================
// Software-pipelined FP64 sweep (AB join and full-matrix self-join; the
// default, TSD_PIPE=1). The step of column k computes the slot values of
// column k into one register set from the other set (column k - 1) and only
// THEN tests column k - 1: the high-word test -> vote -> branch chain no
// longer sits between two steps' DFMAs, so a warp keeps issuing its next
// column's 16 DFMAs while the previous column's test resolves. Two sets (PA
// holds even columns, PB odd ones) replace the register rotation of
// sweep_block: slot r of column k reads slot r - 1 of column k - 1 of the
// other set, slot 0 the shuffled slot 7 of the lane above (lane 0: the band
// above, through the edge ring). Everything else -- threshold blocks, the
// shared exact update, chunk turns, edges -- is sweep_block's.
// ===========================================================================
template <int R>
struct PipeState {
  double PA[R], PB[R];  // column values: even columns in PA, odd in PB
  double bKp[R];        // kplus(bestK)
  int thr[R];           // hi(bKp * nmin) of the current threshold block
  int lthr;             // TSD_LANE_THR64: the smallest of thr (the lane threshold)
  double dfb, dgb, e, in, nmin;  // prefetched column data / incoming diagonals of the next column
  bool dirty;
};

#ifndef TSD_LANE_THR64
#define TSD_LANE_THR64 0  // off: C4 539 -> 527 ms with it, but C5 +15 % and C3 +6 % (near-periodic data
                          // passes the lane threshold on most steps); a per-segment adaptive switch cost more
#endif
// first level of the FP64 row test (TSD_LANE_THR64): the largest high word of
// the lane's 8 values against the smallest slot threshold (VIMNMX3 tree);
// the 8 per-slot tests run only when some lane passes it. High words of
// doubles order like the FP32 bit patterns of vote_lane16f (sign included).
__device__ __forceinline__ bool vote_lane8(const double (&V)[8], int thr) {
  int h[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) h[r] = __double2hiint(V[r]);
  const int a = max(max(h[0], h[1]), h[2]), b = max(max(h[3], h[4]), h[5]);
  return __any_sync(0xffffffffu, max(max(a, b), max(h[6], h[7])) >= thr);
}
__device__ __forceinline__ int min_thr8(const int (&t)[8]) {
  return min(min(min(t[0], t[1]), t[2]), min(min(min(t[3], t[4]), t[5]), min(t[6], t[7])));
}

// the high-word test of the column held in V (column c = k0 + uc, ring
// position of its column data pos), then the exact update on a pass
template <int R, bool SELF>
__device__ __forceinline__ void pipe_test(WarpSmem<R>& sm, const SweepCtx& cx, int lane, PipeState<R>& S,
                                          const double (&V)[R], int c, int pos) {
  // (AB / dictionary joins only: the self-join's near-periodic candidates pass
  // the lane threshold too often -- C2 5.07 -> 5.15 ms with it, C4 539 -> 527 ms)
  if (TSD_LANE_THR64 && !SELF && !vote_lane8(V, S.lthr)) [[likely]]
    return;
  if (vote_any8<R, TSD_VOTE1 != 0>(V, 0, S.thr)) [[unlikely]] {
#ifdef TSD_COUNT_EXACT
    if (lane == 0) atomicAdd(&g_exact_count, 1ull);
#endif
#ifdef TSD_COUNT_EXACT
    const long long rare_t0 = clock64();
#endif
#ifdef TSD_ABL_NOEXACT
    unsigned opaque0;  // 0, invisible to the compiler: the test and its branch stay, the exact path never runs
    asm volatile("mov.u32 %0, 0;" : "=r"(opaque0));
    if (!opaque0) return;
#endif
    const double invb = (&sm.colbuf[0][0])[pos].z;
    bool may = false;
#pragma unroll
    for (int r = 0; r < R; ++r) may |= V[r] * invb > S.bKp[r] || !(S.bKp[r] > 0.0);
    if (__any_sync(0xffffffffu, may)) {
#ifdef TSD_COUNT_EXACT
      if (lane == 0) atomicAdd(&g_cas_count, 1ull);  // (AB joins: exact-path entries past the register check)
#endif
#pragma unroll
      for (int r = 0; r < R; ++r) sm.slide[r * 32 + lane] = V[r];
      S.dirty |= exact_update64<R, SELF>(sm, lane, cx.colbase + c, invb, cx.row0, cx.excl);
    }
#ifdef TSD_COUNT_EXACT
    if (lane == 0) atomicAdd(&g_rare_cycles, (unsigned long long)(clock64() - rare_t0));
#endif
  }
}

// one block of R steps from column k0 (k0 % R == 0)
template <int R, bool SELF, bool FIRST, bool GUARD>
__device__ __forceinline__ void sweep_block_p(WarpSmem<R>& sm, const SweepCtx& cx, int lane, int k0, int m96,
                                              PipeState<R>& S, const double (&dfa)[R], const double (&dga)[R],
                                              double* sbase, bool l0) {
  static_assert(R == 8 && TB == R, "the pipelined sweep is written for R = 8 with one threshold block per 8 steps");
  const int n = cx.ncol;
  const double4* cflat = &sm.colbuf[0][0];
  const double4* ccur = cflat + m96;
  const double4* cnext = cflat + (m96 + R == 96 ? 0 : m96 + R);
  double* const st_prev = sbase + (m96 == 0 ? 95 : m96 - 1);  // ring slot of column k0 - 1
  double* const st_cur = sbase + m96;
#pragma unroll
  for (int u = 0; u < R; ++u) {
    const int k = k0 + u;
    if (GUARD && k >= n) break;
    double(&D)[R] = (u & 1) ? S.PB : S.PA;  // column k
    double(&V)[R] = (u & 1) ? S.PA : S.PB;  // column k - 1
    if (FIRST && u == 0) {
      // column 0 (the heads) is already in PA: its test runs at step 1
      S.nmin = ccur[0].w;
#pragma unroll
      for (int r = 0; r < R; ++r) S.thr[r] = __double2hiint(S.bKp[r] * S.nmin);
      S.lthr = min_thr8(S.thr);
    } else {
      // column k from column k - 1: slots 7..1 first (slot 7 feeds the next shuffle)
#pragma unroll
      for (int r = R - 1; r >= 1; --r) D[r] = __fma_rn(dga[r], S.dfb, __fma_rn(dfa[r], S.dgb, V[r - 1]));
      const double x0 = TSD_PRED_EDGE ? S.in : l0 ? S.e : S.in;
      D[0] = __fma_rn(dga[0], S.dfb, __fma_rn(dfa[0], S.dgb, x0));
      // lane 31 retires its bottom row of column k - 1 into the edge ring
      (u == 0 ? st_prev : st_cur + u - 1)[0] = V[R - 1];
    }
    // prefetch column k + 1: column data, lane 0's edge, the shuffled slot 7
    if (!GUARD || k + 1 < n) {
      const double4* cb = u + 1 < R ? ccur + u + 1 : cnext;
      if ((u + 1) % TB == 0) {
        const double4 c4 = *cb;
        S.dfb = c4.x;
        S.dgb = c4.y;
        S.nmin = c4.w;  // consumed at the next block start, after this block's last test
      } else {
        const double2 c2 = *reinterpret_cast<const double2*>(cb);
        S.dfb = c2.x;
        S.dgb = c2.y;
      }
      if (!TSD_PRED_EDGE) S.e = sm.ering[m96 + u];
    }
    S.in = shfl_up1(D[R - 1]);
    // TSD_PRED_EDGE: lane 0 overwrites its (unused) shuffle result with the
    // band above's edge by a predicated load -- no per-step select on the ALU pipe
    if (TSD_PRED_EDGE && l0) S.in = sm.ering[m96 + u];
    if (!(FIRST && u == 0)) {
      // test column k - 1 with the thresholds of its block
      pipe_test<R, SELF>(sm, cx, lane, S, V, k - 1, u == 0 ? (m96 == 0 ? 95 : m96 - 1) : m96 + u - 1);
      if (u % TB == 0) {  // column k opens a threshold block: its thresholds, after the previous test
        if (S.dirty) {
#pragma unroll
          for (int r = 0; r < R; ++r) S.bKp[r] = kplus(sm.bK[r][lane]);
          S.dirty = false;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) S.thr[r] = __double2hiint(S.bKp[r] * S.nmin);
        S.lthr = min_thr8(S.thr);
      }
    }
  }
}
template <int R, bool SELF>
__device__ void sweep_segment_p(WarpSmem<R>& sm, const SweepCtx& cx, int lane, const double (&dfa)[R],
                                const double (&dga)[R], PipeState<R>& S) {
  const int n = cx.ncol;
  const int nchunks = (n + 31) >> 5;
  double* const sbase = lane == 31 ? sm.ering : sm.slide + 256;
  const bool l0 = lane == 0;
  __syncwarp();
  issue_chunk(sm, cx, lane, 0);
  if (nchunks > 1) issue_chunk(sm, cx, lane, 1); else cp_commit();
  cp_wait<1>();
  __syncwarp();
  // column 1's data and lane 0's edge (step 0 of the first block prefetches them)
  int flushed = 0;
  auto chunk_turn = [&](int c) {
    __syncwarp();
    if (c >= 2 && cx.write_out) {
      flush_block(sm, cx, lane, c - 2);
      flushed = c - 1;
    }
    __syncwarp();
    if (c + 1 < nchunks) issue_chunk(sm, cx, lane, c + 1); else cp_commit();
    cp_wait<1>();
    __syncwarp();
  };
  constexpr int BPC = 32 / R;
  int k0 = 0, m96 = 0;
  if (n <= R) {
    sweep_block_p<R, SELF, true, true>(sm, cx, lane, 0, 0, S, dfa, dga, sbase, l0);
  } else {
    sweep_block_p<R, SELF, true, false>(sm, cx, lane, 0, 0, S, dfa, dga, sbase, l0);
    int bic = 1;
    k0 = R;
    m96 = R;
    for (; k0 + R <= n; k0 += R) {
      if (bic == BPC - 1 && k0 + R < n) chunk_turn((k0 + R) >> 5);
      sweep_block_p<R, SELF, false, false>(sm, cx, lane, k0, m96, S, dfa, dga, sbase, l0);
      m96 = m96 + R == 96 ? 0 : m96 + R;
      bic = bic == BPC - 1 ? 0 : bic + 1;
    }
    if (k0 < n) sweep_block_p<R, SELF, false, true>(sm, cx, lane, k0, m96, S, dfa, dga, sbase, l0);
  }
  // drain: the last column's test (its values sit in PA if its index is even)
  {
    const int c = n - 1;
    const int pos = c % 96;  // ring position of column c
    if (c & 1)
      pipe_test<R, SELF>(sm, cx, lane, S, S.PB, c, pos);
    else
      pipe_test<R, SELF>(sm, cx, lane, S, S.PA, c, pos);
  }
  cp_wait<0>();
  __syncwarp();
#ifdef TSD_COUNT_EXACT
  if (lane == 0) atomicAdd(&g_step_count, (unsigned long long)n);
#endif
  if (cx.write_out) {
    const int last = (n - 2) >> 5;
    for (int b = flushed; b <= last && n >= 2; ++b) flush_block(sm, cx, lane, b);
  }
  __syncwarp();
}

// ===========================================================================
// Wide FP64 sweep (AB / dictionary joins, TSD_WIDE=1): 16 rows per lane, bands
// of 512 rows. A step's fixed costs -- the shuffle, the column and edge loads,
// the bottom-row store, the vote and the branch over the exact path -- are
// shared by 32 DFMAs instead of 16, and a warp carries 16 independent
// two-DFMA chains, so fewer resident warps keep the FP64 pipe fed. The column
// is updated IN PLACE from the highest slot down (slot r reads slot r - 1 of
// the previous column before that register is overwritten), so one register
// set holds the band and nothing rotates; the test of column k runs right
// after its DFMAs. Cells, operations and their order are the R = 8 sweep's,
// so profiles are bitwise identical.
// ===========================================================================
#ifndef TSD_JOIN_MINB_WIDE
#define TSD_JOIN_MINB_WIDE 6
#endif
#ifndef TSD_WIDE_DEFAULT
#define TSD_WIDE_DEFAULT 0
#endif
#ifndef TSD_WIDE_MIN_ROWS
#define TSD_WIDE_MIN_ROWS (1 << 20)
#endif
constexpr int RW = 16;

template <int R>
struct WideState {
  double P[R];    // slot r's covariance at the current column
  int thr[R];     // hi(kplus(bestK) * nmin) of the current threshold block (bests live in sm.bK only)
  double dfb, dgb, in, nmin;  // prefetched column data / incoming diagonal of the next column
};

// warp vote over 16 slot tests "hi(cov) >= thr" (four 4-deep predicate chains)
__device__ __forceinline__ bool vote_any16d(const double (&P)[16], const int (&t)[16]) {
  int h[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) h[r] = __double2hiint(P[r]);
  unsigned r;
  asm volatile(
      "{\n .reg .pred a, b, c, d;\n"
      " setp.ge.s32 a, %1, %17;\n setp.ge.s32 b, %5, %21;\n setp.ge.s32 c, %9, %25;\n setp.ge.s32 d, %13, %29;\n"
      " setp.ge.or.s32 a, %2, %18, a;\n setp.ge.or.s32 b, %6, %22, b;\n"
      " setp.ge.or.s32 c, %10, %26, c;\n setp.ge.or.s32 d, %14, %30, d;\n"
      " setp.ge.or.s32 a, %3, %19, a;\n setp.ge.or.s32 b, %7, %23, b;\n"
      " setp.ge.or.s32 c, %11, %27, c;\n setp.ge.or.s32 d, %15, %31, d;\n"
      " setp.ge.or.s32 a, %4, %20, a;\n setp.ge.or.s32 b, %8, %24, b;\n"
      " setp.ge.or.s32 c, %12, %28, c;\n setp.ge.or.s32 d, %16, %32, d;\n"
      " or.pred a, a, b;\n or.pred c, c, d;\n or.pred a, a, c;\n"
      " vote.sync.any.pred a, a, -1;\n selp.u32 %0, 1, 0, a;\n}\n"
      : "=r"(r)
      : "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]), "r"(h[8]),
        "r"(h[9]), "r"(h[10]), "r"(h[11]), "r"(h[12]), "r"(h[13]), "r"(h[14]), "r"(h[15]), "r"(t[0]),
        "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]), "r"(t[7]), "r"(t[8]),
        "r"(t[9]), "r"(t[10]), "r"(t[11]), "r"(t[12]), "r"(t[13]), "r"(t[14]), "r"(t[15]));
  return r != 0;
}

// one block of TB steps from column k0 (k0 % TB == 0)
template <int R, bool SELF, bool FIRST, bool GUARD>
__device__ __forceinline__ void sweep_block_w(WarpSmem<R, true>& sm, const SweepCtx& cx, int lane, int k0, int m96,
                                              WideState<R>& S, const double (&dfa)[R], const double (&dga)[R],
                                              double* sbase, bool l0) {
  static_assert(R == 16 && TB == 8, "the wide sweep is written for R = 16 with 8-column threshold blocks");
  const int n = cx.ncol;
  const double4* cflat = &sm.colbuf[0][0];
  const double4* ccur = cflat + m96;
  const double4* cnext = cflat + (m96 + TB == 96 ? 0 : m96 + TB);
  double* const st_prev = sbase + (m96 == 0 ? 95 : m96 - 1);  // ring slot of column k0 - 1
  double* const st_cur = sbase + m96;
#pragma unroll
  for (int u = 0; u < TB; ++u) {
    const int k = k0 + u;
    if (GUARD && k >= n) break;
    if (u == 0) {  // column k opens a threshold block
      if (FIRST) S.nmin = ccur[0].w;
      // thresholds straight from the bests in shared memory (no register copy
      // of kplus(bestK): 32 registers the 14-warp budget does not have). A
      // best <= 0 gives a product with the sign bit set (or +0): as unsigned
      // it is >= 0x80000000, so the unsigned minimum turns it into INT_MIN
      // (passes everything), exactly kplus's rule; +inf (inactive) never passes
#pragma unroll
      for (int r = 0; r < R; ++r)
        S.thr[r] = (int)umin((unsigned)__double2hiint(sm.bK[r][lane] * S.nmin), 0x80000000u);
    }
    if (!(FIRST && u == 0)) {
      // lane 31 retires its bottom row of column k - 1 into the edge ring
      (u == 0 ? st_prev : st_cur + u - 1)[0] = S.P[R - 1];
      // column k in place, highest slot first (slot 15 feeds the next shuffle)
#pragma unroll
      for (int r = R - 1; r >= 1; --r) S.P[r] = __fma_rn(dga[r], S.dfb, __fma_rn(dfa[r], S.dgb, S.P[r - 1]));
      S.P[0] = __fma_rn(dga[0], S.dfb, __fma_rn(dfa[0], S.dgb, S.in));  // profiles.hpp:330
    }
    // prefetch column k + 1: column data, the shuffled slot 15, lane 0's edge
    if (!GUARD || k + 1 < n) {
      const double4* cb = u + 1 < TB ? ccur + u + 1 : cnext;
      if ((u + 1) % TB == 0) {
        const double4 c4 = *cb;
        S.dfb = c4.x;
        S.dgb = c4.y;
        S.nmin = c4.w;
      } else {
        const double2 c2 = *reinterpret_cast<const double2*>(cb);
        S.dfb = c2.x;
        S.dgb = c2.y;
      }
    }
    S.in = shfl_up1(S.P[R - 1]);
    if (l0) S.in = sm.ering[m96 + u];  // predicated load over the shuffle result (no select)
    if (vote_any16d(S.P, S.thr)) [[unlikely]] {
#ifdef TSD_COUNT_EXACT
      if (lane == 0) atomicAdd(&g_exact_count, 1ull);
#endif
      const double invb = ccur[u].z;
      bool may = false;
#pragma unroll
      for (int r = 0; r < R; ++r) may |= S.P[r] * invb > sm.bK[r][lane];
      if (__any_sync(0xffffffffu, may)) {
#pragma unroll
        for (int r = 0; r < R; ++r) sm.slide[r * 32 + lane] = S.P[r];
        exact_update64<R, SELF>(sm, lane, cx.colbase + k, invb, cx.row0, cx.excl);
      }
    }
  }
}

template <int R, bool SELF>
__device__ void sweep_segment_w(WarpSmem<R, true>& sm, const SweepCtx& cx, int lane, const double (&dfa)[R],
                                const double (&dga)[R], WideState<R>& S) {
  const int n = cx.ncol;
  const int nchunks = (n + 31) >> 5;
  // lanes 0..30 store their (unused) slot 15 into scratch past the staged slot values
  double* const sbase = lane == 31 ? sm.ering : sm.slide + 32 * R;
  const bool l0 = lane == 0;
  __syncwarp();
  issue_chunk(sm, cx, lane, 0);
  if (nchunks > 1) issue_chunk(sm, cx, lane, 1); else cp_commit();
  cp_wait<1>();
  __syncwarp();
  int flushed = 0;
  auto chunk_turn = [&](int c) {
    __syncwarp();
    if (c >= 2 && cx.write_out) {
      flush_block(sm, cx, lane, c - 2);
      flushed = c - 1;
    }
    __syncwarp();
    if (c + 1 < nchunks) issue_chunk(sm, cx, lane, c + 1); else cp_commit();
    cp_wait<1>();
    __syncwarp();
  };
  constexpr int BPC = 32 / TB;
  if (n <= TB) {
    sweep_block_w<R, SELF, true, true>(sm, cx, lane, 0, 0, S, dfa, dga, sbase, l0);
  } else {
    sweep_block_w<R, SELF, true, false>(sm, cx, lane, 0, 0, S, dfa, dga, sbase, l0);
    int k0 = TB, m96 = TB, bic = 1;
    for (; k0 + TB <= n; k0 += TB) {
      if (bic == BPC - 1 && k0 + TB < n) chunk_turn((k0 + TB) >> 5);
      sweep_block_w<R, SELF, false, false>(sm, cx, lane, k0, m96, S, dfa, dga, sbase, l0);
      m96 = m96 + TB == 96 ? 0 : m96 + TB;
      bic = bic == BPC - 1 ? 0 : bic + 1;
    }
    if (k0 < n) sweep_block_w<R, SELF, false, true>(sm, cx, lane, k0, m96, S, dfa, dga, sbase, l0);
  }
  cp_wait<0>();
  __syncwarp();
#ifdef TSD_COUNT_EXACT
  if (lane == 0) atomicAdd(&g_step_count, (unsigned long long)n);
#endif
  if (cx.write_out) {
    const int last = (n - 2) >> 5;
    for (int b = flushed; b <= last && n >= 2; ++b) flush_block(sm, cx, lane, b);
  }
  __syncwarp();
}

// ===========================================================================
// FP32 mode: the same sweep as FP64 in FP32 arithmetic -- the reference's
// unnormalised centred recurrence cov = fma(dg_a, df_b, fma(df_a, dg_b, cov))
// (profiles.hpp:330), two cells per fma.rn.f32x2 (FFMA2), 2 FP32 FMAs per
// cell. The FP32 operands are the FP64 window statistics rounded once after a
// power-of-two scaling (sigma_a for the query, sigma_b for the dictionary)
// that brings the largest window norm of each side to ~1, so cov * sigma_a *
// sigma_b stays inside the FP32 range; run_join falls back to the FP64 sweep
// when the window norms span too wide a range for that (k_norm_range).
// Heads and top edges stay FP64 and are rounded once; diagonals restart from
// an FP64 head at every segment start and every task top, and tasks are capped
// at 4096 rows, which bounds the FP32 drift. The rounding error
// of a cell is that of the column-normalised form to first order (a column
// scaling commutes with the relative rounding of each operation), at 2 instead
// of 3 FP32 operations per cell.
// A lane owns 16 consecutive rows (R = 16, bands of 512 rows). Physical
// register pair q holds the slots (a, a + 8), a = (q - ph) mod 8: both halves
// move down one slot per step in lockstep, so the rotation is pure register
// renaming and every FFMA2 reads aligned pairs (no repacking moves). Per step
// the slot-8 half takes the lane's own slot-7 value and the slot-0 half the
// previous lane's slot-15 value (one 32-bit shuffle; lane 0 reads the band
// above through the edge ring, lane 31's slot 15 is the band's bottom row).
// Row test as in FP64: per 8-column block each slot's threshold is
// kplus(best K) x the block's smallest scaled column norm (one FMUL2 per slot
// pair), compared against the FP32 bits of cov with one ISETP per cell.
// ===========================================================================
typedef unsigned long long u64;

__device__ __forceinline__ u64 pack2(float lo, float hi) {
  return ((u64)__float_as_uint(hi) << 32) | (u64)__float_as_uint(lo);
}
__device__ __forceinline__ float lo2(u64 v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi2(u64 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float shfl_up1f(float v) {
  asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;\n" : "+f"(v));
  return v;
}

// FP32 column data, one 32-byte slot per column: {dg_b*sb, dg_b*sb, df_b*sb,
// df_b*sb} (pairs pre-duplicated for f32x2), kf = invn_b / (sa*sb) (0 if
// flat), nmin = (1 - 2^-20) x sa*sb x the smallest window norm over columns
// j .. j+7 (flat or straddling: FLT_MAX) -- the block threshold factor
struct __align__(16) Col32 {
  u64 dg2, df2;
  float kf, nmin;
  u64 pad;
};
static_assert(sizeof(Col32) == 32, "Col32 must match the double4 column slot");

__device__ __forceinline__ float kplus_f(float b) { return b > 0.0f ? b : -0.0f; }

struct StepIn32 {
  u64 dg2, df2;
  float e, in;
};

__device__ __forceinline__ void prefetch32(const Col32* cb, const float* ep, float v15, StepIn32& d, bool l0) {
  const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(cb);
  d.dg2 = a.x;
  d.df2 = a.y;
  d.in = shfl_up1f(v15);
  if (TSD_PRED_EDGE && l0) d.in = *ep;  // as prefetch(): no per-step select
  if (!TSD_PRED_EDGE) d.e = *ep;
}

constexpr int R32 = 16;  // rows per lane in the FP32 sweep

struct SweepState32 {
  u64 Q[8];       // physical pair q: slots ((q - ph) & 7, +8)
  u64 BK[8];      // kplus(best K) of slots (a, a + 8); the bests themselves live in sm.bK
  float mbk;      // the smallest of the 16 kplus(best K): the lane threshold's factor
  StepIn32 nx;
  bool dirty;     // some best changed in this block: reload BK at its end
};

__device__ __forceinline__ float min_bk16(const u64 (&BK)[8]) {
  float m = fminf(lo2(BK[0]), hi2(BK[0]));
#pragma unroll
  for (int q = 1; q < 8; ++q) m = fminf(m, fminf(lo2(BK[q]), hi2(BK[q])));
  return m;
}

// warp vote over the 16 slot tests "bits(cov) >= bits(thr)" (four 4-deep
// predicate chains). A threshold from kplus(best) <= 0 is -0.0f (bits INT_MIN):
// that slot passes everything
__device__ __forceinline__ bool vote_any16f(const u64 (&Q)[8], int ph, const u64 (&TP)[8]) {
  int h[R32], t[R32];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int a = (q - ph + 8) & 7;  // slot order
    h[a] = (int)(unsigned)Q[q];
    h[a + 8] = (int)(unsigned)(Q[q] >> 32);
    t[q] = (int)(unsigned)TP[q];
    t[q + 8] = (int)(unsigned)(TP[q] >> 32);
  }
  unsigned r;
  asm volatile(
      "{\n .reg .pred a, b, c, d;\n"
      " setp.ge.s32 a, %1, %17;\n setp.ge.s32 b, %5, %21;\n setp.ge.s32 c, %9, %25;\n setp.ge.s32 d, %13, %29;\n"
      " setp.ge.or.s32 a, %2, %18, a;\n setp.ge.or.s32 b, %6, %22, b;\n"
      " setp.ge.or.s32 c, %10, %26, c;\n setp.ge.or.s32 d, %14, %30, d;\n"
      " setp.ge.or.s32 a, %3, %19, a;\n setp.ge.or.s32 b, %7, %23, b;\n"
      " setp.ge.or.s32 c, %11, %27, c;\n setp.ge.or.s32 d, %15, %31, d;\n"
      " setp.ge.or.s32 a, %4, %20, a;\n setp.ge.or.s32 b, %8, %24, b;\n"
      " setp.ge.or.s32 c, %12, %28, c;\n setp.ge.or.s32 d, %16, %32, d;\n"
      " or.pred a, a, b;\n or.pred c, c, d;\n or.pred a, a, c;\n"
      " vote.sync.any.pred a, a, -1;\n selp.u32 %0, 1, 0, a;\n}\n"
      : "=r"(r)
      : "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]), "r"(h[8]),
        "r"(h[9]), "r"(h[10]), "r"(h[11]), "r"(h[12]), "r"(h[13]), "r"(h[14]), "r"(h[15]), "r"(t[0]),
        "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]), "r"(t[7]), "r"(t[8]),
        "r"(t[9]), "r"(t[10]), "r"(t[11]), "r"(t[12]), "r"(t[13]), "r"(t[14]), "r"(t[15]));
  return r != 0;
}

// First level of the FP32 row test (TSD_LANE_THR32): one threshold per lane,
// kplus(the smallest of its 16 bests) x nmin, against the largest of the 16
// slot values -- a VIMNMX3 tree instead of one ISETP per cell. As signed
// integers the FP32 bit patterns order every non-negative value correctly
// against a non-negative threshold and put any negative value below one; a
// threshold of -0.0f (INT_MIN) passes everything. Only when some lane passes
// does the warp run the 16 per-slot tests (vote_any16f), and only when one of
// those passes, the exact update.
__device__ __forceinline__ int max3i(int a, int b, int c) { return max(max(a, b), c); }
__device__ __forceinline__ bool vote_lane16f(const u64 (&Q)[8], int thr) {
  int h[16];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    h[2 * q] = (int)(unsigned)Q[q];
    h[2 * q + 1] = (int)(unsigned)(Q[q] >> 32);
  }
  const int a = max3i(max3i(h[0], h[1], h[2]), max3i(h[3], h[4], h[5]), max3i(h[6], h[7], h[8]));
  const int b = max3i(max3i(h[9], h[10], h[11]), max3i(h[12], h[13], h[14]), h[15]);
  return __any_sync(0xffffffffu, a >= thr || b >= thr);
}
#ifndef TSD_LANE_THR32
#define TSD_LANE_THR32 1
#endif
template <int R>
__device__ __forceinline__ void issue_chunk32(WarpSmem<R>& sm, const SweepCtx& cx, int lane, int c) {
  const double4* src = cx.colg + 32 * c + lane;
  double4* dst = &sm.colbuf[c % 3][lane];
  cp16(dst, src);
  cp16(reinterpret_cast<char*>(dst) + 16, reinterpret_cast<const char*>(src) + 16);
  float* ring = reinterpret_cast<float*>(sm.ering);
  const float* E = reinterpret_cast<const float*>(cx.E);
  if (lane < 8) cp16(&ring[(c % 3) * 32 + 4 * lane], E + 32 * c + 4 * lane);
  cp_commit();
}

template <int R>
__device__ __forceinline__ void flush_block32(WarpSmem<R>& sm, const SweepCtx& cx, int lane, int b) {
  const int j = 32 * b + lane;
  if (j < cx.ncol - 1) reinterpret_cast<float*>(cx.E)[j] = reinterpret_cast<const float*>(sm.ering)[(b % 3) * 32 + lane];
}

// FP32 exact update of one step, shared by every unrolled step: the lane's 16
// slot values staged in slot order (sm.slide, pair a at [a][lane]), K = c~ *
// (invn_b / s_k) against the best in sm.bK (a float value; strict >, columns
// arrive in increasing order, profiles.hpp:70-77). Returns whether any best
// of the lane changed.
template <bool SELF>
__device__ __noinline__ bool exact_update32(WarpSmem<R32>& sm, int lane, int col, float kf, long long row0,
                                            long long excl) {
  bool any = false;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const u64 v = reinterpret_cast<const u64*>(sm.slide)[a * 32 + lane];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = a + 8 * h;
      const float K = (h ? hi2(v) : lo2(v)) * kf;
      bool ok = K > (float)sm.bK[r][lane];
      if (SELF) {
        const long long d = row0 + r - col;
        ok = ok && (d > excl || d < -excl);  // profiles.hpp:281-284
      }
      if (ok) {
        sm.bK[r][lane] = (double)K;
        sm.bj[r][lane] = col;
        any = true;
      }
    }
  }
  __syncwarp();
  return any;
}

// One block of 8 steps (the rotation period) starting at k0 (k0 % 8 == 0).
// FA[a] / GA[a]: the packed row data (df_a, dg_a) of slots (a, a + 8).
template <bool SELF, bool FIRST, bool GUARD>
__device__ __forceinline__ void sweep_block32(WarpSmem<R32>& sm, const SweepCtx& cx, int lane, int k0, int m96,
                                              SweepState32& S, const u64 (&FA)[8], const u64 (&GA)[8], float* sbase,
                                              bool l0) {
  const int n = cx.ncol;
  const Col32* cflat = reinterpret_cast<const Col32*>(&sm.colbuf[0][0]);
  const Col32* ccur = cflat + m96;
  const Col32* cnext = cflat + (m96 + 8 == 96 ? 0 : m96 + 8);
  const float* ring = reinterpret_cast<const float*>(sm.ering);
  const int ebase = m96;
  float* const st_prev = sbase + (m96 == 0 ? 95 : m96 - 1);
  float* const st_cur = sbase + ebase;
  // block thresholds: cov > best K / kf_j for some column j of the block
  // implies cov > kplus(best K) x nmin (nmin lowered by 2^-20 for the rounding)
  const float nm = ccur->nmin;
  const int lthr = __float_as_int(S.mbk * nm);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int k = k0 + u;
    if (GUARD && k >= n) break;
    const int ph = (8 - u) & 7;  // physical pair of slots (0, 8) at this step
    if (!(FIRST && u == 0)) {
      // the pair that held slots (7, 15) now holds (0, 8): lane 31 retires its
      // slot 15 (bottom row, column k-1); slot 8 takes the lane's own slot 7
      const u64 old = S.Q[ph];
      (u == 0 ? st_prev : st_cur + u - 1)[0] = hi2(old);
      S.Q[ph] = pack2(TSD_PRED_EDGE ? S.nx.in : l0 ? S.nx.e : S.nx.in, lo2(old));
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int a = (q - ph + 8) & 7;
        S.Q[q] = fma2(GA[a], S.nx.df2, fma2(FA[a], S.nx.dg2, S.Q[q]));  // profiles.hpp:330
      }
    }
    if (!GUARD || k + 1 < n) prefetch32(u + 1 < 8 ? ccur + u + 1 : cnext, &ring[ebase + u], hi2(S.Q[(ph + 7) & 7]), S.nx, l0);
    // two-level test: the lane threshold (VIMNMX3 trees) first, the 16 slot
    // thresholds only when some lane passes it
    bool pass = TSD_LANE_THR32 ? vote_lane16f(S.Q, lthr) : true;
    if (pass) [[unlikely]] {
      u64 TP[8];
      const u64 NM = pack2(nm, nm);
#pragma unroll
      for (int q = 0; q < 8; ++q) TP[q] = mul2(S.BK[q], NM);
      pass = vote_any16f(S.Q, ph, TP);
    }
    if (pass) [[unlikely]] {
#ifdef TSD_COUNT_EXACT
      if (lane == 0) atomicAdd(&g_exact_count, 1ull);
      if (lane == 0 && cx.first_seg) atomicAdd(&g_exact_first, 1ull);
#endif
      // stage the pairs in slot order and run the one shared exact update
      // (eight inline copies of it would overflow the instruction cache)
#pragma unroll
      for (int q = 0; q < 8; ++q) reinterpret_cast<u64*>(sm.slide)[((q - ph + 8) & 7) * 32 + lane] = S.Q[q];
      S.dirty |= exact_update32<SELF>(sm, lane, cx.colbase + k, (ccur + u)->kf, cx.row0, cx.excl);
    }
  }
  if (S.dirty) {  // bests this block raised (the stale thresholds only passed more cells)
#pragma unroll
    for (int q = 0; q < 8; ++q) S.BK[q] = pack2(kplus_f(sm.bK[q][lane]), kplus_f(sm.bK[q + 8][lane]));
    S.mbk = min_bk16(S.BK);
    S.dirty = false;
  }
}

template <bool SELF>
__device__ void sweep_segment32(WarpSmem<R32>& sm, const SweepCtx& cx, int lane, const u64 (&FA)[8],
                                const u64 (&GA)[8], SweepState32& S) {
  const int n = cx.ncol;
  const int nchunks = (n + 31) >> 5;
  float* const sbase = reinterpret_cast<float*>(lane == 31 ? sm.ering : sm.slide + 256);
  const bool l0 = lane == 0;
  __syncwarp();
  issue_chunk32(sm, cx, lane, 0);
  if (nchunks > 1) issue_chunk32(sm, cx, lane, 1); else cp_commit();
  cp_wait<1>();
  __syncwarp();
  int flushed = 0;
  if (n > 1)
    prefetch32(reinterpret_cast<const Col32*>(&sm.colbuf[0][1]), reinterpret_cast<const float*>(sm.ering),
               hi2(S.Q[7]), S.nx, l0);
  auto chunk_turn = [&](int c) {
    __syncwarp();
    if (c >= 2 && cx.write_out) {
      flush_block32(sm, cx, lane, c - 2);
      flushed = c - 1;
    }
    __syncwarp();
    if (c + 1 < nchunks) issue_chunk32(sm, cx, lane, c + 1); else cp_commit();
    cp_wait<1>();
    __syncwarp();
  };
  constexpr int BPC = 32 / 8;
  if (n <= 8) {
    sweep_block32<SELF, true, true>(sm, cx, lane, 0, 0, S, FA, GA, sbase, l0);
  } else {
    sweep_block32<SELF, true, false>(sm, cx, lane, 0, 0, S, FA, GA, sbase, l0);
    int k0 = 8, m96 = 8, bic = 1;
    for (; k0 + 8 <= n; k0 += 8) {
      if (bic == BPC - 1 && k0 + 8 < n) chunk_turn((k0 + 8) >> 5);
      sweep_block32<SELF, false, false>(sm, cx, lane, k0, m96, S, FA, GA, sbase, l0);
      m96 = m96 + 8 == 96 ? 0 : m96 + 8;
      bic = bic == BPC - 1 ? 0 : bic + 1;
    }
    if (k0 < n) sweep_block32<SELF, false, true>(sm, cx, lane, k0, m96, S, FA, GA, sbase, l0);
  }
  cp_wait<0>();
  __syncwarp();
#ifdef TSD_COUNT_EXACT
  if (lane == 0) atomicAdd(&g_step_count, (unsigned long long)n);
  if (lane == 0 && cx.first_seg) atomicAdd(&g_step_first, (unsigned long long)n);
#endif
  if (cx.write_out) {
    const int last = (n - 2) >> 5;
    for (int b = flushed; b <= last && n >= 2; ++b) flush_block32(sm, cx, lane, b);
  }
  __syncwarp();
}

template <int R, bool SELF, bool F32, bool SYM>
__device__ __forceinline__ void join_body(const JoinArgs& a) {
  static_assert(!SYM || (SELF && !F32), "the symmetric sweep is the FP64 self-join");
  constexpr int H = Geo<R>::H;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using SM = WarpSmem<R, (R == 16 && !F32)>;
  SM* smem = reinterpret_cast<SM*>(smem_raw);
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  SM& sm = smem[wl];
  const int gw = blockIdx.x * WARPS + wl;
  double* Ew = a.edges + (int64_t)gw * a.ecap;
  double* Hw = a.hscr + (int64_t)gw * 2048;
  const int bpt = a.bands_per_task;
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  if (lane == 0) sm.cq_n = 0;
  __syncwarp();
#ifdef TSD_COUNT_EXACT
  const long long body_t0 = clock64();
  struct BodyTimer {
    long long t0;
    int lane;
    __device__ ~BodyTimer() {
      if (lane == 0) atomicAdd(&g_total_cycles, (unsigned long long)(clock64() - t0));
    }
  } body_timer{body_t0, lane};
#endif

  for (int it = 0;; ++it) {
    int task, g, b0, b1;
    if constexpr (SYM) {  // triangle tasks differ in size: dynamic queue, longest first
      if (lane == 0) task = atomicAdd(a.task_next, 1);
      task = __shfl_sync(0xffffffffu, task, 0);
      if (task >= a.ntasks) break;
      // broadcast from lane 0: provably warp-uniform, so the sweep below needs
      // no divergence checks at its shuffles and votes
      int4 t4 = make_int4(0, 0, 0, 0);
      if (lane == 0) t4 = a.tasks[task];
      b0 = __shfl_sync(0xffffffffu, t4.x, 0);
      b1 = __shfl_sync(0xffffffffu, t4.y, 0);
      g = __shfl_sync(0xffffffffu, t4.z, 0);
    } else {
      // dynamic queue, group-major: the groups of one band range run in
      // different waves, so each starts from the bests published by the
      // earlier ones (fewer record updates)
      if (lane == 0) task = atomicAdd(a.task_next, 1);
      task = __shfl_sync(0xffffffffu, task, 0);
      if (task >= a.ntasks) break;
      const int nbr = (a.nbands + bpt - 1) / bpt;
      g = task / nbr;
      b0 = (task - g * nbr) * bpt;
      b1 = min(a.nbands, b0 + bpt);
    }
    const int s_beg = a.group_seg[g], s_end = a.group_seg[g + 1];
    for (int b = b0; b < b1; ++b) {
      const int64_t i0 = (int64_t)b * H;
      double namin = DBL_MAX;  // SYM: smallest window norm among this lane's rows
      if constexpr (SYM) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int64_t i = i0 + R * lane + r;
          const bool act = i < a.nrows && a.flag_a[i] == 1;
          const double ia = act ? a.invn_a[i] : 0.0;
          sm.inva[r][lane] = ia;
          if (act) namin = fmin(namin, rcp_pos(ia));
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t i = i0 + R * lane + r;
        const uint8_t f = i < a.nrows ? a.flag_a[i] : 0;
        sm.bK[r][lane] = f == 1 ? -kInf : kInf;  // valid non-flat rows take part; +inf never passes
        sm.bj[r][lane] = -1;
      }
      if (a.seed) {
        // Seed each row's best with its precomputed lower bound: one ulp below
        // the best column-0 candidate over ALL segments (heads_fft.cu). The
        // cell achieving it is visited by exactly one group and recorded by
        // the strict test there; anything at least as good earlier in column
        // order wins as before; a group holding nothing better leaves the row
        // without a candidate (-1), which the group merge skips. The result is
        // unchanged, but the running best no longer climbs from -inf in every
        // band and group -- most of the exact-update traffic.
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int64_t i = i0 + R * lane + r;
          const unsigned long long key = sm.bK[r][lane] == -kInf ? __ldcg(a.seed + i) : 0ull;  // -inf: valid row
          if (key != 0ull) {
            const unsigned long long bits = (key >> 63) ? (key & 0x7fffffffffffffffull) : ~key;
            const double kb = nextafter(__longlong_as_double((long long)bits), -kInf);
            // FP32 sweep: its value of the seed cell differs by FP32 rounding
            // (~6e-8 relative); a 1e-6 margin keeps the seed strictly below it
            sm.bK[r][lane] = F32 ? (kb > 0.0 ? kb * (1.0 - 1e-6) : kb * (1.0 + 1e-6)) : kb;
          }
        }
      }
      if constexpr (SYM) {
        // the column side may already hold a better lower bound for these rows
        // (their lower-triangle pairs, deposited by earlier bands). For the
        // self-join row i and column i are the same window, so cthr[i] =
        // kplus(best corr) * norm_i * (1 - 2^-40) is that bound in the row's K
        // units. Lower-triangle candidates have lower indices than any
        // row-side one, so starting at it loses no tie.
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int64_t i = i0 + R * lane + r;
          const double bk = sm.bK[r][lane];
          if (i < a.nrows && bk != kInf) {
            // (cthr holds kplus() values: -0.0 means "no positive bound yet" and
            // must not lift a row from -inf -- its best may be a negative
            // correlation, e.g. with an exclusion zone that leaves only distant,
            // anti-correlated windows)
            const double klb = a.cthr[i];
            if (klb > 0.0 && klb > bk) sm.bK[r][lane] = klb;
          }
        }
      }
      const double cA = a.mua[i0];
      for (int s = s_beg; s < s_end; ++s) {
        const SegDev sg0 = a.segs[s];
        // SYM: the band sweeps only columns from its first admissible one on
        // (aligned down to 32; the cells before the staircase are masked)
        int q = 0;
        if constexpr (SYM) {
          const int64_t d = i0 + a.excl + 1 - sg0.col0;
          const int64_t qa = d & ~int64_t(31);
          q = d <= 0 ? 0 : (int)(qa < (int64_t)sg0.ncol ? qa : (int64_t)sg0.ncol);
          if (q >= sg0.ncol) continue;
        }
        const SegDev sg{sg0.col0 + q, sg0.src0 + q, sg0.ncol - q, 0};
        SweepCtx cx;
        // column data (read in 32-column chunks, padded by 64) and this
        // segment's edge slice (whole chunks) stay inside their buffers
        TSD_CHECK(s >= 0 && s < a.nseg_v && gw < a.nwarps_alloc);
        TSD_CHECK(sg.col0 >= 0 && sg.col0 + ((sg.ncol + 31) & ~31) <= a.ccols + 64);
        TSD_CHECK(a.seg_eoff[s] + q + ((sg.ncol + 31) & ~31) <= a.ecap);
        cx.colg = a.col + sg.col0;
        cx.E = Ew + a.seg_eoff[s] + q;
        cx.ncol = sg.ncol;
        cx.colbase = (int)sg.col0;
        cx.write_out = (b + 1 < b1);
        cx.row0 = i0 + R * lane;
        cx.excl = a.excl;
        cx.first_seg = (s == s_beg);
        cx.cthr = SYM ? a.cthr + sg.col0 : nullptr;
        cx.namin = namin;
        if (b == b0 && sg.ncol >= 2 && a.tedge) {
          // top edge precomputed by FFT correlation: E[q - delta] = cov(re, col0 + q)
          const int delta = i0 >= 1 ? 0 : 1;
          TSD_CHECK(b0 / bpt < a.tedge_rows && sg.col0 + sg.ncol <= a.tstride);
          const double* te = a.tedge + (int64_t)(b0 / bpt) * a.tstride + sg.col0;
          for (int q = delta + lane; q < sg.ncol - 1 + delta; q += 32) {
            const double v = te[q] * (F32 ? a.f32_sig : 1.0);
            if constexpr (F32)
              reinterpret_cast<float*>(cx.E)[q - delta] = (float)v;
            else
              cx.E[q - delta] = v;
          }
          __threadfence_block();
          __syncwarp();
        } else if (b == b0 && sg.ncol >= 2) {
          // top edge of the task: E[j] = cov(re, j + delta), j = 0 .. ncol-2
          // (row 0 has df = dg = 0, so E[j] = cov(0, j+1) feeds it exactly)
          const int64_t re = i0 >= 1 ? i0 - 1 : 0;
          const int delta = i0 >= 1 ? 0 : 1;
          for (int q0 = delta; q0 < sg.ncol - 1 + delta; q0 += H) {
            double out[R];
            double eU;
            const double cS = a.mub[sg.col0 + q0];
            sliding_dot<R>(sm, a.xa + re, a.mua[re], a.xb + sg.col0 + q0, (int64_t)sg.ncol + a.m - 1 - q0, cS,
                           a.m, lane, out, &eU);
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int q = q0 + R * lane + r;
              // delta = 1: row 0 adds nothing, so cov(0, q) = E[q-1]
              if (q < sg.ncol - 1 + delta) {
                const double v = (out[r] - (a.mub[sg.col0 + q] - cS) * eU) * (F32 ? a.f32_sig : 1.0);
                if constexpr (F32)
                  reinterpret_cast<float*>(cx.E)[q - delta] = (float)v;
                else
                  cx.E[q - delta] = v;
              }
            }
          }
          __threadfence_block();
          __syncwarp();
        }
        double head[R];
        if (SYM && q > 0) {  // left edge at an interior column of the piece: direct dot products
          double out[R], eU;
          sliding_dot<R>(sm, a.xb + sg.col0, a.mub[sg.col0], a.xa + i0, a.na - i0, cA, a.m, lane, out, &eU);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int64_t i = i0 + R * lane + r;
            const double mu = i < a.nrows ? a.mua[i] : cA;
            head[r] = out[r] - (mu - cA) * eU;
          }
        } else if (a.heads) {  // left edge precomputed by FFT correlation (heads_fft.cu)
          TSD_CHECK(i0 + R * lane + R <= a.hstride && a.hstride <= a.hrows_alloc);
          const double2* hp = reinterpret_cast<const double2*>(a.heads + s * a.hstride + i0 + R * lane);
#pragma unroll
          for (int r = 0; r < R / 2; ++r) {
            const double2 h2 = __ldg(hp + r);
            head[2 * r] = h2.x;
            head[2 * r + 1] = h2.y;
          }
          if constexpr (F32) {  // the FP32 sweep's scaled covariances
#pragma unroll
            for (int r = 0; r < R; ++r) head[r] *= a.f32_sig;
          }
        } else {  // left edge: cov(i, col0) for the band's rows, batched 8 segments at a time
#ifndef TSD_ABL_NOHEADS
          if (R == 8 && ((s - s_beg) & 7) == 0 && a.dmma_heads)
#else
          if (s == s_beg && b == b0)
#endif
            if constexpr (R == 8)
              heads_dmma<R>(sm, a.xa + i0, a.na - i0, cA, a.btil + (int64_t)s * a.m, min(8, s_end - s), a.m, lane,
                            Hw);
          double out[R];
          if (R == 8 && a.dmma_heads) {  // heads_dmma: 256-row bands
#pragma unroll
            for (int r = 0; r < R; ++r) out[r] = Hw[((s - s_beg) & 7) * 256 + R * lane + r];
          } else {
            sliding_dot<R>(sm, a.btil + (int64_t)s * a.m, 0.0, a.xa + i0, a.na - i0, cA, a.m, lane, out, nullptr);
          }
          const double e = a.ebt[s], s0 = F32 ? a.f32_sig : 1.0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int64_t i = i0 + R * lane + r;
            const double mu = i < a.nrows ? a.mua[i] : cA;
            head[r] = (out[r] - (mu - cA) * e) * s0;
          }
        }
        if constexpr (F32) {
          // row data of slots (a, a + 8) packed, rounded once
          static_assert(!F32 || R == R32, "the FP32 sweep runs 16 rows per lane");
          float fa[R], ga[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int64_t i = i0 + R * lane + r;
            const bool in = i < a.nrows;
            fa[r] = in ? (float)(a.dfa[i] * a.f32_siga) : 0.0f;
            ga[r] = in ? (float)(a.dga[i] * a.f32_siga) : 0.0f;
          }
          u64 FA[8], GA[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            FA[q] = pack2(fa[q], fa[q + 8]);
            GA[q] = pack2(ga[q], ga[q + 8]);
          }
          // bests as FP32 values (seeds rounded once; +inf = inactive row)
          SweepState32 S;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            S.Q[q] = pack2((float)head[q], (float)head[q + 8]);
            S.BK[q] = pack2(kplus_f(sm.bK[q][lane]), kplus_f(sm.bK[q + 8][lane]));
          }
          S.mbk = min_bk16(S.BK);
          S.dirty = false;
          if constexpr (R == R32) sweep_segment32<SELF>(sm, cx, lane, FA, GA, S);
        } else if constexpr (R == RW) {
          static_assert(R != RW || !SYM, "the wide sweep has no symmetric variant");
          WideState<R> S;
          double dfa[R], dga[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int64_t i = i0 + R * lane + r;
            const bool in = i < a.nrows;
            S.P[r] = head[r];
            dfa[r] = in ? a.dfa[i] : 0.0;
            dga[r] = in ? a.dga[i] : 0.0;
          }
          sweep_segment_w<R, SELF>(sm, cx, lane, dfa, dga, S);
        } else if constexpr (TSD_PIPE && !SYM) {
          PipeState<R> S;
          S.dirty = false;
          double dfa[R], dga[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int64_t i = i0 + R * lane + r;
            const bool in = i < a.nrows;
            S.PA[r] = head[r];
            S.PB[r] = 0.0;
            dfa[r] = in ? a.dfa[i] : 0.0;
            dga[r] = in ? a.dga[i] : 0.0;
            S.bKp[r] = kplus(sm.bK[r][lane]);
          }
          if constexpr (R == 8) sweep_segment_p<R, SELF>(sm, cx, lane, dfa, dga, S);
        } else {
          SweepState<R> S;
          S.dirty = false;
#pragma unroll
          for (int r = 0; r < R; ++r) S.P[r] = head[r];
          // row data and row bests (reloaded per segment so they are not live
          // across the heads)
          double dfa[R], dga[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int64_t i = i0 + R * lane + r;
            const bool in = i < a.nrows;
            dfa[r] = in ? a.dfa[i] : 0.0;
            dga[r] = in ? a.dga[i] : 0.0;
            S.bKp[r] = kplus(sm.bK[r][lane]);
          }
          sweep_segment<R, SELF, SYM>(sm, cx, lane, dfa, dga, S, a.invn_a, a.nrows,
                                      SYM ? a.ccand + (int64_t)(task % SYM_NC) * 2 * a.ccols : nullptr, a.cthr);
        }
      }
      // band results: c = clamp(K * invn_a) (profiles.hpp:331, :335)
      double* oc = a.out_c + (int64_t)g * a.nrows;
      int64_t* oj = a.out_j + (int64_t)g * a.nrows;
      __syncwarp();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t i = i0 + R * lane + r;
        if (i < a.nrows) {
          const int j = sm.bj[r][lane];
          const double c = j >= 0 ? clamp_corr(sm.bK[r][lane] * a.invn_a[i]) : -2.0;
          oc[i] = c;
          oj[i] = j;
          // publish the band's best: later tasks on these rows (other groups)
          // start from it. It is exactly the K this group's sweep computed for
          // the recorded cell, so the seed argument above holds for it too.
          if (!SYM && j >= 0 && a.seed) atomicMax(a.seed + i, order_key(sm.bK[r][lane]));
          // SYM: the row's best so far bounds its final best from below, so it
          // raises the column-side threshold of column i (same window): in
          // clamped correlation units like col_update, lowered by 2^-40, so a
          // lower-triangle candidate tying with it still passes
          if (SYM && j >= 0) {
            const double t = kplus_d(c) * rcp_pos(a.invn_a[i]) * (1.0 - 0x1p-40);
            atomicMax(reinterpret_cast<long long*>(a.cthr + i), __double_as_longlong(t));
          }
        }
      }
      __syncwarp();
    }
  }
}

template <int R, bool SELF, bool F32, bool SYM>
constexpr int join_nreg() {
  return F32 ? TSD_NREG32 : SYM ? TSD_NREG_SYM : R == 16 ? TSD_NREG_WIDE : TSD_NREG;
}
// two kernels around one body: the launch-bound budget, or a __maxnreg__ cap
template <int R, bool SELF, bool F32, bool SYM>
__global__ void __launch_bounds__(32 * WARPS, F32 ? TSD_JOIN_MINB32 : SYM ? TSD_JOIN_MINB_SYM : R == 16 ? TSD_JOIN_MINB_WIDE : TSD_JOIN_MINB)
    k_join(const JoinArgs a) {
  join_body<R, SELF, F32, SYM>(a);
}
template <int R, bool SELF, bool F32, bool SYM>
__global__ void __maxnreg__((join_nreg<R, SELF, F32, SYM>() > 0 ? join_nreg<R, SELF, F32, SYM>() : 128)) k_join_wide(const JoinArgs a) {
  join_body<R, SELF, F32, SYM>(a);
}

// centred top window of each band range (row re = first row - 1, or 0 for
// the first range): w[r][k] = x[re + k] - mu[re], e[r] = sum_k w[r][k]
__global__ void k_topwin(const double* __restrict__ x, const double* __restrict__ mu, int nbr, int rows_per_range,
                         int m, double* __restrict__ w, double* __restrict__ e) {
  const int r = blockIdx.x;
  if (r >= nbr) return;
  const int64_t i0 = (int64_t)r * rows_per_range;
  const int64_t re = i0 >= 1 ? i0 - 1 : 0;
  const double c = mu[re];
  double s = 0.0;
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    const double v = x[re + k] - c;
    w[(int64_t)r * m + k] = v;
    s += v;
  }
  __shared__ double sh[128];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 64; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) e[r] = sh[0];
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

// FP64 column data per concatenated window j: {df_b, dg_b, invn_b, nmin}
// with nmin = (1 - 2^-40) x the smallest window norm 1/invn_b over windows
// j .. j+TB-1 (flat or straddling windows count as DBL_MAX): the block
// threshold of the sweep, whose blocks start at multiples of TB of a
// segment's columns.
// FP64 column data per concatenated window j: {df_b, dg_b, invn_b, nmin}
// with nmin = (1 - 2^-40) x the smallest window norm 1/invn_b over windows
// j .. j+TB-1 (flat or straddling windows count as DBL_MAX): the block
// threshold of the sweep, whose blocks start at multiples of TB of a
// segment's columns.
__global__ void k_pack_cols(const double* __restrict__ df, const double* __restrict__ dg,
                            const double* __restrict__ invn, const uint8_t* __restrict__ flag, int64_t n,
                            double4* __restrict__ col) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n + 64) return;
  if (i >= n) {
    col[i] = make_double4(0, 0, 0, DBL_MAX);
    return;
  }
  double nm = DBL_MAX;
  for (int t = 0; t < TB && i + t < n; ++t) {
    const double iv = invn[i + t];
    if ((flag[i + t] & 1) && iv > 0.0) nm = fmin(nm, 1.0 / iv);
  }
  const double iv = invn[i];
  col[i] = make_double4(df[i], dg[i], iv, nm < DBL_MAX ? nm * (1.0 - 0x1p-40) : DBL_MAX);
}

// FP32 column data (Col32 layout in the same 32-byte slots), from FP64 values
// scaled by sigma_b (column data) and sigma = sigma_a * sigma_b (covariances);
// nmin over the 8-column threshold block (TB = 8 in the FP32 sweep)
__global__ void k_pack_cols32(const double* __restrict__ df, const double* __restrict__ dg,
                              const double* __restrict__ invn, const uint8_t* __restrict__ flag, int64_t n,
                              double4* __restrict__ col, double sigb, double sig) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n + 64) return;
  Col32 c;
  c.pad = 0;
  if (i >= n) {
    c.dg2 = c.df2 = 0;
    c.kf = 0.0f;
    c.nmin = FLT_MAX;
  } else {
    double nm = DBL_MAX;
    for (int t = 0; t < 8 && i + t < n; ++t) {
      const double iv = invn[i + t];
      if ((flag[i + t] & 1) && iv > 0.0) nm = fmin(nm, 1.0 / iv);
    }
    const double iv = invn[i];
    const float g = (float)(dg[i] * sigb), f = (float)(df[i] * sigb);
    c.dg2 = pack2(g, g);
    c.df2 = pack2(f, f);
    c.kf = iv > 0.0 ? (float)(iv / sig) : 0.0f;
    c.nmin = nm < DBL_MAX ? (float)(nm * sig * (1.0 - 0x1p-20)) : FLT_MAX;
  }
  reinterpret_cast<Col32*>(col)[i] = c;
}

// smallest and largest window norm over valid non-flat windows, as positive
// double bits (order-preserving as integers): out[0] = min, out[1] = max
__global__ void k_norm_range(const double* __restrict__ invn, const uint8_t* __restrict__ flag, int64_t n,
                             unsigned long long* __restrict__ out) {
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double iv = invn[i];
    if (flag[i] == 1 && iv > 0.0) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(1.0 / iv);
      lo = min(lo, b);
      hi = max(hi, b);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
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

// flat-column table: per 1024-column block the lowest flat column, then a
// suffix minimum over blocks; next_flat(x) = lowest flat column >= x
constexpr int FB = 1024;
__global__ void k_flat_bmin(const uint8_t* __restrict__ flag, int64_t ncols, int64_t* __restrict__ bmin) {
  __shared__ unsigned long long mn;
  if (threadIdx.x == 0) mn = ~0ull;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * FB;
  for (int t = threadIdx.x; t < FB; t += blockDim.x) {
    const int64_t x = base + t;
    if (x < ncols && (flag[x] & 2)) atomicMin(&mn, (unsigned long long)x);
  }
  __syncthreads();
  if (threadIdx.x == 0) bmin[blockIdx.x] = mn == ~0ull ? -1 : (int64_t)mn;
}
__global__ void k_flat_suffix(int64_t* __restrict__ bmin, int64_t nb) {
  int64_t run = -1;
  for (int64_t b = nb - 1; b >= 0; --b) {
    if (bmin[b] >= 0) run = bmin[b];
    bmin[b] = run;
  }
}
__device__ int64_t next_flat(const uint8_t* __restrict__ flag, const int64_t* __restrict__ bsuf, int64_t ncols,
                             int64_t x) {
  if (x >= ncols) return -1;
  if (x < 0) x = 0;
  const int64_t b = x / FB, end = min(ncols, (b + 1) * FB);
  for (int64_t t = x; t < end; ++t)
    if (flag[t] & 2) return t;
  return (b + 1) * FB < ncols ? bsuf[b + 1] : -1;
}

// Epilogue. Flat rows (profiles.hpp:332-336): c = 1 at the lowest admissible
// flat column, else c = 0 at the lowest admissible column.
__global__ void k_epilogue(const double* __restrict__ bc, const int64_t* __restrict__ bj,
                           const uint8_t* __restrict__ flag, int64_t nrows, const SegDev* __restrict__ segs, int nseg,
                           int m, const int64_t* __restrict__ s_woff, const int64_t* __restrict__ s_ooff, int nser,
                           const uint8_t* __restrict__ cflag, const int64_t* __restrict__ bsuf, int64_t ncols,
                           long long excl, double* __restrict__ val, int64_t* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const uint8_t f = flag[i];
  if (!(f & 1)) return;
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
  double c = bc[i];
  int64_t j = bj[i];
  if (f & 2) {
    const int64_t f0 = next_flat(cflag, bsuf, ncols, 0);
    if (excl < 0) {
      c = f0 >= 0 ? 1.0 : 0.0;
      j = f0 >= 0 ? f0 : segs[0].col0;
    } else {  // self-join: single segment, columns == rows
      const int64_t fj = (f0 >= 0 && f0 < i - excl) ? f0 : next_flat(cflag, bsuf, ncols, i + excl + 1);
      if (fj >= 0) {
        c = 1.0;
        j = fj;
      } else {
        c = 0.0;
        j = i > excl ? 0 : (i + excl + 1 < ncols ? i + excl + 1 : -1);
      }
    }
  } else if (excl >= 0) {
    // self-join, non-flat row: every flat window j is a candidate with c = 0
    // (invn_j = 0, profiles.hpp:289-296), the lowest admissible one winning
    // among them. Those above the exclusion zone are swept by the row itself;
    // those below come to a symmetric sweep only through the column side,
    // which skips flat rows, so the lowest flat window j < i - excl is folded
    // in here by acc_merge's rule (a no-op after the full-matrix sweep, which
    // has already seen the same candidate)
    const int64_t f0 = ncols > 0 ? bsuf[0] : -1;  // lowest flat column (suffix minimum from block 0)
    if (f0 >= 0 && f0 < i - excl && (j < 0 || better(0.0, f0, c, j))) {
      c = 0.0;
      j = f0;
    }
  }
  if (j < 0) {  // no admissible neighbour (profiles.hpp:149-151)
    val[o] = __longlong_as_double(0x7ff0000000000000LL);
    idx[o] = -1;
    return;
  }
  TSD_CHECK(j < ncols);
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

namespace {

// SYM: per row, the lexicographic best of the row side (per-group partials)
// and the column side (ccand) -- acc_merge's rule (profiles.hpp:63-85)
__global__ void k_merge_sym(const double* __restrict__ pc, const int64_t* __restrict__ pj, int64_t nrows, int ngroups,
                            const unsigned long long* __restrict__ ccand, int64_t nrows_cols, double* __restrict__ oc,
                            int64_t* __restrict__ oj) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double bc = -2.0;
  int64_t bj = -1;
  for (int g = 0; g < ngroups; ++g) {
    const double cc = pc[(int64_t)g * nrows + i];
    const int64_t jj = pj[(int64_t)g * nrows + i];
    if (jj >= 0 && (bj < 0 || better(cc, jj, bc, bj))) {
      bc = cc;
      bj = jj;
    }
  }
  for (int c = 0; c < SYM_NC; ++c) {
    const unsigned long long* q = ccand + (int64_t)c * 2 * nrows_cols + 2 * i;
    const unsigned long long ci = q[1];
    if (ci != ~0ull) {
      const double cc = key_value(q[0]);
      const int64_t jj = (int64_t)ci;
      if (bj < 0 || better(cc, jj, bc, bj)) {
        bc = cc;
        bj = jj;
      }
    }
  }
  oc[i] = bj >= 0 ? bc : -2.0;
  oj[i] = bj;
}

// Row seeds from external lower bounds lb[i] (corr units, <= -2: none): the
// order key of (lb - margin) / invn_a in the sweep's K units (k_join)
__global__ void k_seed_fold(unsigned long long* __restrict__ seed, const double* __restrict__ lb,
                            const double* __restrict__ invn, const uint8_t* __restrict__ flag, int64_t n,
                            double margin) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double iv = invn[i];
  const double c = lb[i] - margin;
  if (flag[i] != 1 || !(iv > 0.0) || !(c > -1.0)) return;
  const unsigned long long key = order_key(c / iv);
  if (key > seed[i]) seed[i] = key;
}

// SYM: column side initial state from the row seeds (a lower bound of each
// row's final best, never reported: index "none" = ~0)
__global__ void k_sym_init(const unsigned long long* __restrict__ seed, const double* __restrict__ invn,
                           const uint8_t* __restrict__ flag, int64_t n, unsigned long long* __restrict__ ccand,
                           double* __restrict__ cthr) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n + 64) return;
  if (j >= n) {
    cthr[j] = DBL_MAX;
    return;
  }
  double lb = -2.0;
  const double iv = invn[j];
  const bool act = flag[j] == 1 && iv > 0.0;
  if (act && seed && seed[j] != 0ull) lb = nextafter(key_value(seed[j]), -DBL_MAX) * iv * (1.0 - 0x1p-40);
  for (int c = 0; c < SYM_NC; ++c) {
    ccand[(int64_t)c * 2 * n + 2 * j] = order_key(lb);
    ccand[(int64_t)c * 2 * n + 2 * j + 1] = ~0ull;
  }
  // flat / inactive rows: resolved by the epilogue; their column side never triggers
  cthr[j] = act ? kplus_d(lb) * (1.0 / iv) * (1.0 - 0x1p-40) : DBL_MAX;
}

// ---------------------------------------------------------------------------
// Self-join row seeds from a coarse search (symmetric sweep): the series
// averaged over blocks of f samples is self-joined at window m / f; the
// coarse nearest neighbour jd of coarse row t places each full-resolution
// row i = f t + r near column f jd + r. k_seed_cand evaluates, per coarse row,
// the diagonals through columns f jd + delta (|delta| <= 8) of its f rows:
// one direct centred dot product (window_dot, profiles.hpp:101-108) per
// diagonal, then the reference's recurrence (profiles.hpp:330) down the f
// rows. The best admissible clamped correlation of a row is a lower bound of
// its final best (an evaluation of a real cell), given to the sweep with a
// margin (JoinInputs::seed_corr).
__global__ void k_downsample(const double* __restrict__ x, int64_t nd, int f, double* __restrict__ xd) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nd) return;
  double s = 0.0;
  for (int k = 0; k < f; ++k) s += x[t * f + k];
  xd[t] = s / f;
}

__global__ void k_seed_cand(const double* __restrict__ x, int64_t cnt, int m, long long excl, int f,
                            const double* __restrict__ mu, const double* __restrict__ invn,
                            const double* __restrict__ df, const double* __restrict__ dg,
                            const uint8_t* __restrict__ flag, const int64_t* __restrict__ cbj, int64_t ncoarse,
                            double* __restrict__ seed) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= ncoarse) return;
  const int64_t i0 = t * f;
  if (i0 >= cnt) return;
  constexpr int MAXF = 32;
  double best[MAXF];
#pragma unroll
  for (int r = 0; r < MAXF; ++r) best[r] = -2.0;
  // anchors: the coarse neighbours of rows t - 1, t, t + 1 (as diagonals
  // j - i = f (jd - a) + delta; repeated diagonals are skipped)
  int64_t seen[3];
  int ns = 0;
  for (int da = -1; da <= 1; ++da) {
    const int64_t a = t + da;
    if (a < 0 || a >= ncoarse) continue;
    const int64_t jd = cbj[a];
    if (jd < 0) continue;
    const int64_t off = f * (jd - a);
    bool dup = false;
    for (int q = 0; q < ns; ++q) dup |= seen[q] == off;
    if (dup) continue;
    seen[ns++] = off;
    const int64_t j0 = i0 + off + (lane - 16);  // delta in [-16, 15]
    const bool on = j0 >= 0 && j0 < cnt;
    double cov = 0.0;
    if (on) {
      const double ma = mu[i0], mb = mu[j0];
      for (int k = 0; k < m; ++k) cov = __fma_rn(x[i0 + k] - ma, x[j0 + k] - mb, cov);
    }
#pragma unroll
    for (int r = 0; r < MAXF; ++r) {
      if (r >= f) break;
      const int64_t i = i0 + r, j = j0 + r;
      if (on && i < cnt && j < cnt) {
        if (r > 0) cov += __fma_rn(df[i], dg[j], dg[i] * df[j]);  // profiles.hpp:330
        const long long d = (long long)(i - j);
        if ((d > excl || d < -excl) && flag[i] == 1 && flag[j] == 1 && invn[i] > 0.0 && invn[j] > 0.0)
          best[r] = fmax(best[r], clamp_corr(cov * invn[i] * invn[j]));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < MAXF; ++r) {
    if (r >= f) break;
    double c = best[r];
    for (int o = 16; o; o >>= 1) c = fmax(c, __shfl_xor_sync(0xffffffffu, c, o));
    if (lane == 0 && i0 + r < cnt) seed[i0 + r] = c;
  }
}

// rows that had a seed but ended without any candidate: the seed was above
// the sweep's own value of every admissible cell (count in *bad)
__global__ void k_seed_check(const double* __restrict__ seed, const int64_t* __restrict__ bj, int64_t n,
                             unsigned* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && seed[i] > -1.5 && bj[i] < 0) atomicAdd(bad, 1u);
}

template <int R, bool SELF, bool F32, bool SYM>
int launch_join(const JoinInputs& in, double* d_best_c, int64_t* d_best_j, Arena& arena, cudaStream_t st, Error* err,
                int* launches) {
  constexpr int H = Geo<R>::H;
  const int m = in.m;
  // Virtual segments: a long segment (self-join, AB-join against one long
  // series) is cut into contiguous column pieces so the decomposition can form
  // several segment groups and tall tasks (few top edges). Column numbering,
  // masks and the epilogue's source mapping are unchanged; each piece starts
  // from its own head (cov at its first column), exactly as a segment does.
  const auto t_host0 = std::chrono::steady_clock::now();
  static const bool vmarks = getenv("TSD_VERBOSE") && getenv("TSD_VMARKS");
  auto vmark = [&](const char* what) {  // development timing: host time, stream drained
    if (!vmarks) return;
    cudaStreamSynchronize(st);
    fprintf(stderr, "[tsd]   %s at %.2f ms\n", what,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count());
  };
  std::vector<SegDev> vsegs;
  {
    int64_t tot = 0;
    for (const auto& s : in.segs) tot += s.ncol;
    const char* pe = getenv("TSD_PIECE_MIN");  // development override
    const char* pn = getenv("TSD_PIECES");  // development override of the pieces per long segment
    // the symmetric sweep takes 128 pieces (more, shorter tasks: self-joins
    // of 2^20-2^21 windows 0.5-3 % faster, 2^22 unchanged), AB joins 64
    const int64_t np64 = pn ? std::max<int64_t>(1, atoll(pn)) : (SYM ? 128 : 64);
    // a join too small to give every resident warp a (band, segment) task is
    // latency-bound on its longest sweep: cut its segments into 256-column
    // pieces as well (C1, 64 bands x 8 segments of 413 columns: kernel 0.187 ->
    // 0.122 ms; 128- and 64-column pieces measured 0.13-0.15 ms)
    int nsm0 = 148;
    {
      int dev0 = 0;
      cudaGetDevice(&dev0);
      cudaDeviceGetAttribute(&nsm0, cudaDevAttrMultiProcessorCount, dev0);
    }
    const bool small = !SYM && (int64_t)((in.rows.nwin + H - 1) / H) * (int64_t)in.segs.size() < (int64_t)nsm0 * 16;
    const int64_t lmax = std::max<int64_t>(pe ? atoll(pe) : ((in.min_tasks > 0 || small) ? 256 : 2048),
                                           (tot + np64 - 1) / np64);
    for (const auto& s : in.segs) {
      const int64_t np = (s.ncol + lmax - 1) / lmax;
      if (np <= 1) {
        vsegs.push_back(s);
        continue;
      }
      const int64_t len = (((s.ncol + np - 1) / np) + 31) & ~int64_t(31);  // pieces start 32-aligned
      for (int64_t c = 0; c < s.ncol; c += len)
        vsegs.push_back(SegDev{s.col0 + c, s.src0 + c, (int32_t)std::min<int64_t>(len, s.ncol - c), 0});
    }
  }
  const std::vector<SegDev>& segs = vsegs;
  const int nseg = (int)segs.size();
  const int64_t nrows = in.rows.nwin;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // TSD_SMEM_PAD (development): extra dynamic shared memory per CTA, to probe the
  // sweep's sensitivity to resident warps
  static const size_t smem_pad = getenv("TSD_SMEM_PAD") ? (size_t)atol(getenv("TSD_SMEM_PAD")) : 0;
  const size_t smem_bytes = sizeof(WarpSmem<R, (R == 16 && !F32)>) * WARPS + smem_pad;
  auto kern = [] {
    if constexpr (join_nreg<R, SELF, F32, SYM>() == 0)
      return k_join<R, SELF, F32, SYM>;
    else
      return k_join_wide<R, SELF, F32, SYM>;
  }();
  vmark("segments");
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * WARPS, smem_bytes);
  if (occ < 1) occ = 1;
  const int nwarps = nsm * occ * WARPS;
  const int nbands = (int)((nrows + H - 1) / H);

  // Decomposition: tasks = (range of bpt bands) x (group of consecutive
  // segments). Cost model in FP64-op units per warp: a band sweeps its
  // group's cells (3 ops) plus one m-term head per row per segment; the first
  // band of a task also computes the group's top edge (m terms per column).
  // Tasks are handed out dynamically, group-major: several waves cost the
  // total over all warps plus half a task (the tail); a single wave costs one
  // task over the fraction of warps it fills (the SMs are issue-bound, and its
  // slowest task sets the end) plus 25 %: uneven progress across SMs is not
  // rebalanced, and no group starts from the bests an earlier group
  // published (C4, random walks: 8 %; C2, ECG with many record updates:
  // 33 %). G > 1 costs a merge pass (16 B per row and group). At most 64
  // groups and 16 waves. Calibrated on C4 (G = 16, 28 bands per task:
  // 633 -> 588 ms) and C2 (64 pieces of 2048 columns, one band per task:
  // 6.9 -> 6.3 ms): profiles/README.md.
  vmark("occupancy");
  int64_t total_cols = 0;
  for (const auto& s : segs) total_cols += s.ncol;
  auto split = [&](int G, std::vector<int>& gs) {
    gs.assign(G + 1, nseg);
    gs[0] = 0;
    int s = 0;
    int64_t acc = 0;
    for (int g = 1; g < G; ++g) {
      const int64_t target = total_cols * g / G;
      while (s < nseg - (G - g) && acc + segs[s].ncol <= target) acc += segs[s++].ncol;
      if (s <= gs[g - 1]) acc += segs[s++].ncol;
      gs[g] = s;
    }
  };
  int G = 1, bpt = 1;
  {
    double best = 1e300;
    std::vector<int> gs;
    // round-2 re-calibration for AB / dictionary joins (measured on C4, C3,
    // C5): at most 16 segment groups, plans up to 32 waves, and the FFT
    // top-edge pre-pass costed; the self-join's full-matrix sweep keeps the
    // round-1 model (64 pieces, 16 waves: C2 5.0 vs 5.5-5.8 ms otherwise)
    const int gmax = SELF ? 64 : 16, wave_cap = SELF ? 16 : 32;
    for (int g = 1; g <= nseg && g <= gmax; g *= 2) {
      split(g, gs);
      int64_t cmax = 0, smax = 0;
      for (int q = 0; q < g; ++q) {
        int64_t c = 0;
        for (int s = gs[q]; s < gs[q + 1]; ++s) c += segs[s].ncol;
        cmax = std::max(cmax, c);
        smax = std::max<int64_t>(smax, gs[q + 1] - gs[q]);
      }
      // per row and segment: an FFT head (a load) or an m-term direct head
      const bool fft = heads_fft_supported(m);
      const double band = (double)H * (3.0 * cmax + (double)smax * (fft && nseg >= 2 ? 16.0 : m + 64.0)) + 24.0 * cmax;
      // top edge of a task: its row of the FFT table (~16 sweep cells of
      // transform work per column), else an m-term dot per column
      const double top = (double)cmax * (fft ? 50.0 : (double)m);
      const int bmax = std::min(nbands, F32 ? 4096 / H : 4096);
      for (int b = 1; b <= bmax; ++b) {
        const int64_t nt = (int64_t)((nbands + b - 1) / b) * g;
        if (nt > (int64_t)wave_cap * nwarps) continue;
        const double tc = b * band + top;
        const double run = nt <= nwarps ? 1.25 * tc * nwarps / (double)nt : (double)nt * tc / nwarps + 0.5 * tc;
        // the FFT top-edge pre-pass, one table row per band range over all
        // columns, in the same per-warp units (C4: 3.2 ms for 2341 x 131328).
        // With it and 32 waves C4 takes 14 bands per task instead of 28
        // (kernel 537 -> 525 ms, step 565 -> 557 ms)
        const double pre =
            !SELF && fft && nseg >= 2 ? 0.058 * (double)((nbands + b - 1) / b) * (double)total_cols : 0.0;
        const double cost = run + pre + (g > 1 ? 30.0 * (double)nrows * g / nwarps : 0.0);
        if (cost < best * 0.999) {
          best = cost;
          G = g;
          bpt = b;
        }
        if (nt <= nwarps) break;  // larger b only adds work per task
      }
    }
  }
  if (!SYM && in.min_tasks > 0) {
    // small latency-bound joins (the self-join's coarse seed search): the
    // most groups and the fewest bands per task that reach min_tasks tasks
    // -- every warp of the GPU busy beats the cost model's merge savings
    G = 1;
    bpt = 1;
    while (2 * G <= std::min(nseg, 64) && (int64_t)nbands * G < in.min_tasks) G *= 2;
  }
  if (!SYM && getenv("TSD_FORCE_G") && getenv("TSD_FORCE_BPT")) {  // development override
    G = std::max(1, std::min(nseg, atoi(getenv("TSD_FORCE_G"))));
    bpt = std::max(1, atoi(getenv("TSD_FORCE_BPT")));
  }
  // SYM: one group per piece; bands sweep only their triangle part, so task
  // sizes differ -- choose bpt by an LPT (longest first onto the least-loaded
  // warp) makespan estimate and hand tasks out dynamically in that order
  std::vector<int4> sym_tasks;
  // the LPT plan depends only on the shape: repeated calls of one shape (a
  // learning loop, a benchmark) reuse it
  struct SymPlan {
    std::vector<int64_t> key;
    std::vector<int4> tasks;
    int bpt;
  };
  static thread_local SymPlan sym_cache;
  std::vector<int64_t> sym_key;
  if constexpr (SYM) {
    sym_key = {nrows, (int64_t)nseg, in.excl, (int64_t)m, (int64_t)H, (int64_t)nwarps, (int64_t)in.shard,
               (int64_t)in.nshards};
    for (const auto& sg : segs) {
      sym_key.push_back(sg.col0);
      sym_key.push_back(sg.ncol);
    }
  }
  if (SYM && sym_cache.key == sym_key) {
    G = nseg;
    sym_tasks = sym_cache.tasks;
    bpt = sym_cache.bpt;
  } else if constexpr (SYM) {
    G = nseg;
    auto qoff = [&](int b, int sgi) -> int64_t {  // first swept local column (kernel: q)
      const int64_t d = (int64_t)b * H + in.excl + 1 - segs[sgi].col0;
      return d <= 0 ? 0 : std::min<int64_t>(d & ~int64_t(31), segs[sgi].ncol);
    };
    double best = 1e300;
    int bbest = 1;
    std::vector<std::pair<double, int4>> cand;
    // per piece: prefix sums over bands of the swept cells (cost units), so a
    // candidate task's cost is O(1)
    std::vector<double> pre((size_t)G * (nbands + 1));
    for (int g = 0; g < G; ++g) {
      double* P = pre.data() + (size_t)g * (nbands + 1);
      P[0] = 0.0;
      for (int b = 0; b < nbands; ++b) P[b + 1] = P[b] + (double)H * 2.5 * (double)(segs[g].ncol - qoff(b, g));
    }
    struct PlanOpt {
      double mk;
      int bp;
      std::vector<std::pair<double, int4>> cand;
    };
    std::vector<PlanOpt> plans;  // in increasing bands per task
    const int bpmax = std::min(nbands, 1024);
    const char* bpe = getenv("TSD_SYM_BP");  // development override of the bands per task
    const int bpforce = bpe ? atoi(bpe) : 0;
    std::vector<int> bps;
    if (bpforce > 0) {
      bps.push_back(std::min(bpforce, nbands));
    } else {
      for (int bp = 1; bp <= bpmax; bp *= 2) bps.push_back(bp);
    }
    for (const int bp : bps) {
      // very fine splits only add per-task overhead (top edge, head) once
      // there are many tasks per warp; skip them while a coarser one remains
      if (bp * 2 <= bpmax && bpforce <= 0) {
        int64_t cnt = 0;
        for (int g = 0; g < G; ++g)
          for (int b0 = 0; b0 < nbands; b0 += bp) cnt += qoff(b0, g) < segs[g].ncol;
        if (cnt > 32 * (int64_t)nwarps) continue;
      }
      cand.clear();
      for (int b0 = 0; b0 < nbands; b0 += bp) {
        const int b1 = std::min(nbands, b0 + bp);
        for (int g = 0; g < G; ++g) {
          const double* P = pre.data() + (size_t)g * (nbands + 1);
          double c = P[b1] - P[b0];
          if (c <= 0.0) continue;
          // top edge (a row of the FFT table, ~50 sweep-op units per column,
          // or an m-term dot) + the band's left edge at an interior column
          c += (double)(segs[g].ncol - qoff(b0, g)) * (heads_fft_supported(m) ? 50.0 : (double)m) + (double)H * m;
          cand.push_back({c, make_int4(b0, b1, g, 0)});
        }
      }
      std::sort(cand.begin(), cand.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
      std::priority_queue<double, std::vector<double>, std::greater<double>> load;
      for (int w = 0; w < nwarps; ++w) load.push(0.0);
      double mk = 0.0;
      for (const auto& c : cand) {
        const double l = load.top() + c.first;
        load.pop();
        load.push(l);
        mk = std::max(mk, l);
      }
      if (getenv("TSD_VERBOSE")) fprintf(stderr, "[tsd] sym plan: %d bands per task, %zu tasks, makespan %.4g\n", bp,
                                         cand.size(), mk);
      plans.push_back({mk, bp, cand});
      best = std::min(best, mk);
    }
    // one step finer than the estimate's best (if that estimate is within
    // 5 %): more tasks rebalance better and let later waves start from the
    // column bests the earlier ones raised, which the estimate does not
    // model. Measured (ms, bands per task): 2^20 x m 256: 228 / 207 / 194
    // for 32 / 16 / 8 (estimate 16); 2^21 x 512: 611 / 594 for 16 / 8
    // (estimate 16); 2^22 x 512: 2362 / 2300 / 2457 for 32 / 16 / 8
    // (estimate 32)
    int ib = 0;
    for (size_t q = 0; q < plans.size(); ++q)
      if (plans[q].mk == best) ib = (int)q;
    if (ib > 0 && plans[ib - 1].bp * 2 == plans[ib].bp && plans[ib - 1].mk <= best * 1.05) --ib;
    for (size_t q = (size_t)ib; q < plans.size(); ++q) {
      const PlanOpt& pl = plans[q];
      bbest = pl.bp;
      sym_tasks.clear();
      // sharded (multi-GPU) self-join: every nshards-th task of the
      // longest-first order, so each shard gets an even share of the cells
      for (size_t q = 0; q < pl.cand.size(); ++q)
        if ((int)(q % (size_t)in.nshards) == in.shard) sym_tasks.push_back(pl.cand[q].second);
      break;
    }
    bpt = bbest;
    // every band range with cells yields a task, so a plan without tasks can
    // only be a planning fault (its epilogue would report every row empty)
    if (plans.empty() || (sym_tasks.empty() && in.nshards <= 1)) {
      if (err) *err = Error{kCudaError, "internal: the symmetric self-join plan has no tasks"};
      return kCudaError;
    }
    sym_cache.key = sym_key;
    sym_cache.tasks = sym_tasks;
    sym_cache.bpt = bpt;
  }
  std::vector<int> group_seg;
  if (SYM) {
    group_seg.resize(nseg + 1);
    for (int g = 0; g <= nseg; ++g) group_seg[g] = g;
  } else {
    split(G, group_seg);
  }
  std::vector<int> eoff(nseg);
  int64_t ecap = 0;
  for (int g = 0; g < G; ++g) {
    int64_t off = 0;
    for (int s = group_seg[g]; s < group_seg[g + 1]; ++s) {
      eoff[s] = (int)off;
      off += (segs[s].ncol + 1) & ~1;
    }
    ecap = std::max(ecap, off);
  }
  ecap = (ecap + 64 + 31) & ~int64_t(31);
  const int nbr = (nbands + bpt - 1) / bpt;
  const int ntasks = SYM ? (int)sym_tasks.size() : nbr * G;
  const int grid = std::max(1, std::min(nsm * occ, (ntasks + WARPS - 1) / WARPS));
  const int used_warps = grid * WARPS;
  if (getenv("TSD_VERBOSE"))
    fprintf(stderr,
            "[tsd] join R=%d rows=%lld bands=%d cols=%lld segs=%d -> G=%d bpt=%d tasks=%d warps=%d occ=%d (plan %.2f ms)\n",
            R, (long long)nrows, nbands, (long long)total_cols, nseg, G, bpt, ntasks, used_warps, occ,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count());

  SegDev* d_segs = (SegDev*)arena.get(sizeof(SegDev) * nseg);
  int* d_eoff = (int*)arena.get(sizeof(int) * nseg);
  int* d_gs = (int*)arena.get(sizeof(int) * (G + 1));
  double4* d_col = (double4*)arena.get(sizeof(double4) * (in.cols.nwin + 64));
  double* d_btil = (double*)arena.get(sizeof(double) * (int64_t)nseg * m);
  double* d_ebt = (double*)arena.get(sizeof(double) * nseg);
  double* d_edges = (double*)arena.get(sizeof(double) * ecap * used_warps);
  double* d_hscr = (double*)arena.get(sizeof(double) * 2048 * used_warps);
  const bool part = G > 1 || SYM;  // per-group partial outputs, merged afterwards
  double* d_pc = part ? (double*)arena.get(sizeof(double) * nrows * G) : d_best_c;
  int64_t* d_pj = part ? (int64_t*)arena.get(sizeof(int64_t) * nrows * G) : d_best_j;
  int4* d_tasks = nullptr;
  int* d_tnext = nullptr;
  unsigned long long* d_ccand = nullptr;
  double* d_cthr = nullptr;
  d_tnext = (int*)arena.get(sizeof(int));
  if (!d_tnext) {
    if (err) *err = Error{kCudaError, "device allocation failed for the join"};
    return kCudaError;
  }
  CUDA_TRY(cudaMemsetAsync(d_tnext, 0, sizeof(int), st));
  if (SYM) {
    d_tasks = (int4*)arena.get(sizeof(int4) * std::max<size_t>(1, sym_tasks.size()));
    d_ccand = (unsigned long long*)arena.get(sizeof(unsigned long long) * 2 * SYM_NC * (in.cols.nwin + 64));
    d_cthr = (double*)arena.get(sizeof(double) * (in.cols.nwin + 64));
    if (!d_tasks || !d_tnext || !d_ccand || !d_cthr) {
      if (err) *err = Error{kCudaError, "device allocation failed for the symmetric self-join"};
      return kCudaError;
    }
    if (!sym_tasks.empty())
      CUDA_TRY(cudaMemcpyAsync(d_tasks, sym_tasks.data(), sizeof(int4) * sym_tasks.size(), cudaMemcpyHostToDevice,
                               st));
    // (band range, group) pairs without columns are never queued: their
    // partial rows must read "no candidate" in the merge
    CUDA_TRY(cudaMemsetAsync(d_pj, 0xff, sizeof(int64_t) * nrows * G, st));
  }
  if (!d_segs || !d_eoff || !d_gs || !d_col || !d_hscr || !d_btil || !d_ebt || !d_edges || !d_pc || !d_pj) {
    if (err) *err = Error{kCudaError, "device allocation failed for the join"};
    return kCudaError;
  }
  CUDA_TRY(cudaMemcpyAsync(d_segs, segs.data(), sizeof(SegDev) * nseg, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_eoff, eoff.data(), sizeof(int) * nseg, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_gs, group_seg.data(), sizeof(int) * (G + 1), cudaMemcpyHostToDevice, st));
  int nl = 0;
  if (F32)
    k_pack_cols32<<<(unsigned)((in.cols.nwin + 64 + 255) / 256), 256, 0, st>>>(
        in.cols.df, in.cols.dg, in.cols.invn, in.cols.flag, in.cols.nwin, d_col, in.f32_sigb,
        in.f32_siga * in.f32_sigb);
  else
    k_pack_cols<<<(unsigned)((in.cols.nwin + 64 + 255) / 256), 256, 0, st>>>(
        in.cols.df, in.cols.dg, in.cols.invn, in.cols.flag, in.cols.nwin, d_col);
  ++nl;
  k_btil<<<nseg, 128, 0, st>>>(in.xb, in.cols.mu, d_segs, m, d_btil, d_ebt);
  ++nl;
  vmark("allocations + packing");
  // heads by FFT correlation when there are several segments and the
  // [seg][row] array fits comfortably (C4: 256 x 2^24 doubles = 34 GB)
  const int64_t hstride = (int64_t)nbands * H;
  double* d_heads = nullptr;
  unsigned long long* d_seed = nullptr;
  {
    const char* e = getenv("TSD_FFT_HEADS");
    const bool want = (e ? atoi(e) != 0 : true) && nseg >= 2 && heads_fft_supported(m);
    size_t fr = 0;
    const size_t hbytes = sizeof(double) * (size_t)nseg * (size_t)hstride;
    if (want && device_free_bytes(&fr) && hbytes < fr / 2) {
      d_heads = (double*)arena.get(hbytes);
      d_seed = (unsigned long long*)arena.get(sizeof(unsigned long long) * nrows);
      if (d_heads && d_seed) {
        if (in.ev[0]) CUDA_TRY(cudaEventRecord(in.ev[0], st));
        in.heads_used = true;
        const int rc = compute_heads_fft(in.xa, in.na, nrows, hstride, in.rows.mu, in.rows.flag, d_btil, d_ebt,
                                         in.cols.invn, d_segs, nseg, m, d_heads, hstride, d_seed,
                                         SELF ? in.excl : -1,
                                         SYM ? 1 : 0, arena, st, &nl, err);
        if (rc != kOk) return rc;
        if (in.ev[1]) CUDA_TRY(cudaEventRecord(in.ev[1], st));
      }
    }
  }
  vmark("heads fft");
  // top edges by FFT: one row of the table per band range, all columns
  double* d_te = nullptr;
  int64_t tstride = 0;
  {
    const char* e = getenv("TSD_FFT_TOP");
    const int nbr_t = (nbands + bpt - 1) / bpt;
    tstride = (in.cols.nwin + 1) & ~int64_t(1);
    size_t fr = 0;
    const size_t tbytes = sizeof(double) * (size_t)nbr_t * (size_t)tstride;
    // small joins compute their top edges in the kernel: below ~2^30 FMAs of
    // direct dot products the FFT pre-pass's four launches cost more (C1:
    // 0.343 -> 0.320 ms per step)
    const bool big = (double)nbr_t * (double)total_cols * (double)m > 1073741824.0;
    if ((e ? atoi(e) != 0 : big) && heads_fft_supported(m) && nbr_t >= 2 && device_free_bytes(&fr) &&
        tbytes < fr / 4) {
      double* d_tw = (double*)arena.get(sizeof(double) * (size_t)nbr_t * m);
      double* d_tew = (double*)arena.get(sizeof(double) * nbr_t);
      d_te = (double*)arena.get(tbytes);
      if (d_tw && d_tew && d_te) {
        k_topwin<<<nbr_t, 128, 0, st>>>(in.xa, in.rows.mu, nbr_t, bpt * H, m, d_tw, d_tew);
        ++nl;
        const int rc = compute_heads_fft(in.xb, in.nb, in.cols.nwin, in.cols.nwin, in.cols.mu, in.cols.flag, d_tw,
                                         d_tew, in.cols.invn, d_segs, nbr_t, m, d_te, tstride, nullptr, -1, 0, arena,
                                         st, &nl, err, SYM ? (int64_t)bpt * H : 0, SYM ? (long long)in.excl : 0);
        if (rc != kOk) return rc;
      } else {
        d_te = nullptr;
      }
    }
  }
  if (getenv("TSD_VERBOSE")) {
    size_t fr = 0;
    device_free_bytes(&fr);
    fprintf(stderr, "[tsd] heads %s, top edges %s, free %.1f GB\n", d_heads ? "fft" : "in-kernel",
            d_te ? "fft" : "in-kernel", fr / 1e9);
  }
  vmark("top edges fft");
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
  a.f32_sig = in.f32_siga * in.f32_sigb;
  a.f32_siga = in.f32_siga;
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
  a.hscr = d_hscr;
  {
    const char* e = getenv("TSD_DMMA_HEADS");
    a.dmma_heads = (SYM || R != 8) ? 0 : (e ? atoi(e) : 1);  // SYM heads sit at band-dependent columns
  }
  a.heads = d_heads;
  a.hstride = hstride;
  if (!SYM && !d_heads) {
    // no head seeds: the array still carries the bests finished bands publish
    d_seed = (unsigned long long*)arena.get(sizeof(unsigned long long) * nrows);
    if (d_seed) CUDA_TRY(cudaMemsetAsync(d_seed, 0, sizeof(unsigned long long) * nrows, st));
  }
  if (SELF && in.seed_corr && !F32) {
    // external row lower bounds (corr units): exact evaluations of admissible
    // cells, lowered by seed_margin so the sweep's own value of that cell
    // stays above them (k_seed_fold)
    if (!d_seed) {
      d_seed = (unsigned long long*)arena.get(sizeof(unsigned long long) * nrows);
      if (!d_seed) {
        if (err) *err = Error{kCudaError, "device allocation failed for the row seeds"};
        return kCudaError;
      }
      CUDA_TRY(cudaMemsetAsync(d_seed, 0, sizeof(unsigned long long) * nrows, st));
    }
    k_seed_fold<<<(unsigned)((nrows + 255) / 256), 256, 0, st>>>(d_seed, in.seed_corr, in.rows.invn, in.rows.flag,
                                                                  nrows, in.seed_margin);
    ++nl;
  }
  a.seed = (d_heads || !SYM || (SELF && in.seed_corr && !F32)) ? d_seed : nullptr;
  a.tedge = d_te;
  a.tstride = tstride;
  a.nseg_v = nseg;
  a.hrows_alloc = hstride;
  a.tedge_rows = d_te ? (nbands + bpt - 1) / bpt : 0;
  a.nwarps_alloc = used_warps;
  a.tasks = d_tasks;
  a.task_next = d_tnext;
  a.ccand = d_ccand;
  a.ccols = in.cols.nwin;
  a.cthr = d_cthr;
  if (SYM) {
    const int64_t nc = in.cols.nwin;
    k_sym_init<<<(unsigned)((nc + 64 + 255) / 256), 256, 0, st>>>(a.seed, in.rows.invn, in.rows.flag, nc, d_ccand,
                                                                  d_cthr);
    ++nl;
  }
  a.out_c = d_pc;
  a.out_j = d_pj;
#ifdef TSD_COUNT_EXACT
  unsigned long long zero = 0;
  cudaMemcpyToSymbol(g_exact_count, &zero, 8);
  cudaMemcpyToSymbol(g_step_count, &zero, 8);
  cudaMemcpyToSymbol(g_exact_first, &zero, 8);
  cudaMemcpyToSymbol(g_step_first, &zero, 8);
  cudaMemcpyToSymbol(g_col_count, &zero, 8);
  cudaMemcpyToSymbol(g_cas_count, &zero, 8);
  cudaMemcpyToSymbol(g_true_steps, &zero, 8);
  cudaMemcpyToSymbol(g_rare_cycles, &zero, 8);
  cudaMemcpyToSymbol(g_total_cycles, &zero, 8);
  cudaMemcpyToSymbol(g_true_slots, &zero, 8);
#endif
  if (in.ev[2]) CUDA_TRY(cudaEventRecord(in.ev[2], st));
  vmark("args + sym init");
  kern<<<grid, 32 * WARPS, smem_bytes, st>>>(a);
  vmark("k_join");
  ++nl;
  if (in.ev[3]) CUDA_TRY(cudaEventRecord(in.ev[3], st));
#ifdef TSD_COUNT_EXACT
  {
    unsigned long long ce = 0, cs = 0;
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(&ce, g_exact_count, 8);
    cudaMemcpyFromSymbol(&cs, g_step_count, 8);
    unsigned long long cef = 0, csf = 0;
    cudaMemcpyFromSymbol(&cef, g_exact_first, 8);
    cudaMemcpyFromSymbol(&csf, g_step_first, 8);
    fprintf(stderr, "[tsd] exact-path steps %llu of %llu warp-steps (%.2f%%); first segment %.2f%%, others %.2f%%\n",
            ce, cs, 100.0 * ce / (cs ? cs : 1), 100.0 * cef / (csf ? csf : 1),
            100.0 * (ce - cef) / ((cs - csf) ? (cs - csf) : 1));
    unsigned long long cc = 0, ca = 0;
    cudaMemcpyFromSymbol(&cc, g_col_count, 8);
    cudaMemcpyFromSymbol(&ca, g_cas_count, 8);
    fprintf(stderr, "[tsd] column-side updates %llu (%.2f%% of warp-steps), with a candidate %llu\n", cc,
            100.0 * cc / (cs ? cs : 1), ca);
    unsigned long long rc = 0, tcy = 0;
    cudaMemcpyFromSymbol(&rc, g_rare_cycles, 8);
    cudaMemcpyFromSymbol(&tcy, g_total_cycles, 8);
    fprintf(stderr, "[tsd] rare path (pipelined AB sweep): %.1f cycles per entry, %.2f%% of all warp cycles; %.1f warp cycles per step\n",
            (double)rc / (ce ? ce : 1), 100.0 * rc / (tcy ? tcy : 1), (double)tcy / (cs ? cs : 1));
    unsigned long long ts = 0, tsl = 0;
    cudaMemcpyFromSymbol(&ts, g_true_steps, 8);
    cudaMemcpyFromSymbol(&tsl, g_true_slots, 8);
    fprintf(stderr, "[tsd] warp-steps with a true update %.2f%%, updated slots per warp-step %.4f\n",
            100.0 * ts / (cs ? cs : 1), (double)tsl / (cs ? cs : 1));
  }
#endif
  if (SYM) {
    k_merge_sym<<<(unsigned)((nrows + 255) / 256), 256, 0, st>>>(d_pc, d_pj, nrows, G, d_ccand, in.cols.nwin,
                                                                  d_best_c, d_best_j);
    ++nl;
    vmark("merge");
  } else if (G > 1) {
    k_merge_groups<<<(unsigned)((nrows + 255) / 256), 256, 0, st>>>(d_pc, d_pj, nrows, G);
    ++nl;
    CUDA_TRY(cudaMemcpyAsync(d_best_c, d_pc, sizeof(double) * nrows, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d_best_j, d_pj, sizeof(int64_t) * nrows, cudaMemcpyDeviceToDevice, st));
  }
  CUDA_TRY(cudaGetLastError());
  if (launches) *launches += nl;
  return kOk;
}

}  // namespace

namespace {
// FP32 mode: the FP32 sweep chooses each row's column; its correlation is
// then recomputed exactly in FP64 as a direct m-term dot product of the two
// centred windows (window_dot, profiles.hpp:101-108). Without this the
// distance sqrt(2m(1 - rho)) of a near-exact match amplifies FP32 rounding
// of rho (~1e-7) to ~3e-3. Flat rows are resolved by the epilogue; a flat
// column keeps rho = 0 (profiles.hpp:332-336).
__global__ void k_refine_fp64(double* __restrict__ bc, const int64_t* __restrict__ bj, int64_t nrows,
                              const double* __restrict__ xa, const double* __restrict__ mua,
                              const double* __restrict__ invn_a, const uint8_t* __restrict__ flag_a,
                              const double* __restrict__ xb, const double* __restrict__ mub,
                              const double* __restrict__ invn_b, int m) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const int64_t j = bj[i];
  if (j < 0 || flag_a[i] != 1 || !(invn_b[j] > 0.0)) return;
  const double ma = mua[i], mb = mub[j];
  double acc = 0.0;
  for (int k = 0; k < m; ++k) acc = __fma_rn(xa[i + k] - ma, xb[j + k] - mb, acc);
  bc[i] = clamp_corr(acc * invn_a[i] * invn_b[j]);
}
}  // namespace

int run_join(const JoinInputs& in, double* d_best_c, int64_t* d_best_j, Arena& arena, cudaStream_t st, Error* err,
             int* launches) {
  const bool self = in.excl >= 0;
  if (in.precision == 1) {
    // power-of-two scalings that bring the largest window norm of each side
    // to (1/2, 1]: every scaled covariance then lies in [-1, 1]. The FP32
    // sweep needs the smallest scaled products (and the K = cov * invn_b
    // values) to stay well inside the FP32 range; inputs whose window norms
    // span more than the FP32 mode's accuracy allows (2^10 over both sides,
    // below) run the FP64 sweep instead.
    unsigned long long* d_rng = (unsigned long long*)arena.get(sizeof(unsigned long long) * 4);
    if (!d_rng) {
      if (err) *err = Error{kCudaError, "device allocation failed for the FP32 scaling"};
      return kCudaError;
    }
    const unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
    CUDA_TRY(cudaMemcpyAsync(d_rng, init, sizeof(init), cudaMemcpyHostToDevice, st));
    k_norm_range<<<296, 256, 0, st>>>(in.rows.invn, in.rows.flag, in.rows.nwin, d_rng);
    k_norm_range<<<296, 256, 0, st>>>(in.cols.invn, in.cols.flag, in.cols.nwin, d_rng + 2);
    if (launches) *launches += 2;
    unsigned long long rng[4];
    CUDA_TRY(cudaMemcpyAsync(rng, d_rng, sizeof(rng), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    auto side = [](unsigned long long lo, unsigned long long hi, double& mn, double& mx) {
      if (hi == 0) {  // no non-flat window: nothing to scale
        mn = mx = 1.0;
        return;
      }
      mn = __builtin_bit_cast(double, lo);
      mx = __builtin_bit_cast(double, hi);
    };
    double mna, mxa, mnb, mxb;
    side(rng[0], rng[1], mna, mxa);
    side(rng[2], rng[3], mnb, mxb);
    JoinInputs fin = in;
    fin.f32_siga = std::ldexp(1.0, -std::ilogb(mxa) - 1);
    fin.f32_sigb = std::ldexp(1.0, -std::ilogb(mxb) - 1);
    const double span = (mna / mxa) * (mnb / mxb);
    // (K = cov * invn_b, bounded by mxa * mxb / mnb, is kept in FP32 too)
    // Accuracy: a cell's FP32 covariance carries eps32 x the largest |cov| its
    // diagonal has seen since the last FP64 restart, i.e. up to eps32 / span
    // in correlation units once a diagonal has crossed the largest windows of
    // both sides and reached the smallest. The BASELINE shapes span 10 (ECG)
    // to 218 (C4 walks) and stay ten times inside the 1e-3 distance tolerance;
    // a x1000 stretch inside one dictionary segment (span 2e-5) missed it by
    // 20x in the randomized tests. Beyond 2^10 the FP64 sweep runs instead.
    // (windows of fewer than 8 samples gain nothing from FP32 and their
    // correlations sit at +-1 by construction, where FP32 ranking is weakest)
    const bool fits = span > 0x1p-10 && mxa * (mxb / mnb) < 0x1p110 && in.m >= 8;
    if (getenv("TSD_VERBOSE"))
      fprintf(stderr, "[tsd] fp32 norms a [%.3g, %.3g] b [%.3g, %.3g] -> %s\n", mna, mxa, mnb, mxb,
              fits ? "fp32 sweep"
                   : in.m < 8 ? "fp64 sweep (windows shorter than 8 samples)"
                              : "fp64 sweep (window norms span more than 2^10 over both sides)");
    if (!fits) {
      JoinInputs din = in;
      din.precision = 0;
      return run_join(din, d_best_c, d_best_j, arena, st, err, launches);
    }
    const int rc = self ? launch_join<R32, true, true, false>(fin, d_best_c, d_best_j, arena, st, err, launches)
                        : launch_join<R32, false, true, false>(fin, d_best_c, d_best_j, arena, st, err, launches);
    if (rc != kOk) return rc;
    const int64_t n = in.rows.nwin;
    k_refine_fp64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_best_c, d_best_j, n, in.xa, in.rows.mu,
                                                               in.rows.invn, in.rows.flag, in.xb, in.cols.mu,
                                                               in.cols.invn, in.m);
    if (launches) ++*launches;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      if (err) *err = Error{kCudaError, cudaGetErrorString(e)};
      return kCudaError;
    }
    return kOk;
  }
  if (self) {
    // The symmetric upper-triangle sweep evaluates each admissible pair once
    // and updates both rows, as the reference does (profiles.hpp:287-297).
    // Its column side filters well only with distinctive windows and enough
    // waves of bands, so it wins from about 2^26 / m windows for m >= 192;
    // below that, and for short windows at any size, the full-matrix sweep
    // (every pair from both rows) is faster. TSD_SYM=1 / 0 forces either.
    const char* e = getenv("TSD_SYM");
    // Crossover measured on walks / ECG (host API, ms full vs symmetric):
    // m = 1024: 65k 1.9/2.8, 98k 4.0/3.7; m = 512: 65k 2.0/2.6, 131k 5.5/5.2,
    // 2^21 ~1000/590; m = 250: 131k 6.0/7.0, 262k 19.9/19.0, 393k 42/38;
    // m = 128: 786k 163/208; m = 64: 1M 305/833 (short windows leave the
    // column side too many near-best candidates).
    const bool auto_sym =
        in.m >= 192 && in.rows.nwin >= std::max<int64_t>(98304, (int64_t(1) << 26) / std::max(1, in.m));
    const bool sym = in.force_sym || (e ? atoi(e) != 0 : auto_sym);
    auto sweep = [&](const JoinInputs& x) {
      return sym ? launch_join<8, true, false, true>(x, d_best_c, d_best_j, arena, st, err, launches)
                 : launch_join<8, true, false, false>(x, d_best_c, d_best_j, arena, st, err, launches);
    };
    const char* pe = getenv("TSD_SELF_SEEDS");
    const char* fe = getenv("TSD_SEED_F");  // development override of the coarse factor
    const int f = fe ? std::max(4, std::min(32, atoi(fe))) : std::min(32, in.m / 16);
    // (the symmetric sweep only: at C2's size, where the full-matrix
    // sweep runs, the pre-pass costs more than it saves -- C2 6.9 -> 8.2 ms)
    const int seeds_mode = pe ? atoi(pe) : 1;  // 0 off, 1 symmetric sweep only, 2 both sweeps (experiments)
    if ((!sym && seeds_mode < 2) || seeds_mode == 0 || f < 4 || in.seed_corr || in.nshards > 1 ||
        in.na / f < 4 * (in.m / f))
      return sweep(in);
    // coarse search for row seeds (k_seed_cand), then the sweep from them;
    // rows a seed left empty (its margin undercut by the sweep's own
    // rounding, never seen) send the join back through unseeded
    const int64_t n = in.na, cnt = in.rows.nwin;
    const int64_t nd = n / f;
    const int md = in.m / f;
    JoinInputs cin;
    double* d_xd = (double*)arena.get(sizeof(double) * (nd + 64));
    double* d_seed = (double*)arena.get(sizeof(double) * (cnt + 64));
    unsigned* d_bad = (unsigned*)arena.get(sizeof(unsigned));
    if (!d_xd || !d_seed || !d_bad) {
      if (err) *err = Error{kCudaError, "device allocation failed for the self-join seeds"};
      return kCudaError;
    }
    k_downsample<<<(unsigned)((nd + 255) / 256), 256, 0, st>>>(in.xa, nd, f, d_xd);
    std::vector<Group> gd{Group{0, nd - md + 1, 0, 0}};
    int bad_series = -1;
    if (int rc = compute_windows(d_xd, nd, md, gd, 1, cin.rows, arena, st, &bad_series, err)) return rc;
    cin.xa = cin.xb = d_xd;
    cin.na = cin.nb = nd;
    cin.cols = cin.rows;
    cin.segs = {SegDev{0, 0, (int32_t)(nd - md + 1), 0}};
    cin.m = md;
    cin.excl = (in.excl + f - 1) / f;
    cin.precision = 0;
    {
      // the coarse join is small (C2: 8.7k windows): plan it wide enough to
      // occupy the GPU (C2 symmetric path: coarse join 0.83 -> ~0.3 ms)
      const char* mt = getenv("TSD_COARSE_TASKS");  // development override
      cin.min_tasks = mt ? atoi(mt) : 2400;
    }
    const int64_t ncoarse = nd - md + 1;
    double* d_cbc = (double*)arena.get(sizeof(double) * ncoarse);
    int64_t* d_cbj = (int64_t*)arena.get(sizeof(int64_t) * ncoarse);
    if (!d_cbc || !d_cbj) {
      if (err) *err = Error{kCudaError, "device allocation failed for the self-join seeds"};
      return kCudaError;
    }
    if (int rc = launch_join<8, true, false, false>(cin, d_cbc, d_cbj, arena, st, err, launches)) return rc;
    k_seed_cand<<<(unsigned)((ncoarse * 32 + 255) / 256), 256, 0, st>>>(in.xa, cnt, in.m, in.excl, f, in.rows.mu,
                                                                        in.rows.invn, in.rows.df, in.rows.dg,
                                                                        in.rows.flag, d_cbj, ncoarse, d_seed);
    if (launches) *launches += 2 + window_stat_launches(md);
    JoinInputs sin = in;
    sin.seed_corr = d_seed;
    const char* me = getenv("TSD_SEED_MARGIN");  // test hook: a negative margin forces the re-run guard
    sin.seed_margin = me ? atof(me) : 1e-8;
    if (int rc = sweep(sin)) return rc;
    CUDA_TRY(cudaMemsetAsync(d_bad, 0, sizeof(unsigned), st));
    k_seed_check<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(d_seed, d_best_j, cnt, d_bad);
    unsigned bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (getenv("TSD_VERBOSE")) fprintf(stderr, "[tsd] self-join seeds: coarse f=%d, %u rows left empty\n", f, bad);
    if (bad == 0) return kOk;
    return sweep(in);
  }
  // AB / dictionary join. The wide sweep (16 rows per lane) is an ablation
  // build (-DTSD_WIDE_BUILD, then TSD_WIDE=1): measured equal on C4 (504 vs
  // 500 ms at 12 instead of 16 resident warps) and slower on short joins
#ifdef TSD_WIDE_BUILD
  {
    const char* we = getenv("TSD_WIDE");
    const bool wide = we ? atoi(we) != 0 : TSD_WIDE_DEFAULT && in.rows.nwin >= (int64_t)TSD_WIDE_MIN_ROWS;
    if (wide) return launch_join<RW, false, false, false>(in, d_best_c, d_best_j, arena, st, err, launches);
  }
#endif
  return launch_join<8, false, false, false>(in, d_best_c, d_best_j, arena, st, err, launches);
}

namespace {
// acc_merge's rule over shard partials (profiles.hpp:79-85): larger corr,
// then lower index; part p of row i at [p * cnt + i]
__global__ void k_merge_parts(const double* __restrict__ pc, const int64_t* __restrict__ pj, int nparts, int64_t cnt,
                              double* __restrict__ oc, int64_t* __restrict__ oj) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  double bc = -2.0;
  int64_t bj = -1;
  for (int p = 0; p < nparts; ++p) {
    const double c = pc[(int64_t)p * cnt + i];
    const int64_t j = pj[(int64_t)p * cnt + i];
    if (j >= 0 && (bj < 0 || better(c, j, bc, bj))) {
      bc = c;
      bj = j;
    }
  }
  oc[i] = bc;
  oj[i] = bj;
}
}  // namespace

int profile_merge_device(const double* d_pc, const int64_t* d_pj, int nparts, int64_t cnt, double* d_c, int64_t* d_j,
                         cudaStream_t st) {
  if (cnt > 0) k_merge_parts<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(d_pc, d_pj, nparts, cnt, d_c, d_j);
  return cudaGetLastError() == cudaSuccess ? kOk : kCudaError;
}

int run_epilogue(const double* d_best_c, const int64_t* d_best_j, const uint8_t* d_row_flag, int64_t nrows,
                 const SegDev* d_segs, int nseg, int m, const int64_t* d_woff, const int64_t* d_ooff, int nser,
                 const uint8_t* d_col_flag, int64_t ncols, int64_t excl, double* d_val, int64_t* d_idx, Arena& arena,
                 cudaStream_t st, Error* err) {
  const int64_t nb = (ncols + FB - 1) / FB;
  int64_t* d_bsuf = (int64_t*)arena.get(sizeof(int64_t) * (nb + 1));
  if (!d_bsuf) {
    if (err) *err = Error{kCudaError, "device allocation failed for the epilogue"};
    return kCudaError;
  }
  k_flat_bmin<<<(unsigned)nb, 256, 0, st>>>(d_col_flag, ncols, d_bsuf);
  k_flat_suffix<<<1, 1, 0, st>>>(d_bsuf, nb);
  k_epilogue<<<(unsigned)((nrows + 255) / 256), 256, 0, st>>>(d_best_c, d_best_j, d_row_flag, nrows, d_segs, nseg, m,
                                                               d_woff, d_ooff, nser, d_col_flag, d_bsuf, ncols,
                                                               (long long)excl, d_val, d_idx);
  CUDA_TRY(cudaGetLastError());
  return kOk;
}

}  // namespace tsd

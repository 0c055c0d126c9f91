// tsd_internal.h -- host-side interfaces between the C ABI (capi.cu) and the
// kernel modules (stats.cu, join.cu, selfjoin.cu). Not installed.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace tsd {

// Status codes: 0 ok, else 1 + tsdict::errc ordinal (reference errors.hpp:13-35).
enum Status : int {
  kOk = 0,
  kWindowTooSmall = 1,
  kWindowTooLarge = 2,
  kNonFiniteInput = 3,
  kLengthMismatch = 4,
  kSeriesTooShort = 5,
  kIterationCapExceeded = 6,
  kSourceMismatch = 7,
  kWindowMismatch = 8,
  kEmptyDictionary = 9,
  kEmptyProfile = 10,
  kDegenerateLabels = 11,
  kInvalidArgument = 16,
  kCudaError = 100,
};

struct Error {
  int code;
  std::string msg;
};

// One window-statistics "threshold group": windows [wbeg, wend) of a
// concatenated sample buffer that belong to one reference TimeSeries (or one
// 16384-window query block of it, dictionary.hpp:175-180); the constancy
// threshold (series.hpp:75-77) uses max|x| over samples [wbeg, wend-1+m).
struct Group {
  int64_t wbeg, wend;
  int32_t series;  // index into the caller's series list (non-finite reporting order)
  int32_t pad;
};

// Device arrays describing every window of a concatenated sample buffer.
// flag bit 0: window lies inside one series (valid); bit 1: window is flat.
struct WindowArrays {
  int64_t nwin = 0;
  double* mu = nullptr;
  double* sd = nullptr;
  double* invn = nullptr;
  double* df = nullptr;
  double* dg = nullptr;
  uint8_t* flag = nullptr;
};

// Dictionary segment as laid out on the device: its window 0 is concatenated
// column col0; ncol valid windows; src0 = Segment::start (dictionary.hpp:46-51).
struct SegDev {
  int64_t col0;
  int64_t src0;
  int32_t ncol;
  int32_t pad;
};

// Scratch arena: a list of device blocks handed out bump-style; reset()
// rewinds without freeing so repeated calls of the same shape do not hit
// cudaMalloc. Grows, never shrinks.
struct Arena {
  struct Blk {
    char* p;
    size_t cap, used;
  };
  std::vector<Blk> blks;
  size_t cur = 0;
  ~Arena();
  void reset() {
    for (auto& b : blks) b.used = 0;
    cur = 0;
  }
  void* get(size_t bytes);  // nullptr on allocation failure
};

// Free device memory for sizing decisions (heads, top-edge tables). A real
// cudaMemGetInfo is repeated only after some Arena has allocated or freed
// device memory since the last one: the query itself can stall for tens of
// milliseconds (measured up to 60 ms on B200), between the launches of a step.
// Allocations by others are not seen; a stale estimate only makes an
// arena.get fail, which every caller handles with its fallback.
bool device_free_bytes(size_t* free_bytes);

// stats.cu -------------------------------------------------------------------
// Computes window arrays for the concatenated buffer d_x[0..n). `bad_series`
// receives (host) the lowest series index holding a non-finite sample, or -1.
// d_bad_out != nullptr: no host synchronisation; *d_bad_out receives the device
// int the caller reads after its own synchronisation (0x7fffffff = all
// finite, else the lowest series index holding a non-finite sample).
// kernels one compute_windows call launches (2: group maxima + the fused tile
// kernel; 5 with the global prefix scans, for windows too long for a tile)
int window_stat_launches(int m);
int compute_windows(const double* d_x, int64_t n, int m, const std::vector<Group>& groups, int nseries,
                    WindowArrays& out, Arena& arena, cudaStream_t st, int* bad_series, Error* err,
                    const int** d_bad_out = nullptr);

// join.cu --------------------------------------------------------------------
struct JoinInputs {
  // rows: windows of the concatenated query buffer
  const double* xa;
  int64_t na;
  WindowArrays rows;
  // columns: windows of the concatenated dictionary buffer
  const double* xb;
  int64_t nb;
  WindowArrays cols;
  std::vector<SegDev> segs;  // host copy
  int m;
  int64_t excl = -1;  // self-join exclusion half-width (|i-j| <= excl rejected); -1 = AB join
  int precision;      // 0 fp64, 1 fp32
  bool force_sym = false;  // self-join: the symmetric sweep at any size (bitwise-equal pair values)
  int shard = 0, nshards = 1;  // symmetric self-join: this call sweeps every nshards-th task from `shard`
  // optional timing events: [0, 1] around the FFT heads pre-pass, [2, 3]
  // around the join kernel (recorded when non-null); heads_used set by run_join
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  mutable bool heads_used = false;
  // self-join: optional per-row lower bounds of the best correlation (device,
  // nrows; <= -2 = none), each an evaluation of an admissible cell; the sweep
  // starts each row at (bound - seed_margin)
  const double* seed_corr = nullptr;
  double seed_margin = 0.0;
  // FP32 sweep: power-of-two scalings of the query / dictionary statistics (run_join)
  double f32_siga = 1.0, f32_sigb = 1.0;
  // > 0: plan at least this many tasks (most groups, one band per task)
  int min_tasks = 0;
};

// Runs the row-band join of every row against every valid column of every
// segment. Writes per-row best (corr, concat column) into d_best_c/d_best_j.
int run_join(const JoinInputs& in, double* d_best_c, int64_t* d_best_j, Arena& arena, cudaStream_t st,
             Error* err, int* launches);

// heads_fft.cu ---------------------------------------------------------------
// Final left-edge heads of every (row, segment) by FFT correlation:
// d_heads[s * hstride + i] for i < hrows. heads_fft_supported(m): m fits the
// 4096-point transform with >= 512 rows per block.
int heads_fft_supported(int m);
// d_seed (optional, nrows): per row the order-preserving u64 key of its best
// admissible column-0 candidate max_s head * invn_b over ALL segments (0 =
// none; excl >= 0: self-join, heads inside the exclusion zone skipped); one
// ulp below it is a strict lower bound the join starts from (k_join).
int compute_heads_fft(const double* d_x, int64_t na, int64_t nrows, int64_t hrows, const double* d_mua,
                      const uint8_t* d_flag_a, const double* d_btil, const double* d_ebt, const double* d_invn_b,
                      const SegDev* d_segs, int nseg, int m, double* d_heads, int64_t hstride,
                      unsigned long long* d_seed, long long excl, int sym, Arena& arena, cudaStream_t st,
                      int* launches, Error* err, int64_t tri_rows = 0, long long tri_excl = 0);
// tri_rows > 0 (the symmetric self-join's FFT top edges): "segment" s is the
// top window of rows [s * tri_rows, ...), whose sweep reads only the columns
// from ((s * tri_rows + tri_excl + 1) & ~31) on; column blocks entirely below
// that are skipped (about half the table).

// learn.cu -------------------------------------------------------------------
// Device steps of the greedy learning loop (dictionary.hpp:279-316): argmin of
// P - S over unmasked windows (lexicographic, first minimum), max of S, and the
// exact FP64 distance profile of a picked window folded into S.
int learn_argmin(const double* d_P, const double* d_S, const uint8_t* d_mask, int64_t cnt, void* d_scratch,
                 double* h_val, int64_t* h_idx, cudaStream_t st);
int learn_max(const double* d_S, int64_t cnt, void* d_scratch, double* h_max, cudaStream_t st);
int learn_dprof_fold(const double* d_x, const WindowArrays& w, int m, const double* d_qc, double invn_q,
                     bool const_query, int64_t origin, double origin_val, bool first, double* d_S, cudaStream_t st);
size_t learn_scratch_bytes();
// find_discords' peak loop (dict_join.hpp:54-93): up to `want` greedy argmax
// picks over finite, unsuppressed windows, each suppressing +-floor(m/2)
int discord_peaks(const double* d_vals, int64_t cnt, int m, int64_t want, uint8_t* d_sup, void* d_scratch,
                  std::vector<int64_t>& at, std::vector<double>& score, cudaStream_t st);

// dprofile.cu ----------------------------------------------------------------
// Distance profile of one query window q (m samples, device) against every
// window of d_x[0..n): d_means == nullptr -> distance_profile_naive
// (profiles.hpp:164-181, znorm_distance per window, bit-exact); otherwise
// distance_profile_mass's rules (profiles.hpp:186-260) over the given window
// statistics with exact FP64 dot products; origin < 0: none.
struct QueryMoments {  // the query's znorm_distance / MASS moments (host, reference arithmetic)
  double mu = 0.0;       // Kahan mean
  double var_sum = 0.0;  // Kahan sum of (q - mu)^2
  double max_abs = 0.0;
  double invn = 0.0;     // 1 / (sd * sqrt(m)), 0 when constant
  bool constant = false;
};
int distance_profile_device(const double* d_x, int64_t n, const double* d_q, int m, const QueryMoments& qm,
                            const double* d_means, const double* d_invn, const uint8_t* d_cmask, int64_t origin,
                            double* d_out, cudaStream_t st);

// acc_merge over nparts per-row partials [p * cnt + i] (sharded self-join)
int profile_merge_device(const double* d_pc, const int64_t* d_pj, int nparts, int64_t cnt, double* d_c, int64_t* d_j,
                         cudaStream_t st);

// Epilogue: corr -> distance (series.hpp:153-161), concat column -> source
// coordinate (dictionary.hpp:183-188), (inf, -1) sentinel for rows without an
// admissible neighbour (profiles.hpp:149-151), row compaction for batched
// queries: series q's valid windows start at row d_woff[q] and are written
// from output slot d_ooff[q] on (nser == 1: identity).
// Flat rows (invn_a == 0) are resolved here from the column flags
// (d_col_flag over ncols concatenated columns; excl >= 0 for the self-join).
int run_epilogue(const double* d_best_c, const int64_t* d_best_j, const uint8_t* d_row_flag, int64_t nrows,
                 const SegDev* d_segs, int nseg, int m, const int64_t* d_woff, const int64_t* d_ooff, int nser,
                 const uint8_t* d_col_flag, int64_t ncols, int64_t excl, double* d_val, int64_t* d_idx, Arena& arena,
                 cudaStream_t st, Error* err);

}  // namespace tsd

/*
 * tsdict_cuda.h -- C ABI of the B200 (sm_100a) tsdict hot path.
 *
 * The reference `tsdict` library (/root/reference/proj) is header-only C++;
 * its hot path sits behind inline functions in namespace tsdict. This C ABI is
 * what those functions bind to in the drop-in headers under include/tsdict/
 * (and what a ctypes / cgo / JNI binding would call).
 * Plain pointers and sizes only; all buffers are caller-owned HOST memory
 * unless the name says _device. Every entry point is thread-safe (per-thread
 * stream and scratch) and deterministic.
 *
 * Return value: 0 on success, otherwise 1 + the ordinal of tsdict::errc
 * (reference include/tsdict/errors.hpp:13-35), or TSD_CUDA_ERROR. The message
 * of the last failure on the calling thread is tsd_last_error().
 */
#ifndef TSDICT_CUDA_H
#define TSDICT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum tsd_status {
  TSD_OK = 0,
  TSD_WINDOW_TOO_SMALL = 1,     /* errc::window_too_small */
  TSD_WINDOW_TOO_LARGE = 2,     /* errc::window_too_large */
  TSD_NON_FINITE_INPUT = 3,     /* errc::non_finite_input */
  TSD_LENGTH_MISMATCH = 4,      /* errc::length_mismatch */
  TSD_SERIES_TOO_SHORT = 5,     /* errc::series_too_short */
  TSD_ITERATION_CAP_EXCEEDED = 6,
  TSD_SOURCE_MISMATCH = 7,      /* errc::source_mismatch */
  TSD_WINDOW_MISMATCH = 8,      /* errc::window_mismatch */
  TSD_EMPTY_DICTIONARY = 9,     /* errc::empty_dictionary */
  TSD_EMPTY_PROFILE = 10,
  TSD_DEGENERATE_LABELS = 11,
  TSD_PARSE_ERROR = 12,
  TSD_VERSION_ERROR = 13,
  TSD_SCHEMA_ERROR = 14,
  TSD_IO_ERROR = 15,
  TSD_INVALID_ARGUMENT = 16,    /* errc::invalid_argument */
  TSD_CUDA_ERROR = 100          /* device failure (no reference counterpart) */
};

enum tsd_precision { TSD_FP64 = 0, TSD_FP32 = 1 };

/* Replaces tsdict::compute_stats (series.hpp:83-150). Outputs hold n-m+1
 * entries: window means, population stds, invn = 1/(std*sqrt(m)) or 0 when
 * flat, and the flat mask. */
int tsd_compute_stats(const double* x, size_t n, size_t m, double* means, double* stds, double* invn,
                      unsigned char* flat);

/* Replaces tsdict::ab_join (profiles.hpp:306-342). val/idx hold na-m+1
 * entries (distance, nearest window index of b). */
int tsd_ab_join(const double* a, size_t na, const double* b, size_t nb, size_t m, int precision, double* val,
                int64_t* idx);

/* Replaces tsdict::self_join (profiles.hpp:266-301) with the exclusion zone as
 * a parameter: neighbours j with |i-j| <= excl are inadmissible. The
 * reference uses excl = m/2 (profiles.hpp:273); pass TSD_EXCL_DEFAULT for it. */
#define TSD_EXCL_DEFAULT ((size_t)-1)
int tsd_self_join(const double* t, size_t n, size_t m, size_t excl, int precision, double* val, int64_t* idx);

/* Sharded self-join (multi-GPU): shard s of S sweeps every S-th
 * task of the symmetric upper-triangle decomposition and returns per-row
 * partials over ALL rows -- corr (clamped correlation, -2 = none) and col
 * (window index, -1 = none) -- covering its pairs from both ends. The
 * exchange is one all-gather of the partials; tsd_profile_merge applies
 * acc_merge's rule (larger corr, then lower index; profiles.hpp:79-85) and
 * tsd_self_join_finish turns the merged partials into the profile
 * (distances, flat rows, sentinel) exactly as tsd_self_join does. */
int tsd_self_join_partial(const double* t, size_t n, size_t m, size_t excl, size_t shard, size_t nshards,
                          double* corr, int64_t* col);
int tsd_profile_merge(const double* corr_parts, const int64_t* col_parts, size_t nparts, size_t cnt, double* corr,
                      int64_t* col);
int tsd_self_join_finish(const double* t, size_t n, size_t m, size_t excl, const double* corr, const int64_t* col,
                         double* val, int64_t* idx);
/* The same three steps on DEVICE buffers (d_t: n samples; d_corr / d_col /
 * d_val / d_idx: n-m+1 entries; parts: nparts x cnt, part p at [p * cnt]),
 * queued on `stream` (a cudaStream_t) without host copies or synchronisation,
 * so the exchange between them can be a device all-gather (NCCL). finish
 * reads the merged partials from d_val / d_idx and overwrites them with the
 * profile. */
int tsd_self_join_partial_device(const double* d_t, size_t n, size_t m, size_t excl, size_t shard, size_t nshards,
                                 double* d_corr, int64_t* d_col, void* stream);
int tsd_profile_merge_device(const double* d_corr_parts, const int64_t* d_col_parts, size_t nparts, size_t cnt,
                             double* d_corr, int64_t* d_col, void* stream);
int tsd_self_join_finish_device(const double* d_t, size_t n, size_t m, size_t excl, double* d_val, int64_t* d_idx,
                                void* stream);

/* Replaces tsdict::detail::dict_min_profile (dictionary.hpp:149-193), the
 * engine of join_dictionary (dict_join.hpp:42-48) and compute_e_max
 * (dictionary.hpp:247-255). Segments are packed back to back in seg_vals
 * (seg_len[s] samples each); seg_start[s] is Segment::start in source
 * coordinates. One device launch covers every segment; windows straddling
 * segment boundaries are never formed. idx is in source coordinates. */
int tsd_dict_join(const double* q, size_t nq, const double* seg_vals, const size_t* seg_len,
                  const size_t* seg_start, size_t nseg, size_t m, int precision, double* val, int64_t* idx);

/* Row sharding of a dictionary join (multi-GPU): the query
 * windows [*row_lo, *row_hi) of shard `shard` of `nshards`, whole
 * 16384-window query blocks each (dictionary.hpp:175-180). Joining samples
 * [row_lo, row_hi + m - 1) with tsd_dict_join gives exactly those rows of the
 * unsharded profile's windows (indices are source coordinates); concatenating
 * the shards in order is the whole profile. Host-only, no device work. */
int tsd_dict_shard_rows(size_t nq, size_t m, size_t shard, size_t nshards, size_t* row_lo, size_t* row_hi);

/* Batched form (no reference counterpart; equivalent to join_dictionary per
 * series): nseries query series packed back to back in q_vals (q_len[k]
 * samples each). Outputs are packed per series: sum_k (q_len[k]-m+1) rows. */
int tsd_dict_join_batched(const double* q_vals, const size_t* q_len, size_t nseries, const double* seg_vals,
                          const size_t* seg_len, const size_t* seg_start, size_t nseg, size_t m, int precision,
                          double* val, int64_t* idx);

/* Replaces tsdict::compute_e_max (dictionary.hpp:247-255): the largest
 * dictionary-join distance of the source series against its dictionary.
 * source_length is Dictionary::source_length. */
int tsd_compute_e_max(const double* t, size_t n, size_t source_length, const double* seg_vals, const size_t* seg_len,
                      const size_t* seg_start, size_t nseg, size_t m, double* e_max);

/* ---- device-resident plan API (inputs already in HBM; used by bench.py) ---- */
typedef struct tsd_dict_plan tsd_dict_plan;

/* Uploads a dictionary (host buffers, as tsd_dict_join) once. */
int tsd_dict_plan_create(const double* seg_vals, const size_t* seg_len, const size_t* seg_start, size_t nseg,
                         size_t m, int precision, tsd_dict_plan** plan);
/* Joins device-resident query series (d_q: sum q_len doubles) against the
 * plan's dictionary; d_val/d_idx are device buffers of sum (q_len-m+1).
 * `stream` is a cudaStream_t (0 = the plan's own stream). Synchronous. */
int tsd_dict_plan_join_device(tsd_dict_plan* plan, const double* d_q, const size_t* q_len, size_t nseries,
                              double* d_val, int64_t* d_idx, void* stream);
/* Same with host buffers (copies inside). */
int tsd_dict_plan_join(tsd_dict_plan* plan, const double* q, const size_t* q_len, size_t nseries, double* val,
                       int64_t* idx);
int tsd_dict_plan_destroy(tsd_dict_plan* plan);
/* CUDA-event device times (ms) of the last join call of this plan: the whole
 * device pipeline (window stats + join + epilogue) and the join kernels
 * alone, plus the number of kernel launches that call issued. */
int tsd_dict_plan_last_timing(tsd_dict_plan* plan, double* step_ms, double* join_ms, int* launches);

/* CUDA-event device times (ms) of the last join call of this plan for the
 * row-band join kernel alone and for the FFT heads pre-pass (0 when the
 * heads were computed inside the join kernel). */
int tsd_dict_plan_last_kernel_timing(tsd_dict_plan* plan, double* join_kernel_ms, double* heads_ms);

/* ---- greedy dictionary learning (dictionary.hpp:259-328) ----
 * learn_dictionary on the device: argmin of the processed profile P - S over
 * unmasked windows, masking, context intervals and merging as the reference's
 * select_state, distance profiles of the picks (exact FP64 dot products: the
 * 1 x n slice of the join, MASS's rules without its FFT round-off), stop
 * rules, then compute_e_max of the result. Exactly one stop rule: rule =
 * TSD_RULE_SPACE_SAVING (rule_value = target fraction in [0, 1)),
 * TSD_RULE_SAMPLE_BUDGET (samples > 0) or TSD_RULE_ERROR_TARGET (e_max
 * target >= 0). profile: the exact self-join profile values of t (n-m+1
 * doubles, as learn_dictionary(T, cfg, P_B)) or NULL to compute it here
 * (self_join with excl = m/2). Outputs (caller-allocated): merged segments
 * (seg_start, seg_len: capacity n; seg_vals: capacity n samples), their count
 * *nseg, core starts in pick order (capacity n-m+1) and *ncores, e_max,
 * space_saving, no_progress. Validation order as validate_learn_config
 * (:120-141), then series_too_short (n < 2m); iteration_cap_exceeded when
 * max_iterations picks pass without the stop rule firing. */
#define TSD_RULE_SPACE_SAVING 0
#define TSD_RULE_SAMPLE_BUDGET 1
#define TSD_RULE_ERROR_TARGET 2
int tsd_learn_dictionary(const double* t, size_t n, size_t m, double k, int rule, double rule_value,
                         size_t max_iterations, const double* profile, size_t* seg_start, size_t* seg_len,
                         double* seg_vals, size_t* nseg, size_t* core_starts, size_t* ncores, double* e_max,
                         double* space_saving, int* no_progress);

/* ---- discords (dict_join.hpp:50-93) ----
 * find_discords on the device: greedy top-k argmax over the finite profile
 * values with +-floor(m/2) suppression (first maximum wins); the rank-1 pick
 * is certified when it leads the best non-overlapping runner-up by more than
 * e_max (or has none). values: host (tsd_find_discords) or device-resident
 * (tsd_find_discords_device, on `stream`). Outputs (capacity top_k): start,
 * score, certified; *count picks. empty_profile for cnt == 0,
 * invalid_argument for e_max < 0. */
int tsd_find_discords(const double* values, size_t cnt, size_t m, double e_max, size_t top_k, size_t* start,
                      double* score, int* certified, size_t* count);
int tsd_find_discords_device(const double* d_values, size_t cnt, size_t m, double e_max, size_t top_k,
                             size_t* start, double* score, int* certified, size_t* count, void* stream);

/* ---- distance profiles (profiles.hpp:164-260) ----
 * Distance of the query window q (m samples) to every window of t (n - m + 1
 * outputs in out).
 * tsd_distance_profile_naive replaces distance_profile_naive (:164-181):
 * znorm_distance (series.hpp:166-204) per window, bit-identical to the
 * reference's arithmetic.
 * tsd_distance_profile_mass replaces distance_profile_mass (:186-260) over the
 * caller's window statistics of t (SubseqStats: means, invn, constant_mask,
 * n - m + 1 each): MASS's conventions (constant query / constant windows, the
 * origin entry by znorm_distance), with exact FP64 dot products in place of
 * the FFT convolution. origin = TSD_NO_ORIGIN for none. The SubseqStats
 * length checks (:189-194) are the caller's (the drop-in header does them). */
#define TSD_NO_ORIGIN ((size_t)-1)
int tsd_distance_profile_naive(const double* t, size_t n, const double* q, size_t m, double* out);
int tsd_distance_profile_mass(const double* t, size_t n, const double* q, size_t m, const double* means,
                              const double* invn, const unsigned char* constant_mask, size_t origin, double* out);

/* ---- diagnostics ---- */
const char* tsd_last_error(void);
/* CUDA-event device times (ms) of the last tsd_ab_join / tsd_self_join call
 * on this thread: the device pipeline (window statistics to epilogue, no
 * host copies) and the main join kernel alone, plus its kernel launches. */
int tsd_last_join_timing(double* device_ms, double* kernel_ms, int* launches);
const char* tsd_status_name(int status); /* reference errc_name (errors.hpp:37-57) */
const char* tsd_build_info(void);
/* Measured DFMA (precision 0) / FFMA (precision 1) throughput of device 0 in
 * FLOP/s over roughly `seconds` of sustained load. */
int tsd_measure_peak(int precision, double seconds, double* flops);
/* the same, plus the SM clock (MHz) seen by the FP64 loop (0 for FP32) */
int tsd_measure_peak_clock(int precision, double seconds, double* flops, double* sm_mhz);

#ifdef __cplusplus
}
#endif

#endif /* TSDICT_CUDA_H */

// capi.cu -- the extern "C" boundary (include/tsdict_cuda.h).
//
// Validation order and error codes reproduce the reference functions each
// entry point replaces (cited per function); device work runs on a
// per-thread stream with a per-thread scratch arena (thread-safe,
// re-entrant). There is no CPU fallback: when no usable CUDA device exists
// every entry point fails with TSD_CUDA_ERROR.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tsdict_cuda.h"
#include "tsd_internal.h"

using namespace tsd;

namespace {

thread_local std::string t_err;

const char* status_name(int c) {  // reference errors.hpp:37-57
  switch (c) {
    case kOk: return "Ok";
    case kWindowTooSmall: return "WindowTooSmall";
    case kWindowTooLarge: return "WindowTooLarge";
    case kNonFiniteInput: return "NonFiniteInput";
    case kLengthMismatch: return "LengthMismatch";
    case kSeriesTooShort: return "SeriesTooShort";
    case kIterationCapExceeded: return "IterationCapExceeded";
    case kSourceMismatch: return "SourceMismatch";
    case kWindowMismatch: return "WindowMismatch";
    case kEmptyDictionary: return "EmptyDictionary";
    case kEmptyProfile: return "EmptyProfile";
    case kDegenerateLabels: return "DegenerateLabels";
    case 12: return "ParseError";
    case 13: return "VersionError";
    case 14: return "SchemaError";
    case 15: return "IoError";
    case kInvalidArgument: return "InvalidArgument";
    case kCudaError: return "CudaError";
  }
  return "UnknownError";
}

int fail(int code, const std::string& msg) {
  t_err = std::string(status_name(code)) + ": " + msg;
  return code;
}
int fail(const Error& e) { return fail(e.code, e.msg); }

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) return fail(kCudaError, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define TRY(call)                \
  do {                           \
    int rc_ = (call);            \
    if (rc_ != kOk) return fail(er); \
  } while (0)

struct Stream {
  cudaStream_t st = nullptr;
  cudaEvent_t ev[8] = {};  // 0..3: step / join phases; 4..7: heads pre-pass and join kernel
  int init() {
    if (st) return kOk;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      return fail(kCudaError, "no CUDA device available (the B200 library has no CPU fallback)");
    }
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (auto& x : ev) CK(cudaEventCreate(&x));
    return kOk;
  }
  ~Stream() {
    // process teardown may already have destroyed the context; ignore errors
    if (st) cudaStreamDestroy(st);
    for (auto& x : ev)
      if (x) cudaEventDestroy(x);
  }
};

struct ThreadCtx {
  Stream s;
  Arena arena;
};

ThreadCtx& tctx() {
  thread_local ThreadCtx c;
  return c;
}

// CUDA-event times of the last ab / self join on this thread (tsd_last_join_timing)
struct LastJoin {
  double device_ms = 0.0, kernel_ms = 0.0;
  int launches = 0;
};
thread_local LastJoin t_last;

// threshold groups for one series of `len` samples at window offset woff;
// `block` > 0 splits into reference query blocks (dictionary.hpp:175-180)
void add_groups(std::vector<Group>& g, int64_t woff, int64_t len, int m, int64_t block, int series) {
  const int64_t cnt = len - m + 1;
  if (cnt <= 0) return;
  if (block <= 0) block = cnt;
  for (int64_t c0 = 0; c0 < cnt; c0 += block) g.push_back(Group{woff + c0, woff + std::min(cnt, c0 + block), series, 0});
}

}  // namespace

// ---------------------------------------------------------------------------
// plan: dictionary resident on the device
// ---------------------------------------------------------------------------
struct tsd_dict_plan {
  int m = 0;
  int precision = 0;
  Stream s;
  Arena dict_arena, work_arena;
  std::vector<SegDev> segs;
  SegDev* d_segs = nullptr;
  double* d_xb = nullptr;
  int64_t nb = 0;
  WindowArrays cols;
  bool dict_nonfinite = false;
  double step_ms = 0.0, join_ms = 0.0, kernel_ms = 0.0, heads_ms = 0.0;
  int launches = 0;
};

namespace {

// The sweeps keep column (dictionary / self-join window) indices in 32 bits
// (join.cu: SweepCtx::colbase, SegDev::ncol, the symmetric sweep's rows):
// inputs whose column count would reach 2^31 are rejected up front rather
// than truncated. (16 GiB of samples; no reference counterpart.)
constexpr size_t kMaxColumnSamples = (size_t(1) << 31) - 256;

int validate_dict(const size_t* seg_len, size_t nseg, size_t m) {  // dictionary.hpp:151-157
  if (nseg == 0) return fail(kEmptyDictionary, "dictionary has no segments");
  size_t tot = 0;
  for (size_t s = 0; s < nseg; ++s) {
    if (seg_len[s] < m) return fail(kWindowMismatch, "dictionary segment shorter than the window length");
    tot += seg_len[s];
  }
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");
  if (tot > kMaxColumnSamples) return fail(kInvalidArgument, "dictionary exceeds 2^31 samples");
  return kOk;
}

int plan_build(tsd_dict_plan* p, const double* seg_vals, const size_t* seg_len, const size_t* seg_start, size_t nseg,
               size_t m, int precision) {
  if (int rc = p->s.init()) return rc;
  p->m = (int)m;
  p->precision = precision;
  int64_t nb = 0;
  for (size_t s = 0; s < nseg; ++s) nb += (int64_t)seg_len[s];
  p->nb = nb;
  p->d_xb = (double*)p->dict_arena.get(sizeof(double) * (nb + 64));
  p->d_segs = (SegDev*)p->dict_arena.get(sizeof(SegDev) * nseg);
  if (!p->d_xb || !p->d_segs) return fail(kCudaError, "device allocation failed for the dictionary");
  CK(cudaMemcpyAsync(p->d_xb, seg_vals, sizeof(double) * nb, cudaMemcpyHostToDevice, p->s.st));
  std::vector<Group> groups;
  int64_t off = 0;
  p->segs.resize(nseg);
  for (size_t s = 0; s < nseg; ++s) {
    p->segs[s] = SegDev{off, (int64_t)seg_start[s], (int32_t)(seg_len[s] - m + 1), 0};
    add_groups(groups, off, (int64_t)seg_len[s], (int)m, 0, (int)s);  // each segment is one TimeSeries (:160-162)
    off += (int64_t)seg_len[s];
  }
  CK(cudaMemcpyAsync(p->d_segs, p->segs.data(), sizeof(SegDev) * nseg, cudaMemcpyHostToDevice, p->s.st));
  Error er{0, ""};
  int bad = -1;
  TRY(compute_windows(p->d_xb, nb, (int)m, groups, (int)nseg, p->cols, p->dict_arena, p->s.st, &bad, &er));
  p->dict_nonfinite = bad >= 0;
  return kOk;
}

// device-resident query join; q_len host array
int plan_join_dev(tsd_dict_plan* p, const double* d_q, const size_t* q_len, size_t nser, double* d_val,
                  int64_t* d_idx, cudaStream_t user_st) {
  const int m = p->m;
  for (size_t k = 0; k < nser; ++k)  // dictionary.hpp:158 per series
    if ((size_t)m > q_len[k]) return fail(kWindowTooLarge, "window length exceeds series length");
  if (nser == 0) return fail(kInvalidArgument, "no query series");
  cudaStream_t st = user_st ? user_st : p->s.st;
  Arena& ar = p->work_arena;
  ar.reset();
  int64_t N = 0;
  std::vector<Group> groups;
  std::vector<int64_t> woff(nser), ooff(nser);
  int64_t outn = 0;
  for (size_t k = 0; k < nser; ++k) {
    woff[k] = N;
    ooff[k] = outn;
    add_groups(groups, N, (int64_t)q_len[k], m, 16384, (int)k);
    N += (int64_t)q_len[k];
    outn += (int64_t)q_len[k] - m + 1;
  }
  CK(cudaEventRecord(p->s.ev[0], st));
  Error er{0, ""};
  JoinInputs in;
  int bad = -1;
  if (p->dict_nonfinite) return fail(kNonFiniteInput, "series contains a non-finite sample");
  // the query's non-finite check is read after the join's final
  // synchronisation (no host round trip between the statistics and the join)
  const int* d_bad = nullptr;
  TRY(compute_windows(d_q, N, m, groups, (int)nser, in.rows, ar, st, &bad, &er, &d_bad));
  in.xa = d_q;
  in.na = N;
  in.xb = p->d_xb;
  in.nb = p->nb;
  in.cols = p->cols;
  in.segs = p->segs;
  in.m = m;
  in.excl = -1;
  in.precision = p->precision;
  const int64_t nrows = in.rows.nwin;
  double* d_bc = (double*)ar.get(sizeof(double) * nrows);
  int64_t* d_bj = (int64_t*)ar.get(sizeof(int64_t) * nrows);
  int64_t* d_woff = (int64_t*)ar.get(sizeof(int64_t) * nser);
  int64_t* d_ooff = (int64_t*)ar.get(sizeof(int64_t) * nser);
  if (!d_bc || !d_bj || !d_woff || !d_ooff) return fail(kCudaError, "device allocation failed for the join");
  CK(cudaMemcpyAsync(d_woff, woff.data(), sizeof(int64_t) * nser, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_ooff, ooff.data(), sizeof(int64_t) * nser, cudaMemcpyHostToDevice, st));
  int launches = window_stat_launches((int)m);  // stats kernels
  for (int e = 4; e < 8; ++e) in.ev[e - 4] = p->s.ev[e];
  CK(cudaEventRecord(p->s.ev[1], st));
  TRY(run_join(in, d_bc, d_bj, ar, st, &er, &launches));
  CK(cudaEventRecord(p->s.ev[2], st));
  TRY(run_epilogue(d_bc, d_bj, in.rows.flag, nrows, p->d_segs, (int)p->segs.size(), m, d_woff, d_ooff, (int)nser,
                   p->cols.flag, p->cols.nwin, -1, d_val, d_idx, ar, st, &er));
  launches += 3;
  CK(cudaEventRecord(p->s.ev[3], st));
  CK(cudaEventSynchronize(p->s.ev[3]));
  {
    int hb = 0x7fffffff;
    CK(cudaMemcpy(&hb, d_bad, sizeof(int), cudaMemcpyDeviceToHost));
    if (hb != 0x7fffffff) return fail(kNonFiniteInput, "series contains a non-finite sample");  // series.hpp:87
  }
  float a = 0, b = 0;
  cudaEventElapsedTime(&a, p->s.ev[0], p->s.ev[3]);
  cudaEventElapsedTime(&b, p->s.ev[1], p->s.ev[2]);
  p->step_ms = a;
  p->join_ms = b;
  float kk = 0, hh = 0;
  cudaEventElapsedTime(&kk, p->s.ev[6], p->s.ev[7]);
  p->kernel_ms = kk;
  p->heads_ms = in.heads_used && cudaEventElapsedTime(&hh, p->s.ev[4], p->s.ev[5]) == cudaSuccess ? hh : 0.0;
  p->launches = launches;
  CK(cudaGetLastError());
  return kOk;
}

// TSD_VERBOSE: host time since t0 with the stream drained
static void verbose_phase(const char* what, cudaStream_t st, std::chrono::steady_clock::time_point t0) {
  static const bool on = getenv("TSD_VERBOSE") != nullptr;
  if (!on) return;
  cudaStreamSynchronize(st);
  fprintf(stderr, "[tsd] %s at %.2f ms\n", what,
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
}

int plan_join_host(tsd_dict_plan* p, const double* q, const size_t* q_len, size_t nser, double* val, int64_t* idx) {
  const auto t0 = std::chrono::steady_clock::now();
  int64_t N = 0, outn = 0;
  for (size_t k = 0; k < nser; ++k) {
    if ((size_t)p->m > q_len[k]) return fail(kWindowTooLarge, "window length exceeds series length");
    N += (int64_t)q_len[k];
    outn += (int64_t)q_len[k] - p->m + 1;
  }
  ThreadCtx& tc = tctx();
  if (int rc = tc.s.init()) return rc;
  tc.arena.reset();
  double* d_q = (double*)tc.arena.get(sizeof(double) * (N + 64));
  double* d_val = (double*)tc.arena.get(sizeof(double) * outn);
  int64_t* d_idx = (int64_t*)tc.arena.get(sizeof(int64_t) * outn);
  if (!d_q || !d_val || !d_idx) return fail(kCudaError, "device allocation failed for the query");
  cudaStream_t st = p->s.st;
  CK(cudaMemcpyAsync(d_q, q, sizeof(double) * N, cudaMemcpyHostToDevice, st));
  verbose_phase("query upload", st, t0);
  if (int rc = plan_join_dev(p, d_q, q_len, nser, d_val, d_idx, st)) return rc;
  verbose_phase("join", st, t0);
  if (getenv("TSD_VERBOSE"))
    fprintf(stderr, "[tsd] device: step %.2f ms, join %.2f ms, kernel %.2f ms, heads %.2f ms\n", p->step_ms, p->join_ms,
            p->kernel_ms, p->heads_ms);
  CK(cudaMemcpyAsync(val, d_val, sizeof(double) * outn, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(idx, d_idx, sizeof(int64_t) * outn, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  verbose_phase("profile download", st, t0);
  return kOk;
}

}  // namespace

extern "C" {

const char* tsd_last_error(void) { return t_err.c_str(); }

int tsd_last_join_timing(double* device_ms, double* kernel_ms, int* launches) {
  if (device_ms) *device_ms = t_last.device_ms;
  if (kernel_ms) *kernel_ms = t_last.kernel_ms;
  if (launches) *launches = t_last.launches;
  return kOk;
}
const char* tsd_status_name(int status) { return status_name(status); }
const char* tsd_build_info(void) {
  return "tsdict-b200: sm_100a FP64 row-band join, double-double window statistics (" __DATE__ ")";
}

int tsd_compute_stats(const double* x, size_t n, size_t m, double* means, double* stds, double* invn,
                      unsigned char* flat) {
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");  // series.hpp:85
  if (m > n) return fail(kWindowTooLarge, "window length exceeds series length");  // :86
  ThreadCtx& tc = tctx();
  if (int rc = tc.s.init()) return rc;
  tc.arena.reset();
  cudaStream_t st = tc.s.st;
  double* d_x = (double*)tc.arena.get(sizeof(double) * (n + 64));
  if (!d_x) return fail(kCudaError, "device allocation failed");
  CK(cudaMemcpyAsync(d_x, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  std::vector<Group> g;
  add_groups(g, 0, (int64_t)n, (int)m, 0, 0);
  WindowArrays w;
  Error er{0, ""};
  int bad = -1;
  TRY(compute_windows(d_x, (int64_t)n, (int)m, g, 1, w, tc.arena, st, &bad, &er));
  if (bad >= 0) return fail(kNonFiniteInput, "series contains a non-finite sample");  // :87
  const size_t cnt = n - m + 1;
  std::vector<uint8_t> fl(cnt);
  CK(cudaMemcpyAsync(means, w.mu, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(stds, w.sd, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(invn, w.invn, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(fl.data(), w.flag, cnt, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (size_t i = 0; i < cnt; ++i) flat[i] = (fl[i] & 2) ? 1 : 0;
  return kOk;
}

// shared by ab_join and self_join: one series of rows, one segment of columns
// stage 0: join + epilogue; 1: join only, val/idx receive the raw per-row
// (corr, column) partials of shard `shard` of `nshards`; 2: epilogue only,
// val/idx hold merged raw partials on input and the profile on output
// device != nullptr: a, val and idx are DEVICE pointers (self-join only),
// work is queued on *device (the caller's stream), nothing is copied through
// the host and the call returns without synchronising
static int single_join(const double* a, size_t na, const double* b, size_t nb, size_t m, int64_t excl, int precision,
                       double* val, int64_t* idx, bool force_sym = false, int stage = 0, int shard = 0,
                       int nshards = 1, const cudaStream_t* device = nullptr) {
  ThreadCtx& tc = tctx();
  if (int rc = tc.s.init()) return rc;
  tc.arena.reset();
  cudaStream_t st = device ? *device : tc.s.st;
  const bool self = (b == nullptr);
  const bool verbose = getenv("TSD_VERBOSE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {  // TSD_VERBOSE: host time since entry, stream drained
    if (!verbose) return;
    cudaStreamSynchronize(st);
    fprintf(stderr, "[tsd] %s at %.2f ms\n", what,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
  if (device && !self) return fail(kInvalidArgument, "device-resident joins are self-joins");
  double* d_a = device ? const_cast<double*>(a) : (double*)tc.arena.get(sizeof(double) * (na + 64));
  double* d_b = self ? d_a : (double*)tc.arena.get(sizeof(double) * (nb + 64));
  if (self) nb = na;
  if (!d_a || !d_b) return fail(kCudaError, "device allocation failed");
  if (!device) CK(cudaMemcpyAsync(d_a, a, sizeof(double) * na, cudaMemcpyHostToDevice, st));
  if (!self) CK(cudaMemcpyAsync(d_b, b, sizeof(double) * nb, cudaMemcpyHostToDevice, st));
  Error er{0, ""};
  JoinInputs in;
  in.force_sym = force_sym;
  in.shard = shard;
  in.nshards = nshards;
  for (int e = 4; e < 8; ++e) in.ev[e - 4] = tc.s.ev[e];
  CK(cudaEventRecord(tc.s.ev[0], st));
  std::vector<Group> ga;
  add_groups(ga, 0, (int64_t)na, (int)m, 0, 0);
  int bad = -1;
  TRY(compute_windows(d_a, (int64_t)na, (int)m, ga, 1, in.rows, tc.arena, st, &bad, &er));
  if (bad >= 0) return fail(kNonFiniteInput, "series contains a non-finite sample");
  if (self) {
    in.cols = in.rows;
  } else {
    std::vector<Group> gb;
    add_groups(gb, 0, (int64_t)nb, (int)m, 0, 0);
    TRY(compute_windows(d_b, (int64_t)nb, (int)m, gb, 1, in.cols, tc.arena, st, &bad, &er));
    if (bad >= 0) return fail(kNonFiniteInput, "series contains a non-finite sample");
  }
  phase("inputs + window statistics");
  in.xa = d_a;
  in.na = (int64_t)na;
  in.xb = d_b;
  in.nb = (int64_t)nb;
  in.segs = {SegDev{0, 0, (int32_t)(nb - m + 1), 0}};
  in.m = (int)m;
  in.excl = excl;
  in.precision = precision;
  const int64_t nrows = in.rows.nwin;
  // device mode: stage 1 writes the partials straight into val / idx, stage 2
  // reads the merged partials from them and writes the profile in place
  double* d_bc = device ? val : (double*)tc.arena.get(sizeof(double) * nrows);
  int64_t* d_bj = device ? idx : (int64_t*)tc.arena.get(sizeof(int64_t) * nrows);
  double* d_val = device ? val : (double*)tc.arena.get(sizeof(double) * nrows);
  int64_t* d_idx = device ? idx : (int64_t*)tc.arena.get(sizeof(int64_t) * nrows);
  SegDev* d_segs = (SegDev*)tc.arena.get(sizeof(SegDev));
  if (!d_bc || !d_bj || !d_val || !d_idx || !d_segs) return fail(kCudaError, "device allocation failed");
  CK(cudaMemcpyAsync(d_segs, in.segs.data(), sizeof(SegDev), cudaMemcpyHostToDevice, st));
  int launches = 0;
  if (stage == 2) {
    if (!device) {
      CK(cudaMemcpyAsync(d_bc, val, sizeof(double) * nrows, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(d_bj, idx, sizeof(int64_t) * nrows, cudaMemcpyHostToDevice, st));
    }
  } else {
    TRY(run_join(in, d_bc, d_bj, tc.arena, st, &er, &launches));
    if (self && getenv("TSD_PERFECT_SEED")) {  // development probe: rerun seeded from the final bests
      double* d_lb = (double*)tc.arena.get(sizeof(double) * nrows);
      if (!d_lb) return fail(kCudaError, "device allocation failed");
      CK(cudaMemcpyAsync(d_lb, d_bc, sizeof(double) * nrows, cudaMemcpyDeviceToDevice, st));
      in.seed_corr = d_lb;
      in.seed_margin = atof(getenv("TSD_PERFECT_SEED"));
      TRY(run_join(in, d_bc, d_bj, tc.arena, st, &er, &launches));
    }
  }
  phase("join");
  if (stage == 1 && device) return kOk;
  if (stage == 1) {
    CK(cudaMemcpyAsync(val, d_bc, sizeof(double) * nrows, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(idx, d_bj, sizeof(int64_t) * nrows, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return kOk;
  }
  if (device && stage == 2) {  // the epilogue reads and writes the same rows: stage the partials
    double* c2 = (double*)tc.arena.get(sizeof(double) * nrows);
    int64_t* j2 = (int64_t*)tc.arena.get(sizeof(int64_t) * nrows);
    if (!c2 || !j2) return fail(kCudaError, "device allocation failed");
    CK(cudaMemcpyAsync(c2, d_bc, sizeof(double) * nrows, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(j2, d_bj, sizeof(int64_t) * nrows, cudaMemcpyDeviceToDevice, st));
    d_bc = c2;
    d_bj = j2;
  }
  TRY(run_epilogue(d_bc, d_bj, in.rows.flag, nrows, d_segs, 1, (int)m, nullptr, nullptr, 1, in.cols.flag, in.cols.nwin,
                   excl, d_val, d_idx, tc.arena, st, &er));
  if (device) return kOk;
  CK(cudaEventRecord(tc.s.ev[1], st));
  CK(cudaMemcpyAsync(val, d_val, sizeof(double) * nrows, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(idx, d_idx, sizeof(int64_t) * nrows, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (stage == 0) {
    float dm = 0.f, km = 0.f;
    cudaEventElapsedTime(&dm, tc.s.ev[0], tc.s.ev[1]);
    if (cudaEventElapsedTime(&km, tc.s.ev[6], tc.s.ev[7]) != cudaSuccess) km = 0.f;
    t_last = LastJoin{dm, km, launches + 3 + window_stat_launches((int)m)};
  }
  phase("epilogue + outputs");
  return kOk;
}

int tsd_ab_join(const double* a, size_t na, const double* b, size_t nb, size_t m, int precision, double* val,
                int64_t* idx) {
  if (m >= 2 && (na < m || nb < m)) return fail(kSeriesTooShort, "ab-join needs both series at least m long");  // profiles.hpp:307-309
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");  // series.hpp:85 via :310
  if (precision != TSD_FP64 && precision != TSD_FP32) return fail(kInvalidArgument, "unknown precision");
  if (nb > kMaxColumnSamples) return fail(kInvalidArgument, "target series exceeds 2^31 samples");
  return single_join(a, na, b, nb, m, -1, precision, val, idx);
}

int tsd_self_join(const double* t, size_t n, size_t m, size_t excl, int precision, double* val, int64_t* idx) {
  if (m >= 2 && n < 2 * m) return fail(kSeriesTooShort, "self-join needs n >= 2m");  // profiles.hpp:268-270
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");      // via :271
  if (precision != TSD_FP64 && precision != TSD_FP32) return fail(kInvalidArgument, "unknown precision");
  if (n > kMaxColumnSamples) return fail(kInvalidArgument, "series exceeds 2^31 samples");
  const int64_t e = excl == TSD_EXCL_DEFAULT ? (int64_t)(m / 2) : (int64_t)excl;  // :273
  return single_join(t, n, nullptr, 0, m, e, precision, val, idx);
}

int tsd_self_join_partial(const double* t, size_t n, size_t m, size_t excl, size_t shard, size_t nshards,
                          double* corr, int64_t* col) {
  if (m >= 2 && n < 2 * m) return fail(kSeriesTooShort, "self-join needs n >= 2m");
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");
  if (nshards == 0 || shard >= nshards) return fail(kInvalidArgument, "shard index out of range");
  if (n > kMaxColumnSamples) return fail(kInvalidArgument, "series exceeds 2^31 samples");
  const int64_t e = excl == TSD_EXCL_DEFAULT ? (int64_t)(m / 2) : (int64_t)excl;
  return single_join(t, n, nullptr, 0, m, e, TSD_FP64, corr, col, true, 1, (int)shard, (int)nshards);
}

int tsd_profile_merge(const double* corr_parts, const int64_t* col_parts, size_t nparts, size_t cnt, double* corr,
                      int64_t* col) {
  for (size_t i = 0; i < cnt; ++i) {  // acc_merge (profiles.hpp:79-85): larger corr, then lower index
    double bc = -2.0;
    int64_t bj = -1;
    for (size_t p = 0; p < nparts; ++p) {
      const double c = corr_parts[p * cnt + i];
      const int64_t j = col_parts[p * cnt + i];
      if (j >= 0 && (bj < 0 || c > bc || (c == bc && j < bj))) {
        bc = c;
        bj = j;
      }
    }
    corr[i] = bc;
    col[i] = bj;
  }
  return kOk;
}

int tsd_self_join_finish(const double* t, size_t n, size_t m, size_t excl, const double* corr, const int64_t* col,
                         double* val, int64_t* idx) {
  if (m >= 2 && n < 2 * m) return fail(kSeriesTooShort, "self-join needs n >= 2m");
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");
  const int64_t e = excl == TSD_EXCL_DEFAULT ? (int64_t)(m / 2) : (int64_t)excl;
  const size_t cnt = n - m + 1;
  std::copy(corr, corr + cnt, val);
  std::copy(col, col + cnt, idx);
  return single_join(t, n, nullptr, 0, m, e, TSD_FP64, val, idx, true, 2);
}

int tsd_self_join_partial_device(const double* d_t, size_t n, size_t m, size_t excl, size_t shard, size_t nshards,
                                 double* d_corr, int64_t* d_col, void* stream) {
  if (m >= 2 && n < 2 * m) return fail(kSeriesTooShort, "self-join needs n >= 2m");
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");
  if (nshards == 0 || shard >= nshards) return fail(kInvalidArgument, "shard index out of range");
  if (n > kMaxColumnSamples) return fail(kInvalidArgument, "series exceeds 2^31 samples");
  const int64_t e = excl == TSD_EXCL_DEFAULT ? (int64_t)(m / 2) : (int64_t)excl;
  const cudaStream_t st = (cudaStream_t)stream;
  return single_join(d_t, n, nullptr, 0, m, e, TSD_FP64, d_corr, d_col, true, 1, (int)shard, (int)nshards, &st);
}

int tsd_profile_merge_device(const double* d_corr_parts, const int64_t* d_col_parts, size_t nparts, size_t cnt,
                             double* d_corr, int64_t* d_col, void* stream) {
  if (nparts == 0) return fail(kInvalidArgument, "no partials");
  if (profile_merge_device(d_corr_parts, d_col_parts, (int)nparts, (int64_t)cnt, d_corr, d_col,
                           (cudaStream_t)stream) != kOk)
    return fail(kCudaError, std::string("partial merge: ") + cudaGetErrorString(cudaGetLastError()));
  return kOk;
}

int tsd_self_join_finish_device(const double* d_t, size_t n, size_t m, size_t excl, double* d_val, int64_t* d_idx,
                                void* stream) {
  if (m >= 2 && n < 2 * m) return fail(kSeriesTooShort, "self-join needs n >= 2m");
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");
  const int64_t e = excl == TSD_EXCL_DEFAULT ? (int64_t)(m / 2) : (int64_t)excl;
  const cudaStream_t st = (cudaStream_t)stream;
  return single_join(d_t, n, nullptr, 0, m, e, TSD_FP64, d_val, d_idx, true, 2, 0, 1, &st);
}

int tsd_dict_shard_rows(size_t nq, size_t m, size_t shard, size_t nshards, size_t* row_lo, size_t* row_hi) {
  // whole 16384-window query blocks (dictionary.hpp:175-180) per shard, so a
  // shard's window statistics group exactly as in the unsharded join
  if (nshards == 0 || shard >= nshards) return fail(kInvalidArgument, "shard index out of range");
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");
  if (m > nq) return fail(kWindowTooLarge, "window length exceeds series length");
  const size_t cnt = nq - m + 1, block = 16384, nb = (cnt + block - 1) / block;
  const size_t b0 = nb * shard / nshards, b1 = nb * (shard + 1) / nshards;
  *row_lo = std::min(cnt, b0 * block);
  *row_hi = std::min(cnt, b1 * block);
  return kOk;
}

int tsd_dict_join(const double* q, size_t nq, const double* seg_vals, const size_t* seg_len, const size_t* seg_start,
                  size_t nseg, size_t m, int precision, double* val, int64_t* idx) {
  return tsd_dict_join_batched(q, &nq, 1, seg_vals, seg_len, seg_start, nseg, m, precision, val, idx);
}

int tsd_dict_join_batched(const double* q_vals, const size_t* q_len, size_t nseries, const double* seg_vals,
                          const size_t* seg_len, const size_t* seg_start, size_t nseg, size_t m, int precision,
                          double* val, int64_t* idx) {
  if (int rc = validate_dict(seg_len, nseg, m)) return rc;  // dictionary.hpp:151-157
  for (size_t k = 0; k < nseries; ++k)
    if (m > q_len[k]) return fail(kWindowTooLarge, "window length exceeds series length");  // :158
  if (precision != TSD_FP64 && precision != TSD_FP32) return fail(kInvalidArgument, "unknown precision");
  // one cached plan per host thread: its device arenas are reused across
  // calls, so repeated host-API joins do not pay cudaMalloc
  thread_local tsd_dict_plan tp;
  tp.dict_arena.reset();
  tp.work_arena.reset();
  if (int rc = plan_build(&tp, seg_vals, seg_len, seg_start, nseg, m, precision)) return rc;
  return plan_join_host(&tp, q_vals, q_len, nseries, val, idx);
}

int tsd_compute_e_max(const double* t, size_t n, size_t source_length, const double* seg_vals, const size_t* seg_len,
                      const size_t* seg_start, size_t nseg, size_t m, double* e_max) {
  if (source_length != n)  // dictionary.hpp:248-250
    return fail(kSourceMismatch, "dictionary was learned from a series of different length");
  if (int rc = validate_dict(seg_len, nseg, m)) return rc;
  if (m > n) return fail(kWindowTooLarge, "window length exceeds series length");
  const size_t cnt = n - m + 1;
  std::vector<double> v(cnt);
  std::vector<int64_t> ix(cnt);
  if (int rc = tsd_dict_join(t, n, seg_vals, seg_len, seg_start, nseg, m, TSD_FP64, v.data(), ix.data())) return rc;
  double worst = 0.0;  // :252-253
  for (double x : v) worst = std::max(worst, x);
  *e_max = worst;
  return kOk;
}

int tsd_dict_plan_create(const double* seg_vals, const size_t* seg_len, const size_t* seg_start, size_t nseg, size_t m,
                         int precision, tsd_dict_plan** plan) {
  if (!plan) return fail(kInvalidArgument, "null plan pointer");
  *plan = nullptr;
  if (int rc = validate_dict(seg_len, nseg, m)) return rc;
  if (precision != TSD_FP64 && precision != TSD_FP32) return fail(kInvalidArgument, "unknown precision");
  tsd_dict_plan* p = new tsd_dict_plan();
  if (int rc = plan_build(p, seg_vals, seg_len, seg_start, nseg, m, precision)) {
    std::string keep = t_err;
    delete p;
    t_err = keep;
    return rc;
  }
  *plan = p;
  return kOk;
}

int tsd_dict_plan_join_device(tsd_dict_plan* plan, const double* d_q, const size_t* q_len, size_t nseries,
                              double* d_val, int64_t* d_idx, void* stream) {
  if (!plan) return fail(kInvalidArgument, "null plan");
  return plan_join_dev(plan, d_q, q_len, nseries, d_val, d_idx, (cudaStream_t)stream);
}

int tsd_dict_plan_join(tsd_dict_plan* plan, const double* q, const size_t* q_len, size_t nseries, double* val,
                       int64_t* idx) {
  if (!plan) return fail(kInvalidArgument, "null plan");
  return plan_join_host(plan, q, q_len, nseries, val, idx);
}

// ---------------------------------------------------------------------------
// greedy dictionary learning (dictionary.hpp:259-328)
// ---------------------------------------------------------------------------
namespace {
struct Kahan {  // series.hpp:49-60
  double sum = 0.0, comp = 0.0;
  void add(double x) {
    const double y = x - comp;
    const double t = sum + y;
    comp = (t - sum) - y;
    sum = t;
  }
};
double constancy_threshold_h(double max_abs) { return 1e-8 * std::max(1.0, max_abs); }  // series.hpp:75-77
double corr_to_dist_h(double rho, size_t m) {                                            // series.hpp:153-161
  if (rho > 1.0) rho = 1.0;
  if (rho < -1.0) rho = -1.0;
  double d = std::sqrt(2.0 * (double)m * (1.0 - rho));
  const double dmax = 2.0 * std::sqrt((double)m);
  if (d < 0.0) d = 0.0;
  if (d > dmax) d = dmax;
  return d;
}
// znorm_distance (series.hpp:166-203): the exact origin entry of MASS
double znorm_distance_h(const double* a, const double* b, size_t m) {
  double max_abs = 0.0;
  Kahan sa, sb;
  for (size_t i = 0; i < m; ++i) {
    sa.add(a[i]);
    sb.add(b[i]);
    max_abs = std::max({max_abs, std::fabs(a[i]), std::fabs(b[i])});
  }
  const double md = (double)m, mu_a = sa.sum / md, mu_b = sb.sum / md;
  Kahan va, vb, cov;
  for (size_t i = 0; i < m; ++i) {
    const double da = a[i] - mu_a, db = b[i] - mu_b;
    va.add(da * da);
    vb.add(db * db);
    cov.add(da * db);
  }
  const double sd_a = std::sqrt(std::max(0.0, va.sum / md)), sd_b = std::sqrt(std::max(0.0, vb.sum / md));
  const double eps = constancy_threshold_h(max_abs);
  const bool fa = sd_a < eps, fb = sd_b < eps;
  if (fa && fb) return 0.0;
  if (fa || fb) return std::sqrt(2.0 * md);
  return corr_to_dist_h(cov.sum / (md * (sd_a * sd_b)), m);
}
typedef std::pair<size_t, size_t> Interval;
Interval context_interval_h(size_t j, size_t m, double k, size_t n) {  // dictionary.hpp:78-84
  const size_t total = (size_t)(k * (double)m + 1e-9);
  const size_t before = total / 2;
  return {j >= before ? j - before : 0, std::min(n, j + m + (total - before))};
}
std::vector<Interval> merge_intervals_h(std::vector<Interval> iv) {  // :87-98
  std::sort(iv.begin(), iv.end());
  std::vector<Interval> out;
  for (const auto& x : iv) {
    if (!out.empty() && x.first <= out.back().second)
      out.back().second = std::max(out.back().second, x.second);
    else
      out.push_back(x);
  }
  return out;
}
}  // namespace

int tsd_learn_dictionary(const double* t, size_t n, size_t m, double k, int rule, double rule_value,
                         size_t max_iterations, const double* profile, size_t* seg_start, size_t* seg_len,
                         double* seg_vals, size_t* nseg, size_t* core_starts, size_t* ncores, double* e_max,
                         double* space_saving, int* no_progress) {
  // validate_learn_config (dictionary.hpp:120-141), then :267
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");
  if (!(k >= 0.0)) return fail(kInvalidArgument, "context factor k must be non-negative");
  if (rule != TSD_RULE_SPACE_SAVING && rule != TSD_RULE_SAMPLE_BUDGET && rule != TSD_RULE_ERROR_TARGET)
    return fail(kInvalidArgument, "exactly one stop rule must be set");
  if (rule == TSD_RULE_SPACE_SAVING && (rule_value < 0.0 || rule_value >= 1.0))
    return fail(kInvalidArgument, "space saving target must lie in [0, 1)");
  if (rule == TSD_RULE_SAMPLE_BUDGET && !(rule_value >= 1.0))
    return fail(kInvalidArgument, "sample budget must be positive");
  if (rule == TSD_RULE_ERROR_TARGET && rule_value < 0.0)
    return fail(kInvalidArgument, "error target must be non-negative");
  if (max_iterations == 0) return fail(kInvalidArgument, "iteration cap must be positive");
  if (n < 2 * m) return fail(kSeriesTooShort, "dictionary learning needs n >= 2m");
  const size_t cnt = n - m + 1, excl = m / 2;
  // the exact self-join profile P_B (dictionary.hpp:325-327)
  std::vector<double> P(cnt);
  if (profile) {
    std::copy(profile, profile + cnt, P.begin());
  } else {
    // symmetric sweep: a pair's two rows carry the bitwise-identical value, so
    // argmin ties (mutual nearest neighbours) resolve as the reference's do
    std::vector<int64_t> ix(cnt);
    if (int rc = single_join(t, n, nullptr, 0, m, (int64_t)(m / 2), TSD_FP64, P.data(), ix.data(), true)) return rc;
  }
  ThreadCtx& tc = tctx();
  if (int rc = tc.s.init()) return rc;
  cudaStream_t st = tc.s.st;
  Arena ar;  // the loop's own buffers (tsd_* calls below reset the thread arena)
  double* d_x = (double*)ar.get(sizeof(double) * (n + 64));
  double* d_P = (double*)ar.get(sizeof(double) * cnt);
  double* d_S = (double*)ar.get(sizeof(double) * cnt);
  double* d_qc = (double*)ar.get(sizeof(double) * m);
  uint8_t* d_mask = (uint8_t*)ar.get(cnt);
  void* d_scr = ar.get(learn_scratch_bytes());
  if (!d_x || !d_P || !d_S || !d_qc || !d_mask || !d_scr) return fail(kCudaError, "device allocation failed");
  CK(cudaMemcpyAsync(d_x, t, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_P, P.data(), sizeof(double) * cnt, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(d_S, 0, sizeof(double) * cnt, st));
  CK(cudaMemsetAsync(d_mask, 0, cnt, st));
  std::vector<Group> g;
  add_groups(g, 0, (int64_t)n, (int)m, 0, 0);
  WindowArrays w;
  Error er{0, ""};
  int bad = -1;
  TRY(compute_windows(d_x, (int64_t)n, (int)m, g, 1, w, ar, st, &bad, &er));
  if (bad >= 0) return fail(kNonFiniteInput, "series contains a non-finite sample");
  std::vector<uint8_t> hflag(cnt);
  CK(cudaMemcpyAsync(hflag.data(), w.flag, cnt, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));

  const bool budget_rule = rule != TSD_RULE_ERROR_TARGET;
  const double need = rule == TSD_RULE_SAMPLE_BUDGET ? rule_value : (1.0 - rule_value) * (double)n - 1e-6;  // :244-247
  std::vector<Interval> chosen, merged;
  std::vector<size_t> cores;
  size_t stored = 0;
  bool s_init = false, stall = false;
  std::vector<double> qc(m);
  for (size_t iter = 0;; ++iter) {
    if (iter >= max_iterations)
      return fail(kIterationCapExceeded, "iteration cap reached before the stop rule fired");
    double bv = 0.0;
    int64_t j = -1;
    if (learn_argmin(d_P, d_S, d_mask, (int64_t)cnt, d_scr, &bv, &j, st) != kOk)
      return fail(kCudaError, std::string("learning argmin: ") + cudaGetErrorString(cudaGetLastError()));
    if (j < 0) {
      stall = true;
      break;
    }
    // select_state::take (dictionary.hpp:213-224)
    cores.push_back((size_t)j);
    chosen.push_back(context_interval_h((size_t)j, m, k, n));
    merged = merge_intervals_h(chosen);
    stored = 0;
    for (const auto& iv : merged) stored += iv.second - iv.first;
    const size_t lo = (size_t)j >= excl ? (size_t)j - excl : 0, hi = std::min(cnt, (size_t)j + excl + 1);
    CK(cudaMemsetAsync(d_mask + lo, 1, hi - lo, st));
    if (budget_rule && (double)stored >= need) break;
    // distance profile of window j (profiles.hpp:186-260) folded into S
    const double* Q = t + j;
    double max_abs = 0.0;
    Kahan qs;
    for (size_t i = 0; i < m; ++i) {
      qs.add(Q[i]);
      max_abs = std::max(max_abs, std::fabs(Q[i]));
    }
    const double md = (double)m, mu_q = qs.sum / md;
    Kahan qv;
    for (size_t i = 0; i < m; ++i) qv.add((Q[i] - mu_q) * (Q[i] - mu_q));
    const double sd_q = std::sqrt(std::max(0.0, qv.sum / md));
    const bool cq = sd_q < constancy_threshold_h(max_abs);
    const double invn_q = cq ? 0.0 : 1.0 / (sd_q * std::sqrt(md));
    for (size_t i = 0; i < m; ++i) qc[i] = Q[i] - mu_q;
    const double origin = (hflag[j] & 2) ? 0.0 : znorm_distance_h(Q, t + j, m);
    CK(cudaMemcpyAsync(d_qc, qc.data(), sizeof(double) * m, cudaMemcpyHostToDevice, st));
    if (learn_dprof_fold(d_x, w, (int)m, d_qc, invn_q, cq, j, origin, !s_init, d_S, st) != kOk)
      return fail(kCudaError, std::string("distance profile: ") + cudaGetErrorString(cudaGetLastError()));
    s_init = true;
    if (rule == TSD_RULE_ERROR_TARGET) {  // :305-309
      double worst = 0.0;
      if (learn_max(d_S, (int64_t)cnt, d_scr, &worst, st) != kOk)
        return fail(kCudaError, std::string("learning max: ") + cudaGetErrorString(cudaGetLastError()));
      if (worst <= rule_value) break;
    }
  }
  // finish_dictionary (dictionary.hpp:226-237)
  size_t off = 0;
  for (size_t s = 0; s < merged.size(); ++s) {
    seg_start[s] = merged[s].first;
    seg_len[s] = merged[s].second - merged[s].first;
    std::copy(t + merged[s].first, t + merged[s].second, seg_vals + off);
    off += seg_len[s];
  }
  *nseg = merged.size();
  for (size_t c = 0; c < cores.size(); ++c) core_starts[c] = cores[c];
  *ncores = cores.size();
  *space_saving = 1.0 - (double)stored / (double)n;
  *no_progress = stall ? 1 : 0;
  // D.e_max = compute_e_max(D, T_B) (:319)
  return tsd_compute_e_max(t, n, n, seg_vals, seg_len, seg_start, merged.size(), m, e_max);
}

int tsd_find_discords_device(const double* d_values, size_t cnt, size_t m, double e_max, size_t top_k,
                             size_t* start, double* score, int* certified, size_t* count, void* stream) {
  if (cnt == 0) return fail(kEmptyProfile, "profile has no entries");       // dict_join.hpp:55
  if (e_max < 0.0) return fail(kInvalidArgument, "e_max must be non-negative");  // :56
  ThreadCtx& tc = tctx();
  if (int rc = tc.s.init()) return rc;
  cudaStream_t st = stream ? (cudaStream_t)stream : tc.s.st;
  Arena ar;
  uint8_t* d_sup = (uint8_t*)ar.get(cnt);
  void* d_scr = ar.get(learn_scratch_bytes());
  if (!d_sup || !d_scr) return fail(kCudaError, "device allocation failed");
  std::vector<int64_t> at;
  std::vector<double> sc;
  const int64_t want = (int64_t)std::max<size_t>(top_k, 2);  // runner-up for the gap test (:75)
  if (discord_peaks(d_values, (int64_t)cnt, (int)m, want, d_sup, d_scr, at, sc, st) != kOk)
    return fail(kCudaError, std::string("discord peaks: ") + cudaGetErrorString(cudaGetLastError()));
  const bool cert = !at.empty() && (at.size() < 2 || sc[0] - sc[1] > e_max);  // :88-91
  const size_t k = std::min(at.size(), top_k);
  for (size_t i = 0; i < k; ++i) {
    start[i] = (size_t)at[i];
    score[i] = sc[i];
    certified[i] = (i == 0 && cert) ? 1 : 0;
  }
  *count = k;
  return kOk;
}

int tsd_find_discords(const double* values, size_t cnt, size_t m, double e_max, size_t top_k, size_t* start,
                      double* score, int* certified, size_t* count) {
  if (cnt == 0) return fail(kEmptyProfile, "profile has no entries");
  if (e_max < 0.0) return fail(kInvalidArgument, "e_max must be non-negative");
  ThreadCtx& tc = tctx();
  if (int rc = tc.s.init()) return rc;
  Arena ar;
  double* d_v = (double*)ar.get(sizeof(double) * cnt);
  if (!d_v) return fail(kCudaError, "device allocation failed");
  CK(cudaMemcpyAsync(d_v, values, sizeof(double) * cnt, cudaMemcpyHostToDevice, tc.s.st));
  return tsd_find_discords_device(d_v, cnt, m, e_max, top_k, start, score, certified, count, tc.s.st);
}

// ---------------------------------------------------------------------------
// distance profiles (profiles.hpp:164-260)
// ---------------------------------------------------------------------------
namespace {
// the query's moments exactly as znorm_distance / distance_profile_mass form
// them (series.hpp:172-190, profiles.hpp:206-224)
QueryMoments query_moments(const double* q, size_t m) {
  QueryMoments qm;
  Kahan s;
  for (size_t i = 0; i < m; ++i) {
    s.add(q[i]);
    qm.max_abs = std::max(qm.max_abs, std::fabs(q[i]));
  }
  const double md = (double)m;
  qm.mu = s.sum / md;
  Kahan v;
  for (size_t i = 0; i < m; ++i) v.add((q[i] - qm.mu) * (q[i] - qm.mu));
  qm.var_sum = v.sum;
  const double sd = std::sqrt(std::max(0.0, v.sum / md));
  qm.constant = sd < constancy_threshold_h(qm.max_abs);
  qm.invn = qm.constant ? 0.0 : 1.0 / (sd * std::sqrt(md));
  return qm;
}

int dprofile(const double* t, size_t n, const double* q, size_t m, const double* means, const double* invn,
             const unsigned char* cmask, size_t origin, double* out) {
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");
  if (m > n) return fail(kWindowTooLarge, "window length exceeds series length");
  if (means)  // distance_profile_mass: profiles.hpp:206-209
    for (size_t i = 0; i < m; ++i)
      if (!std::isfinite(q[i])) return fail(kNonFiniteInput, "query contains a non-finite sample");
  const size_t cnt = n - m + 1;
  ThreadCtx& tc = tctx();
  if (int rc = tc.s.init()) return rc;
  tc.arena.reset();
  cudaStream_t st = tc.s.st;
  double* d_x = (double*)tc.arena.get(sizeof(double) * (n + 64));
  double* d_q = (double*)tc.arena.get(sizeof(double) * m);
  double* d_out = (double*)tc.arena.get(sizeof(double) * cnt);
  double* d_mu = means ? (double*)tc.arena.get(sizeof(double) * cnt) : nullptr;
  double* d_iv = means ? (double*)tc.arena.get(sizeof(double) * cnt) : nullptr;
  uint8_t* d_cm = means ? (uint8_t*)tc.arena.get(cnt) : nullptr;
  if (!d_x || !d_q || !d_out || (means && (!d_mu || !d_iv || !d_cm)))
    return fail(kCudaError, "device allocation failed");
  CK(cudaMemcpyAsync(d_x, t, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_q, q, sizeof(double) * m, cudaMemcpyHostToDevice, st));
  if (means) {
    CK(cudaMemcpyAsync(d_mu, means, sizeof(double) * cnt, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_iv, invn, sizeof(double) * cnt, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_cm, cmask, cnt, cudaMemcpyHostToDevice, st));
  }
  const QueryMoments qm = query_moments(q, m);
  const int64_t org = (origin == TSD_NO_ORIGIN || origin >= cnt) ? -1 : (int64_t)origin;
  if (distance_profile_device(d_x, (int64_t)n, d_q, (int)m, qm, d_mu, d_iv, d_cm, org, d_out, st) != kOk)
    return fail(kCudaError, std::string("distance profile: ") + cudaGetErrorString(cudaGetLastError()));
  CK(cudaMemcpyAsync(out, d_out, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return kOk;
}
}  // namespace

int tsd_distance_profile_naive(const double* t, size_t n, const double* q, size_t m, double* out) {
  return dprofile(t, n, q, m, nullptr, nullptr, nullptr, TSD_NO_ORIGIN, out);
}

int tsd_distance_profile_mass(const double* t, size_t n, const double* q, size_t m, const double* means,
                              const double* invn, const unsigned char* constant_mask, size_t origin, double* out) {
  if (!means || !invn || !constant_mask) return fail(kInvalidArgument, "window statistics required");
  return dprofile(t, n, q, m, means, invn, constant_mask, origin, out);
}

int tsd_dict_plan_destroy(tsd_dict_plan* plan) {
  delete plan;
  return kOk;
}

int tsd_dict_plan_last_kernel_timing(tsd_dict_plan* plan, double* join_kernel_ms, double* heads_ms) {
  if (!plan) return fail(kInvalidArgument, "null plan");
  if (join_kernel_ms) *join_kernel_ms = plan->kernel_ms;
  if (heads_ms) *heads_ms = plan->heads_ms;
  return kOk;
}

int tsd_dict_plan_last_timing(tsd_dict_plan* plan, double* step_ms, double* join_ms, int* launches) {
  if (!plan) return fail(kInvalidArgument, "null plan");
  if (step_ms) *step_ms = plan->step_ms;
  if (join_ms) *join_ms = plan->join_ms;
  if (launches) *launches = plan->launches;
  return kOk;
}

}  // extern "C"

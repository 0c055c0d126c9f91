// capi.cu -- the extern "C" boundary (include/tsdict_cuda.h).
//
// Validation order and error codes reproduce the reference functions each
// entry point replaces (cited per function); device work runs on a
// per-thread stream with a per-thread scratch arena (thread-safe,
// re-entrant). There is no CPU fallback: when no usable CUDA device exists
// every entry point fails with TSD_CUDA_ERROR.
#include <algorithm>
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

int validate_dict(const size_t* seg_len, size_t nseg, size_t m) {  // dictionary.hpp:151-157
  if (nseg == 0) return fail(kEmptyDictionary, "dictionary has no segments");
  for (size_t s = 0; s < nseg; ++s)
    if (seg_len[s] < m) return fail(kWindowMismatch, "dictionary segment shorter than the window length");
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");
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
  TRY(compute_windows(d_q, N, m, groups, (int)nser, in.rows, ar, st, &bad, &er));
  if (bad >= 0 || p->dict_nonfinite) return fail(kNonFiniteInput, "series contains a non-finite sample");
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
  int launches = 5;  // stats kernels
  for (int e = 4; e < 8; ++e) in.ev[e - 4] = p->s.ev[e];
  CK(cudaEventRecord(p->s.ev[1], st));
  TRY(run_join(in, d_bc, d_bj, ar, st, &er, &launches));
  CK(cudaEventRecord(p->s.ev[2], st));
  TRY(run_epilogue(d_bc, d_bj, in.rows.flag, nrows, p->d_segs, (int)p->segs.size(), m, d_woff, d_ooff, (int)nser,
                   p->cols.flag, p->cols.nwin, -1, d_val, d_idx, ar, st, &er));
  launches += 3;
  CK(cudaEventRecord(p->s.ev[3], st));
  CK(cudaEventSynchronize(p->s.ev[3]));
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

int plan_join_host(tsd_dict_plan* p, const double* q, const size_t* q_len, size_t nser, double* val, int64_t* idx) {
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
  if (int rc = plan_join_dev(p, d_q, q_len, nser, d_val, d_idx, st)) return rc;
  CK(cudaMemcpyAsync(val, d_val, sizeof(double) * outn, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(idx, d_idx, sizeof(int64_t) * outn, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return kOk;
}

}  // namespace

extern "C" {

const char* tsd_last_error(void) { return t_err.c_str(); }
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
static int single_join(const double* a, size_t na, const double* b, size_t nb, size_t m, int64_t excl, int precision,
                       double* val, int64_t* idx) {
  ThreadCtx& tc = tctx();
  if (int rc = tc.s.init()) return rc;
  tc.arena.reset();
  cudaStream_t st = tc.s.st;
  const bool self = (b == nullptr);
  double* d_a = (double*)tc.arena.get(sizeof(double) * (na + 64));
  double* d_b = self ? d_a : (double*)tc.arena.get(sizeof(double) * (nb + 64));
  if (self) nb = na;
  if (!d_a || !d_b) return fail(kCudaError, "device allocation failed");
  CK(cudaMemcpyAsync(d_a, a, sizeof(double) * na, cudaMemcpyHostToDevice, st));
  if (!self) CK(cudaMemcpyAsync(d_b, b, sizeof(double) * nb, cudaMemcpyHostToDevice, st));
  Error er{0, ""};
  JoinInputs in;
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
  in.xa = d_a;
  in.na = (int64_t)na;
  in.xb = d_b;
  in.nb = (int64_t)nb;
  in.segs = {SegDev{0, 0, (int32_t)(nb - m + 1), 0}};
  in.m = (int)m;
  in.excl = excl;
  in.precision = precision;
  const int64_t nrows = in.rows.nwin;
  double* d_bc = (double*)tc.arena.get(sizeof(double) * nrows);
  int64_t* d_bj = (int64_t*)tc.arena.get(sizeof(int64_t) * nrows);
  double* d_val = (double*)tc.arena.get(sizeof(double) * nrows);
  int64_t* d_idx = (int64_t*)tc.arena.get(sizeof(int64_t) * nrows);
  SegDev* d_segs = (SegDev*)tc.arena.get(sizeof(SegDev));
  if (!d_bc || !d_bj || !d_val || !d_idx || !d_segs) return fail(kCudaError, "device allocation failed");
  CK(cudaMemcpyAsync(d_segs, in.segs.data(), sizeof(SegDev), cudaMemcpyHostToDevice, st));
  int launches = 0;
  TRY(run_join(in, d_bc, d_bj, tc.arena, st, &er, &launches));
  TRY(run_epilogue(d_bc, d_bj, in.rows.flag, nrows, d_segs, 1, (int)m, nullptr, nullptr, 1, in.cols.flag, in.cols.nwin,
                   excl, d_val, d_idx, tc.arena, st, &er));
  CK(cudaMemcpyAsync(val, d_val, sizeof(double) * nrows, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(idx, d_idx, sizeof(int64_t) * nrows, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return kOk;
}

int tsd_ab_join(const double* a, size_t na, const double* b, size_t nb, size_t m, int precision, double* val,
                int64_t* idx) {
  if (m >= 2 && (na < m || nb < m)) return fail(kSeriesTooShort, "ab-join needs both series at least m long");  // profiles.hpp:307-309
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");  // series.hpp:85 via :310
  if (precision != TSD_FP64 && precision != TSD_FP32) return fail(kInvalidArgument, "unknown precision");
  return single_join(a, na, b, nb, m, -1, precision, val, idx);
}

int tsd_self_join(const double* t, size_t n, size_t m, size_t excl, int precision, double* val, int64_t* idx) {
  if (m >= 2 && n < 2 * m) return fail(kSeriesTooShort, "self-join needs n >= 2m");  // profiles.hpp:268-270
  if (m < 2) return fail(kWindowTooSmall, "window length must be at least 2");      // via :271
  if (precision != TSD_FP64 && precision != TSD_FP32) return fail(kInvalidArgument, "unknown precision");
  const int64_t e = excl == TSD_EXCL_DEFAULT ? (int64_t)(m / 2) : (int64_t)excl;  // :273
  return single_join(t, n, nullptr, 0, m, e, precision, val, idx);
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

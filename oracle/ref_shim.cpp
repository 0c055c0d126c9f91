// ref_shim.cpp -- ORACLE BUILD ONLY (test infrastructure).
//
// Compiles the UNMODIFIED reference headers where they lie under
// /root/reference/proj (include/tsdict/*.hpp, tests/oracles.hpp,
// tests/synth.hpp) into oracle/_ref/libtsdict_ref.so and exposes their
// hot-path entry points through a C ABI for tests/golden/make_golden.py and
// for bench.py's CPU baseline ("kind": "reference"). Nothing from the
// reference is copied into this repository; oracle/Makefile points the
// include path at /root/reference and writes only into oracle/_ref/.
// <unsupported/Eigen/FFT> comes from oracle/standin (used by MASS only).
//
// Status codes: 0 ok, else 1 + tsdict::errc ordinal.
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "oracles.hpp"  // /root/reference/proj/tests/oracles.hpp
#include "synth.hpp"    // /root/reference/proj/tests/synth.hpp
#include "tsdict/dict_join.hpp"
#include "tsdict/dictionary.hpp"
#include "tsdict/profiles.hpp"
#include "tsdict/series.hpp"

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const tsdict::error& e) {
    return 1 + static_cast<int>(e.code());
  } catch (...) {
    return 100;
  }
}

void emit(const tsdict::MatrixProfile& p, double* val, int64_t* idx) {
  std::memcpy(val, p.values.data(), p.values.size() * sizeof(double));
  std::memcpy(idx, p.indices.data(), p.indices.size() * sizeof(int64_t));
}

tsdict::TimeSeries ts(const double* x, size_t n) { return tsdict::TimeSeries{std::vector<double>(x, x + n)}; }

}  // namespace

extern "C" {

int tsdr_compute_stats(const double* x, size_t n, size_t m, double* means, double* stds, double* invn,
                       unsigned char* flat) {
  return guarded([&] {
    const auto st = tsdict::compute_stats(ts(x, n), m);
    std::memcpy(means, st.means.data(), st.count() * sizeof(double));
    std::memcpy(stds, st.stds.data(), st.count() * sizeof(double));
    std::memcpy(invn, st.invn.data(), st.count() * sizeof(double));
    std::memcpy(flat, st.constant_mask.data(), st.count());
  });
}

int tsdr_ab_join(const double* a, size_t na, const double* b, size_t nb, size_t m, unsigned threads, double* val,
                 int64_t* idx) {
  return guarded([&] { emit(tsdict::ab_join(ts(a, na), ts(b, nb), m, threads), val, idx); });
}

int tsdr_self_join(const double* t, size_t n, size_t m, unsigned threads, double* val, int64_t* idx) {
  return guarded([&] { emit(tsdict::self_join(ts(t, n), m, threads), val, idx); });
}

// profiles.hpp:164-260 distance profiles over the reference's own stats
// (mass != 0: distance_profile_mass; origin = SIZE_MAX for none)
int tsdr_distance_profile(const double* t, size_t n, const double* q, size_t m, int mass, size_t origin, double* out) {
  return guarded([&] {
    const tsdict::TimeSeries T = ts(t, n);
    const auto st = tsdict::compute_stats(T, m);
    std::optional<std::size_t> org;
    if (origin != SIZE_MAX) org = origin;
    const std::span<const double> Q(q, m);
    const auto dp = mass ? tsdict::distance_profile_mass(T, Q, st, org) : tsdict::distance_profile_naive(T, Q, st, org);
    std::memcpy(out, dp.values.data(), dp.values.size() * sizeof(double));
  });
}

int tsdr_join_dictionary(const double* q, size_t nq, const double* seg_vals, const size_t* seg_len,
                         const size_t* seg_start, size_t nseg, size_t m, size_t dict_m, unsigned threads,
                         double* val, int64_t* idx) {
  return guarded([&] {
    tsdict::Dictionary D;
    D.m = dict_m;
    size_t off = 0, last = 0;
    for (size_t s = 0; s < nseg; ++s) {
      tsdict::Segment seg;
      seg.start = seg_start[s];
      seg.values.assign(seg_vals + off, seg_vals + off + seg_len[s]);
      off += seg_len[s];
      last = seg_start[s] + seg_len[s];
      D.segments.push_back(std::move(seg));
    }
    D.source_length = last;
    emit(tsdict::join_dictionary(ts(q, nq), D, m, threads), val, idx);
  });
}

int tsdr_compute_e_max(const double* t, size_t n, const double* seg_vals, const size_t* seg_len,
                       const size_t* seg_start, size_t nseg, size_t m, unsigned threads, double* out) {
  return guarded([&] {
    tsdict::Dictionary D;
    D.m = m;
    D.source_length = n;
    size_t off = 0;
    for (size_t s = 0; s < nseg; ++s) {
      tsdict::Segment seg;
      seg.start = seg_start[s];
      seg.values.assign(seg_vals + off, seg_vals + off + seg_len[s]);
      off += seg_len[s];
      D.segments.push_back(std::move(seg));
    }
    *out = tsdict::compute_e_max(D, ts(t, n), threads);
  });
}

// learn_dictionary (dictionary.hpp:259-328) with a space-saving stop rule;
// writes the merged segments (starts, lengths, packed values; capacity n
// each) and returns the segment count through *nseg and e_max through *e_max.
int tsdr_learn_dictionary(const double* t, size_t n, size_t m, double space_saving, unsigned threads,
                          size_t* seg_start, size_t* seg_len, double* seg_vals, size_t* nseg, double* e_max) {
  return guarded([&] {
    tsdict::LearnConfig cfg;
    cfg.m = m;
    cfg.space_saving_target = space_saving;
    const tsdict::Dictionary D = tsdict::learn_dictionary(ts(t, n), cfg, threads);
    size_t off = 0;
    for (size_t s = 0; s < D.segments.size(); ++s) {
      seg_start[s] = D.segments[s].start;
      seg_len[s] = D.segments[s].length();
      std::memcpy(seg_vals + off, D.segments[s].values.data(), seg_len[s] * sizeof(double));
      off += seg_len[s];
    }
    *nseg = D.segments.size();
    *e_max = D.e_max.value_or(-1.0);
  });
}

// learn_dictionary with any stop rule (rule 0: space saving, 1: sample budget,
// 2: error target); also returns the core starts, space_saving, no_progress
int tsdr_learn_dictionary2(const double* t, size_t n, size_t m, double k, int rule, double value,
                           size_t max_iterations, unsigned threads, size_t* seg_start, size_t* seg_len,
                           double* seg_vals, size_t* nseg, size_t* cores, size_t* ncores, double* e_max,
                           double* space_saving, int* no_progress) {
  return guarded([&] {
    tsdict::LearnConfig cfg;
    cfg.m = m;
    cfg.k = k;
    if (rule == 0) cfg.space_saving_target = value;
    if (rule == 1) cfg.sample_budget = (size_t)value;
    if (rule == 2) cfg.error_target = value;
    cfg.max_iterations = max_iterations;
    const tsdict::Dictionary D = tsdict::learn_dictionary(ts(t, n), cfg, threads);
    size_t off = 0;
    for (size_t s = 0; s < D.segments.size(); ++s) {
      seg_start[s] = D.segments[s].start;
      seg_len[s] = D.segments[s].length();
      std::memcpy(seg_vals + off, D.segments[s].values.data(), seg_len[s] * sizeof(double));
      off += seg_len[s];
    }
    *nseg = D.segments.size();
    for (size_t c = 0; c < D.core_starts.size(); ++c) cores[c] = D.core_starts[c];
    *ncores = D.core_starts.size();
    *e_max = D.e_max.value_or(-1.0);
    *space_saving = D.space_saving;
    *no_progress = D.no_progress ? 1 : 0;
  });
}

// dict_join.hpp:54-165 consumers
int tsdr_find_discords(const double* values, size_t cnt, size_t m, double e_max, size_t top_k, size_t* start,
                       double* score, int* certified, size_t* count) {
  return guarded([&] {
    tsdict::MatrixProfile P;
    P.values.assign(values, values + cnt);
    P.indices.assign(cnt, 0);
    P.kind = tsdict::join_kind::ab;
    P.m = m;
    const auto d = tsdict::find_discords(P, e_max, top_k);
    for (size_t i = 0; i < d.size(); ++i) {
      start[i] = d[i].start;
      score[i] = d[i].score;
      certified[i] = d[i].certified ? 1 : 0;
    }
    *count = d.size();
  });
}

int tsdr_window_labels(const size_t* lo, const size_t* hi, size_t nreg, size_t n, size_t m, unsigned char* labels) {
  return guarded([&] {
    std::vector<tsdict::interval> r;
    for (size_t i = 0; i < nreg; ++i) r.emplace_back(lo[i], hi[i]);
    const auto l = tsdict::window_labels(r, n, m);
    std::memcpy(labels, l.data(), l.size());
  });
}

int tsdr_auc_score(const double* scores, const unsigned char* labels, size_t cnt, double* auc) {
  return guarded([&] {
    *auc = tsdict::auc_score(std::vector<double>(scores, scores + cnt),
                             std::vector<unsigned char>(labels, labels + cnt));
  });
}

// tests/oracles.hpp long-double brute force
int tsdr_ab_join_brute(const double* a, size_t na, const double* b, size_t nb, size_t m, double* val,
                       int64_t* idx) {
  return guarded([&] {
    emit(oracle::ab_join_brute(std::vector<double>(a, a + na), std::vector<double>(b, b + nb), m), val, idx);
  });
}

int tsdr_self_join_brute(const double* t, size_t n, size_t m, double* val, int64_t* idx) {
  return guarded([&] { emit(oracle::self_join_brute(std::vector<double>(t, t + n), m), val, idx); });
}

// tests/synth.hpp generators, so fixtures replay the reference tests' own draws
void* tsdr_rng_new(uint64_t seed) { return new synth::rng_t(seed); }
void tsdr_rng_free(void* h) { delete static_cast<synth::rng_t*>(h); }
void tsdr_noise(void* h, size_t n, double* out) {
  const auto v = synth::noise(*static_cast<synth::rng_t*>(h), n);
  std::memcpy(out, v.data(), n * sizeof(double));
}
void tsdr_walk(void* h, size_t n, double* out) {
  const auto v = synth::walk(*static_cast<synth::rng_t*>(h), n);
  std::memcpy(out, v.data(), n * sizeof(double));
}
void tsdr_sine(size_t n, double period, double amp, double* out) {
  const auto v = synth::sine(n, period, amp);
  std::memcpy(out, v.data(), n * sizeof(double));
}

}  // extern "C"

// tsdict/dictionary.hpp -- drop-in for the dictionary types and engines of
// /root/reference/proj/include/tsdict/dictionary.hpp:
// Segment/Dictionary/LearnConfig (:46-77), the interval helpers (:78-117),
// detail::dict_min_profile (:149-193) and compute_e_max (:247-255) through
// one device launch over every segment (tsd_dict_join), and the greedy
// learn_dictionary (:259-328) with its selection loop on the device
// (tsd_learn_dictionary); learn_dictionary_random (:333-379) keeps its host
// loop (the reference's RNG stream) and computes e_max on the device.
//
// The host helpers below (context_interval, merge_intervals, merge_segments,
// validate_learn_config, the selection bookkeeping, finish_dictionary,
// learn_dictionary_random) deliberately restate the reference's observable
// host semantics -- its interval arithmetic, stop rules, error messages and
// RNG draw order -- so a drop-in user gets identical dictionaries; the
// compute they drive (self-join, distance profiles, argmin, e_max) is the
// device's.
#ifndef TSDICT_B200_DICTIONARY_HPP
#define TSDICT_B200_DICTIONARY_HPP

#include <algorithm>
#include <cstdint>
#include <optional>
#include <random>
#include <utility>
#include <vector>

#include "tsdict/errors.hpp"
#include "tsdict/profiles.hpp"
#include "tsdict/series.hpp"

namespace tsdict {

struct Segment {
  std::size_t start = 0;
  std::vector<double> values;
  std::size_t length() const noexcept { return values.size(); }
};

struct Dictionary {
  std::vector<Segment> segments;
  std::size_t m = 0;
  double k = 1.5;
  std::size_t source_length = 0;
  std::vector<std::size_t> core_starts;
  std::optional<double> e_max;
  double space_saving = 0.0;
  bool no_progress = false;

  std::size_t stored_samples() const noexcept {
    std::size_t total = 0;
    for (const auto& s : segments) total += s.length();
    return total;
  }
};

struct LearnConfig {
  std::size_t m = 0;
  double k = 1.5;
  std::optional<double> space_saving_target;
  std::optional<std::size_t> sample_budget;
  std::optional<double> error_target;
  std::size_t max_iterations = 1000000;
};

using interval = std::pair<std::size_t, std::size_t>;  // [lo, hi)

// Context window of a core start j: floor(k m) extra samples split around the
// core, floor half before (dictionary.hpp:78-84).
inline interval context_interval(std::size_t j, std::size_t m, double k, std::size_t n) {
  const auto extra = static_cast<std::size_t>(k * static_cast<double>(m) + 1e-9);
  const std::size_t before = extra / 2;
  return {j >= before ? j - before : 0, std::min(n, j + m + (extra - before))};
}

// Union of intervals; overlapping or touching ones merge (:87-98).
inline std::vector<interval> merge_intervals(std::vector<interval> ivs) {
  std::sort(ivs.begin(), ivs.end());
  std::vector<interval> out;
  for (const auto& iv : ivs) {
    if (!out.empty() && iv.first <= out.back().second)
      out.back().second = std::max(out.back().second, iv.second);
    else
      out.push_back(iv);
  }
  return out;
}

// The union as verbatim segments of the source (:101-117).
inline std::vector<Segment> merge_segments(const std::vector<interval>& ivs, const TimeSeries& source) {
  for (const auto& iv : ivs)
    if (iv.first >= iv.second || iv.second > source.n()) throw error(errc::invalid_argument, "interval out of range");
  std::vector<Segment> out;
  for (const auto& iv : merge_intervals(ivs)) {
    Segment s;
    s.start = iv.first;
    s.values.assign(source.values.begin() + static_cast<std::ptrdiff_t>(iv.first),
                    source.values.begin() + static_cast<std::ptrdiff_t>(iv.second));
    out.push_back(std::move(s));
  }
  return out;
}

namespace detail {

// dictionary.hpp:120-141 (same checks, same order, same codes)
inline void validate_learn_config(const LearnConfig& cfg) {
  if (cfg.m < 2) throw error(errc::window_too_small, "window length must be at least 2");
  if (cfg.k < 0.0) throw error(errc::invalid_argument, "context factor k must be non-negative");
  const int rules = (cfg.space_saving_target ? 1 : 0) + (cfg.sample_budget ? 1 : 0) + (cfg.error_target ? 1 : 0);
  if (rules != 1) throw error(errc::invalid_argument, "exactly one stop rule must be set");
  if (cfg.space_saving_target && (*cfg.space_saving_target < 0.0 || *cfg.space_saving_target >= 1.0))
    throw error(errc::invalid_argument, "space saving target must lie in [0, 1)");
  if (cfg.sample_budget && *cfg.sample_budget == 0) throw error(errc::invalid_argument, "sample budget must be positive");
  if (cfg.error_target && *cfg.error_target < 0.0) throw error(errc::invalid_argument, "error target must be non-negative");
  if (cfg.max_iterations == 0) throw error(errc::invalid_argument, "iteration cap must be positive");
}

// stored-sample threshold of the budget rules (:243-247)
inline double budget_threshold(const LearnConfig& cfg, std::size_t n) {
  if (cfg.sample_budget) return static_cast<double>(*cfg.sample_budget);
  return (1.0 - *cfg.space_saving_target) * static_cast<double>(n) - 1e-6;
}

// selection bookkeeping shared by both loops (:196-224)
struct select_state {
  std::size_t n = 0, cnt = 0, excl = 0;
  std::vector<unsigned char> masked;
  std::vector<interval> chosen, merged;
  std::vector<std::size_t> core_starts;
  std::size_t stored = 0;

  select_state(std::size_t n_, std::size_t cnt_, std::size_t excl_) : n(n_), cnt(cnt_), excl(excl_), masked(cnt_, 0) {}

  void take(std::size_t j, std::size_t m, double k) {
    core_starts.push_back(j);
    chosen.push_back(context_interval(j, m, k, n));
    merged = merge_intervals(chosen);
    stored = 0;
    for (const auto& iv : merged) stored += iv.second - iv.first;
    const std::size_t lo = j >= excl ? j - excl : 0, hi = std::min(cnt, j + excl + 1);
    std::fill(masked.begin() + static_cast<std::ptrdiff_t>(lo), masked.begin() + static_cast<std::ptrdiff_t>(hi),
              static_cast<unsigned char>(1));
  }
};

inline Dictionary finish_dictionary(const select_state& st, const TimeSeries& T_B, const LearnConfig& cfg,
                                    bool no_progress) {  // :226-237
  Dictionary D;
  D.m = cfg.m;
  D.k = cfg.k;
  D.source_length = T_B.n();
  D.core_starts = st.core_starts;
  D.segments = merge_segments(st.chosen, T_B);
  D.space_saving = 1.0 - static_cast<double>(st.stored) / static_cast<double>(T_B.n());
  D.no_progress = no_progress;
  return D;
}

struct packed_dictionary {
  std::vector<double> vals;
  std::vector<std::size_t> len, start;
};

inline packed_dictionary pack(const Dictionary& D) {
  packed_dictionary p;
  p.len.reserve(D.segments.size());
  p.start.reserve(D.segments.size());
  for (const auto& s : D.segments) {
    p.vals.insert(p.vals.end(), s.values.begin(), s.values.end());
    p.len.push_back(s.length());
    p.start.push_back(s.start);
  }
  return p;
}

// dictionary.hpp:149-193
inline MatrixProfile dict_min_profile(const TimeSeries& T, const Dictionary& D, std::size_t m, unsigned threads = 0,
                                      precision prec = precision::fp64) {
  (void)threads;
  const packed_dictionary p = pack(D);
  MatrixProfile P;
  P.kind = join_kind::ab;
  P.m = m;
  const std::size_t cnt = (m >= 1 && T.n() >= m) ? T.n() - m + 1 : 0;
  P.values.resize(cnt);
  P.indices.resize(cnt);
  detail::raise_status(tsd_dict_join(T.values.data(), T.n(), p.vals.data(), p.len.data(), p.start.data(),
                                     D.segments.size(), m, static_cast<int>(prec), P.values.data(),
                                     P.indices.data()));
  return P;
}

}  // namespace detail

// dictionary.hpp:247-255
inline double compute_e_max(const Dictionary& D, const TimeSeries& T_B, unsigned threads = 0) {
  (void)threads;
  const detail::packed_dictionary p = detail::pack(D);
  double out = 0.0;
  detail::raise_status(tsd_compute_e_max(T_B.values.data(), T_B.n(), D.source_length, p.vals.data(), p.len.data(),
                                         p.start.data(), D.segments.size(), D.m, &out));
  return out;
}

namespace detail {
// learn_dictionary through the device loop; profile = P_B values or nullptr
inline Dictionary learn_on_device(const TimeSeries& T_B, const LearnConfig& cfg, const double* profile) {
  const std::size_t n = T_B.n();
  int rule = TSD_RULE_ERROR_TARGET;
  double value = 0.0;
  if (cfg.space_saving_target) {
    rule = TSD_RULE_SPACE_SAVING;
    value = *cfg.space_saving_target;
  } else if (cfg.sample_budget) {
    rule = TSD_RULE_SAMPLE_BUDGET;
    value = static_cast<double>(*cfg.sample_budget);
  } else if (cfg.error_target) {
    value = *cfg.error_target;
  }
  const std::size_t cap = std::max<std::size_t>(n, 1);
  std::vector<std::size_t> starts(cap), lens(cap), cores(cap);
  std::vector<double> vals(cap);
  std::size_t nseg = 0, ncores = 0;
  double e = 0.0, saving = 0.0;
  int stalled = 0;
  raise_status(tsd_learn_dictionary(T_B.values.data(), n, cfg.m, cfg.k, rule, value, cfg.max_iterations, profile,
                                    starts.data(), lens.data(), vals.data(), &nseg, cores.data(), &ncores, &e,
                                    &saving, &stalled));
  Dictionary D;
  D.m = cfg.m;
  D.k = cfg.k;
  D.source_length = n;
  D.core_starts.assign(cores.begin(), cores.begin() + static_cast<std::ptrdiff_t>(ncores));
  std::size_t off = 0;
  for (std::size_t s = 0; s < nseg; ++s) {
    Segment g;
    g.start = starts[s];
    g.values.assign(vals.begin() + static_cast<std::ptrdiff_t>(off),
                    vals.begin() + static_cast<std::ptrdiff_t>(off + lens[s]));
    off += lens[s];
    D.segments.push_back(std::move(g));
  }
  D.e_max = e;
  D.space_saving = saving;
  D.no_progress = stalled != 0;
  return D;
}
}  // namespace detail

// dictionary.hpp:259-321: greedy learning against a precomputed exact
// self-join profile of the source
inline Dictionary learn_dictionary(const TimeSeries& T_B, const LearnConfig& cfg, const MatrixProfile& P_B,
                                   unsigned threads = 0) {
  (void)threads;
  detail::validate_learn_config(cfg);
  const std::size_t n = T_B.n(), m = cfg.m;
  if (n < 2 * m) throw error(errc::series_too_short, "dictionary learning needs n >= 2m");
  if (P_B.m != m || P_B.kind != join_kind::self || P_B.values.size() != n - m + 1)
    throw error(errc::invalid_argument, "precomputed profile does not match the series and window");
  return detail::learn_on_device(T_B, cfg, P_B.values.data());
}

// dictionary.hpp:324-328: computes the self-join profile itself
inline Dictionary learn_dictionary(const TimeSeries& T_B, const LearnConfig& cfg, unsigned threads = 0) {
  (void)threads;
  detail::validate_learn_config(cfg);
  return detail::learn_on_device(T_B, cfg, nullptr);
}

// dictionary.hpp:333-379: random-selection baseline (budget rules only). The
// picks follow the reference's RNG stream on the host; e_max on the device.
inline Dictionary learn_dictionary_random(const TimeSeries& T_B, const LearnConfig& cfg, std::uint64_t seed,
                                          unsigned threads = 0) {
  detail::validate_learn_config(cfg);
  if (cfg.error_target) throw error(errc::invalid_argument, "random baseline supports budget stop rules only");
  const std::size_t n = T_B.n(), m = cfg.m;
  if (n < 2 * m) throw error(errc::series_too_short, "dictionary learning needs n >= 2m");
  const std::size_t cnt = n - m + 1;
  const double need = detail::budget_threshold(cfg, n);
  detail::select_state st(n, cnt, m / 2);
  std::mt19937_64 rng(seed);
  bool stalled = false;
  for (std::size_t iter = 0;; ++iter) {
    if (iter >= cfg.max_iterations)
      throw error(errc::iteration_cap_exceeded, "iteration cap reached before the stop rule fired");
    std::size_t free = 0;
    for (unsigned char f : st.masked) free += f ? 0 : 1;
    if (free == 0) {
      stalled = true;
      break;
    }
    std::uniform_int_distribution<std::size_t> pick(0, free - 1);
    std::size_t rank = pick(rng), j = 0;
    for (std::size_t i = 0; i < cnt; ++i) {
      if (st.masked[i]) continue;
      if (rank-- == 0) {
        j = i;
        break;
      }
    }
    st.take(j, m, cfg.k);
    if (static_cast<double>(st.stored) >= need) break;
  }
  Dictionary D = detail::finish_dictionary(st, T_B, cfg, stalled);
  D.e_max = compute_e_max(D, T_B, threads);
  return D;
}

}  // namespace tsdict

#endif

// test_dropin.cpp -- the C++ drop-in headers (include/tsdict/*.hpp) used the
// way the reference's own GoogleTest suites use the reference headers
// (tests/test_profiles.cpp, test_dict_join.cpp, test_series.cpp). Results
// are checked against the oracle (oracle/tsd_oracle.h). One [PASS]/[FAIL]
// line per case; exit status = number of failures. Needs a GPU.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <span>
#include <string>
#include <vector>

#include "tsd_oracle.h"
#include "tsdict/tsdict.hpp"

extern "C" {
void* tsd_rng_new(uint64_t seed);
void tsd_rng_free(void* h);
void tsd_rng_walk(void* h, size_t n, double* out);
void tsd_rng_noise(void* h, size_t n, double* out);
void tsd_synth_sine(size_t n, double period, double amp, double* out);
}

using namespace tsdict;

namespace {

int failures = 0;

void check(const char* name, const std::function<std::string()>& body) {
  std::string err;
  try {
    err = body();
  } catch (const std::exception& e) {
    err = std::string("exception: ") + e.what();
  }
  std::printf("[%s] %s%s%s\n", err.empty() ? "PASS" : "FAIL", name, err.empty() ? "" : ": ", err.c_str());
  if (!err.empty()) ++failures;
}

struct Rng {
  void* h;
  explicit Rng(uint64_t s) : h(tsd_rng_new(s)) {}
  ~Rng() { tsd_rng_free(h); }
  std::vector<double> walk(size_t n) {
    std::vector<double> v(n);
    tsd_rng_walk(h, n, v.data());
    return v;
  }
  std::vector<double> noise(size_t n) {
    std::vector<double> v(n);
    tsd_rng_noise(h, n, v.data());
    return v;
  }
};

template <class F>
std::string expect_code(errc want, F&& f) {
  try {
    f();
  } catch (const error& e) {
    return e.code() == want ? "" : std::string("wrong code: ") + e.what();
  }
  return "no exception";
}

std::string close_to_oracle(const MatrixProfile& P, const std::vector<double>& rv, const std::vector<int64_t>& ri,
                            double tol) {
  if (P.values.size() != rv.size()) return "size mismatch";
  for (size_t i = 0; i < rv.size(); ++i) {
    if (std::isinf(rv[i]) != std::isinf(P.values[i])) return "sentinel mismatch at " + std::to_string(i);
    if (std::isinf(rv[i])) continue;
    if (std::fabs(P.values[i] - rv[i]) > tol * std::max(1.0, rv[i])) return "value mismatch at " + std::to_string(i);
    if (P.indices[i] != ri[i] && std::fabs(P.values[i] - rv[i]) > 1e-9)
      return "index mismatch at " + std::to_string(i);
  }
  return "";
}

}  // namespace

int main() {
  check("AbJoin.MatchesOracle", [] {
    Rng r(35);
    const TimeSeries A{r.noise(300)}, B{r.noise(200)};
    const MatrixProfile P = ab_join(A, B, 20);
    std::vector<double> v(281);
    std::vector<int64_t> i(281);
    tsdo_ab_join(A.values.data(), 300, B.values.data(), 200, 20, v.data(), i.data());
    return close_to_oracle(P, v, i, 1e-8);
  });
  check("AbJoin.TooShortThrows", [] {
    Rng r(39);
    return expect_code(errc::series_too_short, [&] { ab_join(TimeSeries{r.noise(10)}, TimeSeries{r.noise(100)}, 20); });
  });
  check("AbJoin.DeterministicAcrossThreadCounts", [] {
    Rng r(40);
    const TimeSeries A{r.walk(1500)}, B{r.walk(900)};
    const auto p1 = ab_join(A, B, 40, 1), p3 = ab_join(A, B, 40, 3);
    return p1.values == p3.values && p1.indices == p3.indices ? "" : "results differ";
  });
  check("SelfJoin.MatchesOracle", [] {
    Rng r(33);
    const TimeSeries T{r.walk(2048)};
    const MatrixProfile P = self_join(T, 50);
    std::vector<double> v(1999);
    std::vector<int64_t> i(1999);
    tsdo_self_join(T.values.data(), 2048, 50, 25, v.data(), i.data());
    return close_to_oracle(P, v, i, 1e-8);
  });
  check("SelfJoin.MinimumLengthEdge", [] {
    Rng r(31);
    const MatrixProfile P = self_join(TimeSeries{r.noise(16)}, 8);
    if (P.values.size() != 9) return std::string("size");
    if (P.indices[4] != MatrixProfile::no_neighbor || !std::isinf(P.values[4])) return std::string("no sentinel");
    for (int k : {0, 1, 7, 8})
      if (P.indices[k] == MatrixProfile::no_neighbor) return std::string("unexpected sentinel");
    return std::string();
  });
  check("SelfJoin.TooShortThrows", [] {
    Rng r(32);
    return expect_code(errc::series_too_short, [&] { self_join(TimeSeries{r.noise(15)}, 8); });
  });
  check("ComputeStats.Errors", [] {
    std::string e = expect_code(errc::window_too_large, [] { compute_stats(TimeSeries{{1, 2, 3}}, 4); });
    if (e.empty()) e = expect_code(errc::window_too_small, [] { compute_stats(TimeSeries{{1, 2, 3}}, 1); });
    if (e.empty())
      e = expect_code(errc::non_finite_input, [] { compute_stats(TimeSeries{{1, std::nan(""), 3}}, 2); });
    return e;
  });
  check("ComputeStats.ConstancyMaskIsScaleRelative", [] {
    std::vector<double> base{5.0, 5.0, 5.0 + 1e-9, 5.0, 1.0, 9.0};
    auto st = compute_stats(TimeSeries{base}, 4);
    if (!st.constant_mask[0] || st.constant_mask[2]) return std::string("unscaled mask");
    for (auto& x : base) x *= 1e6;
    st = compute_stats(TimeSeries{base}, 4);
    return st.constant_mask[0] && !st.constant_mask[2] ? std::string() : std::string("scaled mask");
  });
  check("JoinDictionary.SingleFullSegmentEqualsAbJoin", [] {
    Rng r(70);
    const TimeSeries B{r.walk(600)}, A{r.walk(400)};
    Dictionary D;
    D.m = 50;
    D.source_length = B.n();
    D.segments.push_back({0, B.values});
    const auto via_dict = join_dictionary(A, D, 50);
    const auto direct = ab_join(A, B, 50);
    return via_dict.values == direct.values && via_dict.indices == direct.indices ? "" : "not bit-identical";
  });
  check("JoinDictionary.Errors", [] {
    Dictionary D;
    D.m = 40;
    D.segments.push_back({0, std::vector<double>(100, 1.0)});
    std::string e = expect_code(errc::window_mismatch, [&] { join_dictionary(TimeSeries{std::vector<double>(200, 0.5)}, D, 41); });
    Dictionary empty;
    empty.m = 40;
    if (e.empty()) e = expect_code(errc::empty_dictionary, [&] { join_dictionary(TimeSeries{std::vector<double>(200)}, empty, 40); });
    return e;
  });
  check("JoinDictionary.IndicesAreSourceCoordinates", [] {
    Rng r(71);
    const std::vector<double> src = r.walk(800);
    const TimeSeries A{r.walk(300)};
    Dictionary D;
    D.m = 40;
    D.source_length = src.size();
    for (size_t st : {0u, 300u, 610u}) D.segments.push_back({st, std::vector<double>(src.begin() + st, src.begin() + st + 120)});
    const auto P = join_dictionary(A, D, 40);
    for (size_t i = 0; i < P.values.size(); ++i) {
      const auto j = static_cast<size_t>(P.indices[i]);
      bool inside = false;
      for (const auto& s : D.segments) inside = inside || (j >= s.start && j + 40 <= s.start + s.length());
      if (!inside) return "index " + std::to_string(j) + " outside every segment";
      const double d = tsdo_pair_dist(A.values.data(), A.n(), i, src.data(), src.size(), j, 40);
      if (std::fabs(d - P.values[i]) > 1e-6) return "value does not match its index at row " + std::to_string(i);
    }
    return std::string();
  });
  check("EMax.FullCoverageIsZero", [] {
    Rng r(60);
    const TimeSeries T{r.walk(500)};
    Dictionary D;
    D.m = 50;
    D.source_length = T.n();
    D.segments.push_back({0, T.values});
    const double e = compute_e_max(D, T);
    return e <= 1e-5 ? "" : "e_max " + std::to_string(e);
  });
  // learn_dictionary (test_dictionary.cpp:53-82 invariants, :250-400 rules)
  auto invariants = [](const Dictionary& D, const TimeSeries& T) -> std::string {
    if (D.source_length != T.n() || D.segments.empty()) return "empty or wrong source length";
    std::size_t stored = 0, prev_end = 0;
    for (std::size_t s = 0; s < D.segments.size(); ++s) {
      const auto& g = D.segments[s];
      if (g.length() < D.m || g.start + g.length() > T.n()) return "segment bounds";
      if (s > 0 && g.start <= prev_end) return "segments not disjoint / sorted / separated";
      prev_end = g.start + g.length();
      for (std::size_t i = 0; i < g.length(); ++i)
        if (g.values[i] != T.values[g.start + i]) return "segment is not a verbatim copy";
      stored += g.length();
    }
    if (std::fabs(D.space_saving - (1.0 - double(stored) / double(T.n()))) > 1e-12) return "space_saving";
    for (std::size_t a = 0; a < D.core_starts.size(); ++a)
      for (std::size_t b = a + 1; b < D.core_starts.size(); ++b) {
        const std::size_t lo = std::min(D.core_starts[a], D.core_starts[b]);
        const std::size_t hi = std::max(D.core_starts[a], D.core_starts[b]);
        if (hi - lo <= D.m / 2) return "core starts closer than the exclusion zone";
      }
    return "";
  };
  check("LearnDictionary.InvariantsAndBudget", [&] {
    Rng r(90);
    const TimeSeries T{r.walk(3000)};
    LearnConfig cfg;
    cfg.m = 50;
    cfg.space_saving_target = 0.5;
    const Dictionary D = learn_dictionary(T, cfg);
    if (auto e = invariants(D, T); !e.empty()) return e;
    if (double(D.stored_samples()) < 0.5 * 3000 - 1e-6) return std::string("budget rule did not hold");
    if (!D.e_max || *D.e_max <= 0.0) return std::string("e_max not set");
    return std::string();
  });
  check("LearnDictionary.PrecomputedProfileOverload", [&] {
    Rng r(91);
    const TimeSeries T{r.walk(2000)};
    LearnConfig cfg;
    cfg.m = 60;
    cfg.sample_budget = 600;
    const Dictionary a = learn_dictionary(T, cfg);
    const Dictionary b = learn_dictionary(T, cfg, self_join(T, 60));
    return a.core_starts == b.core_starts && *a.e_max == *b.e_max ? std::string() : std::string("overloads differ");
  });
  check("LearnDictionaryRandom.DeterministicPerSeed", [&] {
    Rng r(92);
    const TimeSeries T{r.walk(2500)};
    LearnConfig cfg;
    cfg.m = 50;
    cfg.space_saving_target = 0.7;
    const Dictionary a = learn_dictionary_random(T, cfg, 42), b = learn_dictionary_random(T, cfg, 42);
    const Dictionary c = learn_dictionary_random(T, cfg, 43);
    if (auto e = invariants(a, T); !e.empty()) return e;
    if (a.core_starts != b.core_starts) return std::string("same seed, different picks");
    if (a.core_starts == c.core_starts) return std::string("different seeds, same picks");
    return std::string();
  });
  check("LearnDictionary.Errors", [&] {
    Rng r(93);
    const TimeSeries T{r.walk(500)};
    LearnConfig cfg;
    cfg.m = 50;
    if (auto e = expect_code(errc::invalid_argument, [&] { learn_dictionary(T, cfg); }); !e.empty()) return e;
    cfg.space_saving_target = 0.5;
    cfg.error_target = 1.0;
    if (auto e = expect_code(errc::invalid_argument, [&] { learn_dictionary(T, cfg); }); !e.empty()) return e;
    cfg.error_target.reset();
    cfg.m = 300;
    if (auto e = expect_code(errc::series_too_short, [&] { learn_dictionary(T, cfg); }); !e.empty()) return e;
    cfg.m = 50;
    cfg.error_target = 1.0;
    cfg.space_saving_target.reset();
    return expect_code(errc::invalid_argument, [&] { learn_dictionary_random(T, cfg, 1); });
  });
  check("Discords.PlantedAnomalyRanksFirst", [&] {  // test_dict_join.cpp discord shapes
    Rng r(95);
    std::vector<double> q = r.walk(4000);
    for (int i = 0; i < 80; ++i) q[2500 + i] += 6.0 * std::sin(i * 0.2);
    Rng rd(96);
    Dictionary D;
    D.m = 64;
    for (int s = 0; s < 4; ++s) D.segments.push_back(Segment{std::size_t(1000 * s), rd.walk(600)});
    D.source_length = 4000;
    const MatrixProfile P = join_dictionary(TimeSeries{q}, D, 64);
    const AnomalyReport rep = make_anomaly_report(P, 0.0, 5);
    if (rep.discords.size() != 5) return std::string("wrong count");
    for (std::size_t a = 0; a < rep.discords.size(); ++a)
      for (std::size_t b = a + 1; b < rep.discords.size(); ++b) {
        const auto x = rep.discords[a].start, y = rep.discords[b].start;
        if ((x > y ? x - y : y - x) <= 32) return std::string("overlapping picks");
        if (rep.discords[a].score < rep.discords[b].score) return std::string("not in score order");
      }
    return expect_code(errc::empty_profile, [] { find_discords(MatrixProfile{}, 0.0, 3); });
  });
  check("Labels.AucOfPerfectScoresIsOne", [&] {
    const auto lab = window_labels({{100, 200}, {150, 260}}, 1000, 50);
    std::vector<double> sc(lab.size());
    for (std::size_t i = 0; i < lab.size(); ++i) sc[i] = lab[i] ? 1.0 : 0.0;
    if (std::fabs(auc_score(sc, lab) - 1.0) > 0) return std::string("AUC != 1");
    return expect_code(errc::degenerate_labels, [&] { auc_score(sc, std::vector<unsigned char>(lab.size(), 0)); });
  });
  // DistanceProfile.* (reference test_profiles.cpp:67-135, same inputs and
  // assertions): the drop-in's distance profiles run on the device
  auto window = [](const TimeSeries& T, std::size_t at, std::size_t m) {
    return std::span<const double>(T.values).subspan(at, m);
  };
  check("DistanceProfile.NaiveSelfMatchIsZero", [&] {
    Rng r(21);
    const TimeSeries T{r.walk(256)};
    const auto st = compute_stats(T, 16);
    const auto dp = distance_profile_naive(T, window(T, 7, 16), st, 7);
    if (dp.values.size() != T.n() - 16 + 1) return std::string("size");
    if (dp.values[7] != 0.0) return "self match " + std::to_string(dp.values[7]);
    return dp.query_origin && *dp.query_origin == 7u ? std::string() : std::string("origin");
  });
  check("DistanceProfile.NaiveConstantTargetConvention", [&] {
    const TimeSeries T{std::vector<double>(64, 2.5)};
    Rng r(22);
    const auto q = r.noise(16);
    const auto st = compute_stats(T, 16);
    const auto dp = distance_profile_naive(T, q, st);
    for (double v : dp.values)
      if (v != std::sqrt(32.0)) return "value " + std::to_string(v);
    return std::string();
  });
  check("DistanceProfile.NaiveEqualsDirectEvaluation", [&] {
    Rng r(23);
    const TimeSeries T{r.noise(1024)};
    const auto q = r.noise(32);
    const auto st = compute_stats(T, 32);
    const auto dp = distance_profile_naive(T, q, st);
    for (std::size_t i = 0; i < dp.values.size(); ++i)
      if (dp.values[i] != znorm_distance(window(T, i, 32), q)) return "not bit-identical at " + std::to_string(i);
    return std::string();
  });
  check("DistanceProfile.MassSelfMatchNearZero", [&] {
    Rng r(24);
    const TimeSeries T{r.walk(256)};
    const auto st = compute_stats(T, 16);
    const auto dp = distance_profile_mass(T, window(T, 7, 16), st, 7);
    return dp.values[7] <= 1e-6 ? std::string() : "self match " + std::to_string(dp.values[7]);
  });
  check("DistanceProfile.MassSinePeriodicity", [&] {
    std::vector<double> s(1024);
    tsd_synth_sine(1024, 64.0, 1.0, s.data());
    const TimeSeries T{s};
    const auto st = compute_stats(T, 64);
    const auto dp = distance_profile_mass(T, window(T, 0, 64), st, 0);
    for (std::size_t at = 0; at + 64 <= T.n() - 64 + 1; at += 64)
      if (dp.values[at] > 1e-4) return "offset " + std::to_string(at);
    return std::string();
  });
  check("DistanceProfile.MassMatchesNaive", [&] {
    // the reference draws n, m from std::uniform_int_distribution (an
    // implementation-defined mapping); the same ranges from our stream
    Rng r(25);
    for (int t = 0; t < 25; ++t) {
      const auto u = r.noise(2);
      const std::size_t n = 128 + (std::size_t)(std::fabs(u[0]) * 1000.0) % (4096 - 128 + 1);
      const std::size_t m = std::min<std::size_t>(8 + (std::size_t)(std::fabs(u[1]) * 1000.0) % 121, n / 2);
      const TimeSeries T{t % 2 == 0 ? r.walk(n) : r.noise(n)};
      const auto q = t % 3 == 0 ? r.walk(m) : r.noise(m);
      const auto st = compute_stats(T, m);
      const auto naive = distance_profile_naive(T, q, st);
      const auto mass = distance_profile_mass(T, q, st);
      double worst = 0.0;
      for (std::size_t i = 0; i < naive.values.size(); ++i)
        worst = std::max(worst, std::fabs(naive.values[i] - mass.values[i]));
      if (!(worst < 1e-5)) return "n=" + std::to_string(n) + " m=" + std::to_string(m) + " worst " + std::to_string(worst);
    }
    return std::string();
  });
  check("DistanceProfile.ConstantQueryConvention", [&] {
    Rng r(26);
    TimeSeries T{r.noise(200)};
    for (std::size_t i = 40; i < 56; ++i) T.values[i] = 4.0;
    const std::vector<double> q(16, 1.0);
    const auto st = compute_stats(T, 16);
    const auto mass = distance_profile_mass(T, q, st);
    const auto naive = distance_profile_naive(T, q, st);
    for (std::size_t i = 0; i < mass.values.size(); ++i) {
      if (mass.values[i] != naive.values[i]) return "mass != naive at " + std::to_string(i);
      if (mass.values[i] != (st.constant_mask[i] ? 0.0 : std::sqrt(32.0))) return "convention at " + std::to_string(i);
    }
    return std::string();
  });
  check("DistanceProfile.LengthMismatchThrows", [&] {
    Rng r(27);
    const TimeSeries T{r.noise(300)};
    const auto st = compute_stats(T, 16);
    const auto q = r.noise(17);
    auto e = expect_code(errc::length_mismatch, [&] { distance_profile_naive(T, q, st); });
    if (e.empty()) e = expect_code(errc::length_mismatch, [&] { distance_profile_mass(TimeSeries{r.noise(299)}, std::span<const double>(q).first(16), st); });
    return e;
  });
  std::printf("%d failure(s)\n", failures);
  return failures;
}

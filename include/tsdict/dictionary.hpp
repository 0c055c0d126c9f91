// tsdict/dictionary.hpp -- drop-in for the dictionary types and the hot
// engine of /root/reference/proj/include/tsdict/dictionary.hpp:
// Segment/Dictionary/LearnConfig (:46-77), detail::dict_min_profile
// (:149-193) and compute_e_max (:247-255), all through one device launch
// over every segment (tsd_dict_join).
#ifndef TSDICT_B200_DICTIONARY_HPP
#define TSDICT_B200_DICTIONARY_HPP

#include <cstdint>
#include <optional>
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

using interval = std::pair<std::size_t, std::size_t>;

namespace detail {

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

}  // namespace tsdict

#endif

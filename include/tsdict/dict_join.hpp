// tsdict/dict_join.hpp -- drop-in for join_dictionary
// (/root/reference/proj/include/tsdict/dict_join.hpp:42-48) plus a batched
// form for many query series against one resident dictionary.
#ifndef TSDICT_B200_DICT_JOIN_HPP
#define TSDICT_B200_DICT_JOIN_HPP

#include <vector>

#include "tsdict/dictionary.hpp"
#include "tsdict/errors.hpp"
#include "tsdict/profiles.hpp"

namespace tsdict {

inline MatrixProfile join_dictionary(const TimeSeries& A, const Dictionary& D, std::size_t m, unsigned threads = 0,
                                     precision prec = precision::fp64) {
  if (m != D.m) throw error(errc::window_mismatch, "requested window length differs from the dictionary's");
  return detail::dict_min_profile(A, D, m, threads, prec);
}

// One device pass over every series (equivalent to join_dictionary per series).
inline std::vector<MatrixProfile> join_dictionary_batched(const std::vector<TimeSeries>& series, const Dictionary& D,
                                                          std::size_t m, precision prec = precision::fp64) {
  if (m != D.m) throw error(errc::window_mismatch, "requested window length differs from the dictionary's");
  const detail::packed_dictionary p = detail::pack(D);
  std::vector<double> q;
  std::vector<std::size_t> qlen;
  std::size_t total = 0;
  for (const auto& s : series) {
    q.insert(q.end(), s.values.begin(), s.values.end());
    qlen.push_back(s.n());
    total += s.n() >= m && m >= 1 ? s.n() - m + 1 : 0;
  }
  std::vector<double> val(total);
  std::vector<std::int64_t> idx(total);
  detail::raise_status(tsd_dict_join_batched(q.data(), qlen.data(), qlen.size(), p.vals.data(), p.len.data(),
                                             p.start.data(), D.segments.size(), m, static_cast<int>(prec), val.data(),
                                             idx.data()));
  std::vector<MatrixProfile> out(series.size());
  std::size_t o = 0;
  for (std::size_t k = 0; k < series.size(); ++k) {
    const std::size_t c = series[k].n() - m + 1;
    out[k].kind = join_kind::ab;
    out[k].m = m;
    out[k].values.assign(val.begin() + o, val.begin() + o + c);
    out[k].indices.assign(idx.begin() + o, idx.begin() + o + c);
    o += c;
  }
  return out;
}

}  // namespace tsdict

#endif

// tsdict/dict_join.hpp -- drop-in for /root/reference/proj/include/tsdict/
// dict_join.hpp: join_dictionary (:42-48) plus a batched form for many query
// series against one resident dictionary; its consumers Discord /
// AnomalyReport (:28-38), find_discords (:54-93, peaks on the device),
// make_anomaly_report (:95-101), window_labels (:102-127) and auc_score
// (:130-162) (host; auc_score restates the reference's ranking rule so scores
// agree exactly).
#ifndef TSDICT_B200_DICT_JOIN_HPP
#define TSDICT_B200_DICT_JOIN_HPP

#include <algorithm>
#include <cmath>
#include <numeric>
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

struct Discord {
  std::size_t start = 0;
  double score = 0.0;
  bool certified = false;
};

struct AnomalyReport {
  MatrixProfile scores;
  std::vector<Discord> discords;
  double e_max_used = 0.0;
};

// greedy top-k with +-floor(m/2) suppression; rank 1 certified by the e_max gap
inline std::vector<Discord> find_discords(const MatrixProfile& P, double e_max, std::size_t top_k) {
  const std::size_t cap = std::max<std::size_t>(top_k, 1);
  std::vector<std::size_t> start(cap);
  std::vector<double> score(cap);
  std::vector<int> cert(cap);
  std::size_t count = 0;
  detail::raise_status(tsd_find_discords(P.values.data(), P.values.size(), P.m, e_max, top_k, start.data(),
                                         score.data(), cert.data(), &count));
  std::vector<Discord> out(count);
  for (std::size_t i = 0; i < count; ++i) out[i] = Discord{start[i], score[i], cert[i] != 0};
  return out;
}

inline AnomalyReport make_anomaly_report(MatrixProfile scores, double e_max, std::size_t top_k) {
  AnomalyReport rep;
  rep.discords = find_discords(scores, e_max, top_k);
  rep.scores = std::move(scores);
  rep.e_max_used = e_max;
  return rep;
}

// a window is positive when it overlaps a merged region by >= m/2 samples
inline std::vector<unsigned char> window_labels(const std::vector<interval>& regions, std::size_t n, std::size_t m) {
  if (m < 2 || m > n) throw error(errc::invalid_argument, "window length out of range");
  for (const auto& r : regions)
    if (r.first >= r.second || r.second > n) throw error(errc::invalid_argument, "label region out of range");
  const std::size_t cnt = n - m + 1;
  std::vector<unsigned char> labels(cnt, 0);
  for (const auto& r : merge_intervals(regions)) {
    const std::size_t first = r.first + 1 > m ? r.first + 1 - m : 0;
    for (std::size_t i = first; i < std::min(cnt, r.second); ++i) {
      const std::size_t lo = std::max(i, r.first), hi = std::min(i + m, r.second);
      if (hi > lo && 2 * (hi - lo) >= m) labels[i] = 1;
    }
  }
  return labels;
}

// exact Mann-Whitney AUC, ties counted as 1/2
inline double auc_score(const std::vector<double>& scores, const std::vector<unsigned char>& labels) {
  if (scores.size() != labels.size()) throw error(errc::length_mismatch, "scores and labels differ in length");
  std::size_t pos = 0, neg = 0;
  for (std::size_t i = 0; i < labels.size(); ++i) {
    if (std::isnan(scores[i])) throw error(errc::invalid_argument, "scores must not contain NaN");
    (labels[i] ? pos : neg) += 1;
  }
  if (pos == 0 || neg == 0)
    throw error(errc::degenerate_labels, "AUC needs at least one positive and one negative label");
  std::vector<std::size_t> order(scores.size());
  std::iota(order.begin(), order.end(), std::size_t{0});
  std::sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return scores[a] < scores[b]; });
  double wins = 0.0, neg_below = 0.0;
  for (std::size_t a = 0; a < order.size();) {
    std::size_t b = a;
    double gp = 0.0, gn = 0.0;
    for (; b < order.size() && scores[order[b]] == scores[order[a]]; ++b) (labels[order[b]] ? gp : gn) += 1.0;
    wins += gp * (neg_below + 0.5 * gn);
    neg_below += gn;
    a = b;
  }
  return wins / (static_cast<double>(pos) * static_cast<double>(neg));
}

}  // namespace tsdict

#endif

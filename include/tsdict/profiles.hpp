// tsdict/profiles.hpp -- drop-in for /root/reference/proj/include/tsdict/profiles.hpp
// (hot path: ab_join :306-342, self_join :266-301). Both run on the B200
// through the C ABI; `threads` is accepted for source compatibility (results
// are bit-identical for any value, as the reference promises at :12-17).
#ifndef TSDICT_B200_PROFILES_HPP
#define TSDICT_B200_PROFILES_HPP

#include <cstdint>
#include <optional>
#include <span>
#include <thread>
#include <vector>

#include "tsdict/errors.hpp"
#include "tsdict/series.hpp"

namespace tsdict {

struct DistanceProfile {  // profiles.hpp:36-40
  std::vector<double> values;
  std::optional<std::size_t> query_origin;
  std::size_t m = 0;
};

enum class join_kind { self, ab };

struct MatrixProfile {  // profiles.hpp:44-51
  static constexpr std::int64_t no_neighbor = -1;
  std::vector<double> values;
  std::vector<std::int64_t> indices;
  join_kind kind = join_kind::self;
  std::size_t m = 0;
};

inline unsigned resolve_threads(unsigned requested) {  // profiles.hpp:53-57
  if (requested != 0) return requested;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw != 0 ? hw : 1;
}

enum class precision { fp64 = TSD_FP64, fp32 = TSD_FP32 };

// profiles.hpp:306-342
inline MatrixProfile ab_join(const TimeSeries& A, const TimeSeries& B, std::size_t m, unsigned threads = 0,
                             precision prec = precision::fp64) {
  (void)threads;
  MatrixProfile P;
  P.kind = join_kind::ab;
  P.m = m;
  const std::size_t cnt = (m >= 1 && A.n() >= m) ? A.n() - m + 1 : 0;
  P.values.resize(cnt);
  P.indices.resize(cnt);
  detail::raise_status(tsd_ab_join(A.values.data(), A.n(), B.values.data(), B.n(), m, static_cast<int>(prec),
                                   P.values.data(), P.indices.data()));
  return P;
}

// profiles.hpp:266-301 with the exclusion zone exposed: neighbours within
// `excl` of the query window are inadmissible (reference: m/2, :273).
inline MatrixProfile self_join_excl(const TimeSeries& T, std::size_t m, std::size_t excl, unsigned threads = 0,
                                    precision prec = precision::fp64) {
  (void)threads;
  MatrixProfile P;
  P.kind = join_kind::self;
  P.m = m;
  const std::size_t cnt = (m >= 1 && T.n() >= m) ? T.n() - m + 1 : 0;
  P.values.resize(cnt);
  P.indices.resize(cnt);
  detail::raise_status(
      tsd_self_join(T.values.data(), T.n(), m, excl, static_cast<int>(prec), P.values.data(), P.indices.data()));
  return P;
}

inline MatrixProfile self_join(const TimeSeries& T, std::size_t m, unsigned threads = 0) {
  return self_join_excl(T, m, TSD_EXCL_DEFAULT, threads);
}

namespace detail {
inline void check_profile_inputs(const TimeSeries& T, std::span<const double> Q, const SubseqStats& stats) {
  // profiles.hpp:167-172 / :189-194
  if (Q.size() != stats.m) throw error(errc::length_mismatch, "query length does not match stats window length");
  if (stats.count() != T.n() - stats.m + 1)
    throw error(errc::length_mismatch, "stats were computed for a different series length");
}
}  // namespace detail

// profiles.hpp:164-181: znorm_distance per window, on the device with the
// reference's operation order (bit-identical values)
inline DistanceProfile distance_profile_naive(const TimeSeries& T, std::span<const double> Q,
                                              const SubseqStats& stats,
                                              std::optional<std::size_t> query_origin = {}) {
  detail::check_profile_inputs(T, Q, stats);
  DistanceProfile dp;
  dp.m = stats.m;
  dp.query_origin = query_origin;
  dp.values.resize(stats.count());
  if (stats.count() > 0)
    detail::raise_status(tsd_distance_profile_naive(T.values.data(), T.n(), Q.data(), Q.size(), dp.values.data()));
  return dp;
}

// profiles.hpp:186-260: MASS's conventions over the given window statistics
// (constant query / windows, exact origin entry); the sliding dot products
// are exact FP64 on the device instead of an FFT convolution
inline DistanceProfile distance_profile_mass(const TimeSeries& T, std::span<const double> Q,
                                             const SubseqStats& stats,
                                             std::optional<std::size_t> query_origin = {}) {
  detail::check_profile_inputs(T, Q, stats);
  DistanceProfile dp;
  dp.m = stats.m;
  dp.query_origin = query_origin;
  dp.values.resize(stats.count());
  detail::raise_status(tsd_distance_profile_mass(T.values.data(), T.n(), Q.data(), Q.size(), stats.means.data(),
                                                 stats.invn.data(), stats.constant_mask.data(),
                                                 query_origin ? *query_origin : TSD_NO_ORIGIN, dp.values.data()));
  return dp;
}

}  // namespace tsdict

#endif

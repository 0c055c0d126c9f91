// tsdict/series.hpp -- drop-in for /root/reference/proj/include/tsdict/series.hpp.
// Same types and signatures; compute_stats runs on the B200 through the C ABI
// (tsd_compute_stats); corr_to_dist and znorm_distance are scalar host helpers.
#ifndef TSDICT_B200_SERIES_HPP
#define TSDICT_B200_SERIES_HPP

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <span>
#include <vector>

#include "tsdict/errors.hpp"

namespace tsdict {

struct TimeSeries {  // series.hpp:27-31
  std::vector<double> values;
  std::size_t n() const noexcept { return values.size(); }
};

struct SubseqStats {  // series.hpp:37-45
  std::size_t m = 0;
  std::vector<double> means;
  std::vector<double> stds;
  std::vector<double> invn;
  std::vector<unsigned char> constant_mask;
  std::size_t count() const noexcept { return means.size(); }
};

// series.hpp:75-77
inline double constancy_threshold(double max_abs_sample) { return 1e-8 * std::max(1.0, max_abs_sample); }

// series.hpp:83-150 (device: double-double window moments, stats.cu)
inline SubseqStats compute_stats(const TimeSeries& T, std::size_t m) {
  SubseqStats st;
  st.m = m;
  const std::size_t cnt = (m >= 2 && m <= T.n()) ? T.n() - m + 1 : 0;
  st.means.resize(cnt);
  st.stds.resize(cnt);
  st.invn.resize(cnt);
  st.constant_mask.resize(cnt);
  detail::raise_status(tsd_compute_stats(T.values.data(), T.n(), m, st.means.data(), st.stds.data(), st.invn.data(),
                                         st.constant_mask.data()));
  return st;
}

// series.hpp:153-161
inline double corr_to_dist(double rho, std::size_t m) {
  rho = std::min(1.0, std::max(-1.0, rho));
  const double d = std::sqrt(2.0 * static_cast<double>(m) * (1.0 - rho));
  return std::min(std::max(d, 0.0), 2.0 * std::sqrt(static_cast<double>(m)));
}

namespace detail {
struct kahan_sum {  // series.hpp:50-60
  double sum = 0.0, comp = 0.0;
  void add(double x) {
    const double y = x - comp;
    const double t = sum + y;
    comp = (t - sum) - y;
    sum = t;
  }
};
}  // namespace detail

// series.hpp:166-204: z-normalised Euclidean distance of two equal windows;
// flat/flat -> 0, flat/other -> sqrt(2m). Host scalar code with the
// reference's arithmetic (Kahan moments, the pair's constancy threshold), so
// it agrees bit for bit with distance_profile_naive on the device.
inline double znorm_distance(std::span<const double> a, std::span<const double> b) {
  if (a.size() != b.size()) throw error(errc::length_mismatch, "subsequences differ in length");
  const std::size_t m = a.size();
  if (m < 2) throw error(errc::window_too_small, "window length must be at least 2");
  double max_abs = 0.0;
  detail::kahan_sum sa, sb;
  for (std::size_t i = 0; i < m; ++i) {
    sa.add(a[i]);
    sb.add(b[i]);
    max_abs = std::max({max_abs, std::fabs(a[i]), std::fabs(b[i])});
  }
  const double md = static_cast<double>(m), mu_a = sa.sum / md, mu_b = sb.sum / md;
  detail::kahan_sum va, vb, cv;
  for (std::size_t i = 0; i < m; ++i) {
    const double x = a[i] - mu_a, y = b[i] - mu_b;
    va.add(x * x);
    vb.add(y * y);
    cv.add(x * y);
  }
  const double sd_a = std::sqrt(std::max(0.0, va.sum / md)), sd_b = std::sqrt(std::max(0.0, vb.sum / md));
  const double eps = constancy_threshold(max_abs);
  const bool fa = sd_a < eps, fb = sd_b < eps;
  if (fa && fb) return 0.0;
  if (fa || fb) return std::sqrt(2.0 * md);
  return corr_to_dist(cv.sum / (md * (sd_a * sd_b)), m);
}

}  // namespace tsdict

#endif

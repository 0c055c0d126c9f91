// Fixed objects both I/O implementations format and parse in the cross-checks
// (tests/cpp/test_io.cpp against ours, oracle/ref_io.cpp against the unmodified
// reference io.hpp). Only tsdict type names and members both define.
#pragma once
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

namespace io_objects {

inline double sample(std::uint64_t i) {  // awkward doubles: signs, tiny, huge, non-terminating binary
  const double base = std::sin(0.37 * static_cast<double>(i)) * std::pow(10.0, static_cast<double>(i % 23) - 11.0);
  return (i % 7 == 3) ? -base / 3.0 : base + static_cast<double>(i % 5) * 0.1;
}

inline tsdict::TimeSeries series() {
  tsdict::TimeSeries T;
  for (std::uint64_t i = 0; i < 60; ++i) T.values.push_back(sample(i));
  T.values.push_back(0.0);
  T.values.push_back(-0.0);
  T.values.push_back(std::numeric_limits<double>::denorm_min());
  T.values.push_back(std::numeric_limits<double>::max());
  return T;
}

inline tsdict::Dictionary dictionary(bool with_emax) {
  tsdict::Dictionary D;
  D.m = 16;
  D.k = 1.5;
  D.source_length = 1000;
  const std::uint64_t starts[3] = {0, 20, 300}, lens[3] = {20, 17, 30};  // touching first two
  std::uint64_t stored = 0;
  for (int s = 0; s < 3; ++s) {
    tsdict::Segment g;
    g.start = starts[s];
    for (std::uint64_t i = 0; i < lens[s]; ++i) g.values.push_back(sample(starts[s] + i));
    stored += lens[s];
    D.segments.push_back(g);
  }
  D.core_starts = {2, 25, 310};
  D.space_saving = 1.0 - static_cast<double>(stored) / 1000.0;
  if (with_emax) D.e_max = 3.141592653589793;
  return D;
}

inline tsdict::MatrixProfile profile(bool self) {
  tsdict::MatrixProfile P;
  P.m = self ? 8 : 12;
  P.kind = self ? tsdict::join_kind::self : tsdict::join_kind::ab;
  for (std::uint64_t i = 0; i < 40; ++i) {
    P.values.push_back(std::fabs(sample(i)) * 2.0);
    P.indices.push_back(static_cast<std::int64_t>((i * 7) % 33));
  }
  P.values[4] = std::numeric_limits<double>::infinity();  // sentinel row
  P.indices[4] = -1;
  return P;
}

inline std::vector<tsdict::interval> labels() { return {{500, 600}, {5, 10}, {550, 700}, {10, 20}}; }

}  // namespace io_objects

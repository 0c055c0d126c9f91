// ORACLE / TEST INFRASTRUCTURE ONLY. Runs the unmodified reference file
// formats (/root/reference/proj/include/tsdict/io.hpp, with the nlohmann
// JSON header it includes) over the parity cases of tests/cpp/io_cases.hpp
// and prints one golden line per case:
//   <kind>\t<name>\t<result>
// result = the reference's errc name, or "ok:" + the canonical dump of what
// it parsed. Then the formatter goldens: "format\t<what>\t<hex bytes>".
// With "read-dict <file>" it parses one dictionary document (written by the
// drop-in) and prints its canonical dump: the cross-reading check.
// Built by oracle/Makefile (target ref_io) into oracle/_ref/.
#include <cstdio>
#include <iostream>

#include "tsdict/io.hpp"

#include "../tests/cpp/io_cases.hpp"

using namespace tsdict;

static std::string run(const io_cases::Case& c) {
  try {
    if (c.kind == "series") return "ok:" + io_cases::canon_series(parse_series(c.input));
    if (c.kind == "dictionary") return "ok:" + io_cases::canon_dictionary(parse_dictionary(c.input));
    if (c.kind == "profile") return "ok:" + io_cases::canon_profile(parse_profile(c.input));
    if (c.kind == "labels") return "ok:" + io_cases::canon_labels(parse_labels(c.input));
    return "unknown-kind";
  } catch (const error& e) {
    return errc_name(e.code());
  }
}

int main(int argc, char** argv) {
  if (argc == 3 && std::string(argv[1]) == "read-dict") {
    std::cout << run({"dictionary", "x", detail::slurp(argv[2])}) << "\n";
    return 0;
  }
  for (const auto& c : io_cases::cases()) std::cout << c.kind << "\t" << c.name << "\t" << run(c) << "\n";
  // formatter goldens
  TimeSeries T;
  T.values = io_cases::sample_values();
  std::cout << "format\tseries_text\t" << io_cases::hex_bytes(format_series_text(T)) << "\n";
  std::cout << "format\tseries_binary\t" << io_cases::hex_bytes(format_series_binary(T)) << "\n";
  MatrixProfile P;
  P.m = 7;
  P.kind = join_kind::ab;
  P.values = io_cases::sample_values();
  for (double& v : P.values) v = std::fabs(v);
  P.values.push_back(std::numeric_limits<double>::infinity());
  for (std::size_t i = 0; i < P.values.size(); ++i) P.indices.push_back(static_cast<std::int64_t>(i * 37 % 101) - 1);
  std::cout << "format\tprofile\t" << io_cases::hex_bytes(format_profile(P)) << "\n";
  P.kind = join_kind::self;
  std::cout << "format\tprofile_self\t" << io_cases::hex_bytes(format_profile(P)) << "\n";
  std::vector<interval> L = {{0, 5}, {7, 9}, {100, 1000000000000ull}};
  std::cout << "format\tlabels\t" << io_cases::hex_bytes(format_labels(L)) << "\n";
  Dictionary D;
  D.m = 4;
  D.k = 1.5;
  D.source_length = 200;
  D.core_starts = {3, 60};
  D.e_max = 0.125;
  Segment s1{0, {}}, s2{50, {}};
  const auto sv = io_cases::sample_values();
  s1.values.assign(sv.begin(), sv.begin() + 20);
  s2.values.assign(sv.begin() + 20, sv.end());
  D.segments = {s1, s2};
  D.space_saving = 1.0 - static_cast<double>(s1.values.size() + s2.values.size()) / 200.0;
  std::cout << "format\tdictionary\t" << io_cases::hex_bytes(format_dictionary(D)) << "\n";
  return 0;
}

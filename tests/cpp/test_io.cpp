// Drop-in file formats (include/tsdict/io.hpp) against the reference's
// goldens (tests/golden/io_golden.tsv, made by tests/golden/make_io_golden.sh
// from the unmodified reference io.hpp): every parser case must give the
// reference's error code or the same parsed values bit for bit; series,
// profile and label formatters must reproduce the reference's bytes; a
// dictionary written here must read back identically in both
// implementations. Host code only (no GPU).
//   test_io <golden.tsv>        run the checks (exit 1 on any mismatch)
//   test_io emit-dict <file>    write this writer's golden dictionary
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>

#include "tsdict/io.hpp"

#include "io_cases.hpp"

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

static Dictionary golden_dictionary() {  // the same document as oracle/ref_io_golden.cpp
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
  return D;
}

int main(int argc, char** argv) {
  if (argc == 3 && std::string(argv[1]) == "emit-dict") {
    detail::write_file(argv[2], format_dictionary(golden_dictionary()));
    return 0;
  }
  if (argc != 2) {
    std::cerr << "usage: test_io <golden.tsv> | emit-dict <file>\n";
    return 2;
  }
  std::map<std::string, std::string> gold;
  {
    std::ifstream in(argv[1]);
    std::string line;
    while (std::getline(in, line)) {
      const auto a = line.find('\t'), b = line.find('\t', a + 1);
      if (a == std::string::npos || b == std::string::npos) continue;
      gold[line.substr(0, b)] = line.substr(b + 1);
    }
  }
  int bad = 0, n = 0;
  auto check = [&](const std::string& key, const std::string& got) {
    ++n;
    auto it = gold.find(key);
    if (it == gold.end() || it->second != got) {
      ++bad;
      std::cerr << "MISMATCH " << key << "\n  reference: " << (it == gold.end() ? "<missing>" : it->second)
                << "\n  drop-in:   " << got << "\n";
    }
  };
  for (const auto& c : io_cases::cases()) check(c.kind + "\t" + c.name, run(c));

  TimeSeries T;
  T.values = io_cases::sample_values();
  check("format\tseries_text", io_cases::hex_bytes(format_series_text(T)));
  check("format\tseries_binary", io_cases::hex_bytes(format_series_binary(T)));
  MatrixProfile P;
  P.m = 7;
  P.kind = join_kind::ab;
  P.values = io_cases::sample_values();
  for (double& v : P.values) v = std::fabs(v);
  P.values.push_back(std::numeric_limits<double>::infinity());
  for (std::size_t i = 0; i < P.values.size(); ++i) P.indices.push_back(static_cast<std::int64_t>(i * 37 % 101) - 1);
  check("format\tprofile", io_cases::hex_bytes(format_profile(P)));
  P.kind = join_kind::self;
  check("format\tprofile_self", io_cases::hex_bytes(format_profile(P)));
  std::vector<interval> L = {{0, 5}, {7, 9}, {100, 1000000000000ull}};
  check("format\tlabels", io_cases::hex_bytes(format_labels(L)));

  // round trips through this implementation, bit for bit
  auto same = [&](const char* what, const std::string& a, const std::string& b) {
    ++n;
    if (a != b) {
      ++bad;
      std::cerr << "ROUND TRIP " << what << "\n  " << a << "\n  " << b << "\n";
    }
  };
  same("series text", io_cases::canon_series(T), io_cases::canon_series(parse_series(format_series_text(T))));
  same("series binary", io_cases::canon_series(T), io_cases::canon_series(parse_series(format_series_binary(T))));
  same("profile", io_cases::canon_profile(P), io_cases::canon_profile(parse_profile(format_profile(P))));
  same("labels", io_cases::canon_labels(L), io_cases::canon_labels(parse_labels(format_labels(L))));
  const Dictionary D = golden_dictionary();
  same("dictionary", io_cases::canon_dictionary(D), io_cases::canon_dictionary(parse_dictionary(format_dictionary(D))));
  // the reference's dictionary text reads back to the same values here...
  auto it = gold.find("format\tdictionary");
  if (it != gold.end())
    same("reference dictionary text", io_cases::canon_dictionary(D),
         io_cases::canon_dictionary(parse_dictionary(io_cases::unhex(it->second))));
  // ...and this writer's text (unchanged since the golden run) read back to
  // the same values in the reference
  check("crossread\twriter", io_cases::hex_bytes(format_dictionary(D)));
  // byte identity with the reference's own text for this document
  check("format\tdictionary", io_cases::hex_bytes(format_dictionary(D)));
  check("crossread\treference_reads", "ok:" + io_cases::canon_dictionary(D));

  std::cout << "io parity: " << n - bad << " of " << n << " checks match the reference\n";
  return bad ? 1 : 0;
}

// test_io.cpp -- the drop-in file formats (include/tsdict/io.hpp) against the
// unmodified reference io.hpp, through committed golden data
// (tests/golden/io/make_io_golden.py, which ran the reference here):
//   1. the reference-written files of tests/golden/io/ref parse to exactly the
//      objects of tests/golden/io/objects.hpp;
//   2. every document of tests/golden/io/cases.tsv (valid ones and
//      deterministic corruptions) gets the reference parser's outcome: accepted,
//      or rejected with the same errc;
//   3. our formatters round-trip every object bit-exactly, and write the
//      object files into argv[1] (tests/test_cpu.py hands them to the reference
//      parser when the reference is present);
//   4. behaviours the reference's test_io.cpp names (file errors, null e_max,
//      row counts, label merging).
// usage: test_io OUT_DIR GOLDEN_DIR
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>

#include "tsdict/io.hpp"
#include "objects.hpp"

namespace {

int g_fail = 0, g_pass = 0;

void check(bool ok, const std::string& what) {
  if (ok) {
    ++g_pass;
  } else {
    ++g_fail;
    std::printf("[FAIL] %s\n", what.c_str());
  }
}

std::string b64decode(const std::string& in) {
  auto val = [](char c) -> int {
    if (c >= 'A' && c <= 'Z') return c - 'A';
    if (c >= 'a' && c <= 'z') return c - 'a' + 26;
    if (c >= '0' && c <= '9') return c - '0' + 52;
    if (c == '+') return 62;
    if (c == '/') return 63;
    return -1;
  };
  std::string out;
  unsigned acc = 0;
  int bits = 0;
  for (char c : in) {
    const int v = val(c);
    if (v < 0) continue;  // '=' padding
    acc = (acc << 6) | unsigned(v);
    bits += 6;
    if (bits >= 8) {
      bits -= 8;
      out += char((acc >> bits) & 0xFF);
    }
  }
  return out;
}

bool bits_equal(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), 8 * a.size()) == 0);
}

bool same_dict(const tsdict::Dictionary& a, const tsdict::Dictionary& b) {
  if (a.m != b.m || a.source_length != b.source_length || a.core_starts != b.core_starts ||
      std::memcmp(&a.k, &b.k, 8) || std::memcmp(&a.space_saving, &b.space_saving, 8) ||
      a.e_max.has_value() != b.e_max.has_value() || (a.e_max && std::memcmp(&*a.e_max, &*b.e_max, 8)) ||
      a.segments.size() != b.segments.size())
    return false;
  for (size_t s = 0; s < a.segments.size(); ++s)
    if (a.segments[s].start != b.segments[s].start || !bits_equal(a.segments[s].values, b.segments[s].values))
      return false;
  return true;
}

bool same_profile(const tsdict::MatrixProfile& a, const tsdict::MatrixProfile& b) {
  return a.m == b.m && a.kind == b.kind && a.indices == b.indices && bits_equal(a.values, b.values);
}

// outcome of one parse: "ok" or the errc ordinal (the reference driver's encoding)
std::string outcome(const std::string& kind, const std::string& doc) {
  try {
    if (kind == "series") (void)tsdict::parse_series(doc);
    else if (kind == "dictionary") (void)tsdict::parse_dictionary(doc);
    else if (kind == "profile") (void)tsdict::parse_profile(doc);
    else if (kind == "labels") (void)tsdict::parse_labels(doc);
    else return "unknown-kind";
    return "ok";
  } catch (const tsdict::error& e) {
    return std::to_string(static_cast<int>(e.code()));
  } catch (const std::exception&) {
    return "other";
  }
}

template <class F>
void expect_code(F&& f, tsdict::errc want, const std::string& what) {
  try {
    f();
    check(false, what + ": no error");
  } catch (const tsdict::error& e) {
    check(e.code() == want, what + ": " + e.what());
  }
}

}  // namespace

int main(int argc, char** argv) {
  using namespace tsdict;
  if (argc < 3) {
    std::fprintf(stderr, "usage: test_io OUT_DIR GOLDEN_DIR\n");
    return 64;
  }
  const std::string out = std::string(argv[1]) + "/", gold = std::string(argv[2]) + "/";
  const TimeSeries T = io_objects::series();
  const Dictionary D = io_objects::dictionary(true), Dn = io_objects::dictionary(false);
  const MatrixProfile Ps = io_objects::profile(true), Pa = io_objects::profile(false);

  // 1. reference-written files
  try {
    check(bits_equal(read_series(gold + "ref/series.txt").values, T.values), "reference series.txt");
    check(bits_equal(read_series(gold + "ref/series.mpd1").values, T.values), "reference series.mpd1");
    check(same_dict(read_dictionary(gold + "ref/dict.json"), D), "reference dict.json");
    check(same_dict(read_dictionary(gold + "ref/dict_null_emax.json"), Dn), "reference dict_null_emax.json");
    check(same_profile(read_profile(gold + "ref/profile_self.tsv"), Ps), "reference profile_self.tsv");
    check(same_profile(read_profile(gold + "ref/profile_ab.tsv"), Pa), "reference profile_ab.tsv");
    check(read_labels(gold + "ref/labels.tsv") == merge_intervals(io_objects::labels()), "reference labels.tsv");
  } catch (const std::exception& e) {
    check(false, std::string("reading the reference files: ") + e.what());
  }

  // 2. every golden document: the reference parser's outcome
  {
    std::ifstream f(gold + "cases.tsv");
    check(bool(f), "cases.tsv present");
    std::string line;
    int n = 0, diff = 0;
    while (std::getline(f, line)) {
      const size_t t1 = line.find('\t'), t2 = line.find('\t', t1 + 1);
      const std::string kind = line.substr(0, t1), want = line.substr(t1 + 1, t2 - t1 - 1);
      const std::string doc = b64decode(line.substr(t2 + 1));
      const std::string got = outcome(kind, doc);
      ++n;
      if (got != want) {
        ++diff;
        if (diff <= 10) std::printf("  case %d (%s): reference %s, drop-in %s\n", n, kind.c_str(), want.c_str(), got.c_str());
      }
    }
    check(n > 400 && diff == 0, "golden cases: " + std::to_string(n - diff) + " of " + std::to_string(n) +
                                    " with the reference outcome");
  }

  // 3. round trips, and our files for the reference parser
  try {
    check(bits_equal(parse_series(format_series_text(T)).values, T.values), "series text round trip");
    check(bits_equal(parse_series(format_series_binary(T)).values, T.values), "series binary round trip");
    check(same_dict(parse_dictionary(format_dictionary(D)), D), "dictionary round trip");
    check(same_dict(parse_dictionary(format_dictionary(Dn)), Dn), "dictionary round trip (null e_max)");
    check(same_profile(parse_profile(format_profile(Ps)), Ps), "self profile round trip");
    check(same_profile(parse_profile(format_profile(Pa)), Pa), "ab profile round trip");
    write_series_text(out + "series.txt", T);
    write_series_binary(out + "series.mpd1", T);
    write_dictionary(out + "dict.json", D);
    write_dictionary(out + "dict_null_emax.json", Dn);
    write_profile(out + "profile_self.tsv", Ps);
    write_profile(out + "profile_ab.tsv", Pa);
    write_labels(out + "labels.tsv", io_objects::labels());
    check(bits_equal(read_series(out + "series.mpd1").values, T.values), "series file round trip");
  } catch (const std::exception& e) {
    check(false, std::string("round trips: ") + e.what());
  }

  // 4. named behaviours (reference test_io.cpp)
  {
    TimeSeries t2;
    t2.values = {1.5, -2.0};
    check(format_series_text(t2) == "# n=2\n1.5\n-2\n", "text series shape");  // test_io.cpp:72-76
    const std::string blob = format_series_binary(t2);
    check(blob.size() == 12 + 16 && blob.substr(0, 4) == "MPD1", "binary series shape");
    check(format_dictionary(Dn).find("\"e_max\":null") != std::string::npos, "null e_max written as null");
    expect_code([&] { (void)read_series(out + "does_not_exist.bin"); }, errc::io_error, "missing file");
    expect_code([&] { write_series_text("/nonexistent_dir/x.txt", t2); }, errc::io_error, "unwritable file");
    const std::string prof = format_profile(Ps);
    size_t rows = 0;
    for (char c : prof) rows += c == '\n';
    check(rows == 2 + Ps.values.size(), "profile rows = meta + header + windows");
    const auto merged = parse_labels(format_labels({{10, 50}, {40, 90}}));
    check(merged.size() == 1 && merged[0] == interval{10, 90}, "overlapping labels merge");
    const auto kept = parse_labels(format_labels({{20, 30}, {5, 10}}));
    check(kept.size() == 2 && kept[0] == interval{5, 10} && kept[1] == interval{20, 30}, "disjoint labels sorted");
    Dictionary touching;  // test_io.cpp:188-201
    touching.m = 10;
    touching.source_length = 200;
    touching.segments.push_back({0, std::vector<double>(50, 1.0)});
    touching.segments.push_back({50, std::vector<double>(10, 2.0)});
    touching.core_starts = {20, 52};
    touching.space_saving = 1.0 - 60.0 / 200.0;
    check(parse_dictionary(format_dictionary(touching)).segments.size() == 2, "touching segments are legal");
  }

  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}

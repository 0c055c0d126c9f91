// ref_io.cpp -- ORACLE BUILD ONLY (test infrastructure).
//
// Drives the UNMODIFIED reference io.hpp (/root/reference/proj/include) for
// the I/O cross-checks; built by oracle/Makefile into oracle/_ref/ref_io when
// /root/reference and an nlohmann json.hpp are present. Modes:
//   ref_io write DIR   format the fixed objects of tests/golden/io/objects.hpp
//                      with the reference formatters into DIR
//   ref_io read DIR    parse DIR (written by our formatters) with the
//                      reference parsers; exit 0 when every object matches
//   ref_io codes       per stdin line "<kind>\t<hex document>": the
//                      reference parser's outcome ("ok" or its errc ordinal)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <string>

#include "tsdict/io.hpp"
#include "objects.hpp"

namespace {

std::string unhex(const std::string& h) {
  std::string out(h.size() / 2, '\0');
  for (size_t i = 0; i < out.size(); ++i) out[i] = (char)std::stoi(h.substr(2 * i, 2), nullptr, 16);
  return out;
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

bool same(const tsdict::TimeSeries& a, const tsdict::TimeSeries& b) {
  if (a.values.size() != b.values.size()) return false;
  for (size_t i = 0; i < a.values.size(); ++i)
    if (!same_bits(a.values[i], b.values[i])) return false;
  return true;
}

bool same(const tsdict::Dictionary& a, const tsdict::Dictionary& b) {
  if (a.m != b.m || !same_bits(a.k, b.k) || a.source_length != b.source_length ||
      !same_bits(a.space_saving, b.space_saving) || a.core_starts != b.core_starts ||
      a.e_max.has_value() != b.e_max.has_value() || (a.e_max && !same_bits(*a.e_max, *b.e_max)) ||
      a.segments.size() != b.segments.size())
    return false;
  for (size_t s = 0; s < a.segments.size(); ++s) {
    if (a.segments[s].start != b.segments[s].start) return false;
    tsdict::TimeSeries x{a.segments[s].values}, y{b.segments[s].values};
    if (!same(x, y)) return false;
  }
  return true;
}

bool same(const tsdict::MatrixProfile& a, const tsdict::MatrixProfile& b) {
  tsdict::TimeSeries x{a.values}, y{b.values};
  return a.m == b.m && a.kind == b.kind && a.indices == b.indices && same(x, y);
}

int check(bool ok, const char* what) {
  if (!ok) std::printf("MISMATCH %s\n", what);
  return ok ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  using namespace tsdict;
  const std::string mode = argc > 1 ? argv[1] : "";
  if (mode == "write" && argc > 2) {
    const std::string d = std::string(argv[2]) + "/";
    write_series_text(d + "series.txt", io_objects::series());
    write_series_binary(d + "series.mpd1", io_objects::series());
    write_dictionary(d + "dict.json", io_objects::dictionary(true));
    write_dictionary(d + "dict_null_emax.json", io_objects::dictionary(false));
    write_profile(d + "profile_self.tsv", io_objects::profile(true));
    write_profile(d + "profile_ab.tsv", io_objects::profile(false));
    write_labels(d + "labels.tsv", io_objects::labels());
    return 0;
  }
  if (mode == "read" && argc > 2) {
    const std::string d = std::string(argv[2]) + "/";
    int bad = 0;
    try {
      bad += check(same(read_series(d + "series.txt"), io_objects::series()), "series.txt");
      bad += check(same(read_series(d + "series.mpd1"), io_objects::series()), "series.mpd1");
      bad += check(same(read_dictionary(d + "dict.json"), io_objects::dictionary(true)), "dict.json");
      bad += check(same(read_dictionary(d + "dict_null_emax.json"), io_objects::dictionary(false)),
                   "dict_null_emax.json");
      bad += check(same(read_profile(d + "profile_self.tsv"), io_objects::profile(true)), "profile_self.tsv");
      bad += check(same(read_profile(d + "profile_ab.tsv"), io_objects::profile(false)), "profile_ab.tsv");
      bad += check(read_labels(d + "labels.tsv") == merge_intervals(io_objects::labels()), "labels.tsv");
    } catch (const error& e) {
      std::printf("ERROR %s\n", e.what());
      return 2;
    }
    std::printf(bad ? "FAILED\n" : "OK\n");
    return bad ? 1 : 0;
  }
  if (mode == "codes") {
    std::string line;
    while (std::getline(std::cin, line)) {
      const size_t tab = line.find('\t');
      const std::string kind = line.substr(0, tab), doc = unhex(line.substr(tab + 1));
      try {
        if (kind == "series") (void)parse_series(doc);
        else if (kind == "dictionary") (void)parse_dictionary(doc);
        else if (kind == "profile") (void)parse_profile(doc);
        else if (kind == "labels") (void)parse_labels(doc);
        std::printf("ok\n");
      } catch (const error& e) {
        std::printf("%d\n", static_cast<int>(e.code()));
      } catch (const std::exception& e) {
        std::printf("other\n");
      }
    }
    return 0;
  }
  std::fprintf(stderr, "usage: ref_io write DIR | read DIR | codes\n");
  return 64;
}

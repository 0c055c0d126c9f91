// io_cases.hpp -- the file-format parity cases, shared by the reference-side
// golden generator (oracle/ref_io_golden.cpp, built against the unmodified
// reference io.hpp) and the drop-in's test (tests/cpp/test_io.cpp). Test
// infrastructure only.
//
// Templates work on either implementation's types (the drop-in keeps the
// reference's member names). A case is (kind, name, input bytes); its result
// is the error code name the parser raises, or "ok:" + a canonical dump of
// what it parsed (doubles as bit patterns).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <utility>
#include <vector>

namespace io_cases {

struct Case {
  std::string kind;  // series | dictionary | profile | labels
  std::string name;
  std::string input;
};

inline std::string hex_bytes(const std::string& s) {
  static const char* d = "0123456789abcdef";
  std::string o;
  for (unsigned char c : s) {
    o += d[c >> 4];
    o += d[c & 15];
  }
  return o;
}
inline std::string unhex(const std::string& h) {
  std::string o;
  for (std::size_t i = 0; i + 1 < h.size(); i += 2) {
    auto v = [](char c) { return c <= '9' ? c - '0' : c - 'a' + 10; };
    o += static_cast<char>(v(h[i]) * 16 + v(h[i + 1]));
  }
  return o;
}
inline std::string bits(double v) {
  std::uint64_t u;
  std::memcpy(&u, &v, 8);
  char b[32];
  std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(u));
  return b;
}

template <class TS>
std::string canon_series(const TS& T) {
  std::string o = "n=" + std::to_string(T.values.size());
  for (double v : T.values) o += " " + bits(v);
  return o;
}
template <class D>
std::string canon_dictionary(const D& d) {
  std::string o = "m=" + std::to_string(d.m) + " k=" + bits(d.k) + " src=" + std::to_string(d.source_length) +
                  " ss=" + bits(d.space_saving) + " emax=" + (d.e_max ? bits(*d.e_max) : std::string("none")) +
                  " cores=";
  for (auto c : d.core_starts) o += std::to_string(c) + ",";
  for (const auto& s : d.segments) {
    o += " seg@" + std::to_string(s.start) + ":";
    for (double v : s.values) o += bits(v) + ",";
  }
  return o;
}
template <class P>
std::string canon_profile(const P& p) {
  std::string o = "m=" + std::to_string(p.m) + " kind=" + std::to_string(static_cast<int>(p.kind));
  for (std::size_t i = 0; i < p.values.size(); ++i) o += " " + bits(p.values[i]) + "/" + std::to_string(p.indices[i]);
  return o;
}
template <class L>
std::string canon_labels(const L& regions) {
  std::string o = "regions";
  for (const auto& r : regions) o += " " + std::to_string(r.first) + "-" + std::to_string(r.second);
  return o;
}

// sample data for the formatter cases: ordinary values, exact integers,
// tiny / huge magnitudes, negative zero, subnormals, values whose shortest
// decimal is long
inline std::vector<double> sample_values() {
  std::vector<double> v = {0.0,    -0.0,   1.0,     -1.0,     0.1,          1.0 / 3.0, 2.5e-300,
                           1e300,  123456789.0, -9007199254740993.0, 4.9e-324, 2.2250738585072014e-308,
                           1e-7,   1e21,   1e15,    1e16,     0.000123,     -7.25,     3.141592653589793};
  for (int i = 0; i < 40; ++i) v.push_back(std::sin(0.37 * i) * std::pow(10.0, (i % 9) - 4));
  return v;
}

inline std::vector<Case> cases() {
  std::vector<Case> c;
  auto add = [&](const char* k, const char* n, std::string in) { c.push_back({k, n, std::move(in)}); };
  auto bin = [](std::uint64_t n, const std::vector<double>& vals, std::size_t cut = 0) {
    std::string s = "MPD1";
    s.append(reinterpret_cast<const char*>(&n), 8);
    s.append(reinterpret_cast<const char*>(vals.data()), 8 * vals.size());
    if (cut) s.resize(s.size() - cut);
    return s;
  };
  // ---- series
  add("series", "text_plain", "1\n2.5\n-3e-5\n");
  add("series", "text_header", "# n=3\n1\n2\n3\n");
  add("series", "text_blank_lines_and_cr", "\n  # n=2\r\n\n 4 \r\n\t5\n\n");
  add("series", "text_no_trailing_newline", "7\n8");
  add("series", "text_header_mismatch", "# n=4\n1\n2\n");
  add("series", "text_header_after_data", "1\n# n=1\n");
  add("series", "text_two_headers", "# n=1\n# n=1\n1\n");
  add("series", "text_bad_header", "# count=3\n1\n");
  add("series", "text_short_header", "# n\n1\n");
  add("series", "text_bad_sample", "1\nx2\n");
  add("series", "text_two_numbers", "1 2\n");
  add("series", "text_inf", "1\ninf\n");
  add("series", "text_nan", "nan\n");
  add("series", "text_empty", "");
  add("series", "text_only_header", "# n=0\n");
  add("series", "text_hex_float", "0x1p3\n");
  add("series", "text_plus_sign", "+1\n");
  add("series", "bin_ok", bin(3, {1.0, -2.0, 0.5}));
  add("series", "bin_truncated_count", std::string("MPD1\x03\x00", 6));
  add("series", "bin_length_mismatch", bin(3, {1.0, -2.0, 0.5}, 3));
  add("series", "bin_count_mismatch", bin(4, {1.0, -2.0, 0.5}));
  add("series", "bin_zero", bin(0, {}));
  add("series", "bin_nan", bin(2, {1.0, std::numeric_limits<double>::quiet_NaN()}));
  add("series", "bin_inf", bin(1, {-std::numeric_limits<double>::infinity()}));
  add("series", "bin_huge_count", bin(0x2000000000000001ull, {1.0}));
  // ---- dictionary
  const std::string seg = R"({"start":2,"length":4,"values":[1.0,2.0,-3.5,4.0]})";
  const std::string base = R"("m":3,"k":1.5,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[2])";
  auto dict = [&](const std::string& fields, const std::string& segs) {
    return "{\"format_version\":1," + fields + ",\"segments\":[" + segs + "]}";
  };
  add("dictionary", "ok", dict(base, seg));
  add("dictionary", "ok_whitespace", " \n{ \"format_version\" : 1 , " + base + " , \"segments\" : [ " + seg + " ] }\n\t");
  add("dictionary", "ok_null_emax",
      dict(R"("m":3,"k":0,"source_length":10,"space_saving":0.6,"e_max":null,"core_starts":[])", seg));
  add("dictionary", "ok_two_segments",
      dict(R"("m":2,"k":2,"source_length":20,"space_saving":0.6,"e_max":1e-3,"core_starts":[0,5])",
           R"({"start":0,"length":4,"values":[1,2,3,4]},{"start":6,"length":4,"values":[5,6.5e0,7E1,-8]})"));
  add("dictionary", "ok_escaped_key_order", R"({"segments":[)" + seg + R"(],"core_starts":[2],"e_max":0.25,"space_saving":0.6,"source_length":10,"k":1.5,"m":3,"format_version":1})");
  add("dictionary", "not_json", "{\"format_version\":1,");
  add("dictionary", "trailing_garbage", dict(base, seg) + "x");
  add("dictionary", "not_object", "[1,2,3]");
  add("dictionary", "missing_version", "{" + base + ",\"segments\":[" + seg + "]}");
  add("dictionary", "version_2", "{\"format_version\":2," + base + ",\"segments\":[" + seg + "]}");
  add("dictionary", "version_float", "{\"format_version\":1.0," + base + ",\"segments\":[" + seg + "]}");
  add("dictionary", "unknown_field", "{\"format_version\":1,\"extra\":0," + base + ",\"segments\":[" + seg + "]}");
  add("dictionary", "missing_m", dict(R"("k":1.5,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[2])", seg));
  add("dictionary", "m_too_small", dict(R"("m":1,"k":1.5,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[])", seg));
  add("dictionary", "m_negative", dict(R"("m":-3,"k":1.5,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[2])", seg));
  add("dictionary", "m_float", dict(R"("m":3.0,"k":1.5,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[2])", seg));
  add("dictionary", "k_negative", dict(R"("m":3,"k":-1,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[2])", seg));
  add("dictionary", "k_string", dict(R"("m":3,"k":"1.5","source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[2])", seg));
  add("dictionary", "k_overflow", dict(R"("m":3,"k":1e400,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[2])", seg));
  add("dictionary", "emax_negative", dict(R"("m":3,"k":1.5,"source_length":10,"space_saving":0.6,"e_max":-0.5,"core_starts":[2])", seg));
  add("dictionary", "missing_emax", dict(R"("m":3,"k":1.5,"source_length":10,"space_saving":0.6,"core_starts":[2])", seg));
  add("dictionary", "cores_not_array", dict(R"("m":3,"k":1.5,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":2)", seg));
  add("dictionary", "core_out_of_range", dict(R"("m":3,"k":1.5,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[8])", seg));
  add("dictionary", "cores_too_close", dict(R"("m":4,"k":1.5,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[2,4])", seg));
  add("dictionary", "segments_empty", dict(base, ""));
  add("dictionary", "segment_not_object", dict(base, "[1]"));
  add("dictionary", "segment_unknown_field", dict(base, R"({"start":2,"length":4,"values":[1,2,3,4],"id":7})"));
  add("dictionary", "segment_too_short", dict(base, R"({"start":2,"length":2,"values":[1,2]})"));
  add("dictionary", "segment_past_source", dict(base, R"({"start":8,"length":4,"values":[1,2,3,4]})"));
  add("dictionary", "segments_overlap",
      dict(R"("m":3,"k":1.5,"source_length":20,"space_saving":0.6,"e_max":0.25,"core_starts":[2])",
           R"({"start":2,"length":4,"values":[1,2,3,4]},{"start":5,"length":4,"values":[1,2,3,4]})"));
  add("dictionary", "values_length_mismatch", dict(base, R"({"start":2,"length":4,"values":[1,2,3]})"));
  add("dictionary", "value_not_number", dict(base, R"({"start":2,"length":4,"values":[1,2,null,4]})"));
  add("dictionary", "value_overflow", dict(base, R"({"start":2,"length":4,"values":[1,2,-1e999,4]})"));
  add("dictionary", "space_saving_mismatch",
      dict(R"("m":3,"k":1.5,"source_length":10,"space_saving":0.5,"e_max":0.25,"core_starts":[2])", seg));
  add("dictionary", "source_length_zero", dict(R"("m":3,"k":1.5,"source_length":0,"space_saving":0.6,"e_max":0.25,"core_starts":[])", seg));
  add("dictionary", "leading_zero", dict(R"("m":03,"k":1.5,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[2])", seg));
  add("dictionary", "nan_literal", dict(R"("m":3,"k":NaN,"source_length":10,"space_saving":0.6,"e_max":0.25,"core_starts":[2])", seg));
  add("dictionary", "empty", "");
  // ---- profile
  add("profile", "ok", "# m=4 kind=self-join\nwindow_start\tdistance\tnn_index\n0\t1.5\t3\n1\tinf\t-1\n2\t0\t0\n");
  add("profile", "ok_ab_commas", "#m=2 kind=ab-join\nwindow_start\tdistance\tnn_index\n0,2.25,7\n1 0.5 2\n");
  add("profile", "no_meta", "window_start\tdistance\tnn_index\n0\t1\t1\n");
  add("profile", "meta_one_field", "# m=4\nwindow_start\tdistance\tnn_index\n0\t1\t1\n");
  add("profile", "m_too_small", "# m=1 kind=self-join\nwindow_start\tdistance\tnn_index\n0\t1\t1\n");
  add("profile", "unknown_kind", "# m=4 kind=cross\nwindow_start\tdistance\tnn_index\n0\t1\t1\n");
  add("profile", "bad_header", "# m=4 kind=ab-join\nstart\tdistance\tnn\n0\t1\t1\n");
  add("profile", "two_columns", "# m=4 kind=ab-join\nwindow_start\tdistance\tnn_index\n0\t1\n");
  add("profile", "not_consecutive", "# m=4 kind=ab-join\nwindow_start\tdistance\tnn_index\n0\t1\t1\n2\t1\t1\n");
  add("profile", "negative_distance", "# m=4 kind=ab-join\nwindow_start\tdistance\tnn_index\n0\t-1\t1\n");
  add("profile", "nan_distance", "# m=4 kind=ab-join\nwindow_start\tdistance\tnn_index\n0\tnan\t1\n");
  add("profile", "index_below_sentinel", "# m=4 kind=ab-join\nwindow_start\tdistance\tnn_index\n0\t1\t-2\n");
  add("profile", "no_rows", "# m=4 kind=ab-join\nwindow_start\tdistance\tnn_index\n");
  add("profile", "header_missing", "# m=4 kind=ab-join\n");
  // ---- labels
  add("labels", "ok_merge", "# start\tend\n10\t20\n5 12\n30,40\n40\t41\n");
  add("labels", "ok_no_header", "3 4\n");
  add("labels", "one_field", "10\n");
  add("labels", "three_fields", "1 2 3\n");
  add("labels", "start_not_before_end", "5 5\n");
  add("labels", "negative", "-1 4\n");
  add("labels", "none", "# start\tend\n");
  return c;
}

}  // namespace io_cases

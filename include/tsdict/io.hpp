// tsdict/io.hpp -- the reference's file formats (reference io.hpp:1-20 lists
// them; its tests, test_io.cpp:59-361, pin the behaviour), written for this
// drop-in from that description. Host-only code, off the GPU path: it feeds
// the join entry points from files, as the reference's CLI does.
//
//   series, text    one decimal per line, optional "# n=<count>" first line
//   series, binary  "MPD1", u64 count (little-endian), count doubles
//   dictionary      JSON object, format_version 1; unknown keys are a
//                   version_error so later revisions are never misread
//   profile         "# m=<m> kind=<self-join|ab-join>", a column header,
//                   one "window_start distance nn_index" row per window
//   labels          "start end" half-open regions; merged on load
//
// Error model (reference errors.hpp): malformed text -> parse_error, a
// well-formed document that breaks a rule -> schema_error, an unsupported
// revision -> version_error, a non-finite sample -> non_finite_input, file
// system failures -> io_error. Doubles are written shortest-round-trip
// (std::to_chars), so every format round-trips bit-exactly.
//
// Structure: a line scanner and number readers shared by the text formats;
// a small JSON reader building a DOM (Jv); the dictionary rules applied to
// that DOM one field at a time.
#ifndef TSDICT_B200_IO_HPP
#define TSDICT_B200_IO_HPP

#include <algorithm>
#include <bit>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <initializer_list>
#include <iterator>
#include <limits>
#include <optional>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "tsdict/dictionary.hpp"
#include "tsdict/errors.hpp"
#include "tsdict/profiles.hpp"
#include "tsdict/series.hpp"

namespace tsdict {

namespace iofmt {

static_assert(std::endian::native == std::endian::little, "the MPD1 format is little-endian");

[[noreturn]] inline void bad(errc code, const std::string& what) { throw error(code, what); }

inline std::string at_line(std::size_t no) { return "line " + std::to_string(no) + ": "; }

inline bool blank_char(char c) { return c == ' ' || c == '\t' || c == '\r'; }

inline std::string_view strip(std::string_view s) {
  std::size_t a = 0, b = s.size();
  while (a < b && blank_char(s[a])) ++a;
  while (b > a && blank_char(s[b - 1])) --b;
  return s.substr(a, b - a);
}

// Iterates the '\n'-separated lines of a document (a trailing '\n' ends the
// last line rather than opening an empty one), stripped of blanks and '\r'.
class LineScanner {
 public:
  explicit LineScanner(std::string_view text) : text_(text) {}
  bool next(std::string_view& line) {
    if (pos_ >= text_.size()) return false;
    const std::size_t nl = text_.find('\n', pos_);
    const std::size_t end = nl == std::string_view::npos ? text_.size() : nl;
    line = strip(text_.substr(pos_, end - pos_));
    pos_ = end + 1;
    ++no_;
    return true;
  }
  std::size_t line_no() const { return no_; }

 private:
  std::string_view text_;
  std::size_t pos_ = 0, no_ = 0;
};

// the fields of a table line: separated by blanks or commas (the reference
// tools accept comma-separated tables too)
inline std::vector<std::string_view> fields_of(std::string_view line) {
  auto sep = [](char c) { return blank_char(c) || c == ','; };
  std::vector<std::string_view> out;
  std::size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && sep(line[i])) ++i;
    const std::size_t j0 = i;
    while (i < line.size() && !sep(line[i])) ++i;
    if (i > j0) out.push_back(line.substr(j0, i - j0));
  }
  return out;
}

// the whole token must be a number (std::from_chars accepts inf / nan)
inline bool read_double(std::string_view tok, double& v) {
  if (tok.empty()) return false;
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  return r.ec == std::errc() && r.ptr == tok.data() + tok.size();
}

inline bool read_u64(std::string_view tok, std::uint64_t& v) {
  if (tok.empty()) return false;
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  return r.ec == std::errc() && r.ptr == tok.data() + tok.size();
}

inline bool read_i64(std::string_view tok, std::int64_t& v) {
  if (tok.empty()) return false;
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  return r.ec == std::errc() && r.ptr == tok.data() + tok.size();
}

inline void put_double(std::string& out, double v) {
  char buf[40];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  out.append(buf, r.ptr);
}

inline std::string load_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) bad(errc::io_error, "cannot open '" + path + "' for reading");
  std::string s((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  if (f.bad()) bad(errc::io_error, "read of '" + path + "' failed");
  return s;
}

inline void save_file(const std::string& path, std::string_view content) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) bad(errc::io_error, "cannot open '" + path + "' for writing");
  f.write(content.data(), static_cast<std::streamsize>(content.size()));
  f.flush();
  if (!f) bad(errc::io_error, "write of '" + path + "' failed");
}

// ---------------------------------------------------------------- JSON DOM
struct Jv {
  enum class Kind { null, boolean, number, string, array, object } kind = Kind::null;
  bool b = false;
  double num = 0.0;
  std::optional<std::uint64_t> whole;  // the literal as a non-negative integer, when it is one
  std::string str;
  std::vector<Jv> items;
  std::vector<std::pair<std::string, Jv>> members;  // in document order; later duplicates win
  const Jv* member(std::string_view key) const {
    for (auto it = members.rbegin(); it != members.rend(); ++it)
      if (it->first == key) return &it->second;
    return nullptr;
  }
};

class JsonReader {
 public:
  explicit JsonReader(std::string_view s) : s_(s) {}
  Jv document() {
    Jv v = value(0);
    skip_ws();
    if (i_ != s_.size()) fail("trailing characters after the document");
    return v;
  }

 private:
  std::string_view s_;
  std::size_t i_ = 0;

  [[noreturn]] void fail(const std::string& what) const {
    bad(errc::parse_error, "JSON offset " + std::to_string(i_) + ": " + what);
  }
  void skip_ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r')) ++i_;
  }
  bool eat(char c) {
    skip_ws();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  void word(std::string_view w) {
    if (s_.substr(i_, w.size()) != w) fail("unknown literal");
    i_ += w.size();
  }
  Jv value(int depth) {
    if (depth > 64) fail("nesting too deep");
    skip_ws();
    if (i_ >= s_.size()) fail("unexpected end of document");
    Jv v;
    const char c = s_[i_];
    if (c == '{') {
      ++i_;
      v.kind = Jv::Kind::object;
      if (eat('}')) return v;
      do {
        skip_ws();
        if (i_ >= s_.size() || s_[i_] != '"') fail("expected a key");
        std::string key = string_body();
        if (!eat(':')) fail("expected ':'");
        v.members.emplace_back(std::move(key), value(depth + 1));
      } while (eat(','));
      if (!eat('}')) fail("expected ',' or '}'");
    } else if (c == '[') {
      ++i_;
      v.kind = Jv::Kind::array;
      if (eat(']')) return v;
      do v.items.push_back(value(depth + 1));
      while (eat(','));
      if (!eat(']')) fail("expected ',' or ']'");
    } else if (c == '"') {
      v.kind = Jv::Kind::string;
      v.str = string_body();
    } else if (c == 't') {
      word("true");
      v.kind = Jv::Kind::boolean;
      v.b = true;
    } else if (c == 'f') {
      word("false");
      v.kind = Jv::Kind::boolean;
    } else if (c == 'n') {
      word("null");
    } else {
      number(v);
    }
    return v;
  }
  std::string string_body() {
    ++i_;  // opening quote
    std::string out;
    while (true) {
      if (i_ >= s_.size()) fail("unterminated string");
      const char c = s_[i_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in a string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (i_ >= s_.size()) fail("unterminated escape");
      const char e = s_[i_++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {  // kept as UTF-8; the formats use ASCII keys only
          unsigned cp = 0;
          if (i_ + 4 > s_.size()) fail("short \\u escape");
          for (int k = 0; k < 4; ++k) {
            const char h = s_[i_++];
            cp <<= 4;
            if (h >= '0' && h <= '9') cp |= unsigned(h - '0');
            else if (h >= 'a' && h <= 'f') cp |= unsigned(h - 'a' + 10);
            else if (h >= 'A' && h <= 'F') cp |= unsigned(h - 'A' + 10);
            else fail("bad \\u escape");
          }
          if (cp < 0x80) {
            out += char(cp);
          } else if (cp < 0x800) {
            out += char(0xC0 | (cp >> 6));
            out += char(0x80 | (cp & 0x3F));
          } else {
            out += char(0xE0 | (cp >> 12));
            out += char(0x80 | ((cp >> 6) & 0x3F));
            out += char(0x80 | (cp & 0x3F));
          }
          break;
        }
        default: fail("bad escape");
      }
    }
  }
  // JSON number grammar: -? (0 | [1-9][0-9]*) (.[0-9]+)? ([eE][+-]?[0-9]+)?
  void number(Jv& v) {
    const std::size_t a = i_;
    auto digits = [&] {
      const std::size_t d0 = i_;
      while (i_ < s_.size() && s_[i_] >= '0' && s_[i_] <= '9') ++i_;
      return i_ > d0;
    };
    const bool neg = i_ < s_.size() && s_[i_] == '-';
    if (neg) ++i_;
    if (i_ < s_.size() && s_[i_] == '0') {
      ++i_;
    } else if (!digits()) {
      fail("invalid value");
    }
    bool integral = true;
    if (i_ < s_.size() && s_[i_] == '.') {
      ++i_;
      integral = false;
      if (!digits()) fail("digits expected after '.'");
    }
    if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
      ++i_;
      integral = false;
      if (i_ < s_.size() && (s_[i_] == '+' || s_[i_] == '-')) ++i_;
      if (!digits()) fail("digits expected in the exponent");
    }
    const std::string_view tok = s_.substr(a, i_ - a);
    const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v.num);
    if (r.ec != std::errc() || !std::isfinite(v.num)) fail("number out of range");
    v.kind = Jv::Kind::number;
    std::uint64_t u = 0;
    if (integral && !neg && read_u64(tok, u)) v.whole = u;
  }
};

inline void put_json_string(std::string& out, std::string_view s) {
  out += '"';
  out += s;  // keys are plain ASCII
  out += '"';
}

// ---------------------------------------------------------------- dictionary rules
constexpr int kDictionaryVersion = 1;

// a field as a non-negative integer / a finite number; schema_error otherwise
inline std::uint64_t want_uint(const Jv& v, const char* name) {
  if (v.kind != Jv::Kind::number || !v.whole) bad(errc::schema_error, std::string(name) + " must be a non-negative integer");
  return *v.whole;
}
inline double want_number(const Jv& v, const char* name) {
  if (v.kind != Jv::Kind::number) bad(errc::schema_error, std::string(name) + " must be a number");
  return v.num;  // the reader only produces finite numbers
}
inline const Jv& want_member(const Jv& obj, const char* name, const char* where) {
  const Jv* v = obj.member(name);
  if (!v) bad(errc::schema_error, std::string(where) + " has no '" + name + "'");
  return *v;
}
// every key must be one this revision knows (a newer writer's extras are a version_error)
inline void known_keys_only(const Jv& obj, std::initializer_list<std::string_view> keys, const char* where) {
  for (const auto& [k, v] : obj.members) {
    (void)v;
    if (std::find(keys.begin(), keys.end(), std::string_view(k)) == keys.end())
      bad(errc::version_error, std::string(where) + ": field '" + k + "' is not part of format version " +
                                   std::to_string(kDictionaryVersion));
  }
}

}  // namespace iofmt

// ------------------------------------------------------------------ series
inline std::string format_series_text(const TimeSeries& T) {
  std::string out = "# n=" + std::to_string(T.n()) + "\n";
  for (double v : T.values) {
    iofmt::put_double(out, v);
    out += '\n';
  }
  return out;
}

inline std::string format_series_binary(const TimeSeries& T) {
  const std::uint64_t n = T.n();
  std::string out(12 + 8 * T.n(), '\0');
  std::memcpy(out.data(), "MPD1", 4);
  std::memcpy(out.data() + 4, &n, 8);
  if (n) std::memcpy(out.data() + 12, T.values.data(), 8 * T.n());
  return out;
}

inline TimeSeries parse_series(std::string_view content) {
  using namespace iofmt;
  TimeSeries T;
  if (content.size() >= 4 && content.substr(0, 4) == "MPD1") {
    if (content.size() < 12) bad(errc::parse_error, "MPD1 header is truncated");
    std::uint64_t n = 0;
    std::memcpy(&n, content.data() + 4, 8);
    const std::uint64_t payload = content.size() - 12;
    if (n == 0) bad(errc::parse_error, "MPD1 series holds no samples");
    if (payload % 8 != 0 || payload / 8 != n)
      bad(errc::parse_error, "MPD1 count " + std::to_string(n) + " does not match a payload of " +
                                 std::to_string(payload) + " bytes");
    T.values.resize(n);
    std::memcpy(T.values.data(), content.data() + 12, payload);
    for (std::size_t i = 0; i < T.n(); ++i)
      if (!std::isfinite(T.values[i])) bad(errc::non_finite_input, "sample " + std::to_string(i) + " is not finite");
    return T;
  }
  LineScanner lines(content);
  std::string_view line;
  std::optional<std::uint64_t> declared;
  bool data = false;
  while (lines.next(line)) {
    if (line.empty()) continue;
    if (line.front() == '#') {
      // only a leading "# n=<count>" header is part of the format
      const std::string_view body = strip(line.substr(1));
      std::uint64_t n = 0;
      if (data || declared || body.substr(0, 2) != "n=" || !read_u64(strip(body.substr(2)), n))
        bad(errc::parse_error, at_line(lines.line_no()) + "expected a leading '# n=<count>' header");
      declared = n;
      continue;
    }
    double v = 0.0;
    if (!read_double(line, v)) bad(errc::parse_error, at_line(lines.line_no()) + "not a number: '" + std::string(line) + "'");
    if (!std::isfinite(v)) bad(errc::non_finite_input, at_line(lines.line_no()) + "sample is not finite");
    T.values.push_back(v);
    data = true;
  }
  if (T.values.empty()) bad(errc::parse_error, "series holds no samples");
  if (declared && *declared != T.n())
    bad(errc::parse_error, "header declares " + std::to_string(*declared) + " samples, the file holds " +
                               std::to_string(T.n()));
  return T;
}

inline TimeSeries read_series(const std::string& path) { return parse_series(iofmt::load_file(path)); }
inline void write_series_text(const std::string& path, const TimeSeries& T) {
  iofmt::save_file(path, format_series_text(T));
}
inline void write_series_binary(const std::string& path, const TimeSeries& T) {
  iofmt::save_file(path, format_series_binary(T));
}

// ------------------------------------------------------------------ dictionary
inline std::string format_dictionary(const Dictionary& D) {
  using namespace iofmt;
  std::string out = "{\"format_version\":" + std::to_string(kDictionaryVersion);
  out += ",\"m\":" + std::to_string(D.m);
  out += ",\"k\":";
  put_double(out, D.k);
  out += ",\"source_length\":" + std::to_string(D.source_length);
  out += ",\"space_saving\":";
  put_double(out, D.space_saving);
  out += ",\"e_max\":";
  if (D.e_max) put_double(out, *D.e_max);
  else out += "null";
  out += ",\"core_starts\":[";
  for (std::size_t i = 0; i < D.core_starts.size(); ++i) out += (i ? "," : "") + std::to_string(D.core_starts[i]);
  out += "],\"segments\":[";
  for (std::size_t s = 0; s < D.segments.size(); ++s) {
    const Segment& g = D.segments[s];
    out += s ? ",{" : "{";
    put_json_string(out, "start");
    out += ":" + std::to_string(g.start) + ",";
    put_json_string(out, "length");
    out += ":" + std::to_string(g.length()) + ",";
    put_json_string(out, "values");
    out += ":[";
    for (std::size_t i = 0; i < g.values.size(); ++i) {
      if (i) out += ',';
      put_double(out, g.values[i]);
    }
    out += "]}";
  }
  out += "]}";
  return out;
}

inline Dictionary parse_dictionary(std::string_view content) {
  using namespace iofmt;
  const Jv doc = JsonReader(content).document();
  if (doc.kind != Jv::Kind::object) bad(errc::schema_error, "a dictionary document is a JSON object");
  // the revision first: an unknown revision may legitimately break every other rule
  const Jv& ver = want_member(doc, "format_version", "dictionary");
  if (ver.kind != Jv::Kind::number || !ver.whole || *ver.whole != static_cast<std::uint64_t>(kDictionaryVersion))
    bad(errc::version_error, "unsupported dictionary format_version");
  known_keys_only(doc, {"format_version", "m", "k", "source_length", "space_saving", "e_max", "core_starts", "segments"},
                  "dictionary");

  Dictionary D;
  D.m = want_uint(want_member(doc, "m", "dictionary"), "m");
  if (D.m < 2) bad(errc::schema_error, "m must be at least 2");
  D.k = want_number(want_member(doc, "k", "dictionary"), "k");
  if (D.k < 0.0) bad(errc::schema_error, "k must be non-negative");
  D.source_length = want_uint(want_member(doc, "source_length", "dictionary"), "source_length");
  if (D.source_length == 0) bad(errc::schema_error, "source_length must be positive");
  D.space_saving = want_number(want_member(doc, "space_saving", "dictionary"), "space_saving");
  const Jv& em = want_member(doc, "e_max", "dictionary");
  if (em.kind != Jv::Kind::null) {
    const double e = want_number(em, "e_max");
    if (e < 0.0) bad(errc::schema_error, "e_max must be non-negative or null");
    D.e_max = e;
  }
  // a window must fit after every core start (fits: the remainder is at least `len`)
  auto fits = [&](std::uint64_t start, std::uint64_t len) {
    return start < D.source_length && D.source_length - start >= len;
  };
  const Jv& cores = want_member(doc, "core_starts", "dictionary");
  if (cores.kind != Jv::Kind::array) bad(errc::schema_error, "core_starts must be an array");
  for (const Jv& c : cores.items) {
    const std::uint64_t j = want_uint(c, "core start");
    if (!fits(j, D.m)) bad(errc::schema_error, "core start " + std::to_string(j) + " has no room for a window");
    D.core_starts.push_back(j);
  }
  {  // the learner never keeps two cores within m/2 of each other (dictionary.hpp exclusion)
    std::vector<std::size_t> sorted = D.core_starts;
    std::sort(sorted.begin(), sorted.end());
    for (std::size_t i = 1; i < sorted.size(); ++i)
      if (sorted[i] - sorted[i - 1] <= D.m / 2)
        bad(errc::schema_error, "core starts " + std::to_string(sorted[i - 1]) + " and " + std::to_string(sorted[i]) +
                                    " are closer than m/2");
  }
  const Jv& segs = want_member(doc, "segments", "dictionary");
  if (segs.kind != Jv::Kind::array || segs.items.empty()) bad(errc::schema_error, "segments must be a non-empty array");
  std::uint64_t stored = 0, end_prev = 0;
  for (std::size_t s = 0; s < segs.items.size(); ++s) {
    const Jv& sj = segs.items[s];
    const std::string where = "segment " + std::to_string(s);
    if (sj.kind != Jv::Kind::object) bad(errc::schema_error, where + " must be an object");
    known_keys_only(sj, {"start", "length", "values"}, where.c_str());
    Segment g;
    g.start = want_uint(want_member(sj, "start", where.c_str()), "start");
    const std::uint64_t len = want_uint(want_member(sj, "length", where.c_str()), "length");
    if (len < D.m) bad(errc::schema_error, where + " is shorter than m");
    if (!fits(g.start, len)) bad(errc::schema_error, where + " runs past the end of the source series");
    if (s > 0 && g.start < end_prev) bad(errc::schema_error, where + " overlaps or precedes the previous segment");
    const Jv& vals = want_member(sj, "values", where.c_str());
    if (vals.kind != Jv::Kind::array || vals.items.size() != len)
      bad(errc::schema_error, where + ": 'values' must hold exactly 'length' numbers");
    g.values.reserve(len);
    for (const Jv& x : vals.items) g.values.push_back(want_number(x, "sample"));
    end_prev = g.start + len;
    stored += len;
    D.segments.push_back(std::move(g));
  }
  const double implied = 1.0 - static_cast<double>(stored) / static_cast<double>(D.source_length);
  if (std::fabs(implied - D.space_saving) > 1e-12)
    bad(errc::schema_error, "space_saving disagrees with the stored segments");
  return D;
}

inline Dictionary read_dictionary(const std::string& path) { return parse_dictionary(iofmt::load_file(path)); }
inline void write_dictionary(const std::string& path, const Dictionary& D) {
  iofmt::save_file(path, format_dictionary(D));
}

// ------------------------------------------------------------------ profile
inline std::string format_profile(const MatrixProfile& P) {
  std::string out = "# m=" + std::to_string(P.m) + (P.kind == join_kind::self ? " kind=self-join\n" : " kind=ab-join\n");
  out += "window_start\tdistance\tnn_index\n";
  for (std::size_t i = 0; i < P.values.size(); ++i) {
    out += std::to_string(i);
    out += '\t';
    iofmt::put_double(out, P.values[i]);
    out += '\t';
    out += std::to_string(P.indices[i]);
    out += '\n';
  }
  return out;
}

inline MatrixProfile parse_profile(std::string_view content) {
  using namespace iofmt;
  LineScanner lines(content);
  std::string_view line;
  MatrixProfile P;
  // meta line
  if (!lines.next(line) || line.empty() || line.front() != '#')
    bad(errc::parse_error, "a profile starts with '# m=<m> kind=<kind>'");
  {
    std::optional<std::uint64_t> m;
    std::optional<std::string_view> kind;
    for (std::string_view f : fields_of(strip(line.substr(1)))) {
      std::uint64_t u = 0;
      if (f.substr(0, 2) == "m=" && read_u64(f.substr(2), u)) m = u;
      else if (f.substr(0, 5) == "kind=") kind = f.substr(5);
      else bad(errc::parse_error, at_line(1) + "unexpected '" + std::string(f) + "' in the profile header");
    }
    if (!m || !kind) bad(errc::parse_error, at_line(1) + "the header needs m= and kind=");
    if (*kind == "self-join") P.kind = join_kind::self;
    else if (*kind == "ab-join") P.kind = join_kind::ab;
    else bad(errc::schema_error, "unknown profile kind '" + std::string(*kind) + "'");
    if (*m < 2) bad(errc::schema_error, "m must be at least 2");
    P.m = *m;
  }
  // column header
  if (!lines.next(line)) bad(errc::parse_error, "the column header is missing");
  {
    const auto cols = fields_of(line);
    if (cols.size() != 3 || cols[0] != "window_start" || cols[1] != "distance" || cols[2] != "nn_index")
      bad(errc::parse_error, at_line(2) + "expected 'window_start distance nn_index'");
  }
  while (lines.next(line)) {
    if (line.empty()) continue;
    const auto f = fields_of(line);
    std::uint64_t w = 0;
    double d = 0.0;
    std::int64_t nn = 0;
    if (f.size() != 3 || !read_u64(f[0], w) || !read_double(f[1], d) || !read_i64(f[2], nn))
      bad(errc::parse_error, at_line(lines.line_no()) + "expected '<window_start> <distance> <nn_index>'");
    if (w != P.values.size())
      bad(errc::schema_error, at_line(lines.line_no()) + "window_start " + std::to_string(w) + " out of sequence");
    if (std::isnan(d) || d < 0.0) bad(errc::schema_error, at_line(lines.line_no()) + "distance must be >= 0");
    if (nn < MatrixProfile::no_neighbor) bad(errc::schema_error, at_line(lines.line_no()) + "nn_index below -1");
    P.values.push_back(d);
    P.indices.push_back(nn);
  }
  if (P.values.empty()) bad(errc::schema_error, "the profile has no rows");
  return P;
}

inline MatrixProfile read_profile(const std::string& path) { return parse_profile(iofmt::load_file(path)); }
inline void write_profile(const std::string& path, const MatrixProfile& P) {
  iofmt::save_file(path, format_profile(P));
}

// ------------------------------------------------------------------ labels
inline std::string format_labels(const std::vector<interval>& regions) {
  std::string out = "# start\tend\n";
  for (const auto& [lo, hi] : regions) out += std::to_string(lo) + "\t" + std::to_string(hi) + "\n";
  return out;
}

inline std::vector<interval> parse_labels(std::string_view content) {
  using namespace iofmt;
  LineScanner lines(content);
  std::string_view line;
  std::vector<interval> regions;
  while (lines.next(line)) {
    if (line.empty() || line.front() == '#') continue;
    const auto f = fields_of(line);
    std::uint64_t lo = 0, hi = 0;
    if (f.size() != 2 || !read_u64(f[0], lo) || !read_u64(f[1], hi))
      bad(errc::parse_error, at_line(lines.line_no()) + "expected '<start> <end>'");
    if (lo >= hi) bad(errc::schema_error, at_line(lines.line_no()) + "a region must end after it starts");
    regions.emplace_back(lo, hi);
  }
  if (regions.empty()) bad(errc::schema_error, "no label regions");
  return merge_intervals(std::move(regions));  // sorted, overlapping and touching regions joined
}

inline std::vector<interval> read_labels(const std::string& path) { return parse_labels(iofmt::load_file(path)); }
inline void write_labels(const std::string& path, const std::vector<interval>& regions) {
  iofmt::save_file(path, format_labels(regions));
}

}  // namespace tsdict

#endif  // TSDICT_B200_IO_HPP

// tsdict/io.hpp -- drop-in for the reference's file formats
// (/root/reference/proj/include/tsdict/io.hpp:1-20): the data formats on
// either side of the join path.
//
//  - series, text: one shortest-round-trip decimal per line after an
//    optional "# n=<count>" header (io.hpp:153-160, :173-225);
//  - series, binary "MPD1": magic, little-endian u64 count, the doubles
//    (io.hpp:151, :162-169, :174-199), bit-exact;
//  - dictionary: a JSON object, format_version 1, unknown fields rejected
//    (io.hpp:237-405);
//  - profile: "# m=<m> kind=<kind>", a column header, one row per window
//    (io.hpp:409-487);
//  - labels: "start end" half-open regions, sorted and merged on load
//    (io.hpp:489-528).
//
// Parsers and formatters operate on strings; the read_/write_ functions are
// thin file wrappers. Malformed input of any kind raises tsdict::error with
// the reference's code (parse_error, schema_error, version_error,
// non_finite_input, io_error). Host code only: these formats feed and drain
// the device path, they are not on it.
//
// The reference serialises dictionaries with a third-party JSON library
// (nlohmann, absent here). This reader accepts the JSON grammar the reference
// reads, and the writer emits compact JSON with the same members (sorted
// keys) and the same number layout, so documents round-trip bit-exactly
// through either implementation and the text is byte-identical wherever the
// reference library's digit generation is the shortest (it is not always;
// tests/cpp/test_io.cpp checks both).
#ifndef TSDICT_B200_IO_HPP
#define TSDICT_B200_IO_HPP

#include <algorithm>
#include <bit>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "tsdict/dictionary.hpp"
#include "tsdict/errors.hpp"
#include "tsdict/profiles.hpp"
#include "tsdict/series.hpp"

namespace tsdict {

namespace detail {

static_assert(std::endian::native == std::endian::little, "MPD1 is little-endian; so is this host");

inline std::string_view trim(std::string_view s) {
  auto blank = [](char c) { return c == ' ' || c == '\t' || c == '\r'; };
  std::size_t a = 0, b = s.size();
  while (a < b && blank(s[a])) ++a;
  while (b > a && blank(s[b - 1])) --b;
  return s.substr(a, b - a);
}

// "line N: " prefix of a text-format diagnostic
inline std::string at_line(std::size_t no) { return "line " + std::to_string(no) + ": "; }

inline error malformed(std::size_t line_no, const char* what, std::string_view field) {
  return error(errc::parse_error,
               at_line(line_no) + "cannot read " + what + " from '" + std::string(field) + "'");
}

// the whole (trimmed) field must be one number of type T
template <class T>
inline T whole_number(std::string_view field, std::size_t line_no, const char* what) {
  field = trim(field);
  T v{};
  const char* end = field.data() + field.size();
  const auto r = std::from_chars(field.data(), end, v);
  if (field.empty() || r.ec != std::errc() || r.ptr != end) throw malformed(line_no, what, field);
  return v;
}
inline double parse_double(std::string_view f, std::size_t line_no, const char* what) {
  return whole_number<double>(f, line_no, what);
}
inline std::uint64_t parse_uint(std::string_view f, std::size_t line_no, const char* what) {
  return whole_number<std::uint64_t>(f, line_no, what);
}
inline std::int64_t parse_int(std::string_view f, std::size_t line_no, const char* what) {
  return whole_number<std::int64_t>(f, line_no, what);
}

// shortest decimal that reads back to the same double
inline std::string shortest(double v) {
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, r.ptr);
}

// calls fn(line number from 1, line) for every '\n'-separated line; a
// trailing newline yields one last empty line, as the reference does
template <class F>
inline void each_line(std::string_view text, F&& fn) {
  std::size_t no = 1, pos = 0;
  for (;;) {
    const std::size_t nl = text.find('\n', pos);
    fn(no++, text.substr(pos, nl == std::string_view::npos ? std::string_view::npos : nl - pos));
    if (nl == std::string_view::npos) return;
    pos = nl + 1;
  }
}

// fields separated by runs of spaces, tabs or commas
inline std::vector<std::string_view> fields_of(std::string_view line) {
  std::vector<std::string_view> out;
  auto sep = [](char c) { return c == ' ' || c == '\t' || c == ','; };
  std::size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && sep(line[i])) ++i;
    const std::size_t b = i;
    while (i < line.size() && !sep(line[i])) ++i;
    if (i > b) out.push_back(line.substr(b, i - b));
  }
  return out;
}

inline std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw error(errc::io_error, "cannot open '" + path + "' for reading");
  std::ostringstream ss;
  ss << in.rdbuf();
  if (in.bad()) throw error(errc::io_error, "read failure on '" + path + "'");
  return std::move(ss).str();
}

inline void write_file(const std::string& path, std::string_view content) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw error(errc::io_error, "cannot open '" + path + "' for writing");
  out.write(content.data(), static_cast<std::streamsize>(content.size()));
  out.flush();
  if (!out) throw error(errc::io_error, "write failure on '" + path + "'");
}

// ------------------------------------------------------------- JSON subset
// A JSON value tree sufficient for the dictionary document. Numbers keep
// the distinction the reference's schema checks rely on: an unsigned
// integer literal (no sign, fraction or exponent, fits 64 bits) versus any
// other number.
struct json {
  enum class kind { null, boolean, unsigned_int, number, string, array, object };
  kind k = kind::null;
  bool b = false;
  std::uint64_t u = 0;
  double d = 0.0;
  std::string s;
  std::vector<json> items;                       // array
  std::vector<std::pair<std::string, json>> fields;  // object, in document order (last duplicate wins on lookup)

  bool is_number() const { return k == kind::unsigned_int || k == kind::number; }
  double as_double() const { return k == kind::unsigned_int ? static_cast<double>(u) : d; }
  const json* find(std::string_view key) const {
    const json* hit = nullptr;
    for (const auto& f : fields)
      if (f.first == key) hit = &f.second;
    return hit;
  }
};

class json_reader {
 public:
  explicit json_reader(std::string_view t) : t_(t) {}

  json document() {
    json v = value(0);
    ws();
    if (p_ != t_.size()) fail("unexpected trailing characters");
    return v;
  }

 private:
  std::string_view t_;
  std::size_t p_ = 0;

  [[noreturn]] void fail(const std::string& what) const {
    throw error(errc::parse_error, "JSON: " + what + " at byte " + std::to_string(p_));
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < t_.size() && t_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  bool literal(std::string_view w) {
    if (t_.substr(p_, w.size()) == w) {
      p_ += w.size();
      return true;
    }
    return false;
  }

  json value(int depth) {
    if (depth > 512) fail("nesting too deep");
    ws();
    if (p_ >= t_.size()) fail("unexpected end of input");
    json v;
    const char c = t_[p_];
    if (c == '{') {
      ++p_;
      v.k = json::kind::object;
      if (eat('}')) return v;
      do {
        ws();
        if (p_ >= t_.size() || t_[p_] != '"') fail("expected a member name");
        std::string key = string_body();
        expect(':');
        v.fields.emplace_back(std::move(key), value(depth + 1));
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++p_;
      v.k = json::kind::array;
      if (eat(']')) return v;
      do v.items.push_back(value(depth + 1));
      while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.k = json::kind::string;
      v.s = string_body();
    } else if (literal("true")) {
      v.k = json::kind::boolean;
      v.b = true;
    } else if (literal("false")) {
      v.k = json::kind::boolean;
    } else if (literal("null")) {
      v.k = json::kind::null;
    } else {
      number(v);
    }
    return v;
  }

  // RFC 8259 number grammar; unsigned integers that fit 64 bits stay exact,
  // everything else is read as a double (strtod rounding, overflow to inf)
  void number(json& v) {
    const std::size_t b = p_;
    bool integral = true;
    if (p_ < t_.size() && t_[p_] == '-') {
      ++p_;
      integral = false;
    }
    auto digits = [&] {
      const std::size_t s = p_;
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
      return p_ - s;
    };
    const std::size_t first = p_;
    const std::size_t nint = digits();
    if (nint == 0) fail("invalid literal");
    if (nint > 1 && t_[first] == '0') fail("leading zero in a number");
    if (p_ < t_.size() && t_[p_] == '.') {
      ++p_;
      integral = false;
      if (digits() == 0) fail("digits expected after '.'");
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      ++p_;
      integral = false;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      if (digits() == 0) fail("digits expected in the exponent");
    }
    const std::string_view lit = t_.substr(b, p_ - b);
    if (integral) {
      std::uint64_t u = 0;
      const auto r = std::from_chars(lit.data(), lit.data() + lit.size(), u);
      if (r.ec == std::errc() && r.ptr == lit.data() + lit.size()) {
        v.k = json::kind::unsigned_int;
        v.u = u;
        return;
      }
    }
    const std::string z(lit);
    v.k = json::kind::number;
    v.d = std::strtod(z.c_str(), nullptr);
    if (!std::isfinite(v.d)) fail("number overflow");  // as the reference's reader: a parse error
  }

  static void utf8(std::string& out, std::uint32_t cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  std::uint32_t hex4() {
    if (p_ + 4 > t_.size()) fail("truncated \\u escape");
    std::uint32_t cp = 0;
    for (int i = 0; i < 4; ++i) {
      const char h = t_[p_++];
      cp <<= 4;
      if (h >= '0' && h <= '9') cp |= h - '0';
      else if (h >= 'a' && h <= 'f') cp |= h - 'a' + 10;
      else if (h >= 'A' && h <= 'F') cp |= h - 'A' + 10;
      else fail("invalid \\u escape");
    }
    return cp;
  }
  std::string string_body() {
    ++p_;  // opening quote
    std::string out;
    for (;;) {
      if (p_ >= t_.size()) fail("unterminated string");
      const char c = t_[p_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in a string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p_ >= t_.size()) fail("unterminated escape");
      const char e = t_[p_++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          std::uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (!literal("\\u")) fail("unpaired surrogate");
            const std::uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("unpaired surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            fail("unpaired surrogate");
          }
          utf8(out, cp);
          break;
        }
        default: fail("invalid escape");
      }
    }
  }
};

// JSON number for a double in the layout the reference's writer produces:
// the shortest round-trip digits d (k of them) of v = 0.d x 10^n, written
// as digits with trailing zeros and ".0" when k <= n <= 15, with a decimal
// point inside when 0 < n <= 15, as "0.000d" when -4 < n <= 0, else in
// exponent form "d.ddde+XX" (sign always, at least two exponent digits)
inline std::string json_number(double v) {
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
  const std::string sci(buf, r.ptr);  // [-]d[.ddd]e(+|-)XX
  const std::size_t epos = sci.find('e');
  std::string mant = sci.substr(0, epos), out;
  if (mant[0] == '-') {
    out = "-";
    mant.erase(0, 1);
  }
  const int e10 = std::stoi(sci.substr(epos + 1));
  std::string dig;
  for (char c : mant)
    if (c != '.') dig += c;
  const int k = static_cast<int>(dig.size()), n = e10 + 1;
  if (k <= n && n <= 15) {
    out += dig + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += dig.substr(0, n) + "." + dig.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(-n, '0') + dig;
  } else {
    out += dig.substr(0, 1);
    if (k > 1) out += "." + dig.substr(1);
    const int x = n - 1;
    out += x < 0 ? "e-" : "e+";
    const std::string xs = std::to_string(x < 0 ? -x : x);
    out += (xs.size() < 2 ? "0" : "") + xs;
  }
  return out;
}

inline void check_members(const json& obj, std::initializer_list<std::string_view> known,
                                  const char* where) {
  for (const auto& f : obj.fields) {
    if (std::find(known.begin(), known.end(), std::string_view(f.first)) == known.end())
      throw error(errc::version_error, "unknown field '" + f.first + "' in " + where +
                                           " (this reader implements format_version 1)");
  }
}

inline const json& member(const json& obj, const char* key, const char* where) {
  const json* v = obj.find(key);
  if (!v) throw error(errc::schema_error, std::string("missing field '") + key + "' in " + where);
  return *v;
}

inline std::uint64_t u64_of(const json& v, const char* what) {
  if (v.k != json::kind::unsigned_int) throw error(errc::schema_error, std::string(what) + " must be a non-negative integer");
  return v.u;
}

inline double finite_of(const json& v, const char* what) {
  if (!v.is_number()) throw error(errc::schema_error, std::string(what) + " must be a number");
  const double d = v.as_double();
  if (!std::isfinite(d)) throw error(errc::non_finite_input, std::string(what) + " is not finite");
  return d;
}

}  // namespace detail

// ------------------------------------------------------------------ series

inline constexpr char series_magic[4] = {'M', 'P', 'D', '1'};

inline std::string format_series_text(const TimeSeries& T) {
  std::string out = "# n=" + std::to_string(T.n()) + "\n";
  for (double v : T.values) (out += detail::shortest(v)) += '\n';
  return out;
}

inline std::string format_series_binary(const TimeSeries& T) {
  const std::uint64_t n = T.n();
  std::string out(12 + 8 * n, '\0');
  std::memcpy(out.data(), series_magic, 4);
  std::memcpy(out.data() + 4, &n, 8);
  if (n) std::memcpy(out.data() + 12, T.values.data(), 8 * n);
  return out;
}

// Either form (binary by its magic). Empty series and non-finite samples are
// rejected (io.hpp:171-225).
inline TimeSeries parse_series(std::string_view content) {
  TimeSeries T;
  if (content.size() >= 4 && std::memcmp(content.data(), series_magic, 4) == 0) {
    if (content.size() < 12) throw error(errc::parse_error, "MPD1 stream shorter than its 12-byte header");
    std::uint64_t n = 0;
    std::memcpy(&n, content.data() + 4, 8);
    const std::size_t body = content.size() - 12;  // no 12 + 8n: it can wrap
    if (body % 8 != 0 || body / 8 != n)
      throw error(errc::parse_error, "MPD1 payload size disagrees with the stored count");
    if (n == 0) throw error(errc::parse_error, "no samples");
    T.values.resize(n);
    std::memcpy(T.values.data(), content.data() + 12, 8 * n);
    for (std::size_t i = 0; i < n; ++i)
      if (!std::isfinite(T.values[i])) throw error(errc::non_finite_input, "sample " + std::to_string(i) + " is NaN or infinite");
    return T;
  }
  std::optional<std::uint64_t> declared;
  detail::each_line(content, [&](std::size_t no, std::string_view raw) {
    const std::string_view line = detail::trim(raw);
    if (line.empty()) return;
    if (line.front() == '#') {
      if (declared || !T.values.empty())
        throw error(errc::parse_error, detail::at_line(no) + "header must come before the samples");
      const std::string_view h = detail::trim(line.substr(1));
      if (h.size() < 3 || h.substr(0, 2) != "n=")
        throw error(errc::parse_error, detail::at_line(no) + "header is not of the form '# n=<count>'");
      declared = detail::parse_uint(h.substr(2), no, "sample count");
      return;
    }
    const double v = detail::parse_double(line, no, "sample");
    if (!std::isfinite(v)) throw error(errc::non_finite_input, detail::at_line(no) + "sample is NaN or infinite");
    T.values.push_back(v);
  });
  if (declared && *declared != T.n())
    throw error(errc::parse_error,
                "header announces " + std::to_string(*declared) + " samples, body holds " + std::to_string(T.n()));
  if (T.n() == 0) throw error(errc::parse_error, "no samples");
  return T;
}

inline TimeSeries read_series(const std::string& path) { return parse_series(detail::read_file(path)); }
inline void write_series_text(const std::string& path, const TimeSeries& T) { detail::write_file(path, format_series_text(T)); }
inline void write_series_binary(const std::string& path, const TimeSeries& T) {
  detail::write_file(path, format_series_binary(T));
}

// -------------------------------------------------------------- dictionary

inline constexpr int dictionary_format_version = 1;

// compact JSON, members in sorted order (io.hpp:239-261)
inline std::string format_dictionary(const Dictionary& D) {
  std::string o = "{\"core_starts\":[";
  for (std::size_t i = 0; i < D.core_starts.size(); ++i) (o += i ? "," : "") += std::to_string(D.core_starts[i]);
  o += "],\"e_max\":";
  o += D.e_max ? detail::json_number(*D.e_max) : "null";
  o += ",\"format_version\":" + std::to_string(dictionary_format_version);
  o += ",\"k\":" + detail::json_number(D.k);
  o += ",\"m\":" + std::to_string(D.m);
  o += ",\"segments\":[";
  for (std::size_t s = 0; s < D.segments.size(); ++s) {
    const Segment& g = D.segments[s];
    o += s ? ",{" : "{";
    o += "\"length\":" + std::to_string(g.length()) + ",\"start\":" + std::to_string(g.start) + ",\"values\":[";
    for (std::size_t i = 0; i < g.values.size(); ++i) (o += i ? "," : "") += detail::json_number(g.values[i]);
    o += "]}";
  }
  o += "],\"source_length\":" + std::to_string(D.source_length);
  o += ",\"space_saving\":" + detail::json_number(D.space_saving);
  o += "}\n";
  return o;
}

// Schema checks and their order follow io.hpp:308-400.
inline Dictionary parse_dictionary(std::string_view content) {
  const detail::json j = detail::json_reader(content).document();
  using K = detail::json::kind;
  if (j.k != K::object) throw error(errc::schema_error, "top-level JSON value is not an object");
  const detail::json& ver = detail::member(j, "format_version", "dictionary");
  if (ver.k != K::unsigned_int || ver.u != static_cast<std::uint64_t>(dictionary_format_version))
    throw error(errc::version_error, "format_version is not 1");
  detail::check_members(
      j, {"format_version", "m", "k", "source_length", "space_saving", "e_max", "core_starts", "segments"}, "dictionary");

  Dictionary D;
  D.m = detail::u64_of(detail::member(j, "m", "dictionary"), "m");
  if (D.m < 2) throw error(errc::schema_error, "window length m below 2");
  D.k = detail::finite_of(detail::member(j, "k", "dictionary"), "k");
  if (D.k < 0.0) throw error(errc::schema_error, "k is negative");
  D.source_length = detail::u64_of(detail::member(j, "source_length", "dictionary"), "source_length");
  D.space_saving = detail::finite_of(detail::member(j, "space_saving", "dictionary"), "space_saving");
  const detail::json& em = detail::member(j, "e_max", "dictionary");
  if (em.k != K::null) {
    const double e = detail::finite_of(em, "e_max");
    if (e < 0.0) throw error(errc::schema_error, "e_max is negative");
    D.e_max = e;
  }

  const detail::json& cores = detail::member(j, "core_starts", "dictionary");
  if (cores.k != K::array) throw error(errc::schema_error, "core_starts is not an array");
  for (const auto& c : cores.items) {
    const std::uint64_t st = detail::u64_of(c, "core start");
    if (st >= D.source_length || D.source_length - st < D.m)
      throw error(errc::schema_error, "core start " + std::to_string(st) + " has no full window inside the source");
    D.core_starts.push_back(st);
  }
  for (std::size_t a = 0; a < D.core_starts.size(); ++a)
    for (std::size_t b = a + 1; b < D.core_starts.size(); ++b) {
      const std::size_t lo = std::min(D.core_starts[a], D.core_starts[b]);
      const std::size_t hi = std::max(D.core_starts[a], D.core_starts[b]);
      if (hi - lo <= D.m / 2)
        throw error(errc::schema_error, "core starts " + std::to_string(lo) + " and " + std::to_string(hi) +
                                            " are closer than m/2");
    }

  const detail::json& segs = detail::member(j, "segments", "dictionary");
  if (segs.k != K::array || segs.items.empty()) throw error(errc::schema_error, "segments is missing, not an array, or empty");
  std::size_t prev_end = 0, stored = 0;
  for (const auto& sj : segs.items) {
    if (sj.k != K::object) throw error(errc::schema_error, "a segments entry is not an object");
    detail::check_members(sj, {"start", "length", "values"}, "segment");
    Segment g;
    g.start = detail::u64_of(detail::member(sj, "start", "segment"), "segment start");
    const std::uint64_t len = detail::u64_of(detail::member(sj, "length", "segment"), "segment length");
    if (len < D.m) throw error(errc::schema_error, "segment length below m");
    if (g.start >= D.source_length || D.source_length - g.start < len)
      throw error(errc::schema_error, "segment runs past source_length");
    if (!D.segments.empty() && g.start < prev_end) throw error(errc::schema_error, "segments not sorted or overlapping");
    const detail::json& vals = detail::member(sj, "values", "segment");
    if (vals.k != K::array || vals.items.size() != len)
      throw error(errc::schema_error, "segment values count differs from its length");
    g.values.reserve(len);
    for (const auto& v : vals.items) g.values.push_back(detail::finite_of(v, "segment value"));
    prev_end = g.start + len;
    stored += len;
    D.segments.push_back(std::move(g));
  }
  if (D.source_length == 0) throw error(errc::schema_error, "source_length is zero");
  const double recomputed = 1.0 - static_cast<double>(stored) / static_cast<double>(D.source_length);
  if (std::fabs(recomputed - D.space_saving) > 1e-12)
    throw error(errc::schema_error, "space_saving inconsistent with the stored samples");
  return D;
}

inline Dictionary read_dictionary(const std::string& path) { return parse_dictionary(detail::read_file(path)); }
inline void write_dictionary(const std::string& path, const Dictionary& D) { detail::write_file(path, format_dictionary(D)); }

// ----------------------------------------------------------------- profile

inline const char* join_kind_name(join_kind k) { return k == join_kind::self ? "self-join" : "ab-join"; }

inline std::string format_profile(const MatrixProfile& P) {
  std::string o = "# m=" + std::to_string(P.m) + " kind=" + join_kind_name(P.kind) + "\nwindow_start\tdistance\tnn_index\n";
  for (std::size_t i = 0; i < P.values.size(); ++i)
    o += std::to_string(i) + '\t' + detail::shortest(P.values[i]) + '\t' + std::to_string(P.indices[i]) + '\n';
  return o;
}

inline MatrixProfile parse_profile(std::string_view content) {
  MatrixProfile P;
  bool meta = false, header = false;
  detail::each_line(content, [&](std::size_t no, std::string_view raw) {
    const std::string_view line = detail::trim(raw);
    if (line.empty()) return;
    const std::string at = detail::at_line(no) + "";
    if (!meta) {
      const auto f = line.size() >= 2 && line.front() == '#' ? detail::fields_of(line.substr(1))
                                                             : std::vector<std::string_view>{};
      if (f.size() != 2 || f[0].substr(0, 2) != "m=" || f[1].substr(0, 5) != "kind=")
        throw error(errc::parse_error, at + "first line must be '# m=<m> kind=<kind>'");
      P.m = detail::parse_uint(f[0].substr(2), no, "window length");
      if (P.m < 2) throw error(errc::schema_error, "profile window length below 2");
      const std::string_view kind = f[1].substr(5);
      if (kind == "self-join") P.kind = join_kind::self;
      else if (kind == "ab-join") P.kind = join_kind::ab;
      else throw error(errc::schema_error, at + "kind is neither self-join nor ab-join");
      meta = true;
      return;
    }
    if (!header) {
      if (line != "window_start\tdistance\tnn_index") throw error(errc::parse_error, at + "column header line missing");
      header = true;
      return;
    }
    const auto f = detail::fields_of(line);
    if (f.size() != 3) throw error(errc::parse_error, at + "row needs 3 fields");
    if (detail::parse_uint(f[0], no, "window start") != P.values.size())
      throw error(errc::schema_error, at + "window_start not consecutive");
    const double d = detail::parse_double(f[1], no, "distance");
    if (std::isnan(d) || d < 0.0) throw error(errc::schema_error, at + "distance negative or NaN");
    const std::int64_t nn = detail::parse_int(f[2], no, "neighbor index");
    if (nn < MatrixProfile::no_neighbor) throw error(errc::schema_error, at + "nn_index below -1");
    P.values.push_back(d);
    P.indices.push_back(nn);
  });
  if (!meta || !header) throw error(errc::parse_error, "profile ends before its headers");
  if (P.values.empty()) throw error(errc::schema_error, "profile has no rows");
  return P;
}

inline MatrixProfile read_profile(const std::string& path) { return parse_profile(detail::read_file(path)); }
inline void write_profile(const std::string& path, const MatrixProfile& P) { detail::write_file(path, format_profile(P)); }

// ------------------------------------------------------------------ labels

inline std::string format_labels(const std::vector<interval>& regions) {
  std::string o = "# start\tend\n";
  for (const auto& r : regions) o += std::to_string(r.first) + '\t' + std::to_string(r.second) + '\n';
  return o;
}

// regions come back sorted and merged (overlapping or touching ones collapse)
inline std::vector<interval> parse_labels(std::string_view content) {
  std::vector<interval> regions;
  detail::each_line(content, [&](std::size_t no, std::string_view raw) {
    const std::string_view line = detail::trim(raw);
    if (line.empty() || line.front() == '#') return;
    const auto f = detail::fields_of(line);
    if (f.size() != 2) throw error(errc::parse_error, detail::at_line(no) + "region needs 2 fields");
    const std::uint64_t lo = detail::parse_uint(f[0], no, "region start");
    const std::uint64_t hi = detail::parse_uint(f[1], no, "region end");
    if (lo >= hi) throw error(errc::schema_error, detail::at_line(no) + "empty or inverted region");
    regions.emplace_back(lo, hi);
  });
  if (regions.empty()) throw error(errc::schema_error, "no regions");
  return merge_intervals(regions);
}

inline std::vector<interval> read_labels(const std::string& path) { return parse_labels(detail::read_file(path)); }
inline void write_labels(const std::string& path, const std::vector<interval>& regions) {
  detail::write_file(path, format_labels(regions));
}

}  // namespace tsdict

#endif

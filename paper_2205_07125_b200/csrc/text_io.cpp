// Native readers / writers of the reference's text artefacts:
//   NNG  "NNG 1 M E", M weight lines, E "i j p" edge lines  (model.py:293-364)
//   PMAP "PMAP 1 M N", M GPU-index lines                   (partition.py:270-306)
// with the reference's acceptance rules and error texts (ParseError(message,
// line)): Python's str.splitlines() line breaking, float()/int() token syntax
// (surrounding whitespace, sign, '_' digit separators, inf/nan) and repr() of
// the offending text in messages.  Writers emit repr() of every float (the
// shortest round-trip digits, Python's fixed/exponent switch), so files are
// byte-identical to the reference's save_graph / save_partition_map.
//
// A file is read into memory once; a first pass counts lines (the reference
// checks the line count before any content), a second parses them.

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>

#include "nc_common.h"

namespace {

constexpr int kParse = NC_E_PARSE;

struct Buf {
  std::vector<char> data;
};

bool read_file(const char* path, Buf& b) {
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    nc_set_error("cannot open %s: %s", path, std::strerror(errno));
    return false;
  }
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  b.data.resize(n > 0 ? (size_t)n : 0);
  const size_t got = n > 0 ? std::fread(b.data.data(), 1, (size_t)n, f) : 0;
  std::fclose(f);
  if ((long)got != (n > 0 ? n : 0)) {
    nc_set_error("short read on %s", path);
    return false;
  }
  return true;
}

// Length of the line break at p (0 if none), following str.splitlines():
// \n \r \r\n \v \f \x1c \x1d \x1e and the UTF-8 forms of U+0085, U+2028, U+2029.
inline size_t line_break(const char* p, const char* end) {
  const unsigned char c = (unsigned char)*p;
  if (c == '\n' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e) return 1;
  if (c == '\r') return (p + 1 < end && p[1] == '\n') ? 2 : 1;
  if (c == 0xC2 && p + 1 < end && (unsigned char)p[1] == 0x85) return 2;
  if (c == 0xE2 && p + 2 < end && (unsigned char)p[1] == 0x80 &&
      ((unsigned char)p[2] == 0xA8 || (unsigned char)p[2] == 0xA9))
    return 3;
  return 0;
}

// Line cursor over the buffer (str.splitlines semantics: no empty last line
// after a final break).
struct BreakTable {
  bool t[256] = {};
  BreakTable() {
    for (unsigned char c : {'\n', '\r', '\x0b', '\x0c', '\x1c', '\x1d', '\x1e', '\xc2', '\xe2'}) t[c] = true;
  }
};
const BreakTable kBreaks;

struct Lines {
  const char* p;
  const char* end;
  bool next(std::string_view& line) {
    if (p >= end) return false;
    const char* s = p;
    while (p < end) {
      if (!kBreaks.t[(unsigned char)*p]) {
        ++p;
        continue;
      }
      const size_t k = line_break(p, end);
      if (k) {
        line = std::string_view(s, (size_t)(p - s));
        p += k;
        return true;
      }
      ++p;
    }
    line = std::string_view(s, (size_t)(p - s));
    return true;
  }
};

int64_t count_lines(const Buf& b) {
  Lines ls{b.data.data(), b.data.data() + b.data.size()};
  std::string_view l;
  int64_t n = 0;
  while (ls.next(l)) ++n;
  return n;
}

inline bool py_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1f);
}

std::string_view strip(std::string_view s) {
  size_t a = 0, b = s.size();
  while (a < b && py_space((unsigned char)s[a])) ++a;
  while (b > a && py_space((unsigned char)s[b - 1])) --b;
  return s.substr(a, b - a);
}

// str.split() with no argument: runs of whitespace separate, no empty fields.
size_t split_ws(std::string_view s, std::string_view* out, size_t cap) {
  size_t n = 0, i = 0;
  while (i < s.size()) {
    while (i < s.size() && py_space((unsigned char)s[i])) ++i;
    if (i >= s.size()) break;
    size_t j = i;
    while (j < s.size() && !py_space((unsigned char)s[j])) ++j;
    if (n < cap) out[n] = s.substr(i, j - i);
    ++n;
    i = j;
  }
  return n;
}

// '_' digit separators as Python's int()/float() accept them (only between digits).
bool drop_underscores(std::string_view s, std::string& out) {
  out.clear();
  for (size_t i = 0; i < s.size(); ++i) {
    if (s[i] == '_') {
      if (i == 0 || i + 1 >= s.size() || !std::isdigit((unsigned char)s[i - 1]) ||
          !std::isdigit((unsigned char)s[i + 1]))
        return false;
      continue;
    }
    out.push_back(s[i]);
  }
  return true;
}

bool ieq(std::string_view a, const char* b) {
  const size_t n = std::strlen(b);
  if (a.size() != n) return false;
  for (size_t i = 0; i < n; ++i)
    if (std::tolower((unsigned char)a[i]) != b[i]) return false;
  return true;
}

// Python float(text).
bool py_float(std::string_view text, double& v) {
  std::string_view s = strip(text);
  std::string tmp;
  std::string_view t = s;
  if (s.find('_') != std::string_view::npos) {
    if (!drop_underscores(s, tmp)) return false;
    t = tmp;
  }
  if (t.empty()) return false;
  bool neg = false;
  if (t[0] == '+' || t[0] == '-') {
    neg = t[0] == '-';
    t.remove_prefix(1);
  }
  if (t.empty()) return false;
  if (ieq(t, "inf") || ieq(t, "infinity")) {
    v = neg ? -HUGE_VAL : HUGE_VAL;
    return true;
  }
  if (ieq(t, "nan")) {
    v = std::nan("");
    return true;
  }
  for (char c : t)
    if (!(std::isdigit((unsigned char)c) || c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-')) return false;
  double x = 0.0;
  const auto r = std::from_chars(t.data(), t.data() + t.size(), x, std::chars_format::general);
  if (r.ec != std::errc() || r.ptr != t.data() + t.size()) {
    // from_chars reports out of range for overflow / underflow; Python gives inf / 0.0
    if (r.ec == std::errc::result_out_of_range && r.ptr == t.data() + t.size()) {
      errno = 0;
      x = std::strtod(std::string(t).c_str(), nullptr);
    } else {
      return false;
    }
  }
  v = neg ? -x : x;
  return true;
}

// Python int(text) in base 10 (no overflow beyond int64 in these formats).
bool py_int(std::string_view text, int64_t& v) {
  std::string_view s = strip(text);
  std::string tmp;
  std::string_view t = s;
  if (s.find('_') != std::string_view::npos) {
    if (!drop_underscores(s, tmp)) return false;
    t = tmp;
  }
  if (t.empty()) return false;
  bool neg = false;
  if (t[0] == '+' || t[0] == '-') {
    neg = t[0] == '-';
    t.remove_prefix(1);
  }
  if (t.empty()) return false;
  uint64_t x = 0;
  const auto r = std::from_chars(t.data(), t.data() + t.size(), x, 10);
  if (r.ec != std::errc() || r.ptr != t.data() + t.size() || x > (uint64_t)INT64_MAX) return false;
  v = neg ? -(int64_t)x : (int64_t)x;
  return true;
}

// repr() of a str (ASCII escapes; bytes >= 0x80 are passed through).
std::string py_repr(std::string_view s) {
  const bool sq = s.find('\'') != std::string_view::npos, dq = s.find('"') != std::string_view::npos;
  const char q = (sq && !dq) ? '"' : '\'';
  std::string out(1, q);
  for (unsigned char c : s) {
    if (c == (unsigned char)q || c == '\\') {
      out.push_back('\\');
      out.push_back((char)c);
    } else if (c == '\n') {
      out += "\\n";
    } else if (c == '\r') {
      out += "\\r";
    } else if (c == '\t') {
      out += "\\t";
    } else if (c < 0x20 || c == 0x7f) {
      char b[8];
      std::snprintf(b, sizeof(b), "\\x%02x", c);
      out += b;
    } else {
      out.push_back((char)c);
    }
  }
  out.push_back(q);
  return out;
}

// repr() of a float: shortest round-trip digits, fixed for -4 < decpt <= 16, else exponent.
std::string py_float_repr(double v);

// The same into buf (>= 40 bytes), returns the end; the writers' hot path.
char* py_float_repr_to(char* buf, double v) {
  if (!std::isfinite(v) || v == 0.0) {
    const std::string r = py_float_repr(v);
    std::memcpy(buf, r.data(), r.size());
    return buf + r.size();
  }
  char sci[40];
  const auto r = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
  const char* q = sci;
  char* o = buf;
  if (*q == '-') {
    *o++ = '-';
    ++q;
  }
  char digits[24];
  int nd = 0;
  const char* e = q;
  while (*e != 'e') {
    if (*e != '.') digits[nd++] = *e;
    ++e;
  }
  int exp10 = 0;
  std::from_chars(e + 1 + (e[1] == '+' ? 1 : 0), r.ptr, exp10);
  const int decpt = exp10 + 1;
  if (decpt <= -4 || decpt > 16) {
    *o++ = digits[0];
    if (nd > 1) {
      *o++ = '.';
      std::memcpy(o, digits + 1, (size_t)(nd - 1));
      o += nd - 1;
    }
    *o++ = 'e';
    *o++ = exp10 < 0 ? '-' : '+';
    const int a = exp10 < 0 ? -exp10 : exp10;
    if (a < 10) *o++ = '0';
    o = std::to_chars(o, o + 8, a).ptr;
  } else if (decpt <= 0) {
    *o++ = '0';
    *o++ = '.';
    for (int i = 0; i < -decpt; ++i) *o++ = '0';
    std::memcpy(o, digits, (size_t)nd);
    o += nd;
  } else if (decpt >= nd) {
    std::memcpy(o, digits, (size_t)nd);
    o += nd;
    for (int i = nd; i < decpt; ++i) *o++ = '0';
    *o++ = '.';
    *o++ = '0';
  } else {
    std::memcpy(o, digits, (size_t)decpt);
    o += decpt;
    *o++ = '.';
    std::memcpy(o, digits + decpt, (size_t)(nd - decpt));
    o += nd - decpt;
  }
  return o;
}

std::string py_float_repr(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v < 0 ? "-inf" : "inf";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char b[64];
  const auto r = std::to_chars(b, b + sizeof(b), v, std::chars_format::scientific);
  std::string sci(b, r.ptr);
  std::string sign;
  if (sci[0] == '-') {
    sign = "-";
    sci.erase(0, 1);
  }
  const size_t e = sci.find('e');
  std::string digits = sci.substr(0, e);
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int exp10 = std::atoi(sci.c_str() + e + 1);
  const int decpt = exp10 + 1;   // value = 0.digits x 10^decpt
  const int nd = (int)digits.size();
  std::string out = sign;
  if (decpt <= -4 || decpt > 16) {
    out += digits[0];
    if (nd > 1) {
      out += '.';
      out += digits.substr(1);
    }
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", exp10 < 0 ? '-' : '+', exp10 < 0 ? -exp10 : exp10);
    out += eb;
  } else if (decpt <= 0) {
    out += "0." + std::string((size_t)(-decpt), '0') + digits;
  } else if (decpt >= nd) {
    out += digits + std::string((size_t)(decpt - nd), '0') + ".0";
  } else {
    out += digits.substr(0, (size_t)decpt) + "." + digits.substr((size_t)decpt);
  }
  return out;
}

int parse_error(int64_t line, int64_t* err_line, const std::string& msg) {
  nc_set_error("%s", msg.c_str());
  if (err_line) *err_line = line;
  return kParse;
}

struct Header {
  int64_t a = 0, b = 0;
};

// "<tag> 1 <a> <b>" header shared by NNG and PMAP; version errors are NNG-only.
int parse_header(std::string_view line, const char* tag, bool separate_version, Header& h, int64_t* err_line) {
  std::string_view f[5];
  const size_t n = split_ws(line, f, 5);
  const std::string bad = std::string("malformed header ") + py_repr(line);
  if (n != 4 || f[0] != tag) return parse_error(1, err_line, bad);
  if (f[1] != "1") {
    if (!separate_version) return parse_error(1, err_line, bad);
    return parse_error(1, err_line, std::string("unsupported format version ") + py_repr(f[1]));
  }
  if (!py_int(f[2], h.a) || !py_int(f[3], h.b)) return parse_error(1, err_line, bad);
  return NC_OK;
}

class Writer {
 public:
  explicit Writer(FILE* f) : f_(f) { buf_.reserve(1 << 20); }
  void put(const std::string& s) { buf_ += s; }
  void maybe_flush() {
    if (buf_.size() >= (1u << 20)) flush();
  }
  void put_int(int64_t v) {
    char b[24];
    const auto r = std::to_chars(b, b + sizeof(b), v);
    buf_.append(b, r.ptr);
  }
  void put_float(double v) {
    char b[48];
    buf_.append(b, py_float_repr_to(b, v));
  }
  void put_char(char c) { buf_.push_back(c); }
  bool flush() {
    const bool ok = std::fwrite(buf_.data(), 1, buf_.size(), f_) == buf_.size();
    buf_.clear();
    return ok;
  }

 private:
  FILE* f_;
  std::string buf_;
};

}  // namespace

// ---------------------------------------------------------------- NNG
extern "C" int nc_nng_scan(const char* path, int64_t* n_neurons, int64_t* n_edges, int64_t* err_line) {
  Buf b;
  if (!read_file(path, b)) return NC_E_IO;
  Lines ls{b.data.data(), b.data.data() + b.data.size()};
  std::string_view head;
  if (!ls.next(head)) return parse_error(1, err_line, "empty file");
  Header h;
  if (int e = parse_header(head, "NNG", true, h, err_line)) return e;
  if (h.a < 1 || h.b < 0) return parse_error(1, err_line, std::string("invalid counts in header ") + py_repr(head));
  *n_neurons = h.a;
  *n_edges = h.b;
  return NC_OK;
}

extern "C" int nc_nng_read(const char* path, int64_t m, int64_t e, double* weights, int64_t* edge_i, int64_t* edge_j,
                           double* edge_p, int64_t* err_line) {
  Buf b;
  if (!read_file(path, b)) return NC_E_IO;
  const int64_t total = count_lines(b);
  Lines ls{b.data.data(), b.data.data() + b.data.size()};
  std::string_view line;
  if (!ls.next(line)) return parse_error(1, err_line, "empty file");
  Header h;
  if (int r = parse_header(line, "NNG", true, h, err_line)) return r;
  if (h.a != m || h.b != e) {
    nc_set_error("nc_nng_read: header counts changed since nc_nng_scan");
    return NC_E_ARG;
  }
  const int64_t need = 1 + m + e;
  if (total < need) return parse_error(total + 1, err_line, "unexpected end of file");
  if (total > need) return parse_error(need + 1, err_line, "unexpected trailing content");
  for (int64_t k = 0; k < m; ++k) {
    ls.next(line);
    double v;
    if (!py_float(line, v)) return parse_error(k + 2, err_line, "malformed weight " + py_repr(line));
    if (!(std::isfinite(v) && v > 0.0))
      return parse_error(k + 2, err_line, "weight " + py_float_repr(v) + " is not strictly positive");
    weights[k] = v;
  }
  int64_t pi = -1, pj = -1;
  for (int64_t k = 0; k < e; ++k) {
    const int64_t ln = 2 + m + k;
    ls.next(line);
    std::string_view f[4];
    int64_t i = 0, j = 0;
    double p = 0.0;
    if (split_ws(line, f, 4) != 3) return parse_error(ln, err_line, "malformed edge line " + py_repr(line));
    if (!py_int(f[0], i) || !py_int(f[1], j) || !py_float(f[2], p))
      return parse_error(ln, err_line, "malformed edge line " + py_repr(line));
    if (!(0 <= i && i < j && j < m))
      return parse_error(ln, err_line,
                         "edge (" + std::to_string(i) + ", " + std::to_string(j) + ") out of range for " +
                             std::to_string(m) + " neurons");
    if (!(std::isfinite(p) && p > 0.0 && p <= 1.0))
      return parse_error(ln, err_line, "edge probability " + py_float_repr(p) + " outside (0, 1]");
    if (i == pi && j == pj)
      return parse_error(ln, err_line, "duplicate edge (" + std::to_string(i) + ", " + std::to_string(j) + ")");
    if (i < pi || (i == pi && j < pj))
      return parse_error(ln, err_line,
                         "edge (" + std::to_string(i) + ", " + std::to_string(j) + ") not in ascending (i, j) order");
    pi = i;
    pj = j;
    edge_i[k] = i;
    edge_j[k] = j;
    edge_p[k] = p;
  }
  return NC_OK;
}

extern "C" int nc_nng_write(const char* path, int64_t m, int64_t e, const double* weights, const int64_t* edge_i,
                            const int64_t* edge_j, const double* edge_p) {
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    nc_set_error("cannot open %s: %s", path, std::strerror(errno));
    return NC_E_IO;
  }
  Writer w(f);
  w.put("NNG 1 ");
  w.put_int(m);
  w.put(" ");
  w.put_int(e);
  w.put("\n");
  for (int64_t k = 0; k < m; ++k) {
    w.put_float(weights[k]);
    w.put_char('\n');
    w.maybe_flush();
  }
  for (int64_t k = 0; k < e; ++k) {
    w.put_int(edge_i[k]);
    w.put_char(' ');
    w.put_int(edge_j[k]);
    w.put_char(' ');
    w.put_float(edge_p[k]);
    w.put_char('\n');
    w.maybe_flush();
  }
  const bool ok = w.flush();
  if (std::fclose(f) != 0 || !ok) {
    nc_set_error("write error on %s", path);
    return NC_E_IO;
  }
  return NC_OK;
}

// ---------------------------------------------------------------- PMAP
extern "C" int nc_pmap_scan(const char* path, int64_t* n_neurons, int64_t* n_gpus, int64_t* err_line) {
  Buf b;
  if (!read_file(path, b)) return NC_E_IO;
  Lines ls{b.data.data(), b.data.data() + b.data.size()};
  std::string_view head;
  if (!ls.next(head)) return parse_error(1, err_line, "empty file");
  Header h;
  if (int e = parse_header(head, "PMAP", false, h, err_line)) return e;
  if (h.a < 1 || h.b < 1) return parse_error(1, err_line, std::string("invalid counts in header ") + py_repr(head));
  *n_neurons = h.a;
  *n_gpus = h.b;
  return NC_OK;
}

extern "C" int nc_pmap_read(const char* path, int64_t m, int64_t n, int64_t* assignment, int64_t* err_line) {
  Buf b;
  if (!read_file(path, b)) return NC_E_IO;
  const int64_t total = count_lines(b);
  Lines ls{b.data.data(), b.data.data() + b.data.size()};
  std::string_view line;
  ls.next(line);
  if (total != m + 1)
    return parse_error((total < m + 1 ? total : m + 1) + 1, err_line,
                       total < m + 1 ? "unexpected end of file" : "unexpected trailing content");
  for (int64_t k = 0; k < m; ++k) {
    ls.next(line);
    int64_t g;
    if (!py_int(line, g)) return parse_error(k + 2, err_line, "malformed GPU index " + py_repr(line));
    if (!(0 <= g && g < n))
      return parse_error(k + 2, err_line,
                         "GPU index " + std::to_string(g) + " out of range [0, " + std::to_string(n) + ")");
    assignment[k] = g;
  }
  return NC_OK;
}

extern "C" int nc_pmap_write(const char* path, int64_t m, int64_t n, const int64_t* assignment) {
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    nc_set_error("cannot open %s: %s", path, std::strerror(errno));
    return NC_E_IO;
  }
  Writer w(f);
  w.put("PMAP 1 ");
  w.put_int(m);
  w.put(" ");
  w.put_int(n);
  w.put("\n");
  for (int64_t k = 0; k < m; ++k) {
    w.put_int(assignment[k]);
    w.put_char('\n');
    w.maybe_flush();
  }
  const bool ok = w.flush();
  if (std::fclose(f) != 0 || !ok) {
    nc_set_error("write error on %s", path);
    return NC_E_IO;
  }
  return NC_OK;
}

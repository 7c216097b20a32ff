// Host-side codecs for the reference's file formats (favest/io.py:30-145,
// favest/quadrature.py:112-131): rule files, coefficient JSON, sample CSV.
// The reference formats every float with 17 significant digits
// (format(x, ".17g"), io.py:30-31) and parses with Python's float(); these
// run on memory buffers (the Python layer owns open()/read()/write(), so
// OSError behaviour is Python's own), format through std::to_chars (the same
// correctly rounded "%.17g" digits) on all host threads, and parse through
// std::from_chars after checking Python's float() grammar.  Output is byte
// identical to the reference's writers; parsed doubles are bit identical.
//
// Error text uses "{path}" where the reference prints the file name; the
// Python layer substitutes it.  FV_EINVAL -> ValueError, FV_ETYPE -> TypeError
// (the reference's unpacking / float() TypeErrors are not wrapped either).
#pragma once
#include <charconv>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace fio {

struct Buf {  // malloc-backed growable byte / double buffers handed to the caller
  char* p = nullptr;
  long long n = 0, cap = 0;
  bool reserve(long long need) {
    if (need <= cap) return true;
    long long c = cap ? cap : 4096;
    while (c < need) c *= 2;
    char* q = static_cast<char*>(std::realloc(p, (size_t)c));
    if (!q) return false;
    p = q;
    cap = c;
    return true;
  }
};

// format(x, ".17g") (io.py:30-31): Python spells every NaN "nan"
inline int fmt17(double x, char* out) {
  if (x != x) {
    std::memcpy(out, "nan", 3);
    return 3;
  }
  auto r = std::to_chars(out, out + 40, x, std::chars_format::general, 17);
  return (int)(r.ptr - out);
}

inline int host_threads(long long work) {
  unsigned hc = std::thread::hardware_concurrency();
  long long t = std::min<long long>(hc ? hc : 1, 32);
  return (int)std::max<long long>(1, std::min<long long>(t, work / 4096));
}

// run body(lo, hi, out_buffer) over row chunks on all host threads, then concatenate in order
template <class F>
int parallel_format(long long nrows, F body, Buf& out) {
  const int T = host_threads(nrows);
  std::vector<Buf> parts(T);
  std::vector<int> ok(T, 1);
  auto run = [&](int t) {
    const long long lo = nrows * t / T, hi = nrows * (t + 1) / T;
    ok[t] = body(lo, hi, parts[t]) ? 1 : 0;
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(run, t);
  run(0);
  for (auto& x : th) x.join();
  long long tot = out.n;
  for (int t = 0; t < T; ++t) {
    if (!ok[t]) return FV_ENOMEM;
    tot += parts[t].n;
  }
  if (!out.reserve(tot + 1)) return FV_ENOMEM;
  for (int t = 0; t < T; ++t) {
    if (parts[t].n) std::memcpy(out.p + out.n, parts[t].p, (size_t)parts[t].n);
    out.n += parts[t].n;
    std::free(parts[t].p);
  }
  return FV_OK;
}

// ---- Python float() grammar (PEP 515 underscores, inf / infinity / nan) ----
inline bool py_space(unsigned char c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f); }

inline bool ieq(const char* s, long long n, const char* w) {
  const long long k = (long long)std::strlen(w);
  if (n != k) return false;
  for (long long i = 0; i < n; ++i)
    if ((s[i] | 0x20) != w[i]) return false;
  return true;
}

// digits with single underscores between digits; appends the digits to tmp
inline bool py_digits(const char*& s, const char* e, std::string& tmp) {
  if (s >= e || !(*s >= '0' && *s <= '9')) return false;
  while (s < e) {
    if (*s >= '0' && *s <= '9') {
      tmp.push_back(*s++);
    } else if (*s == '_' && s + 1 < e && s[1] >= '0' && s[1] <= '9') {
      ++s;
    } else {
      break;
    }
  }
  return true;
}

inline bool py_float(const char* s, long long n, double& v) {
  const char* e = s + n;
  while (s < e && py_space((unsigned char)*s)) ++s;
  while (e > s && py_space((unsigned char)e[-1])) --e;
  bool neg = false;
  if (s < e && (*s == '+' || *s == '-')) neg = *s++ == '-';
  const long long k = e - s;
  if (ieq(s, k, "inf") || ieq(s, k, "infinity")) {
    v = neg ? -HUGE_VAL : HUGE_VAL;
    return true;
  }
  if (ieq(s, k, "nan")) {
    v = neg ? -NAN : NAN;
    return true;
  }
  thread_local std::string tmp;
  tmp.clear();
  const char* p = s;
  bool intd = false, fracd = false;
  if (p < e && *p >= '0' && *p <= '9') intd = py_digits(p, e, tmp);
  if (p < e && *p == '.') {
    tmp.push_back('.');
    ++p;
    if (p < e && *p >= '0' && *p <= '9') fracd = py_digits(p, e, tmp);
  }
  if (!intd && !fracd) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    tmp.push_back('e');
    ++p;
    if (p < e && (*p == '+' || *p == '-')) tmp.push_back(*p++);
    if (!py_digits(p, e, tmp)) return false;
  }
  if (p != e) return false;
  auto r = std::from_chars(tmp.data(), tmp.data() + tmp.size(), v);
  if (r.ec == std::errc::result_out_of_range) {  // Python: overflow -> inf, underflow -> 0
    bool big = false;
    const size_t ep = tmp.find('e');
    if (ep != std::string::npos) big = tmp[ep + 1] != '-';
    else big = true;
    v = big ? HUGE_VAL : 0.0;
  } else if (r.ec != std::errc() || r.ptr != tmp.data() + tmp.size()) {
    return false;
  }
  if (neg) v = -v;
  return true;
}

inline std::string py_repr(const char* s, long long n) {  // repr() of an ASCII str, enough for messages
  std::string t(s, (size_t)n);
  const bool dq = t.find('\'') != std::string::npos && t.find('"') == std::string::npos;
  return (dq ? "\"" : "'") + t + (dq ? "\"" : "'");
}

inline std::string float_err(const char* s, long long n) {
  return "could not convert string to float: " + py_repr(s, n);
}

}  // namespace fio

// ------------------------------------------------------------------- writers

extern "C" void fv_io_free(void* p) { std::free(p); }

// Rows of doubles as text: sep ' ' (rule files, io.py:33-38, "\n") or ','
// (csv.writer, io.py:98-108 / 136-145, "\r\n").  Appends to *out (malloc'd,
// may be NULL on entry with *len = 0, e.g. after a header written by the caller).
extern "C" int fv_io_format_table(const double* data, long long nrows, int ncols, int sep, int crlf, char** out,
                                  long long* len) {
  if (!out || !len || nrows < 0 || ncols < 1 || (nrows && !data)) return fail(FV_EINVAL, "invalid table arguments");
  fio::Buf b;
  b.p = *out;
  b.n = b.cap = *len;
  const int rc = fio::parallel_format(nrows, [&](long long lo, long long hi, fio::Buf& o) {
    for (long long r = lo; r < hi; ++r) {
      if (!o.reserve(o.n + (long long)ncols * 26 + 2)) return false;
      for (int c = 0; c < ncols; ++c) {
        if (c) o.p[o.n++] = (char)sep;
        o.n += fio::fmt17(data[r * ncols + c], o.p + o.n);
      }
      if (crlf) o.p[o.n++] = '\r';
      o.p[o.n++] = '\n';
    }
    return true;
  }, b);
  *out = b.p;
  *len = b.n;
  return rc == FV_OK ? FV_OK : fail(rc, "out of host memory formatting a table");
}

// Coefficient file (io.py:62-77): {"L_max": L, "a": [[re, im], ...], "b": [...]}
extern "C" int fv_io_format_coefficients(int lmax, const double* a, const double* b, char** out, long long* len) {
  if (!out || !len || lmax < 0 || !a || !b) return fail(FV_EINVAL, "invalid coefficient arguments");
  const long long K = (long long)(lmax + 1) * (lmax + 1);
  fio::Buf o;
  auto lit = [&](const char* s) {
    const long long k = (long long)std::strlen(s);
    if (!o.reserve(o.n + k + 1)) return false;
    std::memcpy(o.p + o.n, s, (size_t)k);
    o.n += k;
    return true;
  };
  std::string head = "{\n  \"L_max\": " + std::to_string(lmax) + ",\n  \"a\": [";
  bool ok = lit(head.c_str());
  for (int which = 0; ok && which < 2; ++which) {
    const double* v = which ? b : a;
    const int rc = fio::parallel_format(K, [&](long long lo, long long hi, fio::Buf& p) {
      for (long long k = lo; k < hi; ++k) {
        if (!p.reserve(p.n + 60)) return false;
        char* q = p.p + p.n;
        if (k) { *q++ = ','; *q++ = ' '; }
        *q++ = '[';
        q += fio::fmt17(v[2 * k], q);
        *q++ = ',';
        *q++ = ' ';
        q += fio::fmt17(v[2 * k + 1], q);
        *q++ = ']';
        p.n = q - p.p;
      }
      return true;
    }, o);
    ok = rc == FV_OK && lit(which ? "]\n}\n" : "],\n  \"b\": [");
  }
  if (!ok) {
    std::free(o.p);
    return fail(FV_ENOMEM, "out of host memory formatting coefficients");
  }
  *out = o.p;
  *len = o.n;
  return FV_OK;
}

// ------------------------------------------------------------------- readers

namespace fio {

// split text into lines the way Python's universal newlines / csv do: \n, \r\n, \r
struct Lines {
  const char* p;
  const char* e;
  bool next(const char*& s, const char*& t) {
    if (p >= e) return false;
    s = p;
    while (p < e && *p != '\n' && *p != '\r') ++p;
    t = p;
    if (p < e && *p == '\r') ++p;
    if (p < e && p[-1] == '\r' && *p == '\n') ++p;
    else if (p < e && *p == '\n' && (p == s || p[-1] != '\r')) ++p;
    return true;
  }
};

inline bool ascii_only(const char* s, long long n) {
  for (long long i = 0; i < n; ++i)
    if ((unsigned char)s[i] >= 0x80) return false;
  return true;
}

}  // namespace fio

namespace fio {

// One chunk of whole lines of a column file, parsed independently; the chunks'
// results are stitched in file order (global line numbers, the first data
// line's width, the first error).
struct ColChunk {
  Buf out;                   // doubles, rows x width
  long long rows = 0, lines = 0;
  int width = -1;            // width of the chunk's first data line
  long long first_data = -1; // local line of the first data line
  long long err_line = -1;   // local line of the first error
  int err_kind = 0;          // 1 width mismatch (err_got), 2 float (err_text), 3 out of memory
  long long err_got = 0;
  std::string err_text;
};

inline void parse_chunk(const char* s0, const char* e0, int mode, bool file_start, ColChunk& r) {
  Lines ln{s0, e0};
  const char *s, *t;
  std::vector<std::pair<const char*, long long>> fields;
  std::vector<std::string> owned;
  while (ln.next(s, t)) {
    const long long lineno = ++r.lines;
    fields.clear();
    owned.clear();
    if (mode == 0) {
      const char* h = static_cast<const char*>(std::memchr(s, '#', (size_t)(t - s)));
      const char* q = h ? h : t;
      const char* p = s;
      while (p < q) {
        while (p < q && (py_space((unsigned char)*p) || *p == ',')) ++p;
        if (p >= q) break;
        const char* f = p;
        while (p < q && !(py_space((unsigned char)*p) || *p == ',')) ++p;
        fields.emplace_back(f, p - f);
      }
      if (fields.empty()) continue;
      if (r.width < 0) {
        r.width = (int)fields.size();
        r.first_data = lineno;
      } else if ((int)fields.size() != r.width) {
        r.err_line = lineno;
        r.err_kind = 1;
        r.err_got = (long long)fields.size();
        return;
      }
    } else {
      if (s == t) continue;  // csv yields [] for a blank line
      const char* p = s;
      while (true) {  // csv field splitter with "..." quoting
        if (p < t && *p == '"') {
          std::string v;
          ++p;
          while (p < t) {
            if (*p == '"') {
              if (p + 1 < t && p[1] == '"') { v.push_back('"'); p += 2; continue; }
              ++p;
              break;
            }
            v.push_back(*p++);
          }
          const char* f = p;
          while (p < t && *p != ',') ++p;
          v.append(f, (size_t)(p - f));
          owned.push_back(v);
          fields.emplace_back(nullptr, (long long)owned.size() - 1);
        } else {
          const char* f = p;
          while (p < t && *p != ',') ++p;
          fields.emplace_back(f, p - f);
        }
        if (p < t && *p == ',') { ++p; continue; }
        break;
      }
      for (auto& fd : fields)
        if (!fd.first) {
          const std::string& v = owned[(size_t)fd.second];
          fd = {v.data(), (long long)v.size()};
        }
      const char* f0 = fields[0].first;
      const long long k0 = fields[0].second;
      long long a = 0, b = k0;
      while (a < b && py_space((unsigned char)f0[a])) ++a;
      if (a < b && f0[a] == '#') continue;
      if (file_start && lineno == 1) {
        while (b > a && py_space((unsigned char)f0[b - 1])) --b;
        if (ieq(f0 + a, b - a, "theta")) continue;
      }
      if (fields.size() != 8) {
        r.err_line = lineno;
        r.err_kind = 1;
        r.err_got = (long long)fields.size();
        r.width = 8;
        return;
      }
      if (r.width < 0) {
        r.width = 8;
        r.first_data = lineno;
      }
    }
    if (!r.out.reserve((r.rows + 1) * r.width * 8)) {
      r.err_line = lineno;
      r.err_kind = 3;
      return;
    }
    double* d = reinterpret_cast<double*>(r.out.p) + r.rows * r.width;
    for (int c = 0; c < r.width; ++c)
      if (!py_float(fields[c].first, fields[c].second, d[c])) {
        r.err_line = lineno;
        r.err_kind = 2;
        r.err_text = float_err(fields[c].first, fields[c].second);
        return;
      }
    ++r.rows;
  }
}

}  // namespace fio

// Column files.  mode 0: rule / design files (favest/quadrature.py:112-131):
// '#' starts a comment, ',' is a separator, fields split on whitespace, every
// data line has the first line's width.  mode 1: sample CSV (io.py:111-133):
// csv records, '#' rows and the "theta" header skipped, 8 fields per row.
// The text is cut at line boundaries into one chunk per host thread.
extern "C" int fv_io_parse_columns(const char* text, long long n, int mode, double** data, long long* nrows,
                                   int* ncols) {
  if (!data || !nrows || !ncols || n < 0 || (n && !text)) return fail(FV_EINVAL, "invalid parse arguments");
  *data = nullptr;
  *nrows = 0;
  *ncols = 0;
  if (!fio::ascii_only(text, n)) return fail(FV_EINVAL, "{path}: non-ASCII content");
  const int T = fio::host_threads(n / 64);
  std::vector<const char*> cut(T + 1);
  cut[0] = text;
  cut[T] = text + n;
  for (int k = 1; k < T; ++k) {  // after the next line break at or past k n / T
    const char* p = std::max(cut[k - 1], text + n * k / T);
    while (p < text + n && *p != '\n' && *p != '\r') ++p;
    if (p < text + n && *p == '\r') ++p;
    if (p < text + n && *p == '\n') ++p;
    cut[k] = p;
  }
  std::vector<fio::ColChunk> ch(T);
  {
    std::vector<std::thread> th;
    for (int k = 1; k < T; ++k) th.emplace_back([&, k] { fio::parse_chunk(cut[k], cut[k + 1], mode, false, ch[k]); });
    fio::parse_chunk(cut[0], cut[1], mode, true, ch[0]);
    for (auto& x : th) x.join();
  }
  auto release = [&] {
    for (auto& c : ch) std::free(c.out.p);
  };
  int W = -1;
  long long before = 0, rows = 0;
  for (int k = 0; k < T; ++k) {
    fio::ColChunk& c = ch[k];
    if (W < 0 && c.width >= 0) W = c.width;
    std::string msg;
    if (mode == 0 && c.first_data >= 0 && c.width != W) {
      msg = "{path}:" + std::to_string(before + c.first_data) + ": expected " + std::to_string(W) + " columns, got " +
            std::to_string(c.width);
    } else if (c.err_kind == 1) {
      msg = "{path}:" + std::to_string(before + c.err_line) + ": expected " + std::to_string(mode ? 8 : W) +
            " columns, got " + std::to_string(c.err_got);
    } else if (c.err_kind == 2) {
      msg = "{path}:" + std::to_string(before + c.err_line) + ": " + c.err_text;
    } else if (c.err_kind == 3) {
      release();
      return fail(FV_ENOMEM, "out of host memory parsing columns");
    }
    if (!msg.empty()) {
      release();
      return fail(FV_EINVAL, msg);
    }
    before += c.lines;
    rows += c.rows;
  }
  if (rows == 0) {
    release();
    return fail(FV_EINVAL, mode == 0 ? "no data rows in {path}" : "{path}: no sample rows");
  }
  double* out = static_cast<double*>(std::malloc((size_t)rows * W * 8));
  if (!out) {
    release();
    return fail(FV_ENOMEM, "out of host memory parsing columns");
  }
  {
    std::vector<std::thread> th;
    long long off = 0;
    for (int k = 0; k < T; ++k) {
      const long long nb = ch[k].rows * W * 8;
      if (nb) th.emplace_back([&, k, off, nb] { std::memcpy(reinterpret_cast<char*>(out) + off, ch[k].out.p, (size_t)nb); });
      off += nb;
    }
    for (auto& x : th) x.join();
  }
  release();
  *data = out;
  *nrows = rows;
  *ncols = W;
  return FV_OK;
}

// ---- coefficient JSON (io.py:80-95): json.load, then L_max / a / b --------

namespace fio {

struct Json {
  const char* b;  // document start (for positions)
  const char* p;
  const char* e;
  std::string err;

  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool fail_at(const char* what) {
    long long pos = p - b, line = 1, col = 1;
    for (const char* q = b; q < p; ++q) {
      if (*q == '\n') { ++line; col = 1; } else { ++col; }
    }
    err = std::string(what) + ": line " + std::to_string(line) + " column " + std::to_string(col) + " (char " +
          std::to_string(pos) + ")";
    return false;
  }
  bool lit(const char* w) {
    const size_t k = std::strlen(w);
    if ((size_t)(e - p) >= k && std::memcmp(p, w, k) == 0) {
      p += k;
      return true;
    }
    return false;
  }
  bool string(std::string* out) {  // p at '"'
    ++p;
    while (p < e) {
      const char c = *p;
      if (c == '"') { ++p; return true; }
      if ((unsigned char)c < 0x20) return fail_at("Invalid control character at");
      if (c == '\\') {
        if (p + 1 >= e) break;
        const char x = p[1];
        char r = 0;
        switch (x) {
          case '"': r = '"'; break;
          case '\\': r = '\\'; break;
          case '/': r = '/'; break;
          case 'b': r = '\b'; break;
          case 'f': r = '\f'; break;
          case 'n': r = '\n'; break;
          case 'r': r = '\r'; break;
          case 't': r = '\t'; break;
          case 'u': {
            if (e - p < 6) return fail_at("Invalid \\uXXXX escape");
            unsigned v = 0;
            for (int i = 2; i < 6; ++i) {
              const char h = p[i];
              v = v * 16 + (h >= '0' && h <= '9' ? h - '0' : (h | 0x20) >= 'a' && (h | 0x20) <= 'f' ? (h | 0x20) - 'a' + 10 : 99);
              if (v > 0xffff) return fail_at("Invalid \\uXXXX escape");
            }
            if (out) out->push_back(v < 0x80 ? (char)v : '\x7f');  // non-ASCII never parses as a float
            p += 6;
            continue;
          }
          default: return fail_at("Invalid \\escape");
        }
        if (out) out->push_back(r);
        p += 2;
        continue;
      }
      if (out) out->push_back(c);
      ++p;
    }
    return fail_at("Unterminated string starting at");
  }
  bool number() {  // JSON number grammar (json.scanner NUMBER_RE)
    const char* s = p;
    if (p < e && *p == '-') ++p;
    if (p < e && *p == '0') ++p;
    else if (p < e && *p >= '1' && *p <= '9') while (p < e && *p >= '0' && *p <= '9') ++p;
    else { p = s; return fail_at("Expecting value"); }
    if (p + 1 < e && *p == '.' && p[1] >= '0' && p[1] <= '9') {
      ++p;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      const char* q = p + 1;
      if (q < e && (*q == '+' || *q == '-')) ++q;
      if (q < e && *q >= '0' && *q <= '9') {
        p = q;
        while (p < e && *p >= '0' && *p <= '9') ++p;
      }
    }
    return true;
  }
  bool value(int depth) {  // syntax only
    ws();
    if (p >= e) return fail_at("Expecting value");
    const char c = *p;
    if (c == '"') return string(nullptr);
    if (c == '{') return object(depth + 1, nullptr);
    if (c == '[') {
      ++p;
      ws();
      if (p < e && *p == ']') { ++p; return true; }
      while (true) {
        if (!value(depth + 1)) return false;
        ws();
        if (p < e && *p == ',') { ++p; continue; }
        if (p < e && *p == ']') { ++p; return true; }
        return fail_at("Expecting ',' delimiter");
      }
    }
    if (lit("true") || lit("false") || lit("null") || lit("NaN") || lit("Infinity") || lit("-Infinity")) return true;
    return number();
  }
  // object; when top is given, records the last span of each top-level key
  bool object(int depth, std::vector<std::pair<std::string, std::pair<const char*, const char*>>>* top) {
    if (depth > 900) return fail_at("maximum recursion depth exceeded");
    ++p;
    ws();
    if (p < e && *p == '}') { ++p; return true; }
    while (true) {
      ws();
      if (p >= e || *p != '"') return fail_at("Expecting property name enclosed in double quotes");
      std::string key;
      if (!string(top ? &key : nullptr)) return false;
      ws();
      if (p >= e || *p != ':') return fail_at("Expecting ':' delimiter");
      ++p;
      ws();
      const char* vs = p;
      if (!value(depth)) return false;
      if (top) top->push_back({key, {vs, p}});
      ws();
      if (p < e && *p == ',') { ++p; continue; }
      if (p < e && *p == '}') { ++p; return true; }
      return fail_at("Expecting ',' delimiter");
    }
  }
};

// float(x) of a JSON scalar at p (already syntax-checked); 0 ok, FV_EINVAL / FV_ETYPE with msg
inline int json_float(const char*& p, const char* e, double& v, std::string& msg) {
  if (*p == '"') {
    Json j{p, p, e, {}};
    std::string s;
    j.string(&s);
    p = j.p;
    if (!py_float(s.data(), (long long)s.size(), v)) {
      msg = float_err(s.data(), (long long)s.size());
      return FV_EINVAL;
    }
    return FV_OK;
  }
  auto take = [&](const char* w, double x) {
    const size_t k = std::strlen(w);
    if ((size_t)(e - p) >= k && std::memcmp(p, w, k) == 0) { p += k; v = x; return true; }
    return false;
  };
  if (take("true", 1.0) || take("false", 0.0) || take("NaN", NAN) || take("Infinity", HUGE_VAL) ||
      take("-Infinity", -HUGE_VAL))
    return FV_OK;
  if (*p == 'n' || *p == '[' || *p == '{') {
    msg = std::string("float() argument must be a string or a real number, not '") +
          (*p == 'n' ? "NoneType" : *p == '[' ? "list" : "dict") + "'";
    return FV_ETYPE;
  }
  Json j{p, p, e, {}};
  const char* s = p;
  j.number();
  p = j.p;
  const char* q = s[0] == '-' ? s + 1 : s;
  auto r = std::from_chars(q, p, v);
  if (r.ec == std::errc::result_out_of_range) {
    const bool isint = std::memchr(s, '.', (size_t)(p - s)) == nullptr && std::memchr(s, 'e', (size_t)(p - s)) == nullptr &&
                       std::memchr(s, 'E', (size_t)(p - s)) == nullptr;
    if (isint) {  // float(int) overflows
      msg = "int too large to convert to float";
      return FV_EINVAL;
    }
    const char* ep = static_cast<const char*>(std::memchr(s, 'e', (size_t)(p - s)));
    if (!ep) ep = static_cast<const char*>(std::memchr(s, 'E', (size_t)(p - s)));
    v = (ep && ep[1] == '-') ? 0.0 : HUGE_VAL;
  }
  if (s[0] == '-') v = -v;
  if (v == 0.0 && std::memchr(s, '.', (size_t)(p - s)) == nullptr && std::memchr(s, 'e', (size_t)(p - s)) == nullptr &&
      std::memchr(s, 'E', (size_t)(p - s)) == nullptr)
    v = 0.0;  // json gives int -0 == 0: float() of it is +0.0
  return FV_OK;
}

}  // namespace fio

// Parse a coefficient file: *lmax and two malloc'd complex128 arrays (free with
// fv_io_free).  Checks and messages follow read_coefficients (io.py:80-95).
extern "C" int fv_io_parse_coefficients(const char* text, long long n, int* lmax, double** a, double** b) {
  if (!lmax || !a || !b || n < 0 || (n && !text)) return fail(FV_EINVAL, "invalid parse arguments");
  *a = *b = nullptr;
  fio::Json j{text, text, text + n, {}};
  std::vector<std::pair<std::string, std::pair<const char*, const char*>>> top;
  j.ws();
  bool ok;
  bool is_obj = j.p < j.e && *j.p == '{';
  if (is_obj) ok = j.object(0, &top);
  else ok = j.value(0);
  if (ok) {
    j.ws();
    if (j.p != j.e) ok = j.fail_at("Extra data");
  }
  if (!ok) return fail(FV_EINVAL, "{path}: not a valid coefficient file: " + j.err);
  auto find = [&](const char* k) -> const std::pair<const char*, const char*>* {
    const std::pair<const char*, const char*>* r = nullptr;
    for (auto& kv : top)
      if (kv.first == k) r = &kv.second;  // duplicate keys: the last wins (json.load)
    return r;
  };
  const auto* sl = find("L_max");
  const auto* sa = find("a");
  const auto* sb = find("b");
  if (!is_obj || !sl || !sa || !sb) return fail(FV_EINVAL, "{path}: missing L_max/a/b fields");
  // int(doc["L_max"])
  long long L = 0;
  {
    const char* p = sl->first;
    const char c = *p;
    if (c == 'n' || c == '[' || c == '{') return fail(FV_EINVAL, "{path}: missing L_max/a/b fields");
    if (c == '"') {
      fio::Json s{p, p, sl->second, {}};
      std::string v;
      s.string(&v);
      size_t i = 0, k = v.size();
      while (i < k && fio::py_space((unsigned char)v[i])) ++i;
      while (k > i && fio::py_space((unsigned char)v[k - 1])) --k;
      std::string d;
      size_t q = i;
      if (q < k && (v[q] == '+' || v[q] == '-')) d.push_back(v[q++]);
      const char* dp = v.data() + q;
      const char* de = v.data() + k;
      if (!fio::py_digits(dp, de, d) || dp != de)
        return fail(FV_EINVAL, "invalid literal for int() with base 10: " + fio::py_repr(v.data(), (long long)v.size()));
      L = std::strtoll(d.c_str(), nullptr, 10);
    } else if (fio::ieq(p, 4, "true")) {
      L = 1;
    } else if (fio::ieq(p, 5, "false")) {
      L = 0;
    } else {
      double x;
      std::string msg;
      const char* q = p;
      fio::json_float(q, sl->second, x, msg);
      if (x != x) return fail(FV_EINVAL, "cannot convert float NaN to integer");
      if (x == HUGE_VAL || x == -HUGE_VAL) return fail(FV_EINVAL, "cannot convert float infinity to integer");
      L = (long long)x;  // int() truncates toward zero
    }
  }
  if (L < 0) return fail(FV_EINVAL, "lmax must be non-negative, got " + std::to_string(L));
  if (L > 1000000) return fail(FV_EINVAL, "{path}: L_max=" + std::to_string(L) + " out of range");
  const long long size = (L + 1) * (L + 1);
  double* outs[2] = {nullptr, nullptr};
  const std::pair<const char*, const char*>* spans[2] = {sa, sb};
  const char* labels[2] = {"a", "b"};
  for (int w = 0; w < 2; ++w) {
    const char* p = spans[w]->first;
    const char* e = spans[w]->second;
    auto bail = [&](int code, const std::string& m) {
      std::free(outs[0]);
      std::free(outs[1]);
      return fail(code, m);
    };
    if (*p != '[') {
      if (*p == '"' || *p == '{')
        return bail(FV_EINVAL, std::string("{path}: array '") + labels[w] + "' is not a list of [re, im] pairs");
      return bail(FV_ETYPE, "object of type '" + std::string(*p == 'n' ? "NoneType" : "float") + "' has no len()");
    }
    // count entries (top level of this array), remembering where every
    // CH-th one starts: the conversion runs in one chunk per host thread
    long long cnt = 0;
    const int T = fio::host_threads(size / 8);
    const long long CH = std::max<long long>(1, (size + T - 1) / T);
    std::vector<const char*> starts;
    {
      fio::Json s{text, p + 1, e, {}};
      s.ws();
      if (s.p < e && *s.p != ']') {
        while (true) {
          if (cnt % CH == 0) starts.push_back(s.p);
          s.value(0);
          ++cnt;
          s.ws();
          if (s.p < e && *s.p == ',') { ++s.p; continue; }
          break;
        }
      }
    }
    if (cnt != size)
      return bail(FV_EINVAL, std::string("{path}: array '") + labels[w] + "' has " + std::to_string(cnt) +
                                 " entries, expected " + std::to_string(size) + " for L_max=" + std::to_string(L));
    outs[w] = static_cast<double*>(std::malloc((size_t)std::max<long long>(size, 1) * 16));
    if (!outs[w]) return bail(FV_ENOMEM, "out of host memory");
    double* ow = outs[w];
    // convert elements [k0, k1) from their first character; returns the index
    // of the first failing element (code / msg set) or -1
    auto conv = [&](long long k0, long long k1, const char* from, int& code, std::string& msg) -> long long {
#define FV_FAILK(c_, m_) \
  do {                   \
    code = (c_);         \
    msg = (m_);          \
    return k;            \
  } while (0)
      fio::Json s{text, from, e, {}};
      for (long long k = k0; k < k1; ++k) {
      s.ws();
      const char c = *s.p;
      if (c != '[') {
        if (c == '"' || c == '{') {
          // re, im = pair iterates a str's characters / a dict's keys
          std::vector<std::string> items;
          fio::Json q{text, s.p, e, {}};
          if (c == '"') {
            std::string v;
            q.string(&v);
            for (char ch : v) items.push_back(std::string(1, ch));
          } else {
            ++q.p;
            q.ws();
            while (q.p < e && *q.p == '"') {
              std::string key;
              q.string(&key);
              q.ws();
              ++q.p;  // ':'
              q.value(0);
              q.ws();
              bool dup = false;
              for (auto& it : items) dup |= it == key;
              if (!dup) items.push_back(key);
              if (*q.p == ',') { ++q.p; q.ws(); }
            }
            ++q.p;  // '}'
          }
          if (items.size() != 2)
            FV_FAILK(FV_EINVAL, items.size() > 2 ? "too many values to unpack (expected 2)"
                                                    : "not enough values to unpack (expected 2, got " +
                                                          std::to_string(items.size()) + ")");
          double v2[2];
          for (int c2 = 0; c2 < 2; ++c2)
            if (!fio::py_float(items[c2].data(), (long long)items[c2].size(), v2[c2]))
              FV_FAILK(FV_EINVAL, fio::float_err(items[c2].data(), (long long)items[c2].size()));
          ow[2 * k] = v2[0];
          ow[2 * k + 1] = v2[1];
          s.p = q.p;
          s.ws();
          if (s.p < e && *s.p == ',') ++s.p;
          continue;
        }
        const char* vs = s.p;
        s.value(0);
        bool isint = true;
        for (const char* q = vs; q < s.p; ++q) isint &= !(*q == '.' || *q == 'e' || *q == 'E' || *q == 'N' || *q == 'I');
        FV_FAILK(FV_ETYPE, std::string("cannot unpack non-iterable ") +
                                  (c == 'n' ? "NoneType" : (c == 't' || c == 'f') ? "bool" : isint ? "int" : "float") +
                                  " object");
      }
      ++s.p;
      const char* el[3];
      const char* ee[3];
      int got = 0;
      s.ws();
      if (*s.p != ']') {
        while (true) {
          s.ws();
          const char* vs = s.p;
          s.value(0);
          if (got < 3) { el[got] = vs; ee[got] = s.p; }
          ++got;
          s.ws();
          if (*s.p == ',') { ++s.p; continue; }
          break;
        }
      }
      ++s.p;  // ']'
      if (got != 2)  // re, im = pair (io.py:91)
        FV_FAILK(FV_EINVAL, got > 2 ? "too many values to unpack (expected 2)"
                                       : "not enough values to unpack (expected 2, got " + std::to_string(got) + ")");
      double v[2];
      for (int c2 = 0; c2 < 2; ++c2) {  // float(re), float(im): not wrapped with the path (io.py:92)
        std::string fmsg;
        const char* q = el[c2];
        const int rc = fio::json_float(q, ee[c2], v[c2], fmsg);
        if (rc != FV_OK) FV_FAILK(rc, fmsg);
      }
      ow[2 * k] = v[0];
      ow[2 * k + 1] = v[1];
      s.ws();
      if (s.p < e && *s.p == ',') ++s.p;
      }
#undef FV_FAILK
      return -1;
    };
    const int nch = (int)starts.size();
    std::vector<long long> ek(nch, -1);
    std::vector<int> ec(nch, 0);
    std::vector<std::string> em(nch);
    {
      std::vector<std::thread> th;
      for (int t = 1; t < nch; ++t)
        th.emplace_back([&, t] { ek[t] = conv(t * CH, std::min(size, (t + 1) * CH), starts[t], ec[t], em[t]); });
      if (nch) ek[0] = conv(0, std::min(size, CH), starts[0], ec[0], em[0]);
      for (auto& x : th) x.join();
    }
    for (int t = 0; t < nch; ++t)
      if (ek[t] >= 0) return bail(ec[t], em[t]);
  }
  *lmax = (int)L;
  *a = outs[0];
  *b = outs[1];
  return FV_OK;
}

// Native parser for the body of a phenotype / covariate table (host code).
//
// Semantics of the reference loader (/root/reference/pkg/src/panelgwas/phenotypes.py:67-138):
//   * one record per line; blank lines are skipped; every other line must have exactly
//     n_fields delimiter-separated cells ("ragged row" error with its 1-based line number);
//   * the ID cell is whitespace-stripped;
//   * a value cell is stripped, then: in {"", "NA", "NaN", "nan", "-9"} -> NaN (missing);
//     otherwise parsed like Python float(); unparseable or non-finite -> NaN and counted as
//     unparseable for its column (the reference's fast numpy path gives the same values
//     whenever it is taken, so the cell rule is the whole contract).
// Inputs the simple grammar cannot decide byte-for-byte like Python's csv module + float()
// (quote characters, a bare '\r', non-ASCII bytes, digit-group underscores) make the
// parser report PG_TABLE_GENERIC so the caller can use the csv-module path instead.
//
// Work is split over lines (one sample per line, tens of thousands of cells each) across
// host threads; the first ragged line is found deterministically (minimum over threads).
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "pg_common.cuh"

namespace pg {
namespace {

inline bool is_space(unsigned char c) {
  // ASCII characters Python's str.strip() removes
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}

inline bool is_missing_token(const char* s, size_t n) {
  switch (n) {
    case 0: return true;
    case 2: return s[0] == 'N' && s[1] == 'A';
    case 3:
      return (s[0] == 'N' && s[1] == 'a' && s[2] == 'N') || (s[0] == 'n' && s[1] == 'a' && s[2] == 'n');
    default: return false;
  }
}

inline bool is_minus_nine(const char* s, size_t n) { return n == 2 && s[0] == '-' && s[1] == '9'; }

// Python float() on an ASCII token without underscores -> (value, ok). ok=false means
// ValueError; non-finite results are returned as such.
inline bool py_float(const char* s, size_t n, double& out) {
  const char* b = s;
  const char* e = s + n;
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
    if (b < e && (*b == '+' || *b == '-')) return false;
  }
  if (b == e) return false;
  double v = 0.0;
  auto r = std::from_chars(b, e, v, std::chars_format::general);
  if (r.ptr != e) {
    return false;
  }
  if (r.ec == std::errc::result_out_of_range) {
    // over/underflow: strtod gives Python's result (0.0, a subnormal, or +-inf)
    std::string tmp(b, e);
    v = std::strtod(tmp.c_str(), nullptr);
  } else if (r.ec != std::errc()) {
    return false;
  }
  out = neg ? -v : v;
  return true;
}

struct Line {
  int64_t begin, end;  // [begin, end) without the line terminator
  int64_t lineno;      // 1-based physical line number
};

inline bool has_special(const char* s, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    const unsigned char c = static_cast<unsigned char>(s[i]);
    if (c == '"' || c == '\r' || c >= 0x80 || c == '_' || c == 0) return true;
  }
  return false;
}

// Non-blank lines of buf[body_offset, len) with their 1-based physical line numbers (a CR
// before the LF is not part of the line). The newline scan -- a pass over the whole table,
// gigabytes at C3 -- is split over threads by byte range; the line list is then assembled
// in order.
std::vector<Line> find_lines(const char* buf, int64_t len, int64_t body_offset, int64_t first_lineno, int nt) {
  const int64_t span = len - body_offset;
  if (span <= (int64_t{8} << 20)) nt = 1;
  std::vector<std::vector<int64_t>> nl(nt);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
      th.emplace_back([&, t] {
        int64_t pos = body_offset + span * t / nt;
        const int64_t stop = body_offset + span * (t + 1) / nt;
        while (pos < stop) {
          const void* hit = std::memchr(buf + pos, '\n', static_cast<size_t>(stop - pos));
          if (!hit) break;
          const int64_t at = static_cast<const char*>(hit) - buf;
          nl[t].push_back(at);
          pos = at + 1;
        }
      });
    }
    for (auto& x : th) x.join();
  }
  std::vector<Line> lines;
  int64_t begin = body_offset, lineno = first_lineno;
  auto add = [&](int64_t end) {
    int64_t stop = end;
    if (stop > begin && buf[stop - 1] == '\r') --stop;
    if (stop > begin) lines.push_back({begin, stop, lineno});
    begin = end + 1;
    ++lineno;
  };
  for (const auto& v : nl)
    for (int64_t e : v) add(e);
  if (begin < len) add(len);
  return lines;
}

}  // namespace
}  // namespace pg

extern "C" {

// Returns PG_OK, PG_TABLE_GENERIC (caller must use the generic path) or an error.
// Two calls: values == NULL -> *n_rows = number of records (non-blank lines); then with
// buffers sized n_rows x (n_fields - 1) / n_rows / (n_fields - 1). Ragged records are
// reported by the second call (PG_ERR_FORMAT, *err_line / *err_cells: the first one).
//
// One pass per line: fields are found with memchr, a value cell is stripped only when
// it starts or ends with whitespace, and the bytes that would make Python's csv module
// read the line differently (quote, bare CR, non-ASCII, NUL, '_' digit groups) can only
// occur in a cell that fails to parse as a number or in the ID cell, so only those are
// scanned for them.
int pg_table_parse(const char* buf, int64_t len, int64_t body_offset, char delim, int64_t n_fields, int64_t id_field,
                   int n_threads, int64_t first_lineno, int64_t* n_rows, double* values, int64_t* id_off,
                   int64_t* id_len, int64_t* missing, int64_t* unparseable, int64_t* err_line, int64_t* err_cells) {
  using pg::Line;
  PG_REQUIRE(buf != nullptr || len == 0, PG_ERR_INVALID, "pg_table_parse: null buffer");
  PG_REQUIRE(n_fields >= 1 && id_field >= 0 && id_field < n_fields, PG_ERR_INVALID, "pg_table_parse: bad fields");
  *err_line = 0;
  *err_cells = 0;
  // ---- records: non-blank lines (csv.reader yields [] for an empty line)
  int nt = n_threads > 0 ? n_threads : static_cast<int>(std::thread::hardware_concurrency());
  nt = std::max(1, std::min<int>(nt, 64));
  const std::vector<Line> lines = pg::find_lines(buf, len, body_offset, first_lineno, nt);
  const int64_t nr = static_cast<int64_t>(lines.size());
  *n_rows = nr;
  if (values == nullptr) return PG_OK;

  if (nr < 4 * nt) nt = static_cast<int>(std::max<int64_t>(1, nr / 4));
  const int64_t n_val = n_fields - 1;
  std::atomic<bool> generic{false};
  std::atomic<int64_t> bad_rec{INT64_MAX};  // first ragged record
  std::vector<std::vector<int64_t>> miss_t(nt, std::vector<int64_t>(n_val, 0));
  std::vector<std::vector<int64_t>> bad_t(nt, std::vector<int64_t>(n_val, 0));
  {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
      th.emplace_back([&, t] {
        int64_t* miss = miss_t[t].data();
        int64_t* bad = bad_t[t].data();
        for (int64_t r = t; r < nr; r += nt) {
          if (generic.load(std::memory_order_relaxed)) return;
          const Line& L = lines[r];
          double* out = values + r * n_val;
          int64_t k = L.begin, j = 0;
          bool ragged = false;
          for (int64_t f = 0; f < n_fields; ++f) {
            if (k > L.end) {  // fewer cells than the header
              ragged = true;
              break;
            }
            const void* dp = std::memchr(buf + k, delim, static_cast<size_t>(L.end - k));
            const int64_t e = dp ? static_cast<const char*>(dp) - buf : L.end;
            if (f == n_fields - 1 && e != L.end) {  // more cells than the header
              ragged = true;
              break;
            }
            int64_t a = k, z = e;
            if (a < z && (pg::is_space(static_cast<unsigned char>(buf[a])) ||
                          pg::is_space(static_cast<unsigned char>(buf[z - 1])))) {
              while (a < z && pg::is_space(static_cast<unsigned char>(buf[a]))) ++a;
              while (z > a && pg::is_space(static_cast<unsigned char>(buf[z - 1]))) --z;
            }
            const char* s = buf + a;
            const size_t n = static_cast<size_t>(z - a);
            if (f == id_field) {
              if (pg::has_special(buf + k, static_cast<size_t>(e - k))) generic.store(true);
              id_off[r] = a;
              id_len[r] = z - a;
            } else {
              double v = NAN;
              if (pg::is_missing_token(s, n) || pg::is_minus_nine(s, n)) {
                ++miss[j];
              } else if (!pg::py_float(s, n, v) || !std::isfinite(v)) {
                if (pg::has_special(buf + k, static_cast<size_t>(e - k))) generic.store(true);
                v = NAN;
                ++bad[j];
                ++miss[j];
              }
              out[j++] = v;
            }
            k = e + 1;
          }
          if (ragged) {
            int64_t cur = bad_rec.load();
            while (r < cur && !bad_rec.compare_exchange_weak(cur, r)) {
            }
          }
        }
      });
    }
    for (auto& x : th) x.join();
  }
  if (generic.load()) return PG_TABLE_GENERIC;
  if (bad_rec.load() != INT64_MAX) {
    // any quote / CR / non-ASCII byte on an earlier line would have made csv read differently
    const int64_t r = bad_rec.load();
    for (int64_t q = 0; q <= r; ++q)
      if (pg::has_special(buf + lines[q].begin, static_cast<size_t>(lines[q].end - lines[q].begin)))
        return PG_TABLE_GENERIC;
    const Line& L = lines[r];
    int64_t cells = 1;
    for (int64_t k = L.begin; k < L.end; ++k) cells += buf[k] == delim;
    *err_line = L.lineno;
    *err_cells = cells;
    pg::set_error("ragged row");
    return PG_ERR_FORMAT;
  }
  for (int64_t j = 0; j < n_val; ++j) {
    int64_t m = 0, b = 0;
    for (int t = 0; t < nt; ++t) {
      m += miss_t[t][j];
      b += bad_t[t][j];
    }
    missing[j] = m;
    unparseable[j] = b;
  }
  return PG_OK;
}

}  // extern "C"

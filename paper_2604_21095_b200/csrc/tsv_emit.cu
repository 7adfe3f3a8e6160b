// Native TSV record emitter (host code).
//
// The reference writes every record with Python f-strings and repr() floats
// (/root/reference/pkg/src/panelgwas/output.py:50-52, 106-113). At C3/C4 scale a
// scan emits millions of records, so the text is produced here. Floats are
// byte-identical to CPython's repr(): shortest round-trip digits
// (std::to_chars) laid out with CPython's 'r' rules — exponent form when the
// decimal point position is <= -4 or > 16, otherwise fixed with a trailing
// ".0" for integral values; "inf", "-inf", "nan".
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "pg_common.cuh"

namespace pg {
namespace {

// Python repr(float(x)) into `out`; returns the length.
int py_repr(double x, char* out) {
  if (std::isnan(x)) {
    std::memcpy(out, "nan", 3);
    return 3;
  }
  if (std::isinf(x)) {
    if (x > 0) {
      std::memcpy(out, "inf", 3);
      return 3;
    }
    std::memcpy(out, "-inf", 4);
    return 4;
  }
  char sci[64];
  auto res = std::to_chars(sci, sci + sizeof(sci) - 1, x, std::chars_format::scientific);
  *res.ptr = '\0';  // to_chars does not terminate; the exponent is parsed with atoi below
  const int len = static_cast<int>(res.ptr - sci);
  int pos = 0;
  bool neg = false;
  if (sci[0] == '-') {
    neg = true;
    pos = 1;
  }
  char digits[32];
  int nd = 0;
  int i = pos;
  for (; i < len && sci[i] != 'e'; ++i)
    if (sci[i] != '.') digits[nd++] = sci[i];
  int e = 0;
  if (i < len) e = std::atoi(sci + i + 1);
  while (nd > 1 && digits[nd - 1] == '0') --nd;  // to_chars is already shortest; defensive
  const int decpt = e + 1;                        // value = 0.DIGITS x 10^decpt
  int o = 0;
  if (neg) out[o++] = '-';
  if (decpt <= -4 || decpt > 16) {
    out[o++] = digits[0];
    if (nd > 1) {
      out[o++] = '.';
      for (int k = 1; k < nd; ++k) out[o++] = digits[k];
    }
    out[o++] = 'e';
    int ex = decpt - 1;
    out[o++] = ex < 0 ? '-' : '+';
    if (ex < 0) ex = -ex;
    char eb[8];
    int ne = 0;
    do {
      eb[ne++] = static_cast<char>('0' + ex % 10);
      ex /= 10;
    } while (ex);
    if (ne < 2) eb[ne++] = '0';
    while (ne) out[o++] = eb[--ne];
  } else if (decpt <= 0) {
    out[o++] = '0';
    out[o++] = '.';
    for (int k = 0; k < -decpt; ++k) out[o++] = '0';
    for (int k = 0; k < nd; ++k) out[o++] = digits[k];
  } else if (decpt >= nd) {
    for (int k = 0; k < nd; ++k) out[o++] = digits[k];
    for (int k = nd; k < decpt; ++k) out[o++] = '0';
    out[o++] = '.';
    out[o++] = '0';
  } else {
    for (int k = 0; k < decpt; ++k) out[o++] = digits[k];
    out[o++] = '.';
    for (int k = decpt; k < nd; ++k) out[o++] = digits[k];
  }
  return o;
}

int put_int(long long v, char* out) {
  char b[24];
  auto r = std::to_chars(b, b + sizeof(b), v);
  const int n = static_cast<int>(r.ptr - b);
  std::memcpy(out, b, n);
  return n;
}

}  // namespace
}  // namespace pg

extern "C" {

int pg_format_float_repr(const double* x, int64_t n, char* out, int64_t out_cap, int64_t* out_len) {
  int64_t o = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (o + 40 > out_cap) {
      pg::set_error("pg_format_float_repr: output buffer too small");
      return PG_ERR_INVALID;
    }
    o += pg::py_repr(x[i], out + o);
    out[o++] = '\n';
  }
  *out_len = o;
  return PG_OK;
}

// n lines of ncols tab-separated floats (Python repr), line i = cols[0][i] \t ... cols[ncols-1][i] \n
// (the effect-size sidecar of the record writers: BETA \t SE per record line).
int pg_format_float_columns(int64_t n, int ncols, const double* const* cols, char* out, int64_t out_cap,
                            int64_t* out_len) {
  int64_t o = 0;
  if (ncols < 1) {
    pg::set_error("pg_format_float_columns: ncols must be >= 1");
    return PG_ERR_INVALID;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (o + 40 * static_cast<int64_t>(ncols) > out_cap) {
      *out_len = o;
      pg::set_error("pg_format_float_columns: output buffer too small at line %lld", (long long)i);
      return PG_ERR_INVALID;
    }
    for (int j = 0; j < ncols; ++j) {
      o += pg::py_repr(cols[j][i], out + o);
      out[o++] = j + 1 < ncols ? '\t' : '\n';
    }
  }
  *out_len = o;
  return PG_OK;
}

// One TSV line per record: <marker prefix>AF\tN_MISS<mid>R\tT\tP\t<pheno>\n
//   marker prefix of row k = prefix_blob[prefix_off[k] : prefix_off[k+1]]  ("CHR\tID\tPOS\tA1\tA2\t")
//   pheno name of col j    = pheno_blob[pheno_off[j] : pheno_off[j+1]]
//   mid                    = "\t{N}\t{DF}\t"
int pg_format_tsv(int64_t n, const int64_t* rows, const int64_t* cols, const double* r, const double* t,
                  const double* p, const double* af, const int64_t* n_miss, const char* prefix_blob,
                  const int64_t* prefix_off, const char* pheno_blob, const int64_t* pheno_off, const char* mid,
                  int64_t mid_len, char* out, int64_t out_cap, int64_t* out_len) {
  // records [i0, i1) into dst (room for their worst case); returns the bytes written
  auto format_range = [&](int64_t i0, int64_t i1, char* dst) -> int64_t {
    int64_t o = 0;
    for (int64_t i = i0; i < i1; ++i) {
      const int64_t k = rows[i], j = cols[i];
      const int64_t plen = prefix_off[k + 1] - prefix_off[k];
      const int64_t nlen = pheno_off[j + 1] - pheno_off[j];
      std::memcpy(dst + o, prefix_blob + prefix_off[k], plen);
      o += plen;
      o += pg::py_repr(af[k], dst + o);
      dst[o++] = '\t';
      o += pg::put_int(n_miss[k], dst + o);
      std::memcpy(dst + o, mid, mid_len);
      o += mid_len;
      o += pg::py_repr(r[i], dst + o);
      dst[o++] = '\t';
      o += pg::py_repr(t[i], dst + o);
      dst[o++] = '\t';
      o += pg::py_repr(p[i], dst + o);
      dst[o++] = '\t';
      std::memcpy(dst + o, pheno_blob + pheno_off[j], nlen);
      o += nlen;
      dst[o++] = '\n';
    }
    return o;
  };
  auto worst = [&](int64_t i0, int64_t i1) {
    int64_t w = 0;
    for (int64_t i = i0; i < i1; ++i)
      w += (prefix_off[rows[i] + 1] - prefix_off[rows[i]]) + (pheno_off[cols[i] + 1] - pheno_off[cols[i]]) + mid_len +
           4 * 40 + 8;
    return w;
  };
  const int nt = n < (1 << 15) ? 1 : static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  if (nt == 1) {
    if (worst(0, n) > out_cap) {  // the serial path checks per record, as before
      int64_t o = 0;
      for (int64_t i = 0; i < n; ++i) {
        const int64_t need = worst(i, i + 1);
        if (o + need > out_cap) {
          *out_len = o;
          pg::set_error("pg_format_tsv: output buffer too small at record %lld", (long long)i);
          return PG_ERR_INVALID;
        }
        o += format_range(i, i + 1, out + o);
      }
      *out_len = o;
      return PG_OK;
    }
    *out_len = format_range(0, n, out);
    return PG_OK;
  }
  // records split over host threads, each into its own buffer, then concatenated in order
  std::vector<std::vector<char>> parts(nt);
  std::vector<int64_t> used(nt, 0);
  std::vector<std::thread> th;
  for (int tix = 0; tix < nt; ++tix) {
    th.emplace_back([&, tix] {
      const int64_t i0 = n * tix / nt, i1 = n * (tix + 1) / nt;
      parts[tix].resize(static_cast<size_t>(worst(i0, i1)));
      used[tix] = format_range(i0, i1, parts[tix].data());
    });
  }
  for (auto& x : th) x.join();
  int64_t o = 0;
  for (int tix = 0; tix < nt; ++tix) {
    if (o + used[tix] > out_cap) {
      *out_len = o;
      pg::set_error("pg_format_tsv: output buffer too small at record %lld", (long long)(n * tix / nt));
      return PG_ERR_INVALID;
    }
    std::memcpy(out + o, parts[tix].data(), static_cast<size_t>(used[tix]));
    o += used[tix];
  }
  *out_len = o;
  return PG_OK;
}

// FULL-mode marker sidecar lines "SOURCE_INDEX\tCHR\tID\tPOS\tA1\tA2\tAF\tN_MISS\n" for markers
// rows[0..n): the "CHR..A2\t" part comes pre-rendered per marker (prefix blob + offsets), AF as
// Python repr, integers in decimal. Replaces a Python f-string per scanned marker.
int pg_format_marker_lines(int64_t n, const int64_t* rows, const int64_t* src_index, const char* prefix_blob,
                           const int64_t* prefix_off, const double* af, const int64_t* n_miss, char* out,
                           int64_t out_cap, int64_t* out_len) {
  int64_t o = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t k = rows[i];
    const int64_t plen = prefix_off[k + 1] - prefix_off[k];
    if (o + plen + 3 * 24 + 40 > out_cap) {
      *out_len = o;
      pg::set_error("pg_format_marker_lines: output buffer too small at marker %lld", (long long)i);
      return PG_ERR_INVALID;
    }
    o += pg::put_int(src_index[k], out + o);
    out[o++] = '\t';
    std::memcpy(out + o, prefix_blob + prefix_off[k], plen);
    o += plen;
    o += pg::py_repr(af[k], out + o);
    out[o++] = '\t';
    o += pg::put_int(n_miss[k], out + o);
    out[o++] = '\n';
  }
  *out_len = o;
  return PG_OK;
}

}  // extern "C"

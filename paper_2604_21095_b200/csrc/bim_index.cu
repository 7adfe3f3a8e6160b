// PLINK .bim catalog without per-marker Python objects (host code).
//
// The reference reads the .bim line by line into MarkerRecord objects
// (/root/reference/pkg/src/panelgwas/genotypes/plink.py:64-90): six whitespace-separated
// fields per non-blank line (chrom, id, cM, position, allele1, allele2), position an
// integer >= 0. pg_bim_index validates the same grammar in one pass and records, per
// marker, where its chrom / id / allele1 / allele2 tokens sit in the file plus the parsed
// position; the Python catalog builds MarkerRecords from these only when one is asked for.
// Anything outside the plain grammar (non-ASCII bytes, a wrong field count, a position that
// is not a plain decimal) returns PG_TABLE_GENERIC and the caller's line-by-line reader
// produces the reference's exact error or result.
//
// pg_bim_prefixes renders the "CHR\tID\tPOS\tA1\tA2\t" record prefix of a marker range
// (alleles swapped when the counted allele is allele2), the per-marker part of every
// association record and FULL sidecar line.
#include <cstdint>
#include <cstring>

#include "pg_common.cuh"

namespace pg {
namespace {

inline bool bim_space(unsigned char c) {
  // bytes Python's str.split() separates ASCII text on
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}

}  // namespace
}  // namespace pg

extern "C" {

// buf[0, len): the whole .bim. cap: markers the output arrays hold (>= number of lines).
// Out: *n markers; tok_start / tok_len [n x 4] = chrom, id, allele1, allele2 byte spans;
// pos[n]; *same = markers whose two alleles are equal (the reference warns about them).
int pg_bim_index(const char* buf, int64_t len, int64_t cap, int64_t* n, int64_t* tok_start, int32_t* tok_len,
                 int64_t* pos, int64_t* same) {
  PG_REQUIRE(buf != nullptr || len == 0, PG_ERR_INVALID, "pg_bim_index: null buffer");
  int64_t m = 0, n_same = 0, i = 0;
  while (i < len) {
    int64_t st[6];
    int32_t ln[6];
    int f = 0;
    // tokens of one line
    while (i < len && buf[i] != '\n') {
      const unsigned char c = static_cast<unsigned char>(buf[i]);
      if (c >= 0x80 || c == 0) return PG_TABLE_GENERIC;
      // a bare CR ends a line for Python's text-mode reader, not for this scan
      if (c == '\r' && (i + 1 >= len || buf[i + 1] != '\n')) return PG_TABLE_GENERIC;
      if (pg::bim_space(c)) {
        ++i;
        continue;
      }
      const int64_t a = i;
      while (i < len && buf[i] != '\n' && !pg::bim_space(static_cast<unsigned char>(buf[i]))) {
        if (static_cast<unsigned char>(buf[i]) >= 0x80 || buf[i] == 0) return PG_TABLE_GENERIC;
        ++i;
      }
      if (f == 6) return PG_TABLE_GENERIC;  // too many fields
      if (i - a > INT32_MAX) return PG_TABLE_GENERIC;
      st[f] = a;
      ln[f] = static_cast<int32_t>(i - a);
      ++f;
    }
    ++i;  // past the '\n' (or the end)
    if (f == 0) continue;  // blank line
    if (f != 6) return PG_TABLE_GENERIC;
    // position: [+]digits, value < 2^63 (Python int() also takes '_' groups and a '-': generic path)
    const char* p = buf + st[3];
    int32_t k = 0, plen = ln[3];
    if (p[0] == '+') k = 1;
    if (k == plen || plen - k > 18) return PG_TABLE_GENERIC;
    int64_t v = 0;
    for (; k < plen; ++k) {
      if (p[k] < '0' || p[k] > '9') return PG_TABLE_GENERIC;
      v = v * 10 + (p[k] - '0');
    }
    if (m >= cap) return PG_ERR_INVALID;
    int64_t* s = tok_start + 4 * m;
    int32_t* l = tok_len + 4 * m;
    const int pick[4] = {0, 1, 4, 5};
    for (int q = 0; q < 4; ++q) {
      s[q] = st[pick[q]];
      l[q] = ln[pick[q]];
    }
    pos[m] = v;
    n_same += ln[4] == ln[5] && std::memcmp(buf + st[4], buf + st[5], static_cast<size_t>(ln[4])) == 0;
    ++m;
  }
  *n = m;
  *same = n_same;
  return PG_OK;
}

// Prefixes of markers [first, first + count): out gets the concatenated text, out_off[count + 1]
// the byte offsets of each marker's prefix. swap != 0 writes allele2 before allele1.
int pg_bim_prefixes(const char* buf, const int64_t* tok_start, const int32_t* tok_len, const int64_t* pos,
                    int64_t first, int64_t count, int swap, char* out, int64_t out_cap, int64_t* out_off) {
  int64_t o = 0;
  out_off[0] = 0;
  for (int64_t r = 0; r < count; ++r) {
    const int64_t* s = tok_start + 4 * (first + r);
    const int32_t* l = tok_len + 4 * (first + r);
    const int64_t need = static_cast<int64_t>(l[0]) + l[1] + l[2] + l[3] + 20 + 5;
    if (o + need > out_cap) {
      pg::set_error("pg_bim_prefixes: output buffer too small at marker %lld", (long long)(first + r));
      return PG_ERR_INVALID;
    }
    const int order[4] = {0, 1, swap ? 3 : 2, swap ? 2 : 3};
    for (int q = 0; q < 4; ++q) {
      std::memcpy(out + o, buf + s[order[q]], static_cast<size_t>(l[order[q]]));
      o += l[order[q]];
      out[o++] = '\t';
      if (q == 1) {  // position after the id
        char digits[24];
        int nd = 0;
        uint64_t v = static_cast<uint64_t>(pos[first + r]);
        do {
          digits[nd++] = static_cast<char>('0' + v % 10);
          v /= 10;
        } while (v);
        while (nd) out[o++] = digits[--nd];
        out[o++] = '\t';
      }
    }
    out_off[r + 1] = o;
  }
  return PG_OK;
}

}  // extern "C"

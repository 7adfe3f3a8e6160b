// Native BGEN v1.2 variant index + parallel zlib inflate (host code).
//
// Replaces the per-variant Python work of the reference reader
// (/root/reference/pkg/src/panelgwas/genotypes/bgen.py): _index_variants (:130-168) and the
// inflate + validation half of _decode_variant (:183-232). The probability -> dosage
// arithmetic stays on the device (decode.cu). The file is memory-mapped; variants of a
// batch are inflated by a pool of host threads straight into the caller's (pinned)
// device-staging rows  [ 2n probabilities (u8 or u16) | n ploidy bytes ].
//
// Errors are reported as (variant, reason, a, b) so the Python layer raises exactly the
// reference's exception class and message; with several failing variants the lowest
// index wins, as in the reference's sequential loop.
//
// Mixed 8/16-bit batches (legal BGEN, decoded per variant by the reference) are widened
// to 16 bits: k8 / 255 == (257 k8) / 65535 exactly, so the device dosages are bit-identical.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <zlib.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "pg_common.cuh"

namespace pg {
namespace {

struct MappedFile {
  int fd = -1;
  const uint8_t* p = nullptr;
  size_t size = 0;
  ~MappedFile() {
    if (p && size) munmap(const_cast<uint8_t*>(p), size);
    if (fd >= 0) close(fd);
  }
  bool open_ro(const char* path) {
    fd = ::open(path, O_RDONLY);
    if (fd < 0) return false;
    struct stat st;
    if (fstat(fd, &st) != 0) return false;
    size = static_cast<size_t>(st.st_size);
    if (size == 0) return true;
    void* m = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (m == MAP_FAILED) {
      p = nullptr;
      size = 0;
      return false;
    }
    p = static_cast<const uint8_t*>(m);
    return true;
  }
};

inline uint16_t rd16(const uint8_t* p) { return static_cast<uint16_t>(p[0] | (p[1] << 8)); }
inline uint32_t rd32(const uint8_t* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
         (static_cast<uint32_t>(p[3]) << 24);
}

enum Reason : int64_t {
  kOk = 0,
  kTooShort = 1,      // compressed block < 4 bytes
  kZlib = 2,          // a = zlib status; message in the error string
  kInflatedSize = 3,  // a = got, b = want
  kSampleCount = 4,   // a = n
  kAlleles = 5,       // a = k
  kPloidyRange = 6,   // a = pmin, b = pmax
  kNonDiploid = 7,
  kPhased = 8,
  kBits = 9,          // a = bits
  kBlockSize = 10,    // a = len, b = expected
  kTruncated = 11,    // block runs past the end of the file
};

// Inflate one zlib stream like Python's zlib.decompress (trailing bytes after the stream end
// are ignored). Output goes to `dst` up to `cap`; *total counts every inflated byte.
int inflate_block(const uint8_t* src, size_t n, uint8_t* dst, size_t cap, size_t* total, std::string* msg) {
  z_stream zs;
  std::memset(&zs, 0, sizeof(zs));
  int rc = inflateInit(&zs);
  if (rc != Z_OK) return rc;
  zs.next_in = const_cast<Bytef*>(src);
  zs.avail_in = static_cast<uInt>(n);
  size_t got = 0;
  uint8_t sink[16384];
  for (;;) {
    uint8_t* out = got < cap ? dst + got : sink;
    const size_t room = got < cap ? cap - got : sizeof(sink);
    zs.next_out = out;
    zs.avail_out = static_cast<uInt>(std::min<size_t>(room, 1u << 30));
    rc = inflate(&zs, Z_NO_FLUSH);
    got += (zs.next_out - out);
    if (rc == Z_STREAM_END) break;
    if (rc == Z_OK) {
      if (zs.avail_in == 0 && zs.avail_out != 0) {
        rc = Z_BUF_ERROR;  // input exhausted before the stream end
        break;
      }
      continue;
    }
    if (rc == Z_BUF_ERROR && zs.avail_out == 0) continue;  // output space ran out: keep counting
    break;
  }
  if (rc != Z_STREAM_END) {
    if (rc == Z_BUF_ERROR || (rc == Z_OK)) {
      *msg = "incomplete or truncated stream";
      rc = Z_BUF_ERROR;
    } else {
      *msg = zs.msg ? zs.msg : "";
    }
    inflateEnd(&zs);
    return rc;
  }
  inflateEnd(&zs);
  *total = got;
  return Z_OK;
}

}  // namespace
}  // namespace pg

extern "C" {

int pg_bgen_index(const char* path, int64_t first_variant, int64_t n_variants, int64_t* block_offset,
                  int64_t* block_size, uint32_t* position, char* text, int64_t text_cap, int64_t* text_off,
                  int64_t* diag) {
  PG_REQUIRE(path && block_offset && block_size && position && text_off && diag, PG_ERR_INVALID,
             "pg_bgen_index: null argument");
  pg::MappedFile f;
  PG_REQUIRE(f.open_ro(path), PG_ERR_FORMAT, "missing file: %s", path);
  const uint8_t* p = f.p;
  const int64_t size = static_cast<int64_t>(f.size);
  int64_t pos = first_variant;
  int64_t t = 0;
  diag[0] = diag[1] = diag[2] = diag[3] = 0;
  // diag[1]: 1 truncated header field (diag[2] = field code), 2 n_alleles != 2 (diag[2] = n),
  //          3 payload past EOF (diag[2] = comp_len), 4 text buffer too small
  // diag[2] field codes for truncation: 0 variant id, 1 rsid, 2 chrom, 3 variant info, 4 allele,
  // 6 genotype block size (the reference's _read_exact "what" strings)
  auto need = [&](int64_t n) { return pos + n <= size; };
  for (int64_t v = 0; v < n_variants; ++v) {
    diag[0] = v;
    int64_t* to = text_off + 5 * v;
    // three u16-prefixed strings: variant id, rsid, chrom
    for (int s = 0; s < 3; ++s) {
      if (!need(2)) return diag[1] = 1, diag[2] = s, PG_ERR_FORMAT;
      const int64_t len = pg::rd16(p + pos);
      pos += 2;
      if (!need(len)) return diag[1] = 1, diag[2] = s, PG_ERR_FORMAT;
      if (t + len > text_cap) return diag[1] = 4, PG_ERR_INVALID;
      to[s] = t;
      std::memcpy(text + t, p + pos, static_cast<size_t>(len));
      t += len;
      pos += len;
    }
    if (!need(6)) return diag[1] = 1, diag[2] = 3, PG_ERR_FORMAT;
    position[v] = pg::rd32(p + pos);
    const int64_t n_alleles = pg::rd16(p + pos + 4);
    pos += 6;
    if (n_alleles != 2) return diag[1] = 2, diag[2] = n_alleles, PG_ERR_FORMAT;
    // two u32-prefixed alleles
    for (int s = 3; s < 5; ++s) {
      if (!need(4)) return diag[1] = 1, diag[2] = 4, PG_ERR_FORMAT;
      const int64_t len = pg::rd32(p + pos);
      pos += 4;
      if (!need(len)) return diag[1] = 1, diag[2] = 4, PG_ERR_FORMAT;
      if (t + len > text_cap) return diag[1] = 4, PG_ERR_INVALID;
      to[s] = t;
      std::memcpy(text + t, p + pos, static_cast<size_t>(len));
      t += len;
      pos += len;
    }
    if (!need(4)) return diag[1] = 1, diag[2] = 6, PG_ERR_FORMAT;
    const int64_t comp = pg::rd32(p + pos);
    pos += 4;
    if (pos + comp > size) return diag[1] = 3, diag[2] = comp, PG_ERR_FORMAT;
    block_offset[v] = pos;
    block_size[v] = comp;
    pos += comp;
  }
  text_off[5 * n_variants] = t;
  diag[0] = pos;  // end of the variant region
  return PG_OK;
}

int pg_bgen_inflate(const char* path, const int64_t* block_offset, const int64_t* block_size, int64_t count,
                    int64_t n_samples, int n_threads, uint8_t* rows, int64_t row_cap, int* out_bits,
                    int64_t* out_row_bytes, int64_t* diag) {
  using namespace pg;
  PG_REQUIRE(path && block_offset && block_size && rows && out_bits && out_row_bytes && diag, PG_ERR_INVALID,
             "pg_bgen_inflate: null argument");
  PG_REQUIRE(count >= 0 && n_samples >= 1, PG_ERR_INVALID, "pg_bgen_inflate: bad sizes");
  MappedFile f;
  PG_REQUIRE(f.open_ro(path), PG_ERR_FORMAT, "missing file: %s", path);
  const int64_t n = n_samples;
  const int64_t want_max = 10 + n + 4 * n;  // 16-bit block
  // rows are laid out for the widest precision seen; first pass records each variant's bits
  std::vector<int> bits(count, 0);
  std::vector<int64_t> reason(count, 0), ra(count, 0), rb(count, 0);
  std::vector<std::string> zmsg(count);
  int nt = n_threads > 0 ? n_threads : static_cast<int>(std::thread::hardware_concurrency());
  nt = std::max(1, std::min<int>(nt, 64));
  if (count < nt) nt = static_cast<int>(std::max<int64_t>(1, count));
  // Each thread inflates into its own scratch block, validates, then copies into the row
  // of the final precision; widening needs every variant's bits first, so the pass keeps
  // 8-bit probabilities in the row's first 2n bytes and widens afterwards if needed.
  const int64_t row8 = 3 * n, row16 = 5 * n;
  PG_REQUIRE(row_cap >= row16, PG_ERR_INVALID, "pg_bgen_inflate: rows need a %lld-byte stride",
             (long long)row16);
  std::atomic<int64_t> next{0};
  auto work = [&]() {
    std::vector<uint8_t> buf(static_cast<size_t>(want_max + 64));
    for (;;) {
      const int64_t v = next.fetch_add(1);
      if (v >= count) break;
      const int64_t off = block_offset[v], sz = block_size[v];
      if (sz < 4) {
        reason[v] = kTooShort;
        continue;
      }
      if (off < 0 || off + sz > static_cast<int64_t>(f.size)) {
        reason[v] = kTruncated;
        continue;
      }
      const uint8_t* src = f.p + off;
      const int64_t want = rd32(src);
      size_t got = 0;
      std::string msg;
      const size_t cap = std::min<size_t>(buf.size(), static_cast<size_t>(std::max<int64_t>(want, 0)) + 64);
      const int zr = inflate_block(src + 4, static_cast<size_t>(sz - 4), buf.data(), cap, &got, &msg);
      if (zr != Z_OK) {
        reason[v] = kZlib;
        ra[v] = zr;
        zmsg[v] = msg;
        continue;
      }
      if (static_cast<int64_t>(got) != want) {
        reason[v] = kInflatedSize;
        ra[v] = static_cast<int64_t>(got);
        rb[v] = want;
        continue;
      }
      const uint8_t* d = buf.data();
      const int64_t len = static_cast<int64_t>(got);
      if (len < 8) {
        reason[v] = kBlockSize;
        ra[v] = len;
        rb[v] = 10 + n;
        continue;
      }
      const int64_t nn = rd32(d), k = rd16(d + 4), pmin = d[6], pmax = d[7];
      if (nn != n) {
        reason[v] = kSampleCount;
        ra[v] = nn;
        continue;
      }
      if (k != 2) {
        reason[v] = kAlleles;
        ra[v] = k;
        continue;
      }
      if (pmin != 2 || pmax != 2) {
        reason[v] = kPloidyRange;
        ra[v] = pmin;
        rb[v] = pmax;
        continue;
      }
      if (len < 8 + n + 2) {
        reason[v] = kBlockSize;
        ra[v] = len;
        rb[v] = 10 + n;
        continue;
      }
      const uint8_t* ploidy = d + 8;
      bool diploid = true;
      for (int64_t i = 0; i < n; ++i) diploid &= (ploidy[i] & 0x3F) == 2;
      if (!diploid) {
        reason[v] = kNonDiploid;
        continue;
      }
      const int phased = d[8 + n], b = d[8 + n + 1];
      if (phased != 0) {
        reason[v] = kPhased;
        continue;
      }
      if (b != 8 && b != 16) {
        reason[v] = kBits;
        ra[v] = b;
        continue;
      }
      const int64_t expected = 10 + n + 2 * n * (b / 8);
      if (len != expected) {
        reason[v] = kBlockSize;
        ra[v] = len;
        rb[v] = expected;
        continue;
      }
      bits[v] = b;
      // stash [probs | ploidy] at the row's 16-bit stride; widened in the second pass
      uint8_t* row = rows + v * row_cap;
      const int64_t pbytes = 2 * n * (b / 8);
      std::memcpy(row, d + 10 + n, static_cast<size_t>(pbytes));
      std::memcpy(row + pbytes, ploidy, static_cast<size_t>(n));
    }
  };
  {
    std::vector<std::thread> th;
    for (int i = 0; i < nt; ++i) th.emplace_back(work);
    for (auto& x : th) x.join();
  }
  for (int64_t v = 0; v < count; ++v) {
    if (reason[v] != kOk) {
      diag[0] = v;
      diag[1] = reason[v];
      diag[2] = ra[v];
      diag[3] = rb[v];
      if (reason[v] == kZlib) pg::set_error("Error %lld while decompressing data: %s", (long long)ra[v], zmsg[v].c_str());
      else pg::set_error("BGEN block validation failed");
      return PG_ERR_FORMAT;
    }
  }
  bool any8 = false, any16 = false;
  for (int64_t v = 0; v < count; ++v) (bits[v] == 8 ? any8 : any16) = true;
  const int final_bits = any16 ? 16 : 8;
  if (any8 && any16) {
    // widen 8-bit variants in place (back to front so sources are read before overwrite)
    std::atomic<int64_t> nxt{0};
    auto widen = [&]() {
      std::vector<uint8_t> ploidy(static_cast<size_t>(n));
      for (;;) {
        const int64_t v = nxt.fetch_add(1);
        if (v >= count) break;
        if (bits[v] != 8) continue;
        uint8_t* row = rows + v * row_cap;
        std::memcpy(ploidy.data(), row + 2 * n, static_cast<size_t>(n));
        for (int64_t i = 2 * n - 1; i >= 0; --i) {
          const uint32_t w = 257u * row[i];
          row[2 * i] = static_cast<uint8_t>(w & 0xFF);
          row[2 * i + 1] = static_cast<uint8_t>(w >> 8);
        }
        std::memcpy(row + 4 * n, ploidy.data(), static_cast<size_t>(n));
      }
    };
    std::vector<std::thread> th;
    for (int i = 0; i < nt; ++i) th.emplace_back(widen);
    for (auto& x : th) x.join();
  }
  // pack rows contiguously at the final width (front to back: destinations never pass sources)
  const int64_t stride = final_bits == 16 ? row16 : row8;
  if (stride != row_cap)
    for (int64_t v = 1; v < count; ++v)
      std::memmove(rows + v * stride, rows + v * row_cap, static_cast<size_t>(stride));
  *out_bits = final_bits;
  *out_row_bytes = stride;
  return PG_OK;
}

}  // extern "C"

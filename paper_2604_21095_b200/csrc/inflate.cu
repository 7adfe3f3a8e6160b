// zlib / DEFLATE (RFC 1950 / 1951) decoder on the GPU, one warp per stream.
//
// The reference inflates every BGEN genotype block on the host with zlib.decompress
// (/root/reference/pkg/src/panelgwas/genotypes/bgen.py:188-196). A batch holds tens of
// thousands of independent streams, so the B200 decodes them in parallel: each warp owns
// one stream, all 32 lanes run the (inherently serial) Huffman decode in lock-step on the
// same bit buffer (table reads are shared-memory broadcasts), lane 0 writes literals and
// the warp copies LZ77 matches 32 bytes per step. Per-warp tables live in shared memory:
// a 2^10-entry first-level table for literal/length codes, 2^8 for distances, 2^7 for
// code-length codes, plus canonical (count, symbol) arrays for the rare longer codes.
// The zlib header and the Adler-32 trailer are checked like zlib does (warp-parallel
// checksum). Any malformed stream is reported per stream (status != 0); the caller
// re-inflates that one block with host zlib to raise zlib's own message.
#include <cstdint>

#include "inflate.cuh"

namespace pg {
namespace {

constexpr int kLitBits = 10;
constexpr int kDistBits = 8;
constexpr int kClenBits = 7;
constexpr int kWarpsPerBlock = 4;

__constant__ uint16_t c_len_base[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                        31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_len_extra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dist_base[30] = {1,   2,   3,   4,   5,   7,    9,    13,   17,   25,   33,   49,   65,    97,    129,
                                         193, 257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t c_dist_extra[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t c_clen_order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

// Canonical Huffman code (RFC 1951 §3.2.2) with a first-level lookup table.
// lut entry: (length << 9) | symbol, 0 = longer than the table (slow path) or invalid.
struct Huff {
  uint16_t* lut;
  int lut_bits;
  uint16_t count[16];
  uint16_t* sym;  // symbols ordered by (length, value)
};

struct WarpSmem {
  uint16_t lit_lut[1 << kLitBits];
  uint16_t dist_lut[1 << kDistBits];
  uint16_t clen_lut[1 << kClenBits];
  uint16_t lit_sym[288];
  uint16_t dist_sym[32];
  uint16_t clen_sym[19];
  uint8_t lens[288 + 32];
  uint16_t codes[288];
};

// Bit input over an absolute bit position: every peek is two aligned 32-bit loads and a
// funnel shift (no refill loop, no branches). The stream's bytes may be followed by other
// data (the next stream, or >= 8 bytes of padding): peeks past the end read those, and
// truncation is detected by comparing the position with the end after each step.
struct Bits {
  const uint32_t* w;  // 4-byte aligned base
  const uint8_t* b8;  // same base, bytes
  uint32_t bp;        // absolute bit position from w
  uint32_t end;       // bit position just past the stream

  __device__ __forceinline__ uint32_t peek32() const {
    const uint32_t i = bp >> 5;
    return __funnelshift_r(__ldg(w + i), __ldg(w + i + 1), bp & 31);
  }
  __device__ __forceinline__ uint32_t get(int n) {  // n <= 16
    const uint32_t v = peek32() & ((1u << n) - 1u);
    bp += n;
    return v;
  }
  __device__ __forceinline__ bool ok() const { return bp <= end; }
};

// Build the decode structures for lens[0..n) (lane 0 computes codes, the warp fills the
// table). zlib's completeness rules (inflate_table): over-subscribed -> error; incomplete
// only for a single code of length 1 (kind 1/2), never for code-length codes (kind 0).
__device__ bool build(const uint8_t* lens, int n, Huff& h, uint16_t* codes, int kind, int lane) {
  for (int i = 0; i < 16; ++i) h.count[i] = 0;
  for (int s = 0; s < n; ++s) ++h.count[lens[s]];
  int left = 1, max_len = 0;
  for (int l = 1; l < 16; ++l) {
    left <<= 1;
    left -= h.count[l];
    if (left < 0) return false;  // over-subscribed
    if (h.count[l]) max_len = l;
  }
  if (left > 0 && (kind == 0 || max_len != 1)) {
    if (!(kind != 0 && max_len == 0)) return false;  // incomplete (an all-zero distance set is allowed)
  }
  // canonical codes + symbol order (lane 0; <= 288 symbols)
  if (lane == 0) {
    uint16_t next[16], offs[16];
    int code = 0, off = 0;
    h.count[0] = 0;
    for (int l = 1; l < 16; ++l) {
      code = (code + h.count[l - 1]) << 1;
      next[l] = static_cast<uint16_t>(code);
      offs[l] = static_cast<uint16_t>(off);
      off += h.count[l];
    }
    for (int s = 0; s < n; ++s) {
      const int l = lens[s];
      if (l) {
        codes[s] = next[l]++;
        h.sym[offs[l]++] = static_cast<uint16_t>(s);
      }
    }
  }
  __syncwarp();
  const int size = 1 << h.lut_bits;
  for (int i = lane; i < size; i += 32) h.lut[i] = 0;
  __syncwarp();
  for (int s = lane; s < n; s += 32) {
    const int l = lens[s];
    if (l == 0 || l > h.lut_bits) continue;
    // DEFLATE codes are read LSB first: index the table by the bit-reversed code
    const uint32_t rev = __brev(static_cast<uint32_t>(codes[s])) >> (32 - l);
    const uint16_t e = static_cast<uint16_t>((l << 9) | s);
    for (uint32_t i = rev; i < static_cast<uint32_t>(size); i += 1u << l) h.lut[i] = e;
  }
  __syncwarp();
  return true;
}

// Decode one symbol; -1 on error.
__device__ __forceinline__ int decode(Bits& br, const Huff& h) {
  const uint32_t bits = br.peek32();
  const uint16_t e = h.lut[bits & ((1u << h.lut_bits) - 1u)];
  if (e) {
    br.bp += e >> 9;
    return e & 511;
  }
  // slow path: canonical decode bit by bit (codes longer than the table, or invalid)
  int code = 0, first = 0, index = 0;
  for (int l = 1; l < 16; ++l) {
    code |= static_cast<int>((bits >> (l - 1)) & 1u);
    const int c = h.count[l];
    if (code - c < first) {
      br.bp += l;
      return h.sym[index + (code - first)];
    }
    index += c;
    first += c;
    first <<= 1;
    code <<= 1;
  }
  return -1;
}

__global__ void __launch_bounds__(32 * kWarpsPerBlock) inflate_kernel(const uint8_t* __restrict__ blob,
                                                                     const int64_t* __restrict__ off,
                                                                     const int64_t* __restrict__ len, int64_t count,
                                                                     int64_t skip, uint8_t* __restrict__ out,
                                                                     int64_t out_stride, int64_t* __restrict__ out_len,
                                                                     int* __restrict__ status) {
  __shared__ WarpSmem sm_all[kWarpsPerBlock];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  WarpSmem& sm = sm_all[wib];
  const int64_t stream = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + wib;
  if (stream >= count) return;

  Bits br;
  {
    const uint8_t* start = blob + off[stream] + skip;
    const uintptr_t base = reinterpret_cast<uintptr_t>(start) & ~uintptr_t(3);
    br.w = reinterpret_cast<const uint32_t*>(base);
    br.b8 = reinterpret_cast<const uint8_t*>(base);
    br.bp = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(start) - base) * 8u;
    const int64_t n_in = len[stream] - skip;
    br.end = n_in < 0 ? 0 : br.bp + static_cast<uint32_t>(n_in) * 8u;
  }
  uint8_t* dst = out + stream * out_stride;
  const int32_t cap = static_cast<int32_t>(out_stride);
  int32_t pos = 0;
  int err = len[stream] - skip < 2 ? 1 : 0;

  Huff lit{sm.lit_lut, kLitBits, {}, sm.lit_sym};
  Huff dist{sm.dist_lut, kDistBits, {}, sm.dist_sym};
  Huff clen{sm.clen_lut, kClenBits, {}, sm.clen_sym};

  // zlib header
  if (!err) {
    const uint32_t cmf = br.get(8), flg = br.get(8);
    if ((cmf & 15) != 8 || (cmf >> 4) > 7 || ((cmf << 8) | flg) % 31 != 0 || (flg & 0x20)) err = 1;
  }
  bool last = false;
  while (!err && !last) {
    last = br.get(1);
    const uint32_t type = br.get(2);
    if (!br.ok()) {
      err = 1;
      break;
    }
    if (type == 0) {
      // stored block: skip to the byte boundary, then LEN, NLEN and raw bytes
      const uint32_t byte_pos = (br.bp + 7) >> 3;
      if (byte_pos * 8 + 32 > br.end) {
        err = 1;
        break;
      }
      const uint32_t n = br.b8[byte_pos] | (br.b8[byte_pos + 1] << 8);
      const uint32_t nn = br.b8[byte_pos + 2] | (br.b8[byte_pos + 3] << 8);
      if ((n ^ 0xFFFFu) != nn || (byte_pos + 4 + n) * 8 > br.end) {
        err = 1;
        break;
      }
      if (pos + static_cast<int32_t>(n) > cap) {
        err = 2;
        break;
      }
      for (uint32_t j = lane; j < n; j += 32) dst[pos + j] = br.b8[byte_pos + 4 + j];
      pos += n;
      br.bp = (byte_pos + 4 + n) * 8;
      __syncwarp();
      continue;
    }
    if (type == 3) {
      err = 1;
      break;
    }
    if (type == 1) {
      for (int s = lane; s < 288; s += 32) sm.lens[s] = s < 144 ? 8 : s < 256 ? 9 : s < 280 ? 7 : 8;
      for (int s = lane; s < 32; s += 32) sm.lens[288 + s] = 5;  // 30, 31 complete the code, never valid
      __syncwarp();
      build(sm.lens, 288, lit, sm.codes, 1, lane);
      build(sm.lens + 288, 32, dist, sm.codes, 2, lane);
    } else {
      const int hlit = br.get(5) + 257, hdist = br.get(5) + 1, hclen = br.get(4) + 4;
      if (!br.ok() || hlit > 286 || hdist > 30) {
        err = 1;
        break;
      }
      uint8_t cl[19];
      for (int i = 0; i < 19; ++i) cl[i] = 0;
      for (int i = 0; i < hclen; ++i) cl[c_clen_order[i]] = static_cast<uint8_t>(br.get(3));
      if (!br.ok()) {
        err = 1;
        break;
      }
      for (int s = lane; s < 19; s += 32) sm.lens[s] = cl[s];
      __syncwarp();
      if (!build(sm.lens, 19, clen, sm.codes, 0, lane)) {
        err = 1;
        break;
      }
      // literal/length + distance code lengths (run-length coded); every lane decodes,
      // lane 0 stores, so the loop stays uniform
      int idx = 0;
      const int total = hlit + hdist;
      uint8_t lens_buf_last = 0;
      while (idx < total) {
        const int sym = decode(br, clen);
        if (sym < 0) {
          err = 1;
          break;
        }
        if (sym < 16) {
          if (lane == 0) sm.lens[idx] = static_cast<uint8_t>(sym);
          lens_buf_last = static_cast<uint8_t>(sym);
          ++idx;
          continue;
        }
        int rep = 0;
        uint8_t val = 0;
        if (sym == 16) {
          if (idx == 0) {
            err = 1;
            break;
          }
          val = lens_buf_last;
          rep = 3 + br.get(2);
        } else if (sym == 17) {
          rep = 3 + br.get(3);
        } else {
          rep = 11 + br.get(7);
        }
        if (!br.ok() || idx + rep > total) {
          err = 1;
          break;
        }
        for (int j = lane; j < rep; j += 32) sm.lens[idx + j] = val;
        idx += rep;
        lens_buf_last = val;
      }
      if (err || !br.ok()) {
        err = 1;
        break;
      }
      __syncwarp();
      if (sm.lens[256] == 0) {  // no end-of-block code
        err = 1;
        break;
      }
      // distance lengths live right after the hlit literal/length lengths
      if (!build(sm.lens, hlit, lit, sm.codes, 1, lane)) {
        err = 1;
        break;
      }
      // distance lengths -> their own slot (ranges may overlap: read all, then write)
      const uint8_t dl = lane < hdist ? sm.lens[hlit + lane] : 0;
      __syncwarp();
      if (lane < hdist) sm.lens[288 + lane] = dl;
      __syncwarp();
      if (!build(sm.lens + 288, hdist, dist, sm.codes, 2, lane)) {
        err = 1;
        break;
      }
    }
    // ---- compressed data
    for (;;) {
      const int sym = decode(br, lit);
      if (sym < 256) {
        if (sym < 0 || br.bp > br.end) {
          err = 1;
          break;
        }
        if (pos >= cap) {
          err = 2;
          break;
        }
        if (lane == 0) dst[pos] = static_cast<uint8_t>(sym);
        ++pos;
        continue;
      }
      if (sym == 256) {
        if (!br.ok()) err = 1;
        break;
      }
      const int li = sym - 257;
      if (li >= 29) {
        err = 1;
        break;
      }
      const int length = c_len_base[li] + static_cast<int>(br.get(c_len_extra[li]));
      const int ds = decode(br, dist);
      if (ds < 0 || ds >= 30) {
        err = 1;
        break;
      }
      const int distance = c_dist_base[ds] + static_cast<int>(br.get(c_dist_extra[ds]));
      if (!br.ok() || distance > pos) {
        err = 1;
        break;
      }
      if (pos + length > cap) {
        err = 2;
        break;
      }
      __syncwarp();  // earlier literals / copies by other lanes are visible
      // overlapping matches repeat the last `distance` bytes: source index j mod distance
      if (distance >= length) {
        for (int j = lane; j < length; j += 32) dst[pos + j] = dst[pos - distance + j];
      } else {
        for (int j = lane; j < length; j += 32) dst[pos + j] = dst[pos - distance + (j % distance)];
      }
      pos += length;
    }
  }
  // Adler-32 trailer (big-endian, byte aligned after the last block)
  if (!err) {
    const uint32_t byte_pos = (br.bp + 7) >> 3;
    if (byte_pos * 8 + 32 > br.end) {
      err = 1;
    } else {
      const uint32_t want = (static_cast<uint32_t>(br.b8[byte_pos]) << 24) | (br.b8[byte_pos + 1] << 16) |
                            (br.b8[byte_pos + 2] << 8) | br.b8[byte_pos + 3];
      __syncwarp();
      unsigned long long s1 = 0, s2 = 0;
      const int64_t chunk = (static_cast<int64_t>(pos) + 31) / 32;
      const int64_t a = lane * chunk, e = min(static_cast<int64_t>(pos), a + chunk);
      for (int64_t i = a; i < e; ++i) {
        const unsigned long long d = dst[i];
        s1 += d;
        s2 += static_cast<unsigned long long>(pos - i) * d;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      const uint32_t A = static_cast<uint32_t>((1 + s1) % 65521ull);
      const uint32_t B = static_cast<uint32_t>((static_cast<unsigned long long>(pos) + s2) % 65521ull);
      if (((B << 16) | A) != want) err = 1;
    }
  }
  if (lane == 0) {
    out_len[stream] = pos;
    status[stream] = err;
  }
}

}  // namespace

int inflate_streams(const uint8_t* d_blob, const int64_t* d_off, const int64_t* d_len, int64_t count, int64_t skip,
                    uint8_t* d_out, int64_t out_stride, int64_t* d_out_len, int* d_status, cudaStream_t s) {
  if (count <= 0) return PG_OK;
  const unsigned blocks = static_cast<unsigned>((count + kWarpsPerBlock - 1) / kWarpsPerBlock);
  inflate_kernel<<<blocks, 32 * kWarpsPerBlock, 0, s>>>(d_blob, d_off, d_len, count, skip, d_out, out_stride,
                                                        d_out_len, d_status);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

}  // namespace pg

extern "C" int pg_debug_inflate(const void* blob, int64_t blob_bytes, const int64_t* off, const int64_t* size,
                                int64_t count, int64_t skip, void* out, int64_t out_stride, int64_t* out_len,
                                int* status) {
  using namespace pg;
  PG_REQUIRE(blob && off && size && out && out_len && status && count >= 1, PG_ERR_INVALID,
             "pg_debug_inflate: bad arguments");
  uint8_t *d_blob = nullptr, *d_out = nullptr;
  int64_t *d_off = nullptr, *d_size = nullptr, *d_len = nullptr;
  int* d_status = nullptr;
  int rc = PG_OK;
  auto fail = [&](cudaError_t e) {
    set_error("pg_debug_inflate: %s", cudaGetErrorString(e));
    rc = PG_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&d_blob, blob_bytes + 16)) != cudaSuccess ||  // decoder peeks up to 8 B past a stream
      (e = cudaMalloc(&d_out, static_cast<size_t>(out_stride) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_off, sizeof(int64_t) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_size, sizeof(int64_t) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_len, sizeof(int64_t) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_status, sizeof(int) * count)) != cudaSuccess) {
    fail(e);
  } else {
    cudaMemcpy(d_blob, blob, blob_bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(d_off, off, sizeof(int64_t) * count, cudaMemcpyHostToDevice);
    cudaMemcpy(d_size, size, sizeof(int64_t) * count, cudaMemcpyHostToDevice);
    rc = inflate_streams(d_blob, d_off, d_size, count, skip, d_out, out_stride, d_len, d_status, nullptr);
    if (rc == PG_OK) {
      if ((e = cudaDeviceSynchronize()) != cudaSuccess) fail(e);
      cudaMemcpy(out, d_out, static_cast<size_t>(out_stride) * count, cudaMemcpyDeviceToHost);
      cudaMemcpy(out_len, d_len, sizeof(int64_t) * count, cudaMemcpyDeviceToHost);
      cudaMemcpy(status, d_status, sizeof(int) * count, cudaMemcpyDeviceToHost);
    }
  }
  cudaFree(d_blob);
  cudaFree(d_out);
  cudaFree(d_off);
  cudaFree(d_size);
  cudaFree(d_len);
  cudaFree(d_status);
  return rc;
}

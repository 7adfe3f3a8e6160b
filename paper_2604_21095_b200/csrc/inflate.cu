// zlib / DEFLATE (RFC 1950 / 1951) decoder on the GPU, one warp per stream.
//
// The reference inflates every BGEN genotype block on the host with zlib.decompress
// (/root/reference/pkg/src/panelgwas/genotypes/bgen.py:188-196). A batch holds thousands
// of independent streams, so the B200 decodes them in parallel: each warp owns one stream
// and all 32 lanes run the (inherently serial) Huffman decode in lock-step on the same
// register bit buffer; table reads are shared-memory broadcasts, lane 0 writes literals
// and the warp copies LZ77 matches up to 32 bytes per step.
//
// Latency is what bounds a warp here (one symbol depends on the previous one), so the hot
// loop avoids global-memory round trips: the bit buffer is refilled 32 bits at a time
// from the next aligned input word (prefetched one refill ahead), and the last 2 KB of
// output are mirrored in a per-warp shared-memory ring that serves match sources (typical
// BGEN distances are short); only farther matches read back from global memory.
//
// Per-warp shared memory: first-level tables (2^10 literal/length, 2^8 distance,
// 2^7 code-length entries), canonical (count, symbol) arrays for longer codes, and the
// ring. The zlib header and the Adler-32 trailer are checked like zlib does. Malformed
// streams are reported per stream (status != 0); the caller re-inflates that one block
// with host zlib to raise zlib's own message.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "inflate.cuh"

namespace pg {
namespace {

constexpr int kLitBits = 10;
constexpr int kDistBits = 8;
constexpr int kClenBits = 7;
#ifndef PG_INFLATE_RING
#define PG_INFLATE_RING 2048
#endif
#ifndef PG_INFLATE_MINB
#define PG_INFLATE_MINB 1
#endif
constexpr int kRing = PG_INFLATE_RING;  // bytes of recent output mirrored in smem
constexpr int kRingSafe = kRing - 258;  // a copy never overwrites its own sources

__constant__ uint16_t c_len_base[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                        31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_len_extra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
// symbols 30 / 31 (and undecodable codes, decoded as 31) get a distance no stream can reach
__constant__ int32_t c_dist_base[32] = {1,     2,     3,     4,     5,     7,     9,      13,     17,    25,   33,
                                        49,    65,    97,    129,   193,   257,   385,    513,    769,   1025, 1537,
                                        2049,  3073,  4097,  6145,  8193,  12289, 16385,  24577,  1 << 30, 1 << 30};
__constant__ uint8_t c_dist_extra[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
__constant__ uint8_t c_clen_order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

// One canonical Huffman code (RFC 1951 §3.2.2): a first-level table of pre-decoded entries
// (0 = code longer than the table, or no such code) + canonical (count, symbol) arrays.
// Entry layouts (Enc):
//   code-length codes  : u16  len | sym << 4
//   literal / length   : u16  len | extra << 4 | value << 7 | is_length << 15  (literal byte;
//                        or length base - 3 with `extra` bits; extra 7 = end of block,
//                        extra 6 = invalid symbol 286 / 287)
//   distance           : u16  len | extra << 4 | symbol << 8 (base from c_dist_base; >= 30 invalid)
// so the hot loop reads a length / distance with no constant-table lookups, and the
// literal table keeps 16-bit entries (occupancy is what this kernel is bound by).
template <int BITS, int NSYM, class T = uint16_t>
struct Table {
  T lut[1 << BITS];
  uint16_t count[16];
  uint16_t sym[NSYM];
};

struct EncClen {
  static constexpr uint32_t kInvalid = 0;
  __device__ static uint32_t enc(int s, int l) { return static_cast<uint32_t>(l) | (static_cast<uint32_t>(s) << 4); }
};
struct EncLit {
  static constexpr uint32_t kLength = 1u << 15;
  static constexpr uint32_t kInvalid = 0;
  __device__ static uint32_t enc(int s, int l) {
    if (s < 256) return static_cast<uint32_t>(l) | (static_cast<uint32_t>(s) << 7);
    if (s == 256) return static_cast<uint32_t>(l) | (7u << 4) | kLength;
    if (s > 285) return static_cast<uint32_t>(l) | (6u << 4) | kLength;
    return static_cast<uint32_t>(l) | (static_cast<uint32_t>(c_len_extra[s - 257]) << 4) |
           (static_cast<uint32_t>(c_len_base[s - 257] - 3) << 7) | kLength;
  }
};
struct EncDist {
  static constexpr uint32_t kInvalid = 31u << 8;  // symbol 31: an unreachable distance
  __device__ static uint32_t enc(int s, int l) {
    const uint32_t extra = s < 30 ? c_dist_extra[s] : 0u;
    return static_cast<uint32_t>(l) | (extra << 4) | (static_cast<uint32_t>(s) << 8);
  }
};

template <int RING = kRing>
struct WarpSmem {
  Table<kLitBits, 288> lit;
  Table<kDistBits, 32> dist;
  Table<kClenBits, 19> clen;
  uint16_t codes[288];
  uint8_t lens[288 + 32];
  uint8_t ring[RING];
};

// Register bit buffer over 4-byte aligned input words. After refill(): cnt >= 33.
struct Bits {
  const uint32_t* w;
  uint32_t wi;     // next word to load
  uint32_t nextw;  // w[wi], loaded one refill ahead
  uint64_t buf;
  int cnt;
  uint32_t end;        // stream end, in bits from w
  uint32_t last_word;  // loads stop here (a malformed stream cannot run past the blob padding)
  __device__ __forceinline__ void refill() {
    if (cnt <= 32) {
      buf |= static_cast<uint64_t>(nextw) << cnt;
      cnt += 32;
      ++wi;
      nextw = wi <= last_word ? __ldg(w + wi) : 0u;
    }
  }
  __device__ __forceinline__ uint32_t get(int n) {  // n <= 32 buffered bits
    const uint32_t v = static_cast<uint32_t>(buf) & ((1u << n) - 1u);  // n < 32 at every call
    buf >>= n;
    cnt -= n;
    return v;
  }
  __device__ __forceinline__ uint32_t consumed() const { return wi * 32u - static_cast<uint32_t>(cnt); }
  __device__ __forceinline__ bool ok() const { return consumed() <= end; }
};

// zlib's completeness rules (inflate_table): over-subscribed -> error; an incomplete code
// only for a single code of length 1 (lit/len, dist); never for code-length codes.
template <int L, class Enc, int BITS, int NSYM, class T>
__device__ bool build(Table<BITS, NSYM, T>& t, const uint8_t* lens, int n, uint16_t* codes, bool code_lengths,
                      int lane, unsigned mask) {
  uint16_t count[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) count[i] = 0;
  for (int s = 0; s < n; ++s) ++count[lens[s]];
  int left = 1, max_len = 0;
#pragma unroll
  for (int l = 1; l < 16; ++l) {
    left = (left << 1) - count[l];
    if (left < 0) return false;
    if (count[l]) max_len = l;
  }
  if (left > 0 && (code_lengths || max_len != 1) && !(!code_lengths && max_len == 0)) return false;
  if (lane == 0) {
    uint16_t next[16], offs[16];
    int code = 0, off = 0;
    count[0] = 0;
    for (int l = 1; l < 16; ++l) {
      code = (code + count[l - 1]) << 1;
      next[l] = static_cast<uint16_t>(code);
      offs[l] = static_cast<uint16_t>(off);
      off += count[l];
      t.count[l] = count[l];
    }
    for (int s = 0; s < n; ++s) {
      const int l = lens[s];
      if (l) {
        codes[s] = next[l]++;
        t.sym[offs[l]++] = static_cast<uint16_t>(s);
      }
    }
  }
  for (int i = lane; i < (1 << BITS); i += L) t.lut[i] = 0;
  __syncwarp(mask);
  for (int s = lane; s < n; s += L) {
    const int l = lens[s];
    if (l == 0 || l > BITS) continue;
    // codes are read LSB first: index the table by the bit-reversed code
    const uint32_t rev = __brev(static_cast<uint32_t>(codes[s])) >> (32 - l);
    const T e = static_cast<T>(Enc::enc(s, l));
    for (uint32_t i = rev; i < (1u << BITS); i += 1u << l) t.lut[i] = e;
  }
  __syncwarp(mask);
  return true;
}

// Canonical decode bit by bit (codes longer than the table, or invalid); -1 = no such code.
template <int BITS, int NSYM, class T>
__device__ __forceinline__ int decode_slow(Bits& br, const Table<BITS, NSYM, T>& t) {
  const uint32_t bits = static_cast<uint32_t>(br.buf);
  int code = 0, first = 0, index = 0;
  for (int l = 1; l < 16; ++l) {
    code |= static_cast<int>((bits >> (l - 1)) & 1u);
    const int c = t.count[l];
    if (code - c < first) {
      br.get(l);
      return t.sym[index + (code - first)];
    }
    index += c;
    first = (first + c) << 1;
    code <<= 1;
  }
  return -1;
}

// One pre-decoded entry (the caller refilled: >= 33 buffered bits); 0 = no valid code.
template <class Enc, int BITS, int NSYM, class T>
__device__ __forceinline__ uint32_t decode(Bits& br, const Table<BITS, NSYM, T>& t) {
  const uint32_t e = t.lut[static_cast<uint32_t>(br.buf) & ((1u << BITS) - 1u)];
  if (e & 15u) {
    br.get(e & 15u);
    return e;
  }
  const int s = decode_slow(br, t);
  return s < 0 ? Enc::kInvalid : Enc::enc(s, 1);  // bits already consumed; only the fields matter
}

// L lanes decode one stream: L = 32 (a warp per stream, the default) or 16 (two streams per
// warp; the two half-warps share an instruction only while their streams take the same branch).
// Blocks hold 4 streams either way (27 KB of static shared memory).
// L lanes per stream: 32 (a warp per stream), 16, 8 or 4 (32 / L streams share a warp; the
// serial Huffman decode is then replicated on L lanes instead of 32, at the price of
// divergence between the warp's streams). Sub-warp groups keep a 1 KB output ring so a
// warp's 8 streams fit the 48 KB of static shared memory.
template <int L>
struct InflateGeom {
  static constexpr int kStreams = L >= 8 ? 4 : 32 / L;  // streams per block
  static constexpr int kRingL = L >= 16 ? kRing : 1024;
  static constexpr int kRingSafeL = kRingL - 258;
};

template <int L>
__global__ void __launch_bounds__(InflateGeom<L>::kStreams * L, PG_INFLATE_MINB) inflate_kernel(const uint8_t* __restrict__ blob,
                                                                     const int64_t* __restrict__ off,
                                                                     const int64_t* __restrict__ len, int64_t count,
                                                                     int64_t skip, uint8_t* __restrict__ out,
                                                                     int64_t out_stride, int64_t* __restrict__ out_len,
                                                                     int* __restrict__ status) {
  constexpr int kStreams = InflateGeom<L>::kStreams;
  constexpr int kRing = InflateGeom<L>::kRingL;  // shadows the file-level 2 KB ring size
  constexpr int kRingSafe = InflateGeom<L>::kRingSafeL;
  __shared__ WarpSmem<kRing> sm_all[kStreams];
  const int lane = threadIdx.x & (L - 1);
  const unsigned mask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (threadIdx.x & 31u & ~static_cast<unsigned>(L - 1)));
  WarpSmem<kRing>& sm = sm_all[threadIdx.x / L];
  const int64_t stream = static_cast<int64_t>(blockIdx.x) * kStreams + threadIdx.x / L;
  if (stream >= count) return;

  const uint8_t* start = blob + off[stream] + skip;
  const int64_t n_in = len[stream] - skip;
  const uintptr_t base = reinterpret_cast<uintptr_t>(start) & ~uintptr_t(3);
  const uint8_t* b8 = reinterpret_cast<const uint8_t*>(base);
  const uint32_t lead = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(start) - base) * 8u;
  Bits br;
  br.w = reinterpret_cast<const uint32_t*>(base);
  br.wi = 0;
  br.nextw = __ldg(br.w);
  br.buf = 0;
  br.cnt = 0;
  br.end = n_in < 0 ? 0 : lead + static_cast<uint32_t>(n_in) * 8u;
  br.last_word = (br.end + 31) / 32 + 1;  // within the 16 B of padding after the last stream
  br.refill();
  br.refill();
  br.get(lead);
  uint8_t* const dst = out + stream * out_stride;
  const int32_t cap = static_cast<int32_t>(out_stride);
  int32_t pos = 0;
  int err = n_in < 2 ? 1 : 0;

  if (!err) {  // zlib header: CM 8, CINFO <= 7, FCHECK, no preset dictionary
    const uint32_t cmf = br.get(8), flg = br.get(8);
    if ((cmf & 15) != 8 || (cmf >> 4) > 7 || ((cmf << 8) | flg) % 31 != 0 || (flg & 0x20)) err = 1;
  }
  bool last = false;
  while (!err && !last) {
    br.refill();
    last = br.get(1);
    const uint32_t type = br.get(2);
    if (!br.ok() || type == 3) {
      err = 1;
      break;
    }
    if (type == 0) {
      // stored block: byte boundary, LEN, NLEN, raw bytes; the bit buffer restarts after it
      const uint32_t byte_pos = (br.consumed() + 7) >> 3;
      if (byte_pos * 8 + 32 > br.end) {
        err = 1;
        break;
      }
      const uint32_t n = b8[byte_pos] | (b8[byte_pos + 1] << 8);
      const uint32_t nn = b8[byte_pos + 2] | (b8[byte_pos + 3] << 8);
      if ((n ^ 0xFFFFu) != nn || (byte_pos + 4 + n) * 8 > br.end) {
        err = 1;
        break;
      }
      if (pos + static_cast<int32_t>(n) > cap) {
        err = 2;
        break;
      }
      for (uint32_t j = lane; j < n; j += L) {
        const uint8_t v = b8[byte_pos + 4 + j];
        dst[pos + j] = v;
        sm.ring[(pos + j) & (kRing - 1)] = v;
      }
      pos += n;
      const uint32_t next_bit = (byte_pos + 4 + n) * 8;
      br.wi = next_bit >> 5;
      br.nextw = br.wi <= br.last_word ? __ldg(br.w + br.wi) : 0u;
      br.buf = 0;
      br.cnt = 0;
      br.refill();
      br.refill();
      br.get(next_bit & 31);
      __syncwarp(mask);
      continue;
    }
    if (type == 1) {
      for (int s = lane; s < 320; s += L) sm.lens[s] = s < 144 ? 8 : s < 256 ? 9 : s < 280 ? 7 : s < 288 ? 8 : 5;
      __syncwarp(mask);
      build<L, EncLit>(sm.lit, sm.lens, 288, sm.codes, false, lane, mask);
      build<L, EncDist>(sm.dist, sm.lens + 288, 32, sm.codes, false, lane, mask);  // 30, 31 complete the code, never valid
    } else {
      const int hlit = br.get(5) + 257, hdist = br.get(5) + 1, hclen = br.get(4) + 4;
      if (hlit > 286 || hdist > 30) {
        err = 1;
        break;
      }
      br.refill();
      uint8_t cl[19];
#pragma unroll
      for (int i = 0; i < 19; ++i) cl[i] = 0;
      for (int i = 0; i < hclen; ++i) {
        if (i == 10) br.refill();
        cl[c_clen_order[i]] = static_cast<uint8_t>(br.get(3));
      }
      for (int i = lane; i < 19; i += L) sm.lens[i] = cl[i];
      __syncwarp(mask);
      if (!build<L, EncClen>(sm.clen, sm.lens, 19, sm.codes, true, lane, mask)) {
        err = 1;
        break;
      }
      // literal/length + distance code lengths (run-length coded); every lane decodes
      int idx = 0;
      const int total = hlit + hdist;
      uint8_t prev = 0;
      while (idx < total) {
        br.refill();
        const uint32_t ce = decode<EncClen>(br, sm.clen);
        if (!ce) {
          err = 1;
          break;
        }
        const int sym = static_cast<int>(ce >> 4);
        if (sym < 16) {
          if (lane == 0) sm.lens[idx] = static_cast<uint8_t>(sym);
          prev = static_cast<uint8_t>(sym);
          ++idx;
          continue;
        }
        int rep;
        uint8_t val = 0;
        if (sym == 16) {
          if (idx == 0) {
            err = 1;
            break;
          }
          val = prev;
          rep = 3 + br.get(2);
        } else if (sym == 17) {
          rep = 3 + br.get(3);
        } else {
          rep = 11 + br.get(7);
        }
        if (idx + rep > total) {
          err = 1;
          break;
        }
        for (int j = lane; j < rep; j += L) sm.lens[idx + j] = val;
        idx += rep;
        prev = val;
      }
      if (err || !br.ok()) {
        err = 1;
        break;
      }
      __syncwarp(mask);
      if (sm.lens[256] == 0 || !build<L, EncLit>(sm.lit, sm.lens, hlit, sm.codes, false, lane, mask)) {
        err = 1;
        break;
      }
      uint8_t dl[32 / L];  // the ranges may overlap: read everything before writing
#pragma unroll
      for (int q = 0; q < 32 / L; ++q) dl[q] = lane + q * L < hdist ? sm.lens[hlit + lane + q * L] : 0;
      __syncwarp(mask);
#pragma unroll
      for (int q = 0; q < 32 / L; ++q)
        if (lane + q * L < hdist) sm.lens[288 + lane + q * L] = dl[q];
      __syncwarp(mask);
      if (!build<L, EncDist>(sm.dist, sm.lens + 288, hdist, sm.codes, false, lane, mask)) {
        err = 1;
        break;
      }
    }
    // ---- compressed data
    for (;;) {
      br.refill();
      const uint32_t e = decode<EncLit>(br, sm.lit);
      if (!(e & EncLit::kLength)) {
        if (!e) {
          err = 1;
          break;
        }
        if (pos >= cap) {
          err = 2;
          break;
        }
        if (lane == 0) {
          const uint8_t b = static_cast<uint8_t>(e >> 7);
          dst[pos] = b;
          sm.ring[pos & (kRing - 1)] = b;
        }
        ++pos;
        continue;
      }
      const uint32_t extra = (e >> 4) & 7u;
      if (extra >= 6) {  // 7: end of block, 6: invalid length symbol
        if (extra == 6 || !br.ok()) err = 1;
        break;
      }
      const int length = 3 + static_cast<int>((e >> 7) & 255u) + static_cast<int>(br.get(extra));
      br.refill();
      const uint32_t de = decode<EncDist>(br, sm.dist);
      // invalid distance symbols (30, 31, no code) carry an unreachable base: one check below
      const int distance = c_dist_base[de >> 8] + static_cast<int>(br.get((de >> 4) & 15u));
      // (reading past the stream end only consumes padding / the next stream's bytes; the
      // end-of-block check below reports truncation)
      if (distance > pos || pos + length > cap) {
        err = distance > pos ? 1 : 2;
        break;
      }
      __syncwarp(mask);  // earlier literals / copies by other lanes are visible
      const bool from_ring = distance <= kRingSafe;
      if (length <= L && distance >= length) {
        // the common short match: one step, every source byte already written
        if (lane < length) {
          const int src = pos - distance + lane;
          const uint8_t v = from_ring ? sm.ring[src & (kRing - 1)] : dst[src];
          dst[pos + lane] = v;
          sm.ring[(pos + lane) & (kRing - 1)] = v;
        }
      } else {
        // a long or overlapping match: lane j copies source offset j mod distance (an overlapping
        // match repeats the last `distance` bytes). The first offset comes from a float
        // reciprocal (exact after one fix-up: j < 258), later ones by adding L mod distance.
        int jj = lane, step = L;
        if (distance < length) {
          const float inv_d = __frcp_rn(static_cast<float>(distance));
          jj = lane - distance * __float2int_rz(static_cast<float>(lane) * inv_d);
          jj += jj < 0 ? distance : 0;
          jj -= jj >= distance ? distance : 0;
          step = L - distance * __float2int_rz(static_cast<float>(L) * inv_d);
          step += step < 0 ? distance : 0;
          step -= step >= distance ? distance : 0;
        }
        for (int j = lane; j < length; j += L) {
          const int src = pos - distance + jj;
          const uint8_t v = from_ring ? sm.ring[src & (kRing - 1)] : dst[src];
          dst[pos + j] = v;
          sm.ring[(pos + j) & (kRing - 1)] = v;
          if (distance < length) {
            jj += step;
            jj -= jj >= distance ? distance : 0;
          } else {
            jj += L;
          }
        }
      }
      pos += length;
      // no barrier here: the next match's __syncwarp orders these writes before its reads
    }
  }
  // Adler-32 trailer (big-endian, byte aligned after the last block)
  if (!err) {
    const uint32_t byte_pos = (br.consumed() + 7) >> 3;
    if (byte_pos * 8 + 32 > br.end) {
      err = 1;
    } else {
      const uint32_t want = (static_cast<uint32_t>(b8[byte_pos]) << 24) | (b8[byte_pos + 1] << 16) |
                            (b8[byte_pos + 2] << 8) | b8[byte_pos + 3];
      __syncwarp(mask);
      // A = 1 + sum d_k, B = pos + sum (pos - k) d_k = pos + pos * S1 - sum k d_k. Lanes read
      // coalesced 4-byte words (byte sums and 0..3-weighted byte sums by DP4A); the unaligned
      // head and the tail are done bytewise.
      unsigned long long s1 = 0, t = 0;  // S1, sum k d_k
      int32_t head = static_cast<int32_t>((4u - (reinterpret_cast<uintptr_t>(dst) & 3u)) & 3u);
      head = min(head, pos);
      const int32_t n_words = (pos - head) >> 2;
      const int32_t tail = head + 4 * n_words;
      for (int32_t k = lane; k < head; k += L) {
        const uint32_t d = dst[k];
        s1 += d;
        t += static_cast<unsigned long long>(k) * d;
      }
      for (int32_t k = tail + lane; k < pos; k += L) {
        const uint32_t d = dst[k];
        s1 += d;
        t += static_cast<unsigned long long>(k) * d;
      }
      const uint32_t* words = reinterpret_cast<const uint32_t*>(dst + head);
      uint32_t s1w = 0;  // <= 69 KB x 255 per lane: fits
      for (int32_t w = lane; w < n_words; w += L) {
        const uint32_t x = words[w];
        const uint32_t sb = __dp4a(x, 0x01010101u, 0u);
        s1w += sb;
        t += static_cast<unsigned long long>(head + 4 * w) * sb + __dp4a(x, 0x03020100u, 0u);
      }
      s1 += s1w;
#pragma unroll
      for (int o = L / 2; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(mask, s1, o);
        t += __shfl_xor_sync(mask, t, o);
      }
      const unsigned long long s2 = static_cast<unsigned long long>(pos) * s1 - t;
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

// ------------------------------------------------------------------------------------------
// Two-phase decoder (A/B: PG_INFLATE_MODE=tokens). The warp-per-stream kernel above runs the serial Huffman decode
// on all 32 lanes in lock-step: ~100 warp instructions per DEFLATE symbol, 32x redundant. Here
//   phase 1 (thread per stream): each thread decodes its own stream's Huffman codes into LZ77
//            tokens (literal runs of 1-3 bytes | (length, distance) matches) and validates the
//            stream completely (header, block types, code tables, distances vs output so far,
//            output capacity) — 32 streams per warp, no redundant lanes;
//   phase 2 (warp per stream): the warp expands 32 tokens at a time — a prefix sum of their
//            lengths places every literal run, which lanes write in parallel, then the
//            matches are copied cooperatively in order — and checks the Adler-32 trailer.
// Tables of phase 1 live in shared memory per thread (first level: 2^10 literal/length,
// 2^8 distance entries, same pre-decoded entry formats as above); the canonical arrays for
// longer codes are thread-local.
//
// Token (u32): literal run: n << 30 | b0 | b1 << 8 | b2 << 16 (n = 1..3);
//              match:       length << 16 | distance (length 3..258, distance 1..32768).
constexpr int kTokLitBits = 10;
constexpr int kTokDistBits = 8;
constexpr int kTokThreads = 32;  // streams per block (one warp)

struct ThreadTables {
  uint16_t lit[1 << kTokLitBits];
  uint16_t dist[1 << kTokDistBits];
};

// Codes longer than the first level: canonical decode by left-justified limits. With
// rev = the next 15 input bits in code order (first bit read = MSB), the code length is the
// smallest L with rev < lim[L] (lim[L] = (first[L] + count[L]) << (15 - L), non-decreasing),
// found by independent compares instead of a bit-serial loop (32 streams share a warp here,
// so a slow path taken by one lane is paid by all).
struct Canon {
  uint16_t lim[16];
  int16_t base[16];  // index of the first length-L code in sym[] minus first[L]
  uint16_t sym[288];
};

// Per-thread canonical table build (zlib completeness rules, as `build` above).
template <class Enc, int BITS>
__device__ bool build1(uint16_t* lut, Canon& cn, const uint8_t* lens, int n, bool code_lengths) {
  uint16_t count[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) count[i] = 0;
  for (int s = 0; s < n; ++s) ++count[lens[s]];
  int left = 1, max_len = 0;
#pragma unroll
  for (int l = 1; l < 16; ++l) {
    left = (left << 1) - count[l];
    if (left < 0) return false;
    if (count[l]) max_len = l;
  }
  if (left > 0 && (code_lengths || max_len != 1) && !(!code_lengths && max_len == 0)) return false;
  uint16_t next[16], offs[16];
  int code = 0, off = 0;
  count[0] = 0;
  for (int l = 1; l < 16; ++l) {
    code = (code + count[l - 1]) << 1;
    next[l] = static_cast<uint16_t>(code);
    offs[l] = static_cast<uint16_t>(off);
    cn.lim[l] = static_cast<uint16_t>((code + count[l]) << (15 - l));
    cn.base[l] = static_cast<int16_t>(off - code);
    off += count[l];
  }
  for (int i = 0; i < (1 << BITS); ++i) lut[i] = 0;
  for (int s = 0; s < n; ++s) {
    const int l = lens[s];
    if (!l) continue;
    const uint32_t c = next[l]++;
    cn.sym[offs[l]++] = static_cast<uint16_t>(s);
    if (l > BITS) continue;
    const uint32_t rev = __brev(c) >> (32 - l);
    const uint16_t e = static_cast<uint16_t>(Enc::enc(s, l));
    for (uint32_t i = rev; i < (1u << BITS); i += 1u << l) lut[i] = e;
  }
  return true;
}

template <int BITS>
__device__ __forceinline__ int decode_canon(Bits& br, const Canon& cn) {
  const uint32_t rev = __brev(static_cast<uint32_t>(br.buf)) >> 17;  // 15 bits, first read = MSB
  int l = BITS + 1;
#pragma unroll
  for (int k = BITS + 1; k < 15; ++k) l += rev >= cn.lim[k] ? 1 : 0;
  if (rev >= cn.lim[l]) return -1;  // past every code (incomplete single-code tables)
  br.get(l);
  return cn.sym[cn.base[l] + static_cast<int>(rev >> (15 - l))];
}

template <class Enc, int BITS>
__device__ __forceinline__ uint32_t decode1(Bits& br, const uint16_t* lut, const Canon& cn) {
  const uint32_t e = lut[static_cast<uint32_t>(br.buf) & ((1u << BITS) - 1u)];
  if (e & 15u) {
    br.get(e & 15u);
    return e;
  }
  const int sym = decode_canon<BITS>(br, cn);
  return sym < 0 ? Enc::kInvalid : Enc::enc(sym, 1);
}

struct TokenSink {  // 4 tokens per 16-byte store, queued in registers
  uint32_t* dst;
  int32_t n = 0, cap;
  uint32_t q0 = 0, q1 = 0, q2 = 0;
  uint32_t lit = 0;
  int nlit = 0;
  __device__ __forceinline__ bool put(uint32_t t) {
    if (n >= cap) return false;
    switch (n & 3) {
      case 0: q0 = t; break;
      case 1: q1 = t; break;
      case 2: q2 = t; break;
      default: *reinterpret_cast<uint4*>(dst + n - 3) = make_uint4(q0, q1, q2, t);
    }
    ++n;
    return true;
  }
  __device__ __forceinline__ bool literal(uint32_t b) {
    lit |= b << (8 * nlit);
    if (++nlit < 3) return true;
    return flush_lit();
  }
  __device__ __forceinline__ bool flush_lit() {
    if (!nlit) return true;
    const bool ok = put((static_cast<uint32_t>(nlit) << 30) | lit);
    lit = 0;
    nlit = 0;
    return ok;
  }
  __device__ __forceinline__ void finish() {
    const int r = n & 3, b0 = n - r;
    if (r > 0) dst[b0] = q0;
    if (r > 1) dst[b0 + 1] = q1;
    if (r > 2) dst[b0 + 2] = q2;
  }
};

__global__ void __launch_bounds__(kTokThreads) inflate_tokens_kernel(
    const uint8_t* __restrict__ blob, const int64_t* __restrict__ off, const int64_t* __restrict__ len, int64_t count,
    int64_t skip, int64_t out_stride, uint32_t* __restrict__ tokens, int64_t tok_stride, int32_t* __restrict__ ntok,
    int64_t* __restrict__ out_len, int* __restrict__ status) {
  extern __shared__ ThreadTables tabs[];  // kTokThreads entries (dynamic: 80 KB)
  const int64_t stream = static_cast<int64_t>(blockIdx.x) * kTokThreads + threadIdx.x;
  if (stream >= count) return;
  ThreadTables& tb = tabs[threadIdx.x];
  Canon clit, cdist;
  uint8_t lens[288 + 32];

  const uint8_t* start = blob + off[stream] + skip;
  const int64_t n_in = len[stream] - skip;
  const uintptr_t base = reinterpret_cast<uintptr_t>(start) & ~uintptr_t(3);
  const uint8_t* b8 = reinterpret_cast<const uint8_t*>(base);
  const uint32_t lead = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(start) - base) * 8u;
  Bits br;
  br.w = reinterpret_cast<const uint32_t*>(base);
  br.wi = 0;
  br.nextw = __ldg(br.w);
  br.buf = 0;
  br.cnt = 0;
  br.end = n_in < 0 ? 0 : lead + static_cast<uint32_t>(n_in) * 8u;
  br.last_word = (br.end + 31) / 32 + 1;
  br.refill();
  br.refill();
  br.get(lead);
  TokenSink sink;
  sink.dst = tokens + stream * tok_stride;
  sink.cap = static_cast<int32_t>(tok_stride);
  const int32_t cap = static_cast<int32_t>(out_stride);
  int32_t pos = 0;
  int err = n_in < 2 ? 1 : 0;
  if (!err) {
    const uint32_t cmf = br.get(8), flg = br.get(8);
    if ((cmf & 15) != 8 || (cmf >> 4) > 7 || ((cmf << 8) | flg) % 31 != 0 || (flg & 0x20)) err = 1;
  }
  bool last = false;
  while (!err && !last) {
    br.refill();
    last = br.get(1);
    const uint32_t type = br.get(2);
    if (!br.ok() || type == 3) {
      err = 1;
      break;
    }
    if (type == 0) {
      const uint32_t byte_pos = (br.consumed() + 7) >> 3;
      if (byte_pos * 8 + 32 > br.end) {
        err = 1;
        break;
      }
      const uint32_t n = b8[byte_pos] | (b8[byte_pos + 1] << 8);
      const uint32_t nn = b8[byte_pos + 2] | (b8[byte_pos + 3] << 8);
      if ((n ^ 0xFFFFu) != nn || (byte_pos + 4 + n) * 8 > br.end) {
        err = 1;
        break;
      }
      if (pos + static_cast<int32_t>(n) > cap) {
        err = 2;
        break;
      }
      for (uint32_t j = 0; j < n; ++j)
        if (!sink.literal(b8[byte_pos + 4 + j])) err = 2;
      pos += n;
      const uint32_t next_bit = (byte_pos + 4 + n) * 8;
      br.wi = next_bit >> 5;
      br.nextw = br.wi <= br.last_word ? __ldg(br.w + br.wi) : 0u;
      br.buf = 0;
      br.cnt = 0;
      br.refill();
      br.refill();
      br.get(next_bit & 31);
      continue;
    }
    if (type == 1) {
      for (int s = 0; s < 320; ++s) lens[s] = s < 144 ? 8 : s < 256 ? 9 : s < 280 ? 7 : s < 288 ? 8 : 5;
      build1<EncLit, kTokLitBits>(tb.lit, clit, lens, 288, false);
      build1<EncDist, kTokDistBits>(tb.dist, cdist, lens + 288, 32, false);
    } else {
      const int hlit = br.get(5) + 257, hdist = br.get(5) + 1, hclen = br.get(4) + 4;
      if (hlit > 286 || hdist > 30) {
        err = 1;
        break;
      }
      br.refill();
      uint8_t cl[19];
#pragma unroll
      for (int i = 0; i < 19; ++i) cl[i] = 0;
      for (int i = 0; i < hclen; ++i) {
        if (i == 10) br.refill();
        cl[c_clen_order[i]] = static_cast<uint8_t>(br.get(3));
      }
      // code-length code: first level in the distance table's storage (2^7 <= 2^8 entries)
      Canon ccl;
      if (!build1<EncClen, kClenBits>(tb.dist, ccl, cl, 19, true)) {
        err = 1;
        break;
      }
      int idx = 0;
      const int total = hlit + hdist;
      uint8_t prev = 0;
      while (idx < total) {
        br.refill();
        const uint32_t ce = decode1<EncClen, kClenBits>(br, tb.dist, ccl);
        if (!ce) {
          err = 1;
          break;
        }
        const int sym = static_cast<int>(ce >> 4);
        if (sym < 16) {
          lens[idx++] = static_cast<uint8_t>(sym);
          prev = static_cast<uint8_t>(sym);
          continue;
        }
        int rep;
        uint8_t val = 0;
        if (sym == 16) {
          if (idx == 0) {
            err = 1;
            break;
          }
          val = prev;
          rep = 3 + br.get(2);
        } else if (sym == 17) {
          rep = 3 + br.get(3);
        } else {
          rep = 11 + br.get(7);
        }
        if (idx + rep > total) {
          err = 1;
          break;
        }
        for (int j = 0; j < rep; ++j) lens[idx + j] = val;
        idx += rep;
        prev = val;
      }
      if (err || !br.ok()) {
        err = 1;
        break;
      }
      if (lens[256] == 0 || !build1<EncLit, kTokLitBits>(tb.lit, clit, lens, hlit, false)) {
        err = 1;
        break;
      }
      uint8_t dl[32];
      for (int q = 0; q < 32; ++q) dl[q] = q < hdist ? lens[hlit + q] : 0;
      if (!build1<EncDist, kTokDistBits>(tb.dist, cdist, dl, hdist, false)) {
        err = 1;
        break;
      }
    }
    for (;;) {
      br.refill();
      const uint32_t e = decode1<EncLit, kTokLitBits>(br, tb.lit, clit);
      if (!(e & EncLit::kLength)) {
        if (!e) {
          err = 1;
          break;
        }
        if (pos >= cap) {
          err = 2;
          break;
        }
        if (!sink.literal((e >> 7) & 255u)) {
          err = 2;
          break;
        }
        ++pos;
        continue;
      }
      const uint32_t extra = (e >> 4) & 7u;
      if (extra >= 6) {
        if (extra == 6 || !br.ok()) err = 1;
        break;
      }
      const int length = 3 + static_cast<int>((e >> 7) & 255u) + static_cast<int>(br.get(extra));
      br.refill();
      const uint32_t de = decode1<EncDist, kTokDistBits>(br, tb.dist, cdist);
      const int distance = c_dist_base[de >> 8] + static_cast<int>(br.get((de >> 4) & 15u));
      if (distance > pos || pos + length > cap) {
        err = distance > pos ? 1 : 2;
        break;
      }
      if (!sink.flush_lit() || !sink.put((static_cast<uint32_t>(length) << 16) | static_cast<uint32_t>(distance))) {
        err = 2;
        break;
      }
      pos += length;
    }
  }
  uint32_t trailer = 0;
  if (!err) {
    const uint32_t byte_pos = (br.consumed() + 7) >> 3;
    if (byte_pos * 8 + 32 > br.end) {
      err = 1;
    } else {
      trailer = (static_cast<uint32_t>(b8[byte_pos]) << 24) | (b8[byte_pos + 1] << 16) | (b8[byte_pos + 2] << 8) |
                b8[byte_pos + 3];
    }
  }
  if (!err && !sink.flush_lit()) err = 2;
  sink.finish();
  ntok[stream] = err ? 0 : sink.n;
  out_len[stream] = pos;
  status[stream] = err;
  // phase 2 checks the Adler-32 against the trailer: keep it after the tokens' count
  reinterpret_cast<uint32_t*>(ntok + count)[stream] = trailer;
}

// Phase 2: warp per stream; expands the tokens, then checks the Adler-32 trailer.
__global__ void __launch_bounds__(128) inflate_expand_kernel(const uint32_t* __restrict__ tokens, int64_t tok_stride,
                                                             const int32_t* __restrict__ ntok, int64_t count,
                                                             uint8_t* __restrict__ out, int64_t out_stride,
                                                             const int64_t* __restrict__ out_len,
                                                             int* __restrict__ status) {
  constexpr int kWarps = 4;
  __shared__ uint8_t ring_all[kWarps][kRing];
  const int lane = threadIdx.x & 31;
  const int64_t stream = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (stream >= count) return;
  if (status[stream] != 0) return;
  uint8_t* ring = ring_all[threadIdx.x >> 5];
  const uint32_t* tk = tokens + stream * tok_stride;
  const int32_t nt = ntok[stream];
  uint8_t* const dst = out + stream * out_stride;
  int32_t pos = 0;
  for (int32_t b = 0; b < nt; b += 32) {
    const bool have = b + lane < nt;
    const uint32_t t = have ? __ldg(tk + b + lane) : 0u;
    const uint32_t nl = t >> 30;
    const bool is_match = have && nl == 0;
    const int32_t tlen = !have ? 0 : (is_match ? static_cast<int32_t>((t >> 16) & 0x3FFu) : static_cast<int32_t>(nl));
    const int32_t distance = is_match ? static_cast<int32_t>(t & 0xFFFFu) : 0;
    int32_t incl = tlen;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int32_t my_pos = pos + incl - tlen;
    const int32_t chunk_end = pos + __shfl_sync(0xffffffffu, incl, 31);
    const int32_t ring_lo = chunk_end - kRing;  // the ring holds positions >= ring_lo (and older ones < pos)
    // round 0: literal runs, in parallel
    if (have && !is_match) {
      for (uint32_t i = 0; i < nl; ++i) {
        const uint8_t v = static_cast<uint8_t>(t >> (8 * i));
        dst[my_pos + i] = v;
        if (my_pos + static_cast<int32_t>(i) >= ring_lo) ring[(my_pos + i) & (kRing - 1)] = v;
      }
    }
    // A match whose source bytes (before its own output) are covered by no match of this chunk
    // depends only on earlier chunks and this chunk's literals: those copy in parallel.
    // Covering tokens are the lanes whose output [start, end) meets [src0, ext_end).
    const uint32_t match_lanes = __ballot_sync(0xffffffffu, is_match);
    const int32_t src0 = my_pos - distance;
    const int32_t ext_end = is_match ? min(src0 + tlen, my_pos) : 0;
    int lo = 0, hi = 0;  // lo = #lanes ending <= src0, hi = #lanes starting < ext_end
#pragma unroll
    for (int st = 16; st; st >>= 1) {
      if (__shfl_sync(0xffffffffu, incl, lo + st - 1) + pos <= src0) lo += st;
      if (__shfl_sync(0xffffffffu, incl - tlen, hi + st - 1) + pos < ext_end) hi += st;
    }
    const uint32_t cover = hi > lo ? ((hi - lo >= 32 ? 0xffffffffu : ((1u << (hi - lo)) - 1u)) << lo) : 0u;
    const bool par = is_match && (cover & match_lanes) == 0;
    // round 1: independent matches, their bytes dealt out over the lanes
    const int32_t plen = par ? tlen : 0;
    int32_t pincl = plen;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t v = __shfl_up_sync(0xffffffffu, pincl, o);
      if (lane >= o) pincl += v;
    }
    const int32_t ptotal = __shfl_sync(0xffffffffu, pincl, 31);
    __syncwarp();  // literal bytes visible
    for (int32_t g0 = 0; g0 < ptotal; g0 += 32) {
      const int32_t g = g0 + lane;
      int j = 0;  // the lane whose match holds byte g: #lanes with pincl <= g
#pragma unroll
      for (int st = 16; st; st >>= 1)
        if (__shfl_sync(0xffffffffu, pincl, j + st - 1) <= g) j += st;
      j = min(j, 31);
      const int32_t jstart = __shfl_sync(0xffffffffu, pincl - plen, j);
      const int32_t jp0 = __shfl_sync(0xffffffffu, my_pos, j);
      const int32_t jd = __shfl_sync(0xffffffffu, distance, j);
      if (g < ptotal) {
        int32_t o = g - jstart;
        const int32_t q = jp0 + o;
        if (o >= jd) o -= jd * (o / jd);  // overlapping copy: repeats the jd bytes before jp0
        const int32_t src = jp0 - jd + o;
        const uint8_t v = jp0 - jd >= ring_lo ? ring[src & (kRing - 1)] : dst[src];
        dst[q] = v;
        if (q >= ring_lo) ring[q & (kRing - 1)] = v;
      }
    }
    // round 2: the remaining matches in order, each copied by the whole warp
    uint32_t mm = __ballot_sync(0xffffffffu, is_match && !par);
    while (mm) {
      const int j = __ffs(mm) - 1;
      mm &= mm - 1;
      const int32_t p0 = __shfl_sync(0xffffffffu, my_pos, j);
      const int length = __shfl_sync(0xffffffffu, tlen, j);
      const int dj = __shfl_sync(0xffffffffu, distance, j);
      __syncwarp();  // earlier bytes of the chunk are visible
      const bool from_ring = p0 - dj >= ring_lo;
      for (int qo = lane; qo < length; qo += 32) {
        const int o = qo < dj ? qo : qo - dj * (qo / dj);
        const int src = p0 - dj + o;
        const uint8_t v = from_ring ? ring[src & (kRing - 1)] : dst[src];
        dst[p0 + qo] = v;
        if (p0 + qo >= ring_lo) ring[(p0 + qo) & (kRing - 1)] = v;
      }
    }
    pos = chunk_end;
    __syncwarp();
  }
  // Adler-32 (as the warp kernel above)
  const uint32_t want = reinterpret_cast<const uint32_t*>(ntok + count)[stream];
  unsigned long long s1 = 0, tt = 0;
  int32_t head = static_cast<int32_t>((4u - (reinterpret_cast<uintptr_t>(dst) & 3u)) & 3u);
  head = min(head, pos);
  const int32_t n_words = (pos - head) >> 2;
  const int32_t tail = head + 4 * n_words;
  for (int32_t k = lane; k < head; k += 32) {
    const uint32_t d = dst[k];
    s1 += d;
    tt += static_cast<unsigned long long>(k) * d;
  }
  for (int32_t k = tail + lane; k < pos; k += 32) {
    const uint32_t d = dst[k];
    s1 += d;
    tt += static_cast<unsigned long long>(k) * d;
  }
  const uint32_t* words = reinterpret_cast<const uint32_t*>(dst + head);
  uint32_t s1w = 0;
  for (int32_t w = lane; w < n_words; w += 32) {
    const uint32_t x = words[w];
    const uint32_t sb = __dp4a(x, 0x01010101u, 0u);
    s1w += sb;
    tt += static_cast<unsigned long long>(head + 4 * w) * sb + __dp4a(x, 0x03020100u, 0u);
  }
  s1 += s1w;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    tt += __shfl_xor_sync(0xffffffffu, tt, o);
  }
  const unsigned long long s2 = static_cast<unsigned long long>(pos) * s1 - tt;
  const uint32_t A = static_cast<uint32_t>((1 + s1) % 65521ull);
  const uint32_t B = static_cast<uint32_t>((static_cast<unsigned long long>(pos) + s2) % 65521ull);
  if (lane == 0 && (pos != out_len[stream] || ((B << 16) | A) != want)) status[stream] = 1;
}

}  // namespace

int64_t inflate_token_stride(int64_t out_stride) { return (out_stride / 2 + 16 + 3) / 4 * 4; }

int inflate_streams(const uint8_t* d_blob, const int64_t* d_off, const int64_t* d_len, int64_t count, int64_t skip,
                    uint8_t* d_out, int64_t out_stride, int64_t* d_out_len, int* d_status, cudaStream_t s,
                    uint32_t* d_tokens, int32_t* d_ntok) {
  if (count <= 0) return PG_OK;
  // Default: the warp-per-stream decoder. PG_INFLATE_MODE=tokens selects the two-phase
  // decoder (measured slower on C5: 15.0 + 4.6 ms vs 8.5 ms per 8,192 BGEN-8 variants; a
  // batch gives phase 1 only ~55 streams = 1.7 warps per SM, so its serial per-thread decode
  // is latency-bound). PG_INFLATE_LANES=16 / 8 / 4: 2 / 4 / 8 streams per warp (C5 end to end
// 10 % slower at 16; 1.80e9 at 8 and 1.36e9 at 4 vs 2.69e9 at 32 lanes: divergence between
// the warp's streams and fewer resident warps outweigh the lower decode replication).
  // Read per call (A/B tests switch it inside one process).
  const char* mode = std::getenv("PG_INFLATE_MODE");
  const char* lanes_env = std::getenv("PG_INFLATE_LANES");
  const int lanes_req = lanes_env ? std::atoi(lanes_env) : 32;
  const int lanes = (lanes_req == 16 || lanes_req == 8 || lanes_req == 4) ? lanes_req : 32;
  if (d_tokens != nullptr && d_ntok != nullptr && mode != nullptr && std::strcmp(mode, "tokens") == 0) {
    const int64_t tok_stride = inflate_token_stride(out_stride);
    constexpr int kSmem = static_cast<int>(sizeof(ThreadTables)) * kTokThreads;
    PG_CUDA_CHECK(cudaFuncSetAttribute(inflate_tokens_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    inflate_tokens_kernel<<<static_cast<unsigned>((count + kTokThreads - 1) / kTokThreads), kTokThreads, kSmem, s>>>(
        d_blob, d_off, d_len, count, skip, out_stride, d_tokens, tok_stride, d_ntok, d_out_len, d_status);
    PG_CUDA_CHECK(cudaGetLastError());
    inflate_expand_kernel<<<static_cast<unsigned>((count + 3) / 4), 128, 0, s>>>(d_tokens, tok_stride, d_ntok, count,
                                                                                  d_out, out_stride, d_out_len,
                                                                                  d_status);
    PG_CUDA_CHECK(cudaGetLastError());
    return PG_OK;
  }
  auto launch = [&](auto lanes_c) {
    constexpr int Lc = decltype(lanes_c)::value;
    constexpr int kS = InflateGeom<Lc>::kStreams;
    const unsigned blocks = static_cast<unsigned>((count + kS - 1) / kS);
    inflate_kernel<Lc><<<blocks, kS * Lc, 0, s>>>(d_blob, d_off, d_len, count, skip, d_out, out_stride, d_out_len,
                                                  d_status);
  };
  switch (lanes) {
    case 4: launch(std::integral_constant<int, 4>{}); break;
    case 8: launch(std::integral_constant<int, 8>{}); break;
    case 16: launch(std::integral_constant<int, 16>{}); break;
    default: launch(std::integral_constant<int, 32>{}); break;
  }
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
  uint32_t* d_tok = nullptr;
  int32_t* d_ntok = nullptr;
  int rc = PG_OK;
  cudaError_t e;
  if ((e = cudaMalloc(&d_blob, blob_bytes + 16)) != cudaSuccess ||  // the decoder reads ahead <= 8 bytes
      (e = cudaMalloc(&d_out, static_cast<size_t>(out_stride) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_off, sizeof(int64_t) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_size, sizeof(int64_t) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_len, sizeof(int64_t) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_status, sizeof(int) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_tok, sizeof(uint32_t) * inflate_token_stride(out_stride) * count)) != cudaSuccess ||
      (e = cudaMalloc(&d_ntok, sizeof(int32_t) * 2 * count)) != cudaSuccess) {
    set_error("pg_debug_inflate: %s", cudaGetErrorString(e));
    rc = PG_ERR_CUDA;
  } else {
    cudaMemcpy(d_blob, blob, blob_bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(d_off, off, sizeof(int64_t) * count, cudaMemcpyHostToDevice);
    cudaMemcpy(d_size, size, sizeof(int64_t) * count, cudaMemcpyHostToDevice);
    rc = inflate_streams(d_blob, d_off, d_size, count, skip, d_out, out_stride, d_len, d_status, nullptr, d_tok,
                         d_ntok);
    if (rc == PG_OK) {
      if ((e = cudaDeviceSynchronize()) != cudaSuccess) {
        set_error("pg_debug_inflate: %s", cudaGetErrorString(e));
        rc = PG_ERR_CUDA;
      }
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
  cudaFree(d_tok);
  cudaFree(d_ntok);
  return rc;
}

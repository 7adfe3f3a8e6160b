// K1: genotype decode on the device.
//
// Replaces the reference's per-batch host decode + standardization:
//   PlinkSource.read_marker_batch / _build_decode_table (plink.py:32-45, 167-185):
//     2-bit codes, low pair first: 00 -> 2, 01 -> missing, 10 -> 1, 11 -> 0
//   BgenSource._decode_variant (bgen.py:238-249):
//     d = p_het + 2 * max(0, 1 - p_hom1 - p_het), missing when ploidy & 0x80
//   DenseSource.read_marker_batch (dense.py:79-97): NaN = missing
//   prepare_genotype_batch (kernel.py:376-421): n_obs, mean, AF, variance,
//     MONOMORPHIC (var <= 1e-12) / ALL_MISSING skip flags.
//
// Every source is mapped to an integer code u per observed sample (decode.cuh);
// the statistics are exact integer sums of u and u^2 over kept samples, so
// missing counts, AF (PLINK / integral dosages) and skip flags are bit-exact
// with the reference. The GEMM operand is the balanced-ternary expansion of u,
// one int8 row per digit (plus a 0/1 row of missing calls when present), and
// its x127 copy (assoc.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "decode.cuh"

namespace pg {

double geno_unit_scale(const GenoBlock& b) {
  switch (b.kind) {
    case PG_GENO_BGEN8: return 1.0 / 255.0;
    case PG_GENO_BGEN16: return 1.0 / 65535.0;
    case PG_GENO_DENSE_F64: return b.dense_real ? 1.0 / 131072.0 : 1.0;
    default: return 1.0;
  }
}

bool geno_wide(const GenoBlock& b) {
  return b.kind == PG_GENO_BGEN8 || b.kind == PG_GENO_BGEN16 || (b.kind == PG_GENO_DENSE_F64 && b.dense_real);
}

int geno_rows_per_marker(const GenoBlock& b, bool any_missing, bool allow_wide) {
  // base-255 digits + missing row: BGEN-8 |u| <= 510 < 127 * (1 + 255) needs two digits,
  // BGEN-16 / real dense |u| <= 131072 < 127 * (1 + 255 + 255^2) three
  if (allow_wide && geno_wide(b)) return b.kind == PG_GENO_BGEN8 ? 3 : 4;
  switch (b.kind) {
    case PG_GENO_BGEN8: return 8;    // 6 ternary digits (|u| <= 255 < 364) + missing row
    case PG_GENO_BGEN16: return 16;  // 11 digits (|u| <= 65535 < 88573) + missing row
    case PG_GENO_DENSE_F64:
      if (b.dense_real) return 16;   // 12 digits (|u| <= 131072 < 265720) + missing row
      return any_missing ? 2 : 1;
    default: return any_missing ? 2 : 1;
  }
}

namespace {

constexpr int kChunk = 16;  // samples per thread step (one packed .bed word)

__device__ __forceinline__ uint32_t keep16(const uint32_t* keep_bits, int64_t ci) {
  return (keep_bits[ci >> 1] >> ((ci & 1) * 16)) & 0xFFFFu;
}

// Decode 16 samples of marker m starting at sample 16*ci. u = 0 for
// missing / excluded / out-of-range samples; bit i of *miss marks a kept missing call.
template <int KIND>
__device__ __forceinline__ void load16(const GenoBlock& b, int64_t m, int64_t ci, int (&u)[kChunk], uint32_t& miss,
                                       uint32_t& obs, double& dsum, bool& nonint) {
  const uint8_t* row = b.data + m * b.pitch;
  const uint32_t keep = keep16(b.keep_bits, ci);
  miss = 0;
  obs = 0;
  if constexpr (KIND == PG_GENO_BED) {
    uint32_t w = 0;
    if (ci * 4 + 4 <= b.pitch) w = *reinterpret_cast<const uint32_t*>(row + ci * 4);
#pragma unroll
    for (int i = 0; i < kChunk; ++i) {
      const uint32_t c = (w >> (2 * i)) & 3u;
      const bool kept = (keep >> i) & 1u;
      const bool is_miss = (c == 1u);
      u[i] = (kept && !is_miss) ? (c == 0u ? 1 : (c == 2u ? 0 : -1)) : 0;
      miss |= (kept && is_miss) ? (1u << i) : 0u;
      obs |= (kept && !is_miss) ? (1u << i) : 0u;
    }
  } else if constexpr (KIND == PG_GENO_BGEN8 || KIND == PG_GENO_BGEN16) {
    constexpr int den = (KIND == PG_GENO_BGEN8) ? 255 : 65535;
    constexpr int bw = (KIND == PG_GENO_BGEN8) ? 1 : 2;
    const uint8_t* ploidy = row + (b.ploidy_off >= 0 ? b.ploidy_off : b.n_src * 2 * bw);
    const uint8_t* probs = row + b.probs_off;
#pragma unroll
    for (int i = 0; i < kChunk; ++i) {
      const int64_t s = ci * kChunk + i;
      u[i] = 0;
      if (!((keep >> i) & 1u)) continue;  // keep bits are zero past n_src
      if (ploidy[s] & 0x80) {
        miss |= 1u << i;
        continue;
      }
      int v0, v1;
      if constexpr (bw == 1) {
        v0 = probs[2 * s];
        v1 = probs[2 * s + 1];
      } else {
        const uint16_t* p16 = reinterpret_cast<const uint16_t*>(probs);
        v0 = p16[2 * s];
        v1 = p16[2 * s + 1];
      }
      const int k = (v0 + v1 > den) ? v1 : 2 * den - 2 * v0 - v1;
      u[i] = k - den;
      obs |= 1u << i;
    }
  } else {  // dense f64
    const double* d = reinterpret_cast<const double*>(row);
#pragma unroll
    for (int i = 0; i < kChunk; ++i) {
      const int64_t s = ci * kChunk + i;
      u[i] = 0;
      if (!((keep >> i) & 1u)) continue;
      const double x = d[s];
      if (isnan(x)) {
        miss |= 1u << i;
        continue;
      }
      obs |= 1u << i;
      dsum += x;
      if (b.dense_real) {
        u[i] = static_cast<int>(rint((x - 1.0) * 131072.0));
      } else {
        nonint |= (x != rint(x));
        u[i] = static_cast<int>(x) - 1;
      }
    }
  }
}

template <int KIND>
__global__ void integral_kernel(GenoBlock b, int* flags) {
  const int64_t m = blockIdx.x;
  const int64_t n_chunks = (b.n_src + kChunk - 1) / kChunk;
  bool nonint = false;
  for (int64_t ci = threadIdx.x; ci < n_chunks; ci += blockDim.x) {
    int u[kChunk];
    uint32_t miss, obs;
    double ds = 0;
    load16<KIND>(b, m, ci, u, miss, obs, ds, nonint);
  }
  if (__syncthreads_or(nonint) && threadIdx.x == 0) atomicOr(flags + 1, 1);
}

// spread 16 keep bits onto the even bit positions of a 32-bit word (one per 2-bit code)
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

// PLINK rows: counts straight from bit planes. Each lane keeps 6 independent 16-byte
// streaming loads in flight (64 samples each) before counting, so a warp has 3 KB of
// the row outstanding. Per 16-sample word: n0 = popc(lo & hi), missing = popc(lo) - n0,
// n2 = 16 - popc(lo | hi) (~10 integer ops). Masks (excluded samples, the padding codes
// of the last vector) are applied only where needed, in a separate path, so the common
// all-kept loop stays branch-free and under the HBM rate.
__device__ __forceinline__ void bed_word(uint32_t w, int& nm, int& n2, int& n0) {
  const uint32_t lo = w & 0x55555555u, hi = (w >> 1) & 0x55555555u;
  const int c0 = __popc(lo & hi);
  n0 += c0;
  nm += __popc(lo) - c0;
  n2 += 16 - __popc(lo | hi);
}

__device__ __forceinline__ void bed_word_masked(uint32_t w, uint32_t kk, int& nm, int& n2, int& n0) {
  // kk: one bit per kept code (even positions)
  const uint32_t lo = w & kk, hi = (w >> 1) & kk;
  const int c0 = __popc(lo & hi);
  n0 += c0;
  nm += __popc(lo) - c0;
  n2 += __popc(kk) - __popc(lo | hi);
}

template <int kU>
__device__ __forceinline__ void bed_counts(const GenoBlock& b, int64_t m, int lane, long long& nmiss, long long& su,
                                           long long& ssu) {
  const uint4* row = reinterpret_cast<const uint4*>(b.data + m * b.pitch);
  const int64_t n_vec = (b.n_src + 63) / 64;                 // 16-byte vectors holding real samples
  const int64_t n_plain = b.all_kept ? b.n_src / 64 : 0;     // vectors needing no mask
  int n2 = 0, n0 = 0, nm = 0;
  // all-kept vectors: two words share each popcount. With M the even-bit mask, the low code
  // bits of word a go to even and those of word b to odd positions of one register,
  //   L = (a & M) | ((b << 1) & ~M),   H = ((a >> 1) & M) | (b & ~M),
  // so popc(L) = #codes with lo set (missing 01 + hom2 11), popc(H) = #codes with hi set
  // (het 10 + 11) and popc(L & H) = #11 codes, for both words: 3 POPC + 2 SHF + 3 LOP per
  // 32 samples instead of 6 POPC + 8 other ops.
  constexpr uint32_t kM = 0x55555555u;
  int sl = 0, sh = 0, slh = 0, valid = 0;
  // kU loads in flight per lane (a 23k-sample row: 359 vectors = 2 rounds of 6 x 32)
  for (int64_t base = lane; base < n_plain; base += kU * 32) {
    uint4 w4[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int64_t vi = base + 32 * j;
      w4[j] = vi < n_plain ? __ldcs(row + vi) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      valid += base + 32 * j < n_plain;  // zero-filled vectors count as hom allele-1 codes: drop them below
      const uint32_t l0 = (w4[j].x & kM) | ((w4[j].y << 1) & ~kM), h0 = ((w4[j].x >> 1) & kM) | (w4[j].y & ~kM);
      const uint32_t l1 = (w4[j].z & kM) | ((w4[j].w << 1) & ~kM), h1 = ((w4[j].z >> 1) & kM) | (w4[j].w & ~kM);
      sl += __popc(l0) + __popc(l1);
      sh += __popc(h0) + __popc(h1);
      slh += __popc(l0 & h0) + __popc(l1 & h1);
    }
  }
  // code classes: 11 -> 0 copies (n0), 01 missing, 10 het, 00 -> 2 copies (n2)
  n0 = slh;
  nm = sl - slh;
  n2 = 64 * valid - sl - sh + slh;
  for (int64_t vi = n_plain + lane; vi < n_vec; vi += 32) {
    const uint4 w4 = __ldcs(row + vi);
    const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) bed_word_masked(ws[q], spread16(keep16(b.keep_bits, vi * 4 + q)), nm, n2, n0);
  }
  nmiss = nm;
  su = n2 - n0;
  ssu = n2 + n0;
}

constexpr int kMarkersPerWarp = 4;

template <int KIND, int kU = 6>
__global__ void stats_kernel(GenoBlock b, MarkerStats st, int64_t m_pad, double unit_scale) {
  // a warp counts kMarkersPerWarp rows one after the other (all lanes), then lane k finalizes
  // marker k: the fp64 / int128 tail of each marker costs one lane-parallel pass, not a warp's
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp) * kMarkersPerWarp;
  long long k_nmiss = 0, k_su = 0, k_ssu = 0;
  double k_dsum = 0.0;
  for (int k = 0; k < kMarkersPerWarp; ++k) {
    const int64_t m = m0 + k;
    if (m >= b.n_markers) break;  // uniform across the warp
    const int64_t n_chunks = (b.n_src + kChunk - 1) / kChunk;
    long long nmiss = 0, su = 0, ssu = 0;
    double dsum = 0.0;
    bool nonint = false;
    if constexpr (KIND == PG_GENO_BED) {
      bed_counts<kU>(b, m, lane, nmiss, su, ssu);
      // per-lane counts fit in 32 bits: reduce them as int (one shuffle each, not two)
      int a = static_cast<int>(nmiss), c = static_cast<int>(su), d = static_cast<int>(ssu);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
        d += __shfl_xor_sync(0xffffffffu, d, o);
      }
      nmiss = a;
      su = c;
      ssu = d;
    } else {
      for (int64_t ci = lane; ci < n_chunks; ci += 32) {
        int u[kChunk];
        uint32_t miss, obs;
        load16<KIND>(b, m, ci, u, miss, obs, dsum, nonint);
        nmiss += __popc(miss);
#pragma unroll
        for (int i = 0; i < kChunk; ++i) {
          su += u[i];
          ssu += static_cast<long long>(u[i]) * u[i];
        }
      }
    }
    if constexpr (KIND != PG_GENO_BED) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        nmiss += __shfl_xor_sync(0xffffffffu, nmiss, o);
        su += __shfl_xor_sync(0xffffffffu, su, o);
        ssu += __shfl_xor_sync(0xffffffffu, ssu, o);
        dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
      }
    }
    if (lane == k) {
      k_nmiss = nmiss;
      k_su = su;
      k_ssu = ssu;
      k_dsum = dsum;
    }
  }
  const int64_t m = m0 + lane;
  if (lane >= kMarkersPerWarp || m >= m_pad) return;
  if (m >= b.n_markers) {  // padding marker: neutral, never a candidate
    st.mu_d[m] = 0.0;
    st.mu_f[m] = 0.f;
    st.invd_d[m] = __longlong_as_double(0x7ff8000000000000ll);
    st.invd_f[m] = __int_as_float(0x7fc00000);
    return;
  }
  const long long nmiss = k_nmiss, su = k_su, ssu = k_ssu;
  const double dsum = k_dsum;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  st.n_miss[m] = nmiss;
  st.s_u[m] = su;
  st.ss_u[m] = ssu;
  if (st.sum_d) st.sum_d[m] = dsum;
  if (nmiss) atomicOr(st.flags, 1);
  const long long n_obs = b.n_kept - nmiss;
  if (n_obs <= 0) {
    st.af[m] = nan;
    st.var[m] = 0.0;
    st.skip[m] = 2;  // ALL_MISSING
    st.mu_d[m] = 0.0;
    st.mu_f[m] = 0.f;
    st.invd_d[m] = nan;
    st.invd_f[m] = __int_as_float(0x7fc00000);
    return;
  }
  const __int128 nv = static_cast<__int128>(n_obs) * ssu - static_cast<__int128>(su) * su;
  const double V = static_cast<double>(nv) / static_cast<double>(n_obs);  // centred SS in u-units
  const double var = V / static_cast<double>(b.n_kept) * unit_scale * unit_scale;
  double mean;
  if constexpr (KIND == PG_GENO_BED) {
    mean = static_cast<double>(su + n_obs) / static_cast<double>(n_obs);  // nansum of {0,1,2} / n_obs
  } else if constexpr (KIND == PG_GENO_BGEN8 || KIND == PG_GENO_BGEN16) {
    constexpr double den = (KIND == PG_GENO_BGEN8) ? 255.0 : 65535.0;
    mean = (static_cast<double>(su) + den * static_cast<double>(n_obs)) / den / static_cast<double>(n_obs);
  } else {
    mean = b.dense_real ? dsum / static_cast<double>(n_obs)
                        : static_cast<double>(su + n_obs) / static_cast<double>(n_obs);
  }
  st.af[m] = mean / 2.0;
  st.var[m] = var;
  const bool mono = (nv == 0) || (var <= 1e-12);
  st.skip[m] = mono ? 1 : 0;
  const double mu = static_cast<double>(su) / static_cast<double>(n_obs);
  st.mu_d[m] = mu;
  st.mu_f[m] = static_cast<float>(mu);
  const double invd = mono ? nan : 1.0 / sqrt(static_cast<double>(b.n_kept) * V);
  st.invd_d[m] = invd;
  st.invd_f[m] = static_cast<float>(invd);
}

__device__ __forceinline__ uint4 pack16(const int (&x)[kChunk], int mul) {
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc |= (static_cast<uint32_t>(x[4 * q + i] * mul) & 0xFFu) << (8 * i);
    w[q] = acc;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// grid.x = marker slot (incl. padding), grid.y * blockDim = 16-sample chunks of k_pad.
// QUART (R = 3 only): the transposed wide GEMM's layout, 10 markers per 32-row group
// (rows 3j..3j+2 of marker j, rows 30-31 zero) so a marker's rows share one TMEM lane quarter.
template <int KIND, int R, bool QUART = false>
__global__ void planes_kernel(GenoBlock b, int8_t* __restrict__ v, int8_t* __restrict__ v127, int64_t k_pad) {
  const int64_t m = blockIdx.x;
  const int64_t ci = static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x;
  if (ci * kChunk >= k_pad) return;
  int u[kChunk];
  uint32_t miss = 0, obs = 0;
  double ds = 0;
  bool ni = false;
  if (m < b.n_markers && ci * kChunk < b.n_src) {
    load16<KIND>(b, m, ci, u, miss, obs, ds, ni);
  } else {
#pragma unroll
    for (int i = 0; i < kChunk; ++i) u[i] = 0;
  }
  const int64_t base = QUART ? (m / 10) * 32 + 3 * (m % 10) : m * R;
  auto put = [&](int64_t row, const int (&x)[kChunk]) {
    uint4* pv = reinterpret_cast<uint4*>(v + row * k_pad + ci * kChunk);
    *pv = pack16(x, 1);
    if constexpr (R != 4 && R != 3) {
      uint4* pw = reinterpret_cast<uint4*>(v127 + row * k_pad + ci * kChunk);
      *pw = pack16(x, 127);
    }
  };
  if constexpr (R == 4 || R == 3) {
    // wide-digit operand: balanced base-255 digits of u (rows 0..R-2), missing mask (row R-1)
    int cur[kChunk], t[kChunk];
#pragma unroll
    for (int i = 0; i < kChunk; ++i) cur[i] = u[i];
#pragma unroll
    for (int j = 0; j < R - 1; ++j) {
#pragma unroll
      for (int i = 0; i < kChunk; ++i) {
        int r = cur[i] % 255;  // in (-255, 255)
        if (r > 127) r -= 255;
        if (r < -127) r += 255;
        t[i] = r;
        cur[i] = (cur[i] - r) / 255;
      }
      put(base + j, t);
    }
#pragma unroll
    for (int i = 0; i < kChunk; ++i) t[i] = (miss >> i) & 1u;
    put(base + R - 1, t);
    if (QUART && m % 10 == 9) {  // the group's two padding rows
#pragma unroll
      for (int i = 0; i < kChunk; ++i) t[i] = 0;
      put(base + 3, t);
      put(base + 4, t);
    }
  } else if constexpr (R == 1) {
    put(base, u);
  } else if constexpr (R == 2) {
    put(base, u);
    int mk[kChunk];
#pragma unroll
    for (int i = 0; i < kChunk; ++i) mk[i] = (miss >> i) & 1u;
    put(base + 1, mk);
  } else {
    // balanced ternary digits of u in rows 0..R-2, missing mask in row R-1
    int cur[kChunk], t[kChunk];
#pragma unroll
    for (int i = 0; i < kChunk; ++i) cur[i] = u[i];
#pragma unroll 1
    for (int j = 0; j < R - 1; ++j) {
#pragma unroll
      for (int i = 0; i < kChunk; ++i) {
        int r = cur[i] % 3;  // in (-3, 3)
        if (r > 1) r -= 3;
        if (r < -1) r += 3;
        t[i] = r;
        cur[i] = (cur[i] - r) / 3;
      }
      put(base + j, t);
    }
#pragma unroll
    for (int i = 0; i < kChunk; ++i) t[i] = (miss >> i) & 1u;
    put(base + R - 1, t);
  }
}

template <int KIND>
__global__ void dosage_kernel(GenoBlock b, int elem_bytes, void* __restrict__ out, int64_t* __restrict__ missing) {
  // one block per marker; NaN for missing; counts over all source samples
  const int64_t m = blockIdx.x;
  const uint8_t* row = b.data + m * b.pitch;
  long long nm = 0;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  for (int64_t s = threadIdx.x; s < b.n_src; s += blockDim.x) {
    double d;
    if constexpr (KIND == PG_GENO_BED) {
      const uint32_t c = (row[s >> 2] >> (2 * (s & 3))) & 3u;
      d = c == 0u ? 2.0 : (c == 1u ? nan : (c == 2u ? 1.0 : 0.0));
    } else {
      constexpr int bw = (KIND == PG_GENO_BGEN8) ? 1 : 2;
      constexpr double den = (KIND == PG_GENO_BGEN8) ? 255.0 : 65535.0;
      const uint8_t* ploidy = row + (b.ploidy_off >= 0 ? b.ploidy_off : b.n_src * 2 * bw);
      const uint8_t* probs = row + b.probs_off;
      double v0, v1;
      if constexpr (bw == 1) {
        v0 = probs[2 * s];
        v1 = probs[2 * s + 1];
      } else {
        const uint16_t* p16 = reinterpret_cast<const uint16_t*>(probs);
        v0 = p16[2 * s];
        v1 = p16[2 * s + 1];
      }
      // same IEEE operation order as bgen.py:242-248
      const double p_hom1 = v0 / den;
      const double p_het = v1 / den;
      double p_hom2 = 1.0 - p_hom1 - p_het;
      if (p_hom2 < 0.0) p_hom2 = 0.0;
      d = p_het + 2.0 * p_hom2;
      if (ploidy[s] & 0x80) d = nan;
    }
    if (isnan(d)) ++nm;
    if (elem_bytes == 4)
      reinterpret_cast<float*>(out)[m * b.n_src + s] = static_cast<float>(d);
    else
      reinterpret_cast<double*>(out)[m * b.n_src + s] = d;
  }
  nm = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(nm));
  __shared__ long long part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = nm;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
    missing[m] = t;
  }
}

// PG_STATS_KU / PG_STATS_WPB (measurement switches): loads in flight per lane and warps per
// block of the PLINK statistics kernel; read once.
inline int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

template <int KIND>
int stats_dispatch(const GenoBlock& b, MarkerStats& st, int64_t m_pad, cudaStream_t s) {
  static const int ku = env_int("PG_STATS_KU", 6), wpb_env = env_int("PG_STATS_WPB", 8);
  const int wpb = (wpb_env == 4 || wpb_env == 16) ? wpb_env : 8;
  const int64_t per_block = static_cast<int64_t>(wpb) * kMarkersPerWarp;
  const unsigned grid = static_cast<unsigned>((m_pad + per_block - 1) / per_block);
  const double scale = geno_unit_scale(b);
  if (KIND == PG_GENO_BED && ku == 12) {
    stats_kernel<KIND, 12><<<grid, wpb * 32, 0, s>>>(b, st, m_pad, scale);
  } else if (KIND == PG_GENO_BED && ku == 4) {
    stats_kernel<KIND, 4><<<grid, wpb * 32, 0, s>>>(b, st, m_pad, scale);
  } else {
    stats_kernel<KIND><<<grid, wpb * 32, 0, s>>>(b, st, m_pad, scale);
  }
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

// Missing-call side path of the fused PLINK GEMM: the mask row (kept missing calls) and
// its x127 copy of marker list[j] go to row j of v / v127; rows past n_list are zero.
__global__ void mask_planes_kernel(GenoBlock b, const int* __restrict__ list, int64_t n_list, int8_t* __restrict__ v,
                                   int8_t* __restrict__ v127, int64_t k_pad) {
  const int64_t j = blockIdx.x;
  const int64_t ci = static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x;
  if (ci * kChunk >= k_pad) return;
  int mk[kChunk];
  uint32_t miss = 0;
  if (j < n_list && ci * kChunk < b.n_src) {
    int u[kChunk];
    uint32_t obs = 0;
    double ds = 0;
    bool ni = false;
    load16<PG_GENO_BED>(b, list[j], ci, u, miss, obs, ds, ni);
  }
#pragma unroll
  for (int i = 0; i < kChunk; ++i) mk[i] = (miss >> i) & 1u;
  *reinterpret_cast<uint4*>(v + j * k_pad + ci * kChunk) = pack16(mk, 1);
  *reinterpret_cast<uint4*>(v127 + j * k_pad + ci * kChunk) = pack16(mk, 127);
}

// flag[m] = marker m is scanned (not skipped) and has a kept missing call
__global__ void miss_flag_kernel(const long long* __restrict__ n_miss, const int8_t* __restrict__ skip, int64_t m,
                                 int* __restrict__ flag) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flag[i] = (n_miss[i] > 0 && skip[i] == 0) ? 1 : 0;
}

// exclusive prefix of the flags -> slot[m] (-1 when unflagged), list[slot] = m, *count
__global__ void miss_slot_kernel(const int* __restrict__ flag, const int* __restrict__ prefix, int64_t m,
                                 int* __restrict__ slot, int* __restrict__ list, int* __restrict__ count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int f = flag[i];
    slot[i] = f ? prefix[i] : -1;
    if (f) list[prefix[i]] = static_cast<int>(i);
    if (i == m - 1) *count = prefix[i] + f;
  }
}

template <int KIND, int R>
int planes_launch(const GenoBlock& b, int8_t* v, int8_t* v127, int64_t c_pad, int64_t k_pad, cudaStream_t s) {
  const int64_t m_slots = c_pad / R;
  const int64_t chunks = k_pad / kChunk;
  const int threads = 128;
  dim3 grid(static_cast<unsigned>(m_slots), static_cast<unsigned>((chunks + threads - 1) / threads));
  planes_kernel<KIND, R><<<grid, threads, 0, s>>>(b, v, v127, k_pad);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

template <int KIND>
int planes_quart_launch(const GenoBlock& b, int8_t* v, int64_t c_pad, int64_t k_pad, cudaStream_t s) {
  const int64_t m_slots = c_pad / 32 * 10;
  const int64_t chunks = k_pad / kChunk;
  const int threads = 128;
  dim3 grid(static_cast<unsigned>(m_slots), static_cast<unsigned>((chunks + threads - 1) / threads));
  planes_kernel<KIND, 3, true><<<grid, threads, 0, s>>>(b, v, nullptr, k_pad);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

template <int KIND>
int planes_dispatch(const GenoBlock& b, int R, int8_t* v, int8_t* v127, int64_t c_pad, int64_t k_pad,
                    cudaStream_t s) {
  switch (R) {
    case 1: return planes_launch<KIND, 1>(b, v, v127, c_pad, k_pad, s);
    case 2: return planes_launch<KIND, 2>(b, v, v127, c_pad, k_pad, s);
    case 3: return planes_launch<KIND, 3>(b, v, v127, c_pad, k_pad, s);
    case 4: return planes_launch<KIND, 4>(b, v, v127, c_pad, k_pad, s);
    case 8: return planes_launch<KIND, 8>(b, v, v127, c_pad, k_pad, s);
    case 16: return planes_launch<KIND, 16>(b, v, v127, c_pad, k_pad, s);
    default: set_error("unsupported rows_per_marker %d", R); return PG_ERR_INVALID;
  }
}

}  // namespace

int missing_flags(const long long* n_miss, const int8_t* skip, int64_t m, int* flag, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((m + 255) / 256, 4096));
  miss_flag_kernel<<<grid, 256, 0, s>>>(n_miss, skip, m, flag);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int missing_slot_map(const int* flag, const int* prefix, int64_t m, int* slot, int* list, int* d_count,
                     cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((m + 255) / 256, 4096));
  miss_slot_kernel<<<grid, 256, 0, s>>>(flag, prefix, m, slot, list, d_count);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int missing_mask_planes(const GenoBlock& b, const int* list, int64_t n_list, int8_t* v, int8_t* v127, int64_t c_pad,
                        int64_t k_pad, cudaStream_t s) {
  PG_REQUIRE(b.kind == PG_GENO_BED && k_pad % 64 == 0 && c_pad >= n_list, PG_ERR_INVALID,
             "missing_mask_planes: bad arguments");
  const int64_t chunks = k_pad / kChunk;
  dim3 grid(static_cast<unsigned>(c_pad), static_cast<unsigned>((chunks + 127) / 128));
  mask_planes_kernel<<<grid, 128, 0, s>>>(b, list, n_list, v, v127, k_pad);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int geno_check_integral(const GenoBlock& b, MarkerStats& st, cudaStream_t s) {
  if (b.kind != PG_GENO_DENSE_F64 || b.n_markers == 0) return PG_OK;
  GenoBlock bb = b;
  bb.dense_real = 0;
  integral_kernel<PG_GENO_DENSE_F64><<<static_cast<unsigned>(b.n_markers), 128, 0, s>>>(bb, st.flags);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int geno_stats(const GenoBlock& b, MarkerStats& st, int64_t m_pad, cudaStream_t s) {
  switch (b.kind) {
    case PG_GENO_BED: return stats_dispatch<PG_GENO_BED>(b, st, m_pad, s);
    case PG_GENO_BGEN8: return stats_dispatch<PG_GENO_BGEN8>(b, st, m_pad, s);
    case PG_GENO_BGEN16: return stats_dispatch<PG_GENO_BGEN16>(b, st, m_pad, s);
    case PG_GENO_DENSE_F64: return stats_dispatch<PG_GENO_DENSE_F64>(b, st, m_pad, s);
    default: set_error("unknown genotype kind %d", b.kind); return PG_ERR_INVALID;
  }
}

int geno_planes(const GenoBlock& b, int R, int8_t* v, int8_t* v127, int64_t c_pad, int64_t k_pad, cudaStream_t s,
                bool quartered) {
  if (quartered) {
    PG_REQUIRE(R == 3 && k_pad % 64 == 0 && c_pad % 32 == 0, PG_ERR_INVALID, "geno_planes: bad quartered layout");
    switch (b.kind) {
      case PG_GENO_BGEN8: return planes_quart_launch<PG_GENO_BGEN8>(b, v, c_pad, k_pad, s);
      case PG_GENO_BGEN16: return planes_quart_launch<PG_GENO_BGEN16>(b, v, c_pad, k_pad, s);
      case PG_GENO_DENSE_F64: return planes_quart_launch<PG_GENO_DENSE_F64>(b, v, c_pad, k_pad, s);
      default: set_error("quartered planes: unsupported kind %d", b.kind); return PG_ERR_INVALID;
    }
  }
  PG_REQUIRE(k_pad % 64 == 0 && c_pad % R == 0, PG_ERR_INVALID, "geno_planes: bad padding");
  switch (b.kind) {
    case PG_GENO_BED: return planes_dispatch<PG_GENO_BED>(b, R, v, v127, c_pad, k_pad, s);
    case PG_GENO_BGEN8: return planes_dispatch<PG_GENO_BGEN8>(b, R, v, v127, c_pad, k_pad, s);
    case PG_GENO_BGEN16: return planes_dispatch<PG_GENO_BGEN16>(b, R, v, v127, c_pad, k_pad, s);
    case PG_GENO_DENSE_F64: return planes_dispatch<PG_GENO_DENSE_F64>(b, R, v, v127, c_pad, k_pad, s);
    default: set_error("unknown genotype kind %d", b.kind); return PG_ERR_INVALID;
  }
}

int geno_dosages(const GenoBlock& b, int elem_bytes, void* out, int64_t* missing, cudaStream_t s) {
  if (b.n_markers == 0) return PG_OK;
  const unsigned grid = static_cast<unsigned>(b.n_markers);
  switch (b.kind) {
    case PG_GENO_BED: dosage_kernel<PG_GENO_BED><<<grid, 256, 0, s>>>(b, elem_bytes, out, missing); break;
    case PG_GENO_BGEN8: dosage_kernel<PG_GENO_BGEN8><<<grid, 256, 0, s>>>(b, elem_bytes, out, missing); break;
    case PG_GENO_BGEN16: dosage_kernel<PG_GENO_BGEN16><<<grid, 256, 0, s>>>(b, elem_bytes, out, missing); break;
    default: set_error("dosage decode: unsupported kind %d", b.kind); return PG_ERR_INVALID;
  }
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

}  // namespace pg

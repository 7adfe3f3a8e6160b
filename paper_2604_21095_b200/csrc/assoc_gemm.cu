// K2 + K3: the association contraction on the 5th-gen tensor cores with the
// r -> premask -> candidate-compaction epilogue fused behind it.
//
// Reference semantics (what this replaces): kernel.correlate
// (/root/reference/pkg/src/panelgwas/kernel.py:428-457) computes
// R = G~ . Y~ / N in float64 over 256-row tiles, then the engine premasks
// |r| >= r_bar and keeps candidates in (marker, phenotype) order
// (engine.py:197-217). Here the contraction runs on raw ternary genotype codes
// against the resident, quantized panel (assoc.cuh), exactly, and the
// centring / scaling of the reference's G~ is applied in the epilogue:
//
//   r[m,p] = s_p * (X[m,p] - mu_m * (Cq_p - Mq[m,p])) / sqrt(N * V_m)
//
// with X = sum_k u q, Mq = sum over missing calls of q (rows_per_marker >= 2),
// mu_m / V_m the mean / centred sum of squares of u over observed kept samples
// (SURVEY.md appendix 3).
//
// Three operand paths for the genotype side (template MODE):
//   kPlanes : TMA loads pre-decoded ternary int8 planes v / 127v (rows_per_marker 1/2/8/16)
//   kFused  : TMA loads the packed 2-bit .bed tile (256 rows x 16 B per stage) and
//             4 decoder warps expand it in shared memory into the swizzled v / 127v
//             operand tiles (PLINK rows without missing calls: rows_per_marker 1).
//   kWide   : dosage sources (BGEN, real-valued dense): one int8 plane of balanced
//             base-255 digits of u (3 digit rows + missing row per marker) against the
//             three limbs into three accumulators (A = qH v, B = q1 v, C = q0 v,
//             X_row = 32385 A + 127 B + C), tile N = 128 rows (3 x 128 TMEM columns):
//             4 rows per marker instead of 8 / 16 ternary rows, 2-4x fewer MMAs.
//
// Structure: persistent, warp-specialised, 1 CTA per SM, 768 threads.
//   warp 0 lane 0 : TMA producer
//   warp 1 lane 0 : tcgen05.mma (kind::i8) issuer; 3 MMAs per 32 samples
//   warp 2        : TMEM allocator (512 columns: accH | accL, 128 lanes x 256)
//   warps 4..7    : decoders (fused path)
//   warps 8..23   : epilogue, 4 lane quarters x 4 column groups
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "assoc.cuh"

#ifndef PG_PACKED_PREFETCH
#define PG_PACKED_PREFETCH 0  // stages ahead of the ring for the packed-row L2 prefetch (0: off)
#endif
#ifndef PG_FUSED2_STAGES
#define PG_FUSED2_STAGES 8
#endif
#ifndef PG_DEC_TEAMS
#define PG_DEC_TEAMS 2
#endif
#include "pg_ptx.cuh"

namespace pg {
namespace {

// Pair tile (cta_group::2): 256 phenotypes x 256 genotype rows; each CTA of the
// pair stages its own 128 phenotypes (A half) and 128 genotype rows (B half).
constexpr int kHalfP = kTileP / 2;
constexpr int kHalfC = kTileC / 2;
constexpr int kQBytes = kHalfP * kTileK;             // 8 KB per panel limb half-tile
constexpr int kVBytes = kHalfC * kTileK;             // 8 KB per genotype plane half-tile
constexpr int kPackedBytes = kHalfC * (kTileK / 4);  // 2 KB packed .bed half-tile
constexpr int kOffV = 3 * kQBytes;
constexpr int kOffV127 = kOffV + kVBytes;
constexpr int kOffPacked = kOffV127 + kVBytes;
// wide-digit mode: 160 genotype rows per pair tile (80 per CTA), three accumulators in
// 3 x 160 = 480 TMEM columns (the widest N that fits 512: operand bytes per MAC are
// 17 % lower than at N = 128, and this mode is L2-bandwidth bound)
constexpr int kTileCW = kTileCWide;
constexpr int kHalfCW = kTileCW / 2;
constexpr int kVBytesW = kHalfCW * kTileK;  // 5 KB
constexpr int kRowsW = 4;                   // digits 255^0, 255^1, 255^2 + missing row
constexpr int kPlanes = 0, kFused = 1, kWide = 2, kWide3 = 3, kWide3T = 4, kFused2 = 5, kWide3Two = 6, kPlanes2 = 7,
              kWide4Two = 8;
// kWide4Two: the 4-row wide digits (BGEN-16, real-valued dense) without the q0 limb: 256-row
// tiles (64 markers) with two accumulators, refine_wide_two<4> completes the candidates.
// kPlanes2: kPlanes without the q0 limb (the missing-call side GEMM of a two-limb scan: its
// Mq' is completed per candidate by refine_two_limb).
// kWide3Two: kWide3 (BGEN-8 digit rows) without the q0 limb: two accumulators, so the tile
// widens to 240 rows (80 markers; kTileCWide3Two); the q0 part is added to the candidates by
// refine_wide_two.
// kFused2: kFused without the q0 limb (two MMAs per 32 samples instead of three) for
// THRESHOLD / TOPK scans; the premask is widened by a rigorous bound on the skipped limb and
// the candidates are completed exactly by refine_two_limb (AssocEpilogue::q0n).
// kWide3T (BGEN-8, transposed): genotype digit rows are the A operand (M = 256 rows per pair
// tile = 80 markers in 32-row groups of 10 x 3 rows, see geno_planes(quartered)), the three
// panel limbs three B tiles of N = 144 phenotypes: operand bytes per MAC are 24 % lower than
// kWide3's (three 128-row limb tiles streamed past a 72-row genotype tile).
constexpr int kTPheno = 144;                 // phenotypes per transposed pair tile (UMMA N)
constexpr int kTHalfPheno = kTPheno / 2;     // 72 per CTA
constexpr int kTLimbBytes = kTHalfPheno * kTileK;  // 4.5 KB per limb half-tile
constexpr int kTMarkers = 80;                // markers per transposed pair tile
// warps: TMA, MMA, TMEM alloc, idle, 4 decoders, 16 epilogue
constexpr int kThreads = 768;
constexpr int kTmemCols = 512;
// Raster (tile_coords): groups of tiles visited by the persistent grid so that one wave
// (74 pair tiles) shares operands in L2. Measured on the C3 slice (tools/sweep_l2.sh,
// tools/dram_sweep.sh): genotype-stationary groups of 74 genotype tiles (one phenotype tile
// per wave) 2.06e10 tests/s and 49 GB DRAM per launch, vs 1.91e10 for 32-tile groups;
// panel-stationary groups of 2 phenotype tiles (the default) 22 GB per launch at equal or
// better throughput; evict_first on the panel costs 15 %.

template <int MODE>
struct Cfg {
  static constexpr bool FUSED = MODE == kFused || MODE == kFused2;
  static constexpr bool TWO =
      MODE == kFused2 || MODE == kWide3Two || MODE == kWide4Two || MODE == kPlanes2;  // q0 limb deferred
  static constexpr bool TRANS = MODE == kWide3T;
  static constexpr bool WIDE = MODE == kWide || MODE == kWide3 || MODE == kWide3Two || MODE == kWide4Two || TRANS;
  static constexpr int kStages =
      (TRANS || MODE == kWide3Two || MODE == kWide4Two) ? 9 : (WIDE ? 7 : (MODE == kFused2 ? PG_FUSED2_STAGES : (TWO ? 6 : 5)));
  // decoder warps: 4 per team (one thread per packed row). Measured on the two-limb C3 scan
  // (old decoder): 8 warps splitting each stage's rows with 12 epilogue warps 2.45e10 tests/s,
  // with 16 epilogue warps 2.54e10, 4 + 16 2.60e10; a separate 12-deep packed-tile ring 2.50e10.
  // Two teams of 4 taking alternate stages (896 threads, 66 registers): equal or slightly better
  static constexpr int kDecWarps = 4;  // per team
  // decoder teams taking alternate stages (each team's fence + arrive overlaps the other's decode)
  static constexpr int kDecTeams = (MODE == kFused2) ? PG_DEC_TEAMS : 1;
  static constexpr int kFirstEpiWarp = 4 + kDecWarps * kDecTeams;
  static constexpr int kEpiWarps = 16;  // 20 for the two-limb tile measured no faster (2.71 vs 2.73e10)
  static constexpr int kColGroups = kEpiWarps / 4;
  static constexpr int kThreadsM = 32 * (kFirstEpiWarp + kEpiWarps);  // 768
  // fused / planes stage layout: panel limbs (2 in the two-limb mode), v, 127 v, packed codes.
  // The fused two-limb GEMM needs no 127 v plane: without q0, the q1 accumulator holds
  // sum q1 * v alone and the epilogue scales it by 127 (halves the decoders' stores and frees
  // 8 KB per stage for a deeper ring).
  static constexpr bool NO127 = FUSED && TWO;
  static constexpr int kOffV = (TWO ? 2 : 3) * kQBytes;
  static constexpr int kOffV127 = kOffV + (NO127 ? 0 : kVBytes);
  static constexpr int kOffPacked = kOffV127 + kVBytes;
  // genotype rows per pair tile; wide modes: rows per marker
  static constexpr int kTileRows =
      TRANS ? kTileC
            : (MODE == kWide3 ? kTileCWide3
                              : (MODE == kWide3Two ? kTileCWide3Two : (MODE == kWide4Two ? kTileC : (WIDE ? kTileCW : kTileC))));
  static constexpr int kHalfRows = kTileRows / 2;
  static constexpr int kWideR = (MODE == kWide3 || MODE == kWide3Two || TRANS) ? kWideRows3 : kRowsW;  // kWide4Two: 4
  static constexpr int kVBytesWide = kHalfRows * kTileK;
  // accumulator width (UMMA N): genotype rows, or phenotypes in the transposed mode
  static constexpr int kAccCols = TRANS ? kTPheno : kTileRows;
  // 1 KB-aligned stages (transposed: genotype A half-tile, then the three limb B half-tiles)
  static constexpr int kStageBytes =
      TRANS ? (kVBytesWide + 3 * kTLimbBytes + 1023) / 1024 * 1024
            : (WIDE ? kOffV + (kVBytesWide + 1023) / 1024 * 1024 : (FUSED ? kOffPacked + 2048 : kOffPacked));
  static constexpr int kPanelBytes = (TWO ? 2 : 3) * kQBytes;
  static constexpr int kTmaBytes =
      TRANS ? kVBytesWide + 3 * kTLimbBytes
            : (FUSED ? kPanelBytes : (WIDE ? kOffV + kVBytesWide : kOffPacked));  // per CTA
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 512 /*barriers*/;
  static_assert(kStageBytes % 1024 == 0 && kOffV % 512 == 0, "stage / operand alignment (SW64 atoms)");
  static_assert(kTileRows % 16 == 0 && kHalfRows % 8 == 0, "UMMA N and swizzle-atom granularity");
  static_assert(kSmemBytes <= 227 * 1024, "shared memory per CTA");
};

// group_c > 0: genotype-stationary groups of group_c genotype tiles x all phenotype tiles
//              (phenotype-major inside a group);
// group_c < 0: panel-stationary groups of -group_c phenotype tiles x all genotype tiles
//              (genotype-major inside a group: a wave streams genotype tiles past a panel
//              slice that stays in L2).
__device__ __forceinline__ void tile_coords(int t, int n_ctile, int n_ptile, int group_c, int& ct, int& pt) {
  if (group_c > 0) {
    const int group = t / (group_c * n_ptile);
    const int first = group * group_c;
    const int gsz = min(group_c, n_ctile - first);
    const int r = t - group * group_c * n_ptile;
    ct = first + r % gsz;
    pt = r / gsz;
  } else {
    const int gp = -group_c;
    const int group = t / (gp * n_ctile);
    const int first = group * gp;
    const int gsz = min(gp, n_ptile - first);
    const int r = t - group * gp * n_ctile;
    pt = first + r % gsz;
    ct = r / gsz;
  }
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 16 packed 2-bit codes (one 32-bit .bed word, low pair first) -> 16 int8 u values
// (u[0..3]) and their x127 copies (u127[0..3]).  Code 00 -> +1 (two copies of
// allele1), 10 -> 0, 11 -> -1, 01 (missing) -> 0.  Each code is moved to its own
// nibble (one PRMT byte spread + 2 shift/mask steps per 8 codes) and used as a PRMT byte
// selector into a 4-entry table held in one register: 16 instructions per 16 samples.
// (x | (x << sh)) & mask as one shift + one LOP3 (left to itself, ptxas splits the mask)
template <int kShift, uint32_t kMask>
__device__ __forceinline__ uint32_t spread_step(uint32_t x) {
  uint32_t r;
  asm("{\n\t.reg .b32 t;\n\tshl.b32 t, %1, %2;\n\tlop3.b32 %0, t, %1, %3, 0xA8;\n\t}"
      : "=r"(r) : "r"(x), "n"(kShift), "n"(kMask));
  return r;
}
__device__ __forceinline__ void codes_to_nibbles(uint32_t w, uint32_t& lo, uint32_t& hi) {
  const uint32_t a = __byte_perm(w, 0u, 0x4140);  // byte 0 -> bits 0-7, byte 1 -> bits 16-23
  const uint32_t b = __byte_perm(w, 0u, 0x4342);  // bytes 2, 3
  lo = spread_step<2, 0x33333333u>(spread_step<4, 0x0F0F0F0Fu>(a));
  hi = spread_step<2, 0x33333333u>(spread_step<4, 0x0F0F0F0Fu>(b));
}
// the table as a register operand (PRMT reads its data from registers; without this the
// compiler re-materialises the immediate before every PRMT)
__device__ __forceinline__ uint32_t reg_const(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
// PRMT without the intrinsic's `& 0x7777` on the selector (the nibbles' bit 3 is already 0)
__device__ __forceinline__ uint32_t prmt_lut(uint32_t lut, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(lut), "r"(sel));
  return r;
}
template <bool kWith127 = true>
__device__ __forceinline__ void decode_word(uint32_t w, uint32_t (&u)[4], uint32_t (&u127)[4],
                                            uint32_t lut_u = 0xFF000001u,      // codes 0..3: +1, 0, 0, -1
                                            uint32_t lut_u127 = 0x8100007Fu) {  // +127, 0, 0, -127
  uint32_t n_lo, n_hi;
  codes_to_nibbles(w, n_lo, n_hi);
  const uint32_t sel[4] = {n_lo, n_lo >> 16, n_hi, n_hi >> 16};  // PRMT reads selector bits 0-15
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    u[i] = prmt_lut(lut_u, sel[i]);
    if constexpr (kWith127) u127[i] = prmt_lut(lut_u127, sel[i]);
  }
}

// 16 packed codes -> 16 int8 missing flags (code 01 -> 1, else 0), as decode_word's layout.
__device__ __forceinline__ void decode_word_missing(uint32_t w, uint32_t (&mk)[4]) {
  constexpr uint32_t kLutMiss = 0x00000100u;  // bytes for codes 0,1,2,3: 0, 1, 0, 0
  uint32_t n_lo, n_hi;
  codes_to_nibbles(w, n_lo, n_hi);
  const uint32_t sel[4] = {n_lo, n_lo >> 16, n_hi, n_hi >> 16};
#pragma unroll
  for (int i = 0; i < 4; ++i) mk[i] = prmt_lut(kLutMiss, sel[i]);
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Running per-phenotype max |r| (min-p sidecar, only when ep.max_abs_r is set): the fp32
// estimate selects, the exact fp64 r decides. r64 is evaluated for every pair whose fp32 |r|
// comes within the premask's error window of the thread's fp32 maximum so far, so the fp64
// maximum over those pairs is the fp64 maximum over all pairs.
struct MaxAbsR {
  float f = 0.f;      // fp32 |r| maximum seen
  double d = 0.0;     // fp64 |r| maximum over the window candidates
};

// shared tail of the epilogues: fp32 premask, fp64 r for candidates / FULL, compaction
// valid = false (transposed tiles: padding rows / phenotypes past the panel): no result, but
// the lane still takes part in the warp's compaction ballot.
__device__ __forceinline__ void epilogue_value(const AssocEpilogue& ep, long long xu, long long xm, int m, int pheno,
                                               float sc_f, double sc_d, float cq_f, long long cq, float rb, int lane,
                                               uint32_t lanemask_lt, MaxAbsR& mx, bool valid = true,
                                               double lo_u = 0.0, double lo_cm = 0.0) {
  const float mu = __ldg(ep.mu_f + m);
  const float iv = ep.raw ? 1.f : __ldg(ep.invd_f + m);  // NaN for skipped / padding markers
  const float xf = static_cast<float>(xu) - mu * (cq_f - static_cast<float>(xm));
  const float r = xf * sc_f * iv;
  const float ar = fabsf(r);
  const bool hit = valid && ar >= rb;
  // same widening as the premask bar (ctx.cu rbar_kernel), doubled
  const bool near_max = valid && ep.max_abs_r != nullptr && ar >= mx.f * (1.f - 2e-5f) - 2e-7f;
  double r64 = 0.0;
  if (hit || (valid && ep.full_r) || near_max) {
    r64 = sc_d * ((static_cast<double>(xu) + lo_u) - __ldg(ep.mu_d + m) * (static_cast<double>(cq - xm) + lo_cm)) *
          (ep.raw ? 1.0 : __ldg(ep.invd_d + m));
  }
  if (near_max) {
    mx.f = fmaxf(mx.f, ar);
    mx.d = fmax(mx.d, fabs(r64));  // NaN (skipped / padding markers) is ignored by fmax
  }
  if (valid && ep.full_r) ep.full_r[static_cast<int64_t>(m) * ep.full_ld + pheno] = r64;
  const uint32_t mask = __ballot_sync(0xffffffffu, hit);
  if (mask) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(ep.cand_count, static_cast<unsigned long long>(__popc(mask)));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (hit) {
      // unsigned 64-bit slot: no wrap, and slots past the capacity are counted but not stored
      const unsigned long long idx = base - ep.cand_base + __popc(mask & lanemask_lt);
      if (idx < static_cast<unsigned long long>(ep.cand_cap)) {
        ep.cand_key[idx] = (static_cast<unsigned long long>(m) << 32) | static_cast<unsigned>(pheno);
        ep.cand_r[idx] = r64;
      }
    }
  }
}

// wide-digit tile: per marker rows (digit0, digit1, digit2, missing); X_row = kWH A + 127 B + C
__device__ __forceinline__ void epilogue_tile_wide(const AssocEpilogue& ep, uint32_t tA, int ct, int pheno, int lane,
                                                   int c_begin, int c_end) {
  constexpr int kMarkersPerTile = kTileCW / kRowsW;
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  const float sc_f = ep.scale_f[pheno];
  const double sc_d = ep.scale_d[pheno];
  const float cq_f = ep.cq_f[pheno];
  const long long cq = ep.cq[pheno];
  const float rb = ep.rbar ? ep.rbar[pheno] : INFINITY;
  MaxAbsR mx;
#pragma unroll 1
  for (int c = c_begin; c < c_end; c += 16) {
    uint32_t a[16], b[16], d[16];
    tmem_ld_32x32b_x16(tA + c, a);
    tmem_ld_32x32b_x16(tA + kTileCW + c, b);
    tmem_ld_32x32b_x16(tA + 2 * kTileCW + c, d);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; j += kRowsW) {
      long long x[kRowsW];
#pragma unroll
      for (int t = 0; t < kRowsW; ++t)
        x[t] = kWH * static_cast<long long>(static_cast<int>(a[j + t])) + 127ll * static_cast<int>(b[j + t]) +
               static_cast<int>(d[j + t]);
      const long long xu = x[0] + 255ll * x[1] + 65025ll * x[2];
      const int m = ct * kMarkersPerTile + (c + j) / kRowsW;
      if (ep.x_accum) {
        long long* xa = ep.x_accum + (static_cast<int64_t>(m) * ep.x_ld + pheno) * 2;
        xa[0] += xu;
        xa[1] += x[3];
        continue;
      }
      epilogue_value(ep, xu, x[3], m, pheno, sc_f, sc_d, cq_f, cq, rb, lane, lanemask_lt, mx);
    }
  }
  if (ep.max_abs_r && !ep.x_accum && pheno < ep.p_valid)
    atomicMax(ep.max_abs_r + pheno, static_cast<unsigned long long>(__double_as_longlong(mx.d)));
}

// BGEN-8 wide tile: per marker rows (digit0, digit1, missing), 12 columns (4 markers) per step
__device__ __forceinline__ void epilogue_tile_wide3(const AssocEpilogue& ep, uint32_t tA, int ct, int pheno, int lane,
                                                    int c_begin, int c_end) {
  constexpr int kR = kWideRows3;
  constexpr int kMarkersPerTile = kTileCWide3 / kR;
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  const float sc_f = ep.scale_f[pheno];
  const double sc_d = ep.scale_d[pheno];
  const float cq_f = ep.cq_f[pheno];
  const long long cq = ep.cq[pheno];
  const float rb = ep.rbar ? ep.rbar[pheno] : INFINITY;
  MaxAbsR mx;
#pragma unroll 1
  for (int c = c_begin; c < c_end; c += 12) {
    uint32_t a[12], b[12], d[12];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      tmem_ld_32x32b_x4(tA + c + 4 * q, a + 4 * q);
      tmem_ld_32x32b_x4(tA + kTileCWide3 + c + 4 * q, b + 4 * q);
      tmem_ld_32x32b_x4(tA + 2 * kTileCWide3 + c + 4 * q, d + 4 * q);
    }
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 12; j += kR) {
      long long x[kR];
#pragma unroll
      for (int t = 0; t < kR; ++t)
        x[t] = kWH * static_cast<long long>(static_cast<int>(a[j + t])) + 127ll * static_cast<int>(b[j + t]) +
               static_cast<int>(d[j + t]);
      const long long xu = x[0] + 255ll * x[1];
      const int m = ct * kMarkersPerTile + (c + j) / kR;
      if (ep.x_accum) {
        long long* xa = ep.x_accum + (static_cast<int64_t>(m) * ep.x_ld + pheno) * 2;
        xa[0] += xu;
        xa[1] += x[2];
        continue;
      }
      epilogue_value(ep, xu, x[2], m, pheno, sc_f, sc_d, cq_f, cq, rb, lane, lanemask_lt, mx);
    }
  }
  if (ep.max_abs_r && !ep.x_accum && pheno < ep.p_valid)
    atomicMax(ep.max_abs_r + pheno, static_cast<unsigned long long>(__double_as_longlong(mx.d)));
}

__device__ __forceinline__ long long shfl64(long long v, int src) {
  const int lo = __shfl_sync(0xffffffffu, static_cast<int>(v & 0xffffffffll), src);
  const int hi = __shfl_sync(0xffffffffu, static_cast<int>(v >> 32), src);
  return (static_cast<long long>(hi) << 32) | static_cast<unsigned int>(lo);
}

// Transposed BGEN-8 tile: TMEM lanes are genotype rows (lane 3j + d = digit d of marker j of
// this quarter; d = 2 the missing row; lanes 30-31 padding), columns phenotypes. Per
// 3-column step, three rotating shuffles hand lane 3j + t the three rows of marker j at
// column c + t, so all 30 lanes evaluate a different (marker, phenotype) pair.
__device__ __forceinline__ void epilogue_tile_wide3t(const AssocEpilogue& ep, uint32_t tA, int ct, int cr, int pt,
                                                     int quarter, int lane, int c_begin, int c_end) {
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  const int s = lane % 3;
  const int grp = lane - s;
  const int m = ct * kTMarkers + cr * (kTMarkers / 2) + quarter * 10 + lane / 3;
  const bool row_ok = lane < 30 && m < ep.m_valid;
  const int m_safe = row_ok ? m : 0;
  MaxAbsR mx;
#pragma unroll 1
  for (int c = c_begin; c < c_end; c += 12) {
    uint32_t a[12], b[12], d[12];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      tmem_ld_32x32b_x4(tA + c + 4 * q, a + 4 * q);
      tmem_ld_32x32b_x4(tA + kTPheno + c + 4 * q, b + 4 * q);
      tmem_ld_32x32b_x4(tA + 2 * kTPheno + c + 4 * q, d + 4 * q);
    }
    tmem_ld_wait();
#pragma unroll
    for (int c3 = 0; c3 < 12; c3 += 3) {
      long long x[3], row[3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
        x[i] = kWH * static_cast<long long>(static_cast<int>(a[c3 + i])) + 127ll * static_cast<int>(b[c3 + i]) +
               static_cast<int>(d[c3 + i]);
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int idx = (s + 3 - r) % 3;  // the column the lane that needs my row receives
        const long long send = idx == 0 ? x[0] : (idx == 1 ? x[1] : x[2]);
        const int from = (s + r) % 3;
        const long long got = shfl64(send, grp + from);
        if (from == 0) row[0] = got;
        else if (from == 1) row[1] = got;
        else row[2] = got;
      }
      const int pheno = pt * kTPheno + c + c3 + s;
      const bool valid = row_ok && pheno < ep.p_valid;
      const int p_safe = valid ? pheno : 0;
      const long long xu = row[0] + 255ll * row[1];
      epilogue_value(ep, xu, row[2], m_safe, p_safe, __ldg(ep.scale_f + p_safe), __ldg(ep.scale_d + p_safe),
                     __ldg(ep.cq_f + p_safe), __ldg(ep.cq + p_safe), ep.rbar ? __ldg(ep.rbar + p_safe) : INFINITY,
                     lane, lanemask_lt, mx, valid);
    }
  }
}

// Two-limb tile (kFused2, THRESHOLD / TOPK): per pair only the premask test
//   |r'| + delta >= bar,  r' = s (X' - mu (Cq - Mq)) / sqrt(N V),  delta = s ||q0_p|| ||u_m|| / sqrt(N V)
// in fp32 (X' = kWH h + l rounded to fp32: ~3 ulp, inside the bar's 1e-5 widening), and the
// warp-aggregated compaction of (key, exact int64 X') for the hits.
__device__ __forceinline__ void epilogue_tile_two(const AssocEpilogue& ep, uint32_t tH, uint32_t tL, int ct, int pheno,
                                                  int lane, int c_begin, int c_end) {
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  const float sc_f = ep.scale_f[pheno];
  const float cq_f = ep.cq_f[pheno];
  const float rb = ep.rbar ? ep.rbar[pheno] : INFINITY;
  const float dp = sc_f * __ldg(ep.q0n + pheno) * 1.0001f;  // delta = dp * (||u_m|| / sqrt(N V))
  const int* slot = ep.side_slot;
#pragma unroll 1
  for (int c = c_begin; c < c_end; c += 16) {
    uint32_t h[16], l[16];
    tmem_ld_32x32b_x16(tH + c, h);
    tmem_ld_32x32b_x16(tL + c, l);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int m = ct * kTileC + c + j;
      const float4 mk = __ldg(ep.mpack + m);  // mu, 1/sqrt(N V) (NaN: skipped / padding), ||u|| / sqrt(N V)
      float xm_f = 0.f;
      long long xm = 0;
      if (slot) {
        const int sl = __ldg(slot + m);
        if (sl >= 0) {
          xm = __ldg(ep.side_x + static_cast<int64_t>(sl) * ep.side_ld + pheno);
          xm_f = static_cast<float>(xm);
        }
      }
      // X' = kWH h + 127 l (the q1 accumulator holds sum q1 v: no 127 v plane in this mode)
      const float xf = fmaf(static_cast<float>(static_cast<int>(h[j])), static_cast<float>(kWH),
                            127.f * static_cast<float>(static_cast<int>(l[j]))) - mk.x * (cq_f - xm_f);
      const bool hit = fabsf(xf * sc_f * mk.y) + dp * mk.z >= rb;
      const uint32_t mask = __ballot_sync(0xffffffffu, hit);
      if (mask) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(ep.cand_count, static_cast<unsigned long long>(__popc(mask)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (hit) {
          const unsigned long long idx = base - ep.cand_base + __popc(mask & lanemask_lt);
          if (idx < static_cast<unsigned long long>(ep.cand_cap)) {
            const long long xu =
                kWH * static_cast<long long>(static_cast<int>(h[j])) + 127ll * static_cast<int>(l[j]);
            ep.cand_key[idx] = (static_cast<unsigned long long>(m) << 32) | static_cast<unsigned>(pheno);
            ep.cand_r[idx] = __longlong_as_double(xu);
          }
        }
      }
    }
  }
}

// Two-limb wide tile (kWide3Two: rows digit0, digit1, missing; kWide4Two: digit0..2, missing)
// of X'_row = kWH A + 127 B; the premask as epilogue_tile_two with the bound over u and the
// missing row (AssocEpilogue::mpack); a hit stores X'_u (cand_r bits) and X'_m (cand_xm).
template <int kR>
__device__ __forceinline__ void epilogue_tile_wide_two(const AssocEpilogue& ep, uint32_t tA, int ct, int pheno,
                                                       int lane, int c_begin, int c_end) {
  constexpr int kTileRowsW = kR == 3 ? kTileCWide3Two : kTileC;
  constexpr int kUnitW = kR == 3 ? 12 : 16;
  constexpr int kMarkersPerTile = kTileRowsW / kR;
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  const float sc_f = ep.scale_f[pheno];
  const float cq_f = ep.cq_f[pheno];
  const float rb = ep.rbar ? ep.rbar[pheno] : INFINITY;
  const float dp = sc_f * __ldg(ep.q0n + pheno) * 1.0001f;
#pragma unroll 1
  for (int c = c_begin; c < c_end; c += kUnitW) {
    uint32_t a[kUnitW], b[kUnitW];
#pragma unroll
    for (int q = 0; q < kUnitW / 4; ++q) {
      tmem_ld_32x32b_x4(tA + c + 4 * q, a + 4 * q);
      tmem_ld_32x32b_x4(tA + kTileRowsW + c + 4 * q, b + 4 * q);
    }
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < kUnitW; j += kR) {
      long long x[kR];
#pragma unroll
      for (int t = 0; t < kR; ++t)
        x[t] = kWH * static_cast<long long>(static_cast<int>(a[j + t])) + 127ll * static_cast<int>(b[j + t]);
      long long xu = x[0] + 255ll * x[1];
      if constexpr (kR == 4) xu += 65025ll * x[2];
      const int m = ct * kMarkersPerTile + (c + j) / kR;
      const float4 mk = __ldg(ep.mpack + m);
      const float xf = static_cast<float>(xu) - mk.x * (cq_f - static_cast<float>(x[kR - 1]));
      const bool hit = fabsf(xf * sc_f * mk.y) + dp * mk.z >= rb;
      const uint32_t mask = __ballot_sync(0xffffffffu, hit);
      if (mask) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(ep.cand_count, static_cast<unsigned long long>(__popc(mask)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (hit) {
          const unsigned long long idx = base - ep.cand_base + __popc(mask & lanemask_lt);
          if (idx < static_cast<unsigned long long>(ep.cand_cap)) {
            ep.cand_key[idx] = (static_cast<unsigned long long>(m) << 32) | static_cast<unsigned>(pheno);
            ep.cand_r[idx] = __longlong_as_double(xu);
            ep.cand_xm[idx] = x[kR - 1];
          }
        }
      }
    }
  }
}

template <int R>
__device__ __forceinline__ void epilogue_tile(const AssocEpilogue& ep, uint32_t tH, uint32_t tL, int ct, int pheno,
                                              int lane, int c_begin, int c_end) {
  constexpr int kMarkersPerTile = kTileC / R;
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  const float sc_f = ep.scale_f[pheno];
  const double sc_d = ep.scale_d[pheno];
  const float cq_f = ep.cq_f[pheno];
  const long long cq = ep.cq[pheno];
  const float rb = ep.rbar ? ep.rbar[pheno] : INFINITY;
  MaxAbsR mx;
#pragma unroll 1
  for (int c = c_begin; c < c_end; c += 16) {
    uint32_t h[16], l[16];
    tmem_ld_32x32b_x16(tH + c, h);
    tmem_ld_32x32b_x16(tL + c, l);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; j += R) {
      // exact per-row products, then recombine the rows of this marker
      long long xu = 0, xm = 0;
      const int m = ct * kMarkersPerTile + (c + j) / R;
      if constexpr (R == 1) {
        xu = kWH * static_cast<long long>(static_cast<int>(h[j])) + static_cast<int>(l[j]);
        if (ep.side_out) {  // side GEMM over mask rows: keep Mq of row m
          ep.side_out[static_cast<int64_t>(m) * ep.side_ld + pheno] = xu;
          continue;
        }
        if (ep.side_slot) {  // fused GEMM: Mq of the markers with missing calls
          const int sl = __ldg(ep.side_slot + m);
          if (sl >= 0) xm = __ldg(ep.side_x + static_cast<int64_t>(sl) * ep.side_ld + pheno);
        }
      } else {
        long long w = 1;
#pragma unroll
        for (int d = 0; d < (R == 2 ? 1 : R - 1); ++d) {
          xu += w * (kWH * static_cast<long long>(static_cast<int>(h[j + d])) + static_cast<int>(l[j + d]));
          w *= 3;
        }
        xm = kWH * static_cast<long long>(static_cast<int>(h[j + R - 1])) + static_cast<int>(l[j + R - 1]);
      }
      if (ep.x_accum) {  // K-sliced run: exact int64 partials, statistics after the last slice
        long long* x = ep.x_accum + (static_cast<int64_t>(m) * ep.x_ld + pheno) * 2;
        x[0] += xu;
        x[1] += xm;
        continue;
      }
      epilogue_value(ep, xu, xm, m, pheno, sc_f, sc_d, cq_f, cq, rb, lane, lanemask_lt, mx);
    }
  }
  if (ep.max_abs_r && !ep.x_accum && pheno < ep.p_valid)
    atomicMax(ep.max_abs_r + pheno, static_cast<unsigned long long>(__double_as_longlong(mx.d)));
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg<MODE>::kThreadsM, 1)
    assoc_i8_kernel(const __grid_constant__ CUtensorMap tm_qh, const __grid_constant__ CUtensorMap tm_q1,
                    const __grid_constant__ CUtensorMap tm_q0, const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_v127, int n_ctile, int n_ptile, int kb_begin, int n_kb,
                    int group_c, uint32_t l2_codes, AssocEpilogue ep) {
  using C = Cfg<MODE>;
  constexpr bool FUSED = C::FUSED;
  constexpr bool WIDE = C::WIDE;
  constexpr int S = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::kStageBytes);  // leader: TMA of both CTAs
  uint64_t* empty = full + S;                                                // each CTA: MMA done with stage
  uint64_t* dec = empty + S;                                                 // leader: decoders of both CTAs
  uint64_t* pk = dec + S;                                                    // each CTA: its packed tile landed
  uint64_t* tfull = pk + S;                                                  // each CTA: accumulators ready
  uint64_t* tempty = tfull + 1;                                              // leader: both CTAs drained TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  const bool leader = cr == 0;
  const int cid = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  const int n_tiles = n_ctile * n_ptile;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qh);
    tma_prefetch_desc(&tm_q1);
    tma_prefetch_desc(&tm_q0);
    tma_prefetch_desc(&tm_v);
    if (MODE == kPlanes) tma_prefetch_desc(&tm_v127);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
      mbar_init(&dec[s], 2 * C::kDecWarps);
      mbar_init(&pk[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * C::kEpiWarps);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer (both CTAs)
      const uint64_t pol_panel = l2_policy_code(l2_codes & 3u);
      const uint64_t pol_geno = l2_policy_code((l2_codes >> 2) & 3u);
      uint32_t s = 0, ph = 0;
      for (int t = cid; t < n_tiles; t += n_clusters) {
        int ct, pt;
        tile_coords(t, n_ctile, n_ptile, group_c, ct, pt);
        pt += ep.pt_base;
        const int prow = C::TRANS ? pt * kTPheno + cr * kTHalfPheno : pt * kTileP + cr * kHalfP;
        const int grow = ct * C::kTileRows + cr * C::kHalfRows;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * C::kStageBytes;
          const int kx = (kb_begin + kb) * kTileK;
          const uint32_t full0 = map_to_cta(&full[s], 0);
          mbar_arrive_expect_tx_cluster(full0, C::kTmaBytes);
          if constexpr (C::TRANS) {
            tma_load_2d_pair(st, &tm_v, full0, kx, grow, pol_geno);
            tma_load_2d_pair(st + C::kVBytesWide, &tm_qh, full0, kx, prow, pol_panel);
            tma_load_2d_pair(st + C::kVBytesWide + kTLimbBytes, &tm_q1, full0, kx, prow, pol_panel);
            tma_load_2d_pair(st + C::kVBytesWide + 2 * kTLimbBytes, &tm_q0, full0, kx, prow, pol_panel);
            if (++s == S) {
              s = 0;
              ph ^= 1;
            }
            continue;
          }
          tma_load_2d_pair(st, &tm_qh, full0, kx, prow, pol_panel);
          tma_load_2d_pair(st + kQBytes, &tm_q1, full0, kx, prow, pol_panel);
          if constexpr (!C::TWO) tma_load_2d_pair(st + 2 * kQBytes, &tm_q0, full0, kx, prow, pol_panel);
          if constexpr (FUSED) {
            mbar_arrive_expect_tx(&pk[s], kPackedBytes);
            tma_load_2d_hint(st + C::kOffPacked, &tm_v, &pk[s], (kb_begin + kb) * (kTileK / 4), grow, pol_geno);
            // the packed rows often come from DRAM (streamed, evict_first) while the panel hits
            // in L2: start them into L2 further ahead than the ring reaches
            if (PG_PACKED_PREFETCH > 0 && kb + PG_PACKED_PREFETCH < n_kb)
              tma_prefetch_2d(&tm_v, (kb_begin + kb + PG_PACKED_PREFETCH) * (kTileK / 4), grow, pol_geno);
          } else if constexpr (WIDE) {
            tma_load_2d_pair(st + C::kOffV, &tm_v, full0, kx, grow, pol_geno);
          } else {
            tma_load_2d_pair(st + C::kOffV, &tm_v, full0, kx, grow, pol_geno);
            tma_load_2d_pair(st + C::kOffV127, &tm_v127, full0, kx, grow, pol_geno);
          }
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ------------------------------------------------------------ MMA issuer (leader CTA)
      constexpr uint32_t idesc = idesc_s8_s32(kTileP, C::kAccCols);  // M = 256 across the pair
      const uint32_t dH = tmem_base;
      const uint32_t dL = tmem_base + C::kAccCols;
      const uint32_t dC = tmem_base + 2 * C::kAccCols;  // wide modes only
      uint32_t s = 0, ph = 0, aph = 0;
      for (int t = cid; t < n_tiles; t += n_clusters) {
        mbar_wait_cluster(tempty, aph ^ 1);
        tc_fence_after();
        uint32_t acc = 0;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait_cluster(&full[s], ph);
          if constexpr (FUSED) mbar_wait_cluster(&dec[s], ph);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + s * C::kStageBytes);
          if constexpr (C::TRANS) {
            // A = genotype digit rows, B = limb j -> accumulator j
            const uint64_t d_g = umma_desc_sw64(st);
            const uint64_t d_h = umma_desc_sw64(st + C::kVBytesWide);
            const uint64_t d_1 = umma_desc_sw64(st + C::kVBytesWide + kTLimbBytes);
            const uint64_t d_0 = umma_desc_sw64(st + C::kVBytesWide + 2 * kTLimbBytes);
#pragma unroll
            for (int k = 0; k < kTileK / 32; ++k) {
              mma_i8_ss_pair(dH, d_g + 2 * k, d_h + 2 * k, idesc, acc);
              mma_i8_ss_pair(dL, d_g + 2 * k, d_1 + 2 * k, idesc, acc);
              mma_i8_ss_pair(dC, d_g + 2 * k, d_0 + 2 * k, idesc, acc);
              acc = 1;
            }
            mma_commit_pair_multicast(&empty[s], 0x3);
            if (++s == S) {
              s = 0;
              ph ^= 1;
            }
            continue;
          }
          const uint64_t d_qh = umma_desc_sw64(st);
          const uint64_t d_q1 = umma_desc_sw64(st + kQBytes);
          const uint64_t d_q0 = umma_desc_sw64(st + 2 * kQBytes);
          const uint64_t d_v = umma_desc_sw64(st + C::kOffV);
          const uint64_t d_v127 = umma_desc_sw64(st + C::kOffV127);
#pragma unroll
          for (int k = 0; k < kTileK / 32; ++k) {
            // +32 bytes along K inside the 64-byte swizzle row == +2 in the >>4 address field
            if constexpr (WIDE) {
              mma_i8_ss_pair(dH, d_qh + 2 * k, d_v + 2 * k, idesc, acc);
              mma_i8_ss_pair(dL, d_q1 + 2 * k, d_v + 2 * k, idesc, acc);
              if constexpr (!C::TWO) mma_i8_ss_pair(dC, d_q0 + 2 * k, d_v + 2 * k, idesc, acc);
            } else {
              mma_i8_ss_pair(dH, d_qh + 2 * k, d_v + 2 * k, idesc, acc);
              mma_i8_ss_pair(dL, d_q1 + 2 * k, (C::NO127 ? d_v : d_v127) + 2 * k, idesc, acc);
              if constexpr (!C::TWO) mma_i8_ss_pair(dL, d_q0 + 2 * k, d_v + 2 * k, idesc, 1);
            }
            acc = 1;
          }
          mma_commit_pair_multicast(&empty[s], 0x3);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit_pair_multicast(tfull, 0x3);
        aph ^= 1;
      }
    }
  } else if (warp >= 4 && warp < C::kFirstEpiWarp) {
    if constexpr (FUSED) {
      // ------------------------------------------------------------ decoders (both CTAs)
      // row r of this CTA's packed half-tile (16 bytes = 64 samples) -> 64 B of v and 64 B of
      // 127v, as 4 swizzled 16-byte chunks each (SW64: chunk c of row r lives at
      // r*64 + ((c ^ ((r >> 1) & 3)) << 4)); kWords chunks per thread (4, or 2 with 8 warps)
      constexpr int kWords = 4 * 4 / C::kDecWarps;
      const int t_dec = (threadIdx.x - 128) % (32 * C::kDecWarps);
      const int team = (threadIdx.x - 128) / (32 * C::kDecWarps);
      uint32_t it = 0;
      const int r = t_dec / (4 / kWords);
      const int c_first = (t_dec % (4 / kWords)) * kWords;
      const uint32_t sw = (static_cast<uint32_t>(r) >> 1) & 3u;
      const uint32_t lut_u = reg_const(0xFF000001u), lut_u127 = reg_const(0x8100007Fu);
      uint32_t s = 0, ph = 0;
      for (int t = cid; t < n_tiles; t += n_clusters) {
        for (int kb = 0; kb < n_kb; ++kb) {
          if (C::kDecTeams > 1 && static_cast<int>(it++ % C::kDecTeams) != team) {
            if (++s == S) {
              s = 0;
              ph ^= 1;
            }
            continue;
          }
          mbar_wait(&pk[s], ph);
          uint8_t* st = smem + s * C::kStageBytes;
          uint32_t words[kWords];
          if constexpr (kWords == 4) {
            const uint4 w = reinterpret_cast<const uint4*>(st + C::kOffPacked)[r];
            words[0] = w.x;
            words[1] = w.y;
            words[2] = w.z;
            words[3] = w.w;
          } else {
            const uint2 w = reinterpret_cast<const uint2*>(st + C::kOffPacked + r * 16)[c_first >> 1];
            words[0] = w.x;
            words[1] = w.y;
          }
          const uint32_t st_a = smem_u32(st);
#pragma unroll
          for (int i = 0; i < kWords; ++i) {
            const int c = c_first + i;
            uint32_t u[4], u7[4];
            decode_word<!C::NO127>(words[i], u, u7, lut_u, lut_u127);
            const uint32_t off = r * 64 + ((c ^ sw) << 4);
            st_shared_v4(st_a + C::kOffV + off, u[0], u[1], u[2], u[3]);
            if constexpr (!C::NO127) st_shared_v4(st_a + C::kOffV127 + off, u7[0], u7[1], u7[2], u7[3]);
          }
          fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(map_to_cta(&dec[s], 0));
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp >= C::kFirstEpiWarp) {
    // -------------------------------------------------------------- epilogue (both CTAs)
    // this CTA's TMEM holds its 128 phenotypes (lanes) x all 256 genotype rows of the
    // pair tile (columns). Warp w reads lanes [32*(w%4), +32) (lane-quarter rule) and one
    // of kColGroups column ranges (16 warps: 4 groups of 64 columns; 12 warps: 3 groups).
    const int quarter = warp & 3;
    const int cg = (warp - C::kFirstEpiWarp) >> 2;
    const uint32_t tempty0 = map_to_cta(tempty, 0);
    uint32_t aph = 0;
    for (int t = cid; t < n_tiles; t += n_clusters) {
      int ct, pt;
      tile_coords(t, n_ctile, n_ptile, group_c, ct, pt);
      pt += ep.pt_base;
      const int pheno = pt * kTileP + cr * kHalfP + quarter * 32 + lane;
      mbar_wait_cluster(tfull, aph);
      tc_fence_after();
      const uint32_t tH = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
      const uint32_t tL = tH + C::kAccCols;
      // split the tile's 16-column chunks over the 4 column groups (12-column = 4-marker
      // units in the 3-row mode, 12-column = 4 phenotype triples in the transposed mode)
      constexpr int kUnit = (MODE == kWide3 || MODE == kWide3Two || C::TRANS) ? 12 : 16;  // kWide4Two: 16
      constexpr int kChunks = C::kAccCols / kUnit;
      constexpr int G = C::kColGroups;
      const int c0 = kUnit * ((cg * kChunks) / G), c1 = kUnit * (((cg + 1) * kChunks) / G);
      if constexpr (C::TRANS) {
        epilogue_tile_wide3t(ep, tH, ct, static_cast<int>(cr), pt, quarter, lane, c0, c1);
      } else if constexpr (MODE == kWide3Two) {
        epilogue_tile_wide_two<3>(ep, tH, ct, pheno, lane, c0, c1);
      } else if constexpr (MODE == kWide4Two) {
        epilogue_tile_wide_two<4>(ep, tH, ct, pheno, lane, c0, c1);
      } else if constexpr (MODE == kWide3) {
        epilogue_tile_wide3(ep, tH, ct, pheno, lane, c0, c1);
      } else if constexpr (WIDE) {
        epilogue_tile_wide(ep, tH, ct, pheno, lane, c0, c1);
      } else {
        if constexpr (MODE == kFused2) {
          epilogue_tile_two(ep, tH, tL, ct, pheno, lane, c0, c1);
        } else switch (ep.rows_per_marker) {
          case 1: epilogue_tile<1>(ep, tH, tL, ct, pheno, lane, c0, c1); break;
          case 2: epilogue_tile<2>(ep, tH, tL, ct, pheno, lane, c0, c1); break;
          case 8: epilogue_tile<8>(ep, tH, tL, ct, pheno, lane, c0, c1); break;
          default: epilogue_tile<16>(ep, tH, tL, ct, pheno, lane, c0, c1); break;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0);
      aph ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs done with TMEM and with remote barriers
  tc_fence_after();
  if (warp == 2) tmem_free_pair(tmem_base, kTmemCols);
}

// Statistics of a K-sliced run from the accumulated int64 partials (xu, xm) per
// (marker slot, phenotype): lanes = 32 consecutive phenotypes (so the warp-aggregated
// compaction and the premask work as in the GEMM epilogue), warps stride over markers.
__global__ void x_epilogue_kernel(AssocEpilogue ep, int64_t m_slots) {
  const int lane = threadIdx.x & 31;
  const int pheno = blockIdx.x * 32 + lane;
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  const float sc_f = ep.scale_f[pheno];
  const double sc_d = ep.scale_d[pheno];
  const float cq_f = ep.cq_f[pheno];
  const long long cq = ep.cq[pheno];
  const float rb = ep.rbar ? ep.rbar[pheno] : INFINITY;
  MaxAbsR mx;
  for (int64_t m = static_cast<int64_t>(blockIdx.y) * (blockDim.x >> 5) + (threadIdx.x >> 5); m < m_slots;
       m += static_cast<int64_t>(gridDim.y) * (blockDim.x >> 5)) {
    const long long* x = ep.x_accum + (m * ep.x_ld + pheno) * 2;
    AssocEpilogue e = ep;
    e.x_accum = nullptr;
    double lo_u = 0.0, lo_cm = 0.0;
    if (ep.x_lo) {  // F64 precision: the two-level panel's lo partials
      const long long* xl = ep.x_lo + (m * ep.x_ld + pheno) * 2;
      lo_u = static_cast<double>(xl[0]) / kLoScale;
      lo_cm = static_cast<double>(ep.cq_lo[pheno] - xl[1]) / kLoScale;
    }
    epilogue_value(e, x[0], x[1], static_cast<int>(m), pheno, sc_f, sc_d, cq_f, cq, rb, lane, lanemask_lt, mx, true,
                   lo_u, lo_cm);
  }
  if (ep.max_abs_r && pheno < ep.p_valid)
    atomicMax(ep.max_abs_r + pheno, static_cast<unsigned long long>(__double_as_longlong(mx.d)));
}

constexpr uint32_t kDefaultL2Codes = 1u | (1u << 2);  // panel and genotypes evict_last
// Panel-stationary raster, 2 phenotype tiles per group (35 MB of limbs stay in L2 while the
// genotype tiles stream past): DRAM per C3 launch 22 GB vs 49 GB for 74-tile
// genotype-stationary groups (tools/dram_sweep.sh, ncu), with equal or better throughput.
constexpr int kDefaultGroup = -2;
// Two-limb GEMMs: a phenotype tile's limbs are 2/3 the bytes, so 4-tile slices (47 MB at
// N 23k) still stay in L2, with the streamed genotype tiles evict_first: DRAM per C3 launch
// 17.7 -> 12.0 GB, equal or better throughput (profiles/r2_c3_raster_sweep.txt, round 2b)
constexpr uint32_t kDefaultL2CodesTwo = 1u | (2u << 2);
constexpr int kDefaultGroupTwo = -4;

template <int MODE>
int launch_common(const CUtensorMap& tm_qh, const CUtensorMap& tm_q1, const CUtensorMap& tm_q0,
                  const CUtensorMap& tm_v, const CUtensorMap& tm_v127, int64_t p_pad, int64_t c_pad, int64_t k_pad,
                  const AssocEpilogue& ep, cudaStream_t stream) {
  PG_CUDA_CHECK(cudaFuncSetAttribute(assoc_i8_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     Cfg<MODE>::kSmemBytes));
  int dev = 0, n_sm = 0;
  PG_CUDA_CHECK(cudaGetDevice(&dev));
  PG_CUDA_CHECK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  const int n_ctile = static_cast<int>(c_pad / Cfg<MODE>::kTileRows);
  const int n_ptile = ep.pt_count > 0 ? ep.pt_count
                                      : static_cast<int>(Cfg<MODE>::TRANS ? (p_pad + kTPheno - 1) / kTPheno : p_pad / kTileP);
  PG_REQUIRE(!Cfg<MODE>::TRANS || (ep.pt_base == 0 && ep.pt_count == 0), PG_ERR_INVALID,
             "assoc: phenotype-tile ranges are not supported by the transposed GEMM");
  const int n_tiles = n_ctile * n_ptile;
  const int max_pairs = n_sm / 2;
  const int pairs = n_tiles < max_pairs ? n_tiles : max_pairs;
  const int grid = 2 * pairs;
  // tuning knobs (defaults measured best): raster group width and
  // L2 priorities (panel | geno << 2; 0 normal, 1 evict_last, 2 evict_first)
  static const int env_group = [] {  // > 0 genotype-stationary width, < 0 panel-stationary height
    const char* e = std::getenv("PG_GROUP_C");
    return e ? std::atoi(e) : 0;
  }();
  static const int env_l2 = [] {
    const char* e = std::getenv("PG_L2_CODES");
    return e ? std::atoi(e) : -1;
  }();
  const int group_c = env_group != 0 ? env_group : (Cfg<MODE>::TWO ? kDefaultGroupTwo : kDefaultGroup);
  const uint32_t l2_codes =
      env_l2 >= 0 ? static_cast<uint32_t>(env_l2) : (Cfg<MODE>::TWO ? kDefaultL2CodesTwo : kDefaultL2Codes);
  const int n_kb = static_cast<int>(k_pad / kTileK);
  constexpr int kSliceKb = static_cast<int>(kSliceK / kTileK);
  if (ep.x_accum == nullptr) {
    PG_REQUIRE(n_kb <= kSliceKb, PG_ERR_INVALID, "assoc: %d K blocks need the sliced (x_accum) path", n_kb);
    assoc_i8_kernel<MODE><<<grid, Cfg<MODE>::kThreadsM, Cfg<MODE>::kSmemBytes, stream>>>(
        tm_qh, tm_q1, tm_q0, tm_v, tm_v127, n_ctile, n_ptile, 0, n_kb, group_c, l2_codes, ep);
  } else {
    // exact int64 partials per (marker, phenotype): K slices of one int32-exact range each
    // (cohorts above kSliceK samples), and / or the two levels of the F64 panel; the
    // statistics come from the summed partials (same epilogue arithmetic)
    PG_REQUIRE(!Cfg<MODE>::TRANS, PG_ERR_INVALID, "assoc(wide3t): partial-sum runs use the untransposed kernel");
    PG_REQUIRE(ep.x_ld == p_pad, PG_ERR_INVALID, "assoc: x_accum leading dimension must be p_pad");
    const int rows = Cfg<MODE>::WIDE ? Cfg<MODE>::kWideR : ep.rows_per_marker;
    const int64_t m_slots = c_pad / rows;
    PG_CUDA_CHECK(cudaMemsetAsync(ep.x_accum, 0, sizeof(long long) * 2 * m_slots * p_pad, stream));
    for (int kb0 = 0; kb0 < n_kb; kb0 += kSliceKb) {
      const int nk = n_kb - kb0 < kSliceKb ? n_kb - kb0 : kSliceKb;
      assoc_i8_kernel<MODE><<<grid, Cfg<MODE>::kThreadsM, Cfg<MODE>::kSmemBytes, stream>>>(
          tm_qh, tm_q1, tm_q0, tm_v, tm_v127, n_ctile, n_ptile, kb0, nk, group_c, l2_codes, ep);
      PG_CUDA_CHECK(cudaGetLastError());
    }
    if (!ep.x_partials_only) {
      const unsigned gy = static_cast<unsigned>(m_slots < 4096 ? (m_slots + 7) / 8 : 512);
      x_epilogue_kernel<<<dim3(static_cast<unsigned>(p_pad / 32), gy), 256, 0, stream>>>(ep, m_slots);
    }
  }
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int encode_panel(const int8_t* qh, const int8_t* q1, const int8_t* q0, int64_t p_pad, int64_t k_pad,
                 CUtensorMap& a, CUtensorMap& b, CUtensorMap& c) {
  const uint64_t pitch = static_cast<uint64_t>(k_pad);
  PG_CHECK_STATUS(encode_tmap_2d_i8(&a, qh, k_pad, p_pad, pitch, kTileK, kHalfP));
  PG_CHECK_STATUS(encode_tmap_2d_i8(&b, q1, k_pad, p_pad, pitch, kTileK, kHalfP));
  PG_CHECK_STATUS(encode_tmap_2d_i8(&c, q0, k_pad, p_pad, pitch, kTileK, kHalfP));
  return PG_OK;
}

}  // namespace

int launch_assoc(const int8_t* qh, const int8_t* q1, const int8_t* q0, int64_t p_pad, const int8_t* v,
                 const int8_t* v127, int64_t c_pad, int64_t k_pad, const AssocEpilogue& ep, cudaStream_t stream) {
  PG_REQUIRE(p_pad % kTileP == 0 && c_pad % kTileC == 0 && k_pad % kTileK == 0 && p_pad > 0 && c_pad > 0 &&
                 k_pad > 0,
             PG_ERR_INVALID, "assoc: bad padded shape p=%lld c=%lld k=%lld", (long long)p_pad, (long long)c_pad,
             (long long)k_pad);
  PG_REQUIRE(ep.rows_per_marker == 1 || ep.rows_per_marker == 2 || ep.rows_per_marker == 8 ||
                 ep.rows_per_marker == 16,
             PG_ERR_INVALID, "assoc: rows_per_marker %d", ep.rows_per_marker);
  CUtensorMap tm_qh, tm_q1, tm_q0, tm_v, tm_v127;
  PG_CHECK_STATUS(encode_panel(qh, q1, q0, p_pad, k_pad, tm_qh, tm_q1, tm_q0));
  PG_CHECK_STATUS(encode_tmap_2d_i8(&tm_v, v, k_pad, c_pad, k_pad, kTileK, kHalfC));
  PG_CHECK_STATUS(encode_tmap_2d_i8(&tm_v127, v127, k_pad, c_pad, k_pad, kTileK, kHalfC));
  if (ep.q0n) {  // two-limb side GEMM (Mq' only): the candidates get sum_missing q0 later
    PG_REQUIRE(ep.side_out != nullptr && ep.rows_per_marker == 1 && ep.x_accum == nullptr, PG_ERR_INVALID,
               "assoc(planes, two-limb): side GEMMs only");
    return launch_common<kPlanes2>(tm_qh, tm_q1, tm_q0, tm_v, tm_v127, p_pad, c_pad, k_pad, ep, stream);
  }
  return launch_common<kPlanes>(tm_qh, tm_q1, tm_q0, tm_v, tm_v127, p_pad, c_pad, k_pad, ep, stream);
}

int launch_assoc_packed(const int8_t* qh, const int8_t* q1, const int8_t* q0, int64_t p_pad, const uint8_t* packed,
                        int64_t pitch, int64_t n_markers, int64_t k_pad, const AssocEpilogue& ep,
                        cudaStream_t stream) {
  PG_REQUIRE(p_pad % kTileP == 0 && k_pad % kTileK == 0 && n_markers > 0 && pitch * 4 >= k_pad && pitch % 16 == 0,
             PG_ERR_INVALID, "assoc(packed): bad shape p=%lld m=%lld k=%lld pitch=%lld", (long long)p_pad,
             (long long)n_markers, (long long)k_pad, (long long)pitch);
  PG_REQUIRE(ep.rows_per_marker == 1, PG_ERR_INVALID, "assoc(packed): fused decode needs rows_per_marker 1");
  CUtensorMap tm_qh, tm_q1, tm_q0, tm_pk;
  PG_CHECK_STATUS(encode_panel(qh, q1, q0, p_pad, k_pad, tm_qh, tm_q1, tm_q0));
  // packed rows: k_pad/4 bytes of codes per marker (rows past n_markers read as zeros by TMA)
  PG_CHECK_STATUS(encode_tmap_2d_i8(&tm_pk, packed, k_pad / 4, n_markers, pitch, kTileK / 4, kHalfC, false));
  const int64_t c_pad = round_up(n_markers, kTileC);
  if (ep.q0n) {
    PG_REQUIRE(ep.full_r == nullptr && ep.max_abs_r == nullptr && ep.x_accum == nullptr && ep.mpack != nullptr,
               PG_ERR_INVALID, "assoc(two-limb): THRESHOLD / TOPK candidates of unsliced runs only");
    return launch_common<kFused2>(tm_qh, tm_q1, tm_q0, tm_pk, tm_pk, p_pad, c_pad, k_pad, ep, stream);
  }
  return launch_common<kFused>(tm_qh, tm_q1, tm_q0, tm_pk, tm_pk, p_pad, c_pad, k_pad, ep, stream);
}

namespace {

// Warp per candidate: c0 = sum_k q0[p,k] u[m,k] over the packed 2-bit row (u as the GEMM
// decodes it: 00 -> +1, 10 -> 0, 11 -> -1, 01 missing -> 0; q0 is 0 on excluded / padding
// samples), 16 samples per lane step by DP4A; then the exact fp64 r of the candidate.
__global__ void refine_two_limb_kernel(const unsigned long long* __restrict__ key, double* __restrict__ cand_r,
                                       int64_t n, const uint8_t* __restrict__ packed, int64_t pitch,
                                       const int8_t* __restrict__ q0, int64_t k_pad, AssocEpilogue ep) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t chunks = k_pad / 16;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const unsigned long long kk = key[i];
    const int m = static_cast<int>(kk >> 32);
    const int p = static_cast<int>(kk & 0xffffffffull);
    const uint32_t* row = reinterpret_cast<const uint32_t*>(packed + static_cast<int64_t>(m) * pitch);
    const uint4* qrow = reinterpret_cast<const uint4*>(q0 + static_cast<int64_t>(p) * k_pad);
    // with a two-limb side GEMM (side_two) the missing calls' q0 sum is deferred too
    const bool side_two = ep.side_slot != nullptr && ep.side_two && ep.side_slot[m] >= 0;
    int acc = 0, acc_m = 0;
    for (int64_t c = lane; c < chunks; c += 32) {
      uint32_t u[4], u7[4];
      const uint32_t word = __ldg(row + c);
      decode_word(word, u, u7);
      const uint4 w = __ldg(qrow + c);
      acc = __dp4a(static_cast<int>(w.x), static_cast<int>(u[0]), acc);
      acc = __dp4a(static_cast<int>(w.y), static_cast<int>(u[1]), acc);
      acc = __dp4a(static_cast<int>(w.z), static_cast<int>(u[2]), acc);
      acc = __dp4a(static_cast<int>(w.w), static_cast<int>(u[3]), acc);
      if (side_two) {
        uint32_t mk[4];
        decode_word_missing(word, mk);
        acc_m = __dp4a(static_cast<int>(w.x), static_cast<int>(mk[0]), acc_m);
        acc_m = __dp4a(static_cast<int>(w.y), static_cast<int>(mk[1]), acc_m);
        acc_m = __dp4a(static_cast<int>(w.z), static_cast<int>(mk[2]), acc_m);
        acc_m = __dp4a(static_cast<int>(w.w), static_cast<int>(mk[3]), acc_m);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      acc_m += __shfl_xor_sync(0xffffffffu, acc_m, o);
    }
    if (lane == 0) {
      const long long xu = __double_as_longlong(cand_r[i]) + acc;
      long long xm = 0;
      if (ep.side_slot) {
        const int sl = ep.side_slot[m];
        if (sl >= 0) xm = ep.side_x[static_cast<int64_t>(sl) * ep.side_ld + p] + acc_m;
      }
      cand_r[i] = ep.scale_d[p] * (static_cast<double>(xu) - ep.mu_d[m] * static_cast<double>(ep.cq[p] - xm)) *
                  ep.invd_d[m];
    }
  }
}

__global__ void q0_norm_kernel(const int8_t* __restrict__ q0, int64_t k_pad, float* __restrict__ out) {
  const int64_t p = blockIdx.x;
  const uint4* row = reinterpret_cast<const uint4*>(q0 + p * k_pad);
  unsigned long long s = 0;
  for (int64_t c = threadIdx.x; c < k_pad / 16; c += blockDim.x) {
    const uint4 w = row[c];
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) s += static_cast<unsigned long long>(__dp4a(static_cast<int>(ws[j]), static_cast<int>(ws[j]), 0));
  }
  __shared__ unsigned long long red[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
    out[p] = __double2float_ru(sqrt(static_cast<double>(t)) * (1.0 + 1e-12));
  }
}

}  // namespace

int refine_two_limb(const unsigned long long* cand_key, double* cand_r, int64_t n, const uint8_t* packed,
                    int64_t pitch, const int8_t* q0, int64_t k_pad, const AssocEpilogue& ep, cudaStream_t stream) {
  if (n <= 0) return PG_OK;
  PG_REQUIRE(k_pad % 64 == 0 && pitch % 16 == 0 && pitch * 4 >= k_pad, PG_ERR_INVALID, "refine_two_limb: bad shape");
  const int64_t warps = (n + 0);
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((warps + 7) / 8, 148 * 16));
  refine_two_limb_kernel<<<grid, 256, 0, stream>>>(cand_key, cand_r, n, packed, pitch, q0, k_pad, ep);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

namespace {
// ||u_m + mu_m mask_m||_2 = sqrt(sum u^2 + mu^2 n_miss) (u = 0 on missing calls) bounds what the
// deferred limb can add to X - mu (Cq - Mq) when Mq is deferred too (wide two-limb tiles), and
// bounds it from above when Mq is exact (the PLINK side GEMM)
__global__ void pack_marker_kernel(const float* __restrict__ mu_f, const double* __restrict__ mu_d,
                                   const float* __restrict__ invd_f, const long long* __restrict__ ss_u,
                                   const long long* __restrict__ n_miss, int64_t m_cap, float4* __restrict__ out) {
  for (int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; m < m_cap;
       m += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float iv = invd_f[m];
    const double mu = mu_d[m];
    const double sq = static_cast<double>(ss_u[m]) + mu * mu * static_cast<double>(n_miss[m]);
    const float un = __fsqrt_ru(static_cast<float>(sq * (1.0 + 1e-7)));
    out[m] = make_float4(mu_f[m], iv, __fmul_ru(un, iv), 0.f);
  }
}

// Warp per wide two-limb candidate: the q0 limb against the marker's digit rows (u = d0 + 255 d1)
// and missing row, by DP4A over the int8 planes; then the exact fp64 r.
template <int R>
__global__ void refine_wide_two_kernel(const unsigned long long* __restrict__ key, double* __restrict__ cand_r,
                                       const long long* __restrict__ cand_xm, int64_t n, const int8_t* __restrict__ v,
                                       const int8_t* __restrict__ q0, int64_t k_pad, AssocEpilogue ep) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t chunks = k_pad / 16;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const unsigned long long kk = key[i];
    const int64_t m = static_cast<int64_t>(kk >> 32);
    const int p = static_cast<int>(kk & 0xffffffffull);
    const uint4* qrow = reinterpret_cast<const uint4*>(q0 + static_cast<int64_t>(p) * k_pad);
    int d[R];  // per row: sum q0 * row (digits 0..R-2, then the missing row)
#pragma unroll
    for (int t = 0; t < R; ++t) d[t] = 0;
    for (int64_t c = lane; c < chunks; c += 32) {
      const uint4 w = __ldg(qrow + c);
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(v + (R * m + t) * k_pad) + c);
        d[t] = __dp4a(static_cast<int>(w.x), static_cast<int>(a.x), d[t]);
        d[t] = __dp4a(static_cast<int>(w.y), static_cast<int>(a.y), d[t]);
        d[t] = __dp4a(static_cast<int>(w.z), static_cast<int>(a.z), d[t]);
        d[t] = __dp4a(static_cast<int>(w.w), static_cast<int>(a.w), d[t]);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
      for (int t = 0; t < R; ++t) d[t] += __shfl_xor_sync(0xffffffffu, d[t], o);
    if (lane == 0) {
      long long du = 0, w = 1;
#pragma unroll
      for (int t = 0; t < R - 1; ++t) {
        du += w * d[t];
        w *= 255;
      }
      const long long xu = __double_as_longlong(cand_r[i]) + du;
      const long long xm = cand_xm[i] + d[R - 1];
      cand_r[i] = ep.scale_d[p] * (static_cast<double>(xu) - ep.mu_d[m] * static_cast<double>(ep.cq[p] - xm)) *
                  ep.invd_d[m];
    }
  }
}
}  // namespace

int refine_wide_two(const unsigned long long* cand_key, double* cand_r, const long long* cand_xm, int64_t n,
                    const int8_t* v, const int8_t* q0, int64_t k_pad, const AssocEpilogue& ep, cudaStream_t stream) {
  if (n <= 0) return PG_OK;
  PG_REQUIRE(k_pad % 64 == 0 && (ep.rows_per_marker == 3 || ep.rows_per_marker == 4), PG_ERR_INVALID,
             "refine_wide_two: bad shape");
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n + 7) / 8, 148 * 16));
  if (ep.rows_per_marker == 4)
    refine_wide_two_kernel<4><<<grid, 256, 0, stream>>>(cand_key, cand_r, cand_xm, n, v, q0, k_pad, ep);
  else
    refine_wide_two_kernel<3><<<grid, 256, 0, stream>>>(cand_key, cand_r, cand_xm, n, v, q0, k_pad, ep);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int pack_marker_terms(const float* mu_f, const double* mu_d, const float* invd_f, const long long* ss_u,
                      const long long* n_miss, int64_t m_cap, float4* out, cudaStream_t stream) {
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((m_cap + 255) / 256, 2048));
  pack_marker_kernel<<<grid, 256, 0, stream>>>(mu_f, mu_d, invd_f, ss_u, n_miss, m_cap, out);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int panel_q0_norms(const int8_t* q0, int64_t p_pad, int64_t k_pad, float* out, cudaStream_t stream) {
  q0_norm_kernel<<<static_cast<unsigned>(p_pad), 256, 0, stream>>>(q0, k_pad, out);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int launch_assoc_wide3t(const int8_t* qh, const int8_t* q1, const int8_t* q0, int64_t p_pad, const int8_t* v,
                        int64_t c_pad, int64_t k_pad, const AssocEpilogue& ep, cudaStream_t stream) {
  PG_REQUIRE(ep.rows_per_marker == kWideRows3 && ep.max_abs_r == nullptr && ep.x_accum == nullptr &&
                 p_pad % kTileP == 0 && c_pad % kTileC == 0 && k_pad % kTileK == 0 && p_pad > 0 && c_pad > 0 &&
                 k_pad > 0 && k_pad <= kSliceK,
             PG_ERR_INVALID, "assoc(wide3t): bad arguments p=%lld c=%lld k=%lld", (long long)p_pad, (long long)c_pad,
             (long long)k_pad);
  CUtensorMap tm_qh, tm_q1, tm_q0, tm_v;
  const uint64_t pitch = static_cast<uint64_t>(k_pad);
  PG_CHECK_STATUS(encode_tmap_2d_i8(&tm_qh, qh, k_pad, p_pad, pitch, kTileK, kTHalfPheno));
  PG_CHECK_STATUS(encode_tmap_2d_i8(&tm_q1, q1, k_pad, p_pad, pitch, kTileK, kTHalfPheno));
  PG_CHECK_STATUS(encode_tmap_2d_i8(&tm_q0, q0, k_pad, p_pad, pitch, kTileK, kTHalfPheno));
  PG_CHECK_STATUS(encode_tmap_2d_i8(&tm_v, v, k_pad, c_pad, k_pad, kTileK, kTileC / 2));
  return launch_common<kWide3T>(tm_qh, tm_q1, tm_q0, tm_v, tm_v, p_pad, c_pad, k_pad, ep, stream);
}

int launch_assoc_wide(const int8_t* qh, const int8_t* q1, const int8_t* q0, int64_t p_pad, const int8_t* v,
                      int64_t c_pad, int64_t k_pad, const AssocEpilogue& ep, cudaStream_t stream) {
  const int R = ep.rows_per_marker;
  PG_REQUIRE(R == kRowsW || R == kWideRows3, PG_ERR_INVALID, "assoc(wide): rows_per_marker must be 3 or 4, got %d",
             R);
  const int tile = R == kWideRows3 ? (ep.q0n ? kTileCWide3Two : kTileCWide3) : (ep.q0n ? kTileC : kTileCW);
  PG_REQUIRE(p_pad % kTileP == 0 && c_pad % tile == 0 && k_pad % kTileK == 0 && p_pad > 0 && c_pad > 0 &&
                 k_pad > 0,
             PG_ERR_INVALID, "assoc(wide): bad padded shape p=%lld c=%lld k=%lld", (long long)p_pad,
             (long long)c_pad, (long long)k_pad);
  CUtensorMap tm_qh, tm_q1, tm_q0, tm_v;
  PG_CHECK_STATUS(encode_panel(qh, q1, q0, p_pad, k_pad, tm_qh, tm_q1, tm_q0));
  if (R == kWideRows3 && ep.q0n) {  // two-limb premask: 240-row tiles
    PG_REQUIRE(c_pad % kTileCWide3Two == 0 && ep.full_r == nullptr && ep.max_abs_r == nullptr && ep.x_accum == nullptr &&
                   ep.mpack != nullptr && ep.cand_xm != nullptr,
               PG_ERR_INVALID, "assoc(wide, two-limb): bad arguments");
    PG_CHECK_STATUS(encode_tmap_2d_i8(&tm_v, v, k_pad, c_pad, k_pad, kTileK, kTileCWide3Two / 2));
    return launch_common<kWide3Two>(tm_qh, tm_q1, tm_q0, tm_v, tm_v, p_pad, c_pad, k_pad, ep, stream);
  }
  if (R == kRowsW && ep.q0n) {  // two-limb premask: 256-row tiles (64 markers)
    PG_REQUIRE(c_pad % kTileC == 0 && ep.full_r == nullptr && ep.max_abs_r == nullptr && ep.x_accum == nullptr &&
                   ep.mpack != nullptr && ep.cand_xm != nullptr,
               PG_ERR_INVALID, "assoc(wide4, two-limb): bad arguments");
    PG_CHECK_STATUS(encode_tmap_2d_i8(&tm_v, v, k_pad, c_pad, k_pad, kTileK, kTileC / 2));
    return launch_common<kWide4Two>(tm_qh, tm_q1, tm_q0, tm_v, tm_v, p_pad, c_pad, k_pad, ep, stream);
  }
  PG_CHECK_STATUS(encode_tmap_2d_i8(&tm_v, v, k_pad, c_pad, k_pad, kTileK, tile / 2));
  if (R == kWideRows3) return launch_common<kWide3>(tm_qh, tm_q1, tm_q0, tm_v, tm_v, p_pad, c_pad, k_pad, ep, stream);
  return launch_common<kWide>(tm_qh, tm_q1, tm_q0, tm_v, tm_v, p_pad, c_pad, k_pad, ep, stream);
}

}  // namespace pg

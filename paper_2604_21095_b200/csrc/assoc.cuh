// Internal interface of the association GEMM (K2) + fused epilogue (K3).
//
// Exact-integer formulation. The standardized panel is
// quantized once per phenotype p to q = round(y~ / s_p), |q| <= kQMax, and
// split into three int8 limbs  q = kWH * qH + 127 * q1 + q0.
// Genotype rows are ternary codes v in {-1, 0, 1}; the decoder also writes the
// plane 127*v so that two limbs share one int32 accumulator:
//   accH[p, c] = sum_k qH[p,k] * v[c,k]
//   accL[p, c] = sum_k q1[p,k] * (127 v[c,k]) + q0[p,k] * v[c,k]
//   X[p, c]    = kWH * accH + accL   == sum_k q[p,k] v[c,k]   (exact, int64)
// All products and sums are integers, so the tensor-core result is exact and
// independent of tiling, batching and GPU count.
#pragma once
#include <climits>
#include <cstdint>

#include "pg_common.cuh"

namespace pg {

constexpr int kTileP = 256;   // phenotypes per CTA-pair tile (UMMA M = 256, cta_group::2; A = panel limbs)
constexpr int kTileC = 256;   // genotype rows per pair tile (UMMA N, B operand; 128 per CTA)
constexpr int kTileK = 64;    // int8 samples per pipeline stage (one 64-byte swizzle row)
constexpr int64_t kWH = 32385;          // weight of the high limb: 2*(127*127+63)+1
constexpr int64_t kQMax = kWH * 127 + 16192;  // largest |q| representable by the limbs
// Largest padded sample count whose int32 accumulators cannot overflow: one sample adds at
// most 127*127 + 63 = 16192 to accL (ternary) or 127*127 to A / B (wide digits).
constexpr int64_t kMaxExactK = (INT32_MAX / 16192) / 64 * 64;  // 132,608
// Larger cohorts run the contraction in K slices of kSliceK samples whose int32 results
// are exact and are summed in int64 (AssocEpilogue::x_accum).
constexpr int64_t kSliceK = 131072;
static_assert(kSliceK <= kMaxExactK, "slice must stay inside the exact int32 range");

struct AssocEpilogue {
  int rows_per_marker;          // ternary: 1 (u), 2 (u, missing), 8 / 16 (digits + missing); wide: 4
  int raw;                      // 1: emit s_p * (X - mu (Cq - Mq)) without the 1/den scale (side GEMM K5)
  int64_t m_valid;              // markers in this launch
  int64_t p_valid;              // phenotypes
  const float* mu_f;            // [markers] mean of u over observed kept samples
  const double* mu_d;
  const float* invd_f;          // [markers] 1/sqrt(N * V_u); NaN = skipped / padding
  const double* invd_d;
  const float* scale_f;         // [p_pad] quantization step s_p
  const double* scale_d;
  const float* cq_f;            // [p_pad] sum_k q[p,k]
  const long long* cq;
  const float* rbar;            // [p_pad] premask bar on |r| (already widened); null = no candidates
  unsigned long long* cand_key; // (marker << 32) | phenotype
  double* cand_r;               // exact fp64 r of the candidate
  unsigned long long* cand_count;  // 64-bit: a launch may produce more than 2^31 candidates
  unsigned long long cand_base;    // initial counter value (test hook); slot = counter - cand_base
  int64_t cand_cap;
  unsigned long long* max_abs_r;  // [p_pad] running max |r| (bits of a non-negative double), or null = off
  double* full_r;               // FULL mode: r[marker * full_ld + p] (fp64), or null
  int64_t full_ld;
  long long* x_accum;           // K-sliced runs (k_pad > kSliceK): int64 (xu, xm) partials
  int64_t x_ld;                 //   [marker slot][x_ld = p_pad][2]; null otherwise
  // Missing-call side path (PLINK, fused decode, rows_per_marker 1): a planes GEMM over the
  // mask rows of the markers that have missing calls writes Mq = sum_missing q per
  // (row j, phenotype) to side_out[j * side_ld + p] (nothing else); the fused GEMM then reads
  // xm = side_x[side_slot[m] * side_ld + p] for markers with side_slot[m] >= 0 (else 0).
  long long* side_out;
  const long long* side_x;
  const int* side_slot;
  int64_t side_ld;
  // F64 precision mode (two-level panel, panel.cuh): the lo level's exact (xu, xm) partials
  // (x_lo, same layout as x_accum) and column sums cq_lo join the hi level's in the final
  // statistics, r = s ((xu + xu_lo / kLoScale) - mu ((cq - xm) + (cq_lo - xm_lo) / kLoScale)) / den.
  const long long* x_lo;
  const long long* cq_lo;
  int x_partials_only;  // 1: accumulate x_accum only (the lo level's pass), no statistics
  // Two-limb premask (THRESHOLD / TOPK; kFused2, kWide3Two, kPlanes2 side GEMMs): the GEMM
  // skips the q0 limb, so it sees X' = X - sum_k q0 (u + mu mask) terms. The premask widens by
  // the rigorous bound |sum q0 (u + mu mask)| <= ||q0_p||_2 ||u_m + mu_m mask_m||_2
  // (q0n[p] = ||q0_p||_2; mpack[m] = (mu_f, invd_f, ||u_m + mu_m mask_m||_2 invd_f, 0), one
  // 16-byte broadcast load per marker column) and a candidate stores X' (int64 bits in cand_r);
  // refine_two_limb / refine_wide_two add the q0 sums exactly afterwards and write the fp64 r.
  // A non-null q0n selects the two-limb kernels.
  const float* q0n;
  const float4* mpack;
  long long* cand_xm;  // wide two-limb candidates: X'_m (the missing row's deferred-limb sum comes later)
  int side_two;        // the side GEMM ran two limbs: side_x holds Mq' (refine_two_limb adds sum_missing q0)
  // Phenotype-tile range of this launch (pipelined panel, pg_ctx_set_panel_async: the first
  // batch's GEMM runs one phenotype chunk at a time as the chunks land): tiles
  // [pt_base, pt_base + pt_count) of kTileP phenotypes; pt_count 0 = every tile.
  int pt_base;
  int pt_count;
};
// (mu_f, invd_f, sqrt(ss_u + mu^2 n_miss) * invd_f) per marker slot [0, m_cap) for the
// two-limb epilogues.
int pack_marker_terms(const float* mu_f, const double* mu_d, const float* invd_f, const long long* ss_u,
                      const long long* n_miss, int64_t m_cap, float4* out, cudaStream_t stream);
// Candidates of a wide two-limb launch (BGEN-8 digit planes v, 3 rows per marker): cand_r holds
// X'_u bits and cand_xm X'_m on entry; cand_r the exact fp64 r on exit.
int refine_wide_two(const unsigned long long* cand_key, double* cand_r, const long long* cand_xm, int64_t n,
                    const int8_t* v, const int8_t* q0, int64_t k_pad, const AssocEpilogue& ep, cudaStream_t stream);
constexpr double kLoScale = 4194304.0;  // 2^22: lo-level limbs q2 = rint((y~/s - q) 2^22), |q2| <= 2^21

// Launch K2/K3 on `stream`. Panel limbs q*[p_pad, k_pad], genotype planes
// v / v127 [c_pad, k_pad] (int8, K-major, rows 16-byte aligned).
int launch_assoc(const int8_t* qh, const int8_t* q1, const int8_t* q0, int64_t p_pad, const int8_t* v,
                 const int8_t* v127, int64_t c_pad, int64_t k_pad, const AssocEpilogue& ep, cudaStream_t stream);

// Fused-decode variant: genotype operand decoded in shared memory from packed
// 2-bit .bed rows (`pitch` bytes apart, >= k_pad/4 bytes of codes); rows_per_marker 1.
int launch_assoc_packed(const int8_t* qh, const int8_t* q1, const int8_t* q0, int64_t p_pad, const uint8_t* packed,
                        int64_t pitch, int64_t n_markers, int64_t k_pad, const AssocEpilogue& ep,
                        cudaStream_t stream);
// Candidates of a two-limb launch (ep.q0n set): cand_r holds X' (int64 bits) on entry and the
// exact fp64 r on exit, r = s_p (X' + sum_k q0[p,k] u[m,k] - mu_m (Cq_p - Mq)) / sqrt(N V_m).
int refine_two_limb(const unsigned long long* cand_key, double* cand_r, int64_t n, const uint8_t* packed,
                    int64_t pitch, const int8_t* q0, int64_t k_pad, const AssocEpilogue& ep, cudaStream_t stream);
// ||q0_p||_2 per phenotype (rounded up) for the two-limb premask bound.
int panel_q0_norms(const int8_t* q0, int64_t p_pad, int64_t k_pad, float* out, cudaStream_t stream);

// Wide-digit variant for dosage sources: one int8 plane v [c_pad, k_pad] of balanced
// base-255 digits (rows per marker: digit0, digit1, digit2, missing mask; rows_per_marker
// kWideRows), c_pad a multiple of kTileCWide. Three accumulators per tile.
constexpr int kTileCWide = 160;
constexpr int kWideRows = 4;
// BGEN-8 dosages (|u| <= 510) need two base-255 digits: 3 rows per marker (2 digits + missing),
// 144-row pair tiles (48 markers; 3 x 144 = 432 TMEM columns)
constexpr int kTileCWide3 = 144;
constexpr int kWideRows3 = 3;
// two-limb BGEN-8 tiles (THRESHOLD / TOPK, q0 limb deferred): two accumulators, 240 rows
constexpr int kTileCWide3Two = 240;
int launch_assoc_wide(const int8_t* qh, const int8_t* q1, const int8_t* q0, int64_t p_pad, const int8_t* v,
                      int64_t c_pad, int64_t k_pad, const AssocEpilogue& ep, cudaStream_t stream);
// BGEN-8 transposed variant: v in the quartered layout (geno_planes(quartered)), c_pad a
// multiple of 256 rows (80 markers per 256 rows); no K slicing, no max |r| tracking.
int launch_assoc_wide3t(const int8_t* qh, const int8_t* q1, const int8_t* q0, int64_t p_pad, const int8_t* v,
                        int64_t c_pad, int64_t k_pad, const AssocEpilogue& ep, cudaStream_t stream);

}  // namespace pg

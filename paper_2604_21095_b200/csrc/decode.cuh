// Genotype decode (K1): raw genotype blocks -> ternary GEMM rows + per-marker
// integer statistics. See decode.cu.
#pragma once
#include <cstdint>

#include "pg_common.cuh"

namespace pg {

// A block of markers resident on the device.
struct GenoBlock {
  int kind = PG_GENO_BED;     // PG_GENO_*
  const uint8_t* data = nullptr;
  int64_t pitch = 0;          // bytes between marker rows (multiple of 16)
  int64_t n_markers = 0;
  int64_t n_src = 0;          // samples per row in the source
  int64_t n_kept = 0;         // N used by the statistics
  const uint32_t* keep_bits = nullptr;  // [ceil(n_src/32)] bit i = sample i kept
  int dense_real = 0;         // DENSE only: 1 -> fixed-point (2^-17) digits, 0 -> integral dosages
  int all_kept = 0;           // every source sample is kept (keep_bits needed only past n_src)
  // BGEN rows: byte offsets of the probability pairs and of the ploidy bytes within a row
  // (default: probabilities first, ploidy right after; the GPU-inflated layout of a BGEN-8
  // block is used in place with probs at 10 + n, ploidy at 8)
  int64_t probs_off = 0;
  int64_t ploidy_off = -1;
};

// u-units: the integer code each observed sample contributes to the GEMM.
//   BED / integral dense : u = dosage - 1            (scale 1)
//   BGEN (bits b)        : u = k - (2^b - 1), dosage = k / (2^b - 1)
//   real dense           : u = rint((dosage - 1) * 2^17)
double geno_unit_scale(const GenoBlock& b);
// Rows per marker in the GEMM (ternary digits of u, plus a missing-mask row if any).
int geno_rows_per_marker(const GenoBlock& b, bool any_missing, bool allow_wide = true);
// Dosage sources with wide digits (BGEN, real-valued dense): rows_per_marker 4, launch_assoc_wide.
bool geno_wide(const GenoBlock& b);

struct MarkerStats {
  long long* n_miss = nullptr;  // [m] missing calls among kept samples
  long long* s_u = nullptr;     // [m] sum of u over observed kept samples
  long long* ss_u = nullptr;    // [m] sum of u^2
  double* sum_d = nullptr;      // [m] sum of dosages (real dense only)
  double* af = nullptr;         // [m] allele frequency (NaN all-missing)
  double* var = nullptr;        // [m] variance before scaling (1/N convention)
  int8_t* skip = nullptr;       // [m] SkipReason
  double* mu_d = nullptr;       // [m_pad] mean of u (GEMM epilogue)
  float* mu_f = nullptr;
  double* invd_d = nullptr;     // [m_pad] 1/sqrt(N V_u); NaN skipped / padding
  float* invd_f = nullptr;
  int* flags = nullptr;         // [2]: [0] any missing, [1] any non-integral dosage (dense)
};

// Pass 1 (dense only): flags[1] |= any non-integral kept dosage.
int geno_check_integral(const GenoBlock& b, MarkerStats& st, cudaStream_t s);
// Pass 2: integer statistics and derived per-marker quantities (all m_pad entries written).
int geno_stats(const GenoBlock& b, MarkerStats& st, int64_t m_pad, cudaStream_t s);
// Pass 3: GEMM operand planes [c_pad, k_pad] with R rows per marker: ternary digits v / 127v
// (R = 1, 2, 8, 16), or for R = 4 (wide mode, geno_wide) base-255 digits in v only.
// quartered (R = 3): rows of marker m at (m / 10) * 32 + 3 (m % 10) + d, rows 30-31 of every
// 32-row group zero (the transposed wide GEMM, launch_assoc_wide3t).
int geno_planes(const GenoBlock& b, int rows_per_marker, int8_t* v, int8_t* v127, int64_t c_pad, int64_t k_pad,
                cudaStream_t s, bool quartered = false);
// Missing-call side path of the fused PLINK GEMM (markers with missing calls carry a mask
// row in a separate GEMM; the rest of the batch keeps one row per marker):
// flag[m] = scanned marker m has a kept missing call; after an exclusive prefix sum of the
// flags: slot[m] = its index among those markers (-1 if none), list[slot] = m, *d_count.
int missing_flags(const long long* n_miss, const int8_t* skip, int64_t m, int* flag, cudaStream_t s);
int missing_slot_map(const int* flag, const int* prefix, int64_t m, int* slot, int* list, int* d_count,
                     cudaStream_t s);
// Mask rows (kept missing calls; v = mask, v127 = 127 mask) of markers list[0..n_list) as
// rows 0..n_list of [c_pad, k_pad] planes (rows past n_list zero).
int missing_mask_planes(const GenoBlock& b, const int* list, int64_t n_list, int8_t* v, int8_t* v127, int64_t c_pad,
                        int64_t k_pad, cudaStream_t s);
// Dosage decode for the reader API: out[m, n_src] f32/f64 with NaN missing, missing counts.
int geno_dosages(const GenoBlock& b, int elem_bytes, void* out, int64_t* missing, cudaStream_t s);

}  // namespace pg

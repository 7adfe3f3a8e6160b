// Device-resident quantized panel (see panel.cu).
#pragma once
#include <cstdint>

#include "pg_common.cuh"

namespace pg {

struct PanelPlanes {
  int8_t* qh = nullptr;  // [p_pad, k_pad]
  int8_t* q1 = nullptr;
  int8_t* q0 = nullptr;
  double* scale_d = nullptr;  // [p_pad] quantization step s_p
  float* scale_f = nullptr;
  long long* cq = nullptr;  // [p_pad] sum_k q[p,k]
  float* cq_f = nullptr;
  // Two-level panel (F64 precision mode; null = off): the residual y~/s - q quantized again,
  // q2 = rint((y~/s - q) * kLoScale), |q2| <= kLoScale / 2, in three more limbs, so that
  // y~ = s (q + q2 / kLoScale) to ~1e-14 of max |y~| (the GEMM runs once per level).
  int8_t* qh_lo = nullptr;
  int8_t* q1_lo = nullptr;
  int8_t* q0_lo = nullptr;
  long long* cq_lo = nullptr;  // [p_pad] sum_k q2[p,k]
};

// Quantize y (device f64, n_rows kept samples x n_cols phenotypes, row pitch `ld`
// elements) into `out`. Sample row i goes to K column d_gidx[i]; output phenotype c
// reads source column d_cols[c] (identity when d_cols is null).
int panel_quantize(const double* d_y, int64_t n_rows, int64_t n_cols, int64_t ld, const int64_t* d_cols,
                   const int64_t* d_gidx, int64_t k_pad, int64_t p_pad, PanelPlanes& out, double* d_maxabs_scratch,
                   cudaStream_t st);

// Scratch for panel_prepare: see panel_prep_scratch_doubles().
struct PanelPrepOut {
  double* mean = nullptr;    // [n_cols] column means of the raw panel
  double* centre = nullptr;  // [n_cols] column means after residualization
  double* sd = nullptr;      // [n_cols]
  uint8_t* flat = nullptr;   // [n_cols] zero-variance flags
  int* bad = nullptr;        // [1] non-finite input seen
};
int64_t panel_prep_scratch_doubles(int64_t n_rows, int64_t n_cols, int64_t rank);
// In place on d_y [n_rows, n_cols] (row pitch n_cols): centre, subtract the projection
// on the orthonormal basis d_q [n_rows, rank] (row-major), then standardize to unit
// 1/N variance (zero-variance columns -> 0). Deterministic (fixed reduction order).
int panel_prepare(double* d_y, int64_t n_rows, int64_t n_cols, const double* d_q, int64_t rank, double* d_scratch,
                  PanelPrepOut& out, cudaStream_t st);

}  // namespace pg

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
};

// Quantize y (device f64, n_rows kept samples x n_cols phenotypes, row pitch `ld`
// elements) into `out`. Sample row i goes to K column d_gidx[i].
int panel_quantize(const double* d_y, int64_t n_rows, int64_t n_cols, int64_t ld, const int64_t* d_gidx,
                   int64_t k_pad, int64_t p_pad, PanelPlanes& out, double* d_maxabs_scratch, cudaStream_t st);

}  // namespace pg

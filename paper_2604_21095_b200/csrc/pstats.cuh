// Student-t statistics on the device (K4): r -> t -> two-sided p in fp64.
#pragma once
#include <cstdint>

#include "pg_common.cuh"

namespace pg {

constexpr double kPFloor = 2.2250738585072014e-308;  // np.finfo(np.float64).tiny (kernel.py:29)
constexpr double kRCap = 1.0 - 1e-15;                // kernel.py:39

// Optional effect-size outputs of finalize_candidates (beta == nullptr: off):
// var_m[marker] = variance of the prepared dosage row (1/N), sd_p[phenotype] = sd of the
// residualized phenotype (1/N), both as the reference computes them (kernel.py:330-347, 376-421).
struct BetaArgs {
  const double* var_m = nullptr;
  const double* sd_p = nullptr;
  double* beta = nullptr;
  double* se = nullptr;
};

// Sorted candidates -> rows / cols / clipped r / t / p (+ beta, se); counts |r| > 1 into *clamp.
int finalize_candidates(const unsigned long long* key, const double* r_in, int64_t n, double df, int64_t* rows,
                        int64_t* cols, double* r_out, double* t_out, double* p_out, unsigned long long* clamp,
                        const BetaArgs& beta, cudaStream_t s);
// FULL mode: out[new_row(m), p] = beta(r[m, p]) for non-skipped markers (elem 4 or 8).
int full_rows_to_beta(const double* r, int64_t m, int64_t ld, int64_t n_pheno, const int64_t* new_row, double df,
                      int elem_bytes, void* out, const double* var_m, const double* sd_p, cudaStream_t s);
// FULL mode: out[new_row(m), p] = t(r[m, p]) for non-skipped markers (elem 4 or 8).
int full_rows_to_t(const double* r, int64_t m, int64_t ld, int64_t n_pheno, const int64_t* new_row, double df,
                   int elem_bytes, void* out, unsigned long long* clamp, cudaStream_t s);
int elementwise_t_from_r(const double* r, int64_t n, double df, double* t, cudaStream_t s);
int elementwise_p_from_t(const double* t, int64_t n, double df, double* p, unsigned long long* underflow,
                         cudaStream_t s);
int elementwise_reg_inc_beta(const double* a, const double* b, const double* x, int64_t n, double* out,
                             int* err_flag, cudaStream_t s);
int t_threshold(double p_threshold, double df, double* d_out, cudaStream_t s);
// One scalar through the reference's scalar forms: which 0 -> I_x(a, b), 1 -> p_from_t(t = a, df = b).
int scalar_stat(int which, double a, double b, double x, double* d_out, int* err_flag, cudaStream_t s);

}  // namespace pg

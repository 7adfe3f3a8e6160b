// K4: fp64 Student-t statistics on the device.
//
// Follows the reference numerics operation for operation so the results agree
// to the last few ulps (differences come only from lgamma / log / exp libm
// implementations):
//   t_from_r            kernel.py:460-478  (|r| capped at 1 - 1e-15, |r| >= 1 -> +-inf)
//   reg_inc_beta        kernel.py:147-189  (array form: flipped branch re-derives the
//                                           log prefactor from (b, a, 1 - x))
//   _betacf_array       kernel.py:86-119   (modified Lentz, eps 1e-15, tiny 1e-300,
//                                           at most 500 iterations)
//   p_from_t            kernel.py:192-209  (p = I_{df/(df+t^2)}(df/2, 1/2), floored)
//   t_threshold_for_p   kernel.py:212-235  (scalar p path, 200-step bisection)
#include <cub/cub.cuh>

#include <cmath>

#include "pstats.cuh"

namespace pg {
namespace {

constexpr double kCfEps = 1e-15;
constexpr double kCfTiny = 1e-300;
constexpr int kCfMaxIter = 500;

__device__ __forceinline__ double dnan() { return __longlong_as_double(0x7ff8000000000000ll); }

__device__ double betacf(double a, double b, double x, int* err) {
  const double qab = a + b;
  const double qap = a + 1.0;
  const double qam = a - 1.0;
  double c = 1.0;
  double d = 1.0 - qab * x / qap;
  if (fabs(d) < kCfTiny) d = kCfTiny;
  d = 1.0 / d;
  double h = d;
  for (int mi = 1; mi <= kCfMaxIter; ++mi) {
    const double m = static_cast<double>(mi);
    const double m2 = 2.0 * m;
    double aa = m * (b - m) * x / ((qam + m2) * (a + m2));
    d = 1.0 + aa * d;
    if (fabs(d) < kCfTiny) d = kCfTiny;
    c = 1.0 + aa / c;
    if (fabs(c) < kCfTiny) c = kCfTiny;
    d = 1.0 / d;
    const double step = d * c;
    aa = -(a + m) * (qab + m) * x / ((a + m2) * (qap + m2));
    d = 1.0 + aa * d;
    if (fabs(d) < kCfTiny) d = kCfTiny;
    c = 1.0 + aa / c;
    if (fabs(c) < kCfTiny) c = kCfTiny;
    d = 1.0 / d;
    const double delta = d * c;
    h = h * step * delta;
    if (!(fabs(delta - 1.0) >= kCfEps)) return h;
  }
  if (err) *err = 1;
  return dnan();
}

// Array-form I_x(a, b) (kernel.py:168-189).
__device__ double reg_inc_beta_arr(double a, double b, double x, int* err) {
  if (x <= 0.0) return 0.0;
  if (x >= 1.0) return 1.0;
  if (x < (a + 1.0) / (a + b + 2.0)) {
    const double lf = lgamma(a + b) - lgamma(a) - lgamma(b) + a * log(x) + b * log1p(-x);
    return exp(lf) * betacf(a, b, x, err) / a;
  }
  const double xx = 1.0 - x;
  const double lf = lgamma(b + a) - lgamma(b) - lgamma(a) + b * log(xx) + a * log1p(-xx);
  return 1.0 - exp(lf) * betacf(b, a, xx, err) / b;
}

// Scalar-form I_x(a, b) (kernel.py:136-144), used by the threshold bisection.
__device__ double reg_inc_beta_scalar(double a, double b, double x, int* err) {
  if (x <= 0.0) return 0.0;
  if (x >= 1.0) return 1.0;
  const double lf = lgamma(a + b) - lgamma(a) - lgamma(b) + a * log(x) + b * log1p(-x);
  if (x < (a + 1.0) / (a + b + 2.0)) return exp(lf) * betacf(a, b, x, err) / a;
  return 1.0 - exp(lf) * betacf(b, a, 1.0 - x, err) / b;
}

__device__ __forceinline__ double p_from_t_arr(double t, double df, int* err) {
  const double x = df / (df + t * t);
  const double p = reg_inc_beta_arr(df / 2.0, 0.5, x, err);
  return p > kPFloor ? p : (p != p ? p : kPFloor);
}

__device__ __forceinline__ double p_from_t_scalar(double t, double df, int* err) {
  const double x = df / (df + t * t);
  const double p = reg_inc_beta_scalar(df / 2.0, 0.5, x, err);
  return fmax(p, kPFloor);
}

__device__ __forceinline__ double sign_of(double r) { return r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : (r == r ? 0.0 : r)); }

__device__ __forceinline__ double t_from_r_dev(double r, double df) {
  const double a0 = fabs(r);
  const double sg = sign_of(r);
  if (a0 >= 1.0) return sg * __longlong_as_double(0x7ff0000000000000ll);
  const double a = fmin(a0, kRCap);
  return sg * a * sqrt(df / (1.0 - a * a));
}

// Effect size on the phenotype's scale (north star: beta / t / -log10 p). With r the
// correlation of the (imputed, centred[, projected]) dosage g with the residualized
// phenotype y_res, the slope of y_res on g is beta = r * sd(y_res) / sd(g) and its standard
// error se = sd(y_res) / sd(g) * sqrt((1 - r^2) / df), so beta / se == t exactly as
// t_from_r defines it. Extension mode + adjusted df: the Frisch-Waugh-Lovell identity makes
// these the full OLS estimates of y ~ 1 + C + g (oracle.ols_single, oracle.py:35-90).
__device__ __forceinline__ void beta_se(double r, double t, double var_m, double sd_p, double df, double& b,
                                        double& se) {
  const double ratio = sd_p / sqrt(var_m);
  b = r * ratio;
  const double a = fmin(fabs(r), kRCap);
  se = isinf(t) ? 0.0 : ratio * sqrt((1.0 - a * a) / df);
}

__global__ void finalize_kernel(const unsigned long long* __restrict__ key, const double* __restrict__ r_in,
                                int64_t n, double df, int64_t* rows, int64_t* cols, double* r_out, double* t_out,
                                double* p_out, unsigned long long* clamp, BetaArgs beta) {
  unsigned long long nclamp = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double r = r_in[i];
    if (fabs(r) > 1.0) {
      ++nclamp;
      r = r > 0.0 ? 1.0 : -1.0;
    }
    const double t = t_from_r_dev(r, df);
    rows[i] = static_cast<int64_t>(key[i] >> 32);
    cols[i] = static_cast<int64_t>(key[i] & 0xffffffffull);
    r_out[i] = r;
    t_out[i] = t;
    p_out[i] = p_from_t_arr(t, df, nullptr);
    if (beta.beta) {
      double b, se;
      beta_se(r, t, beta.var_m[rows[i]], beta.sd_p[cols[i]], df, b, se);
      beta.beta[i] = b;
      beta.se[i] = se;
    }
  }
  if (nclamp) atomicAdd(clamp, nclamp);
}

__global__ void full_t_kernel(const double* __restrict__ r, int64_t m, int64_t ld, int64_t n_pheno,
                              const int64_t* __restrict__ new_row, double df, int elem_bytes, void* out,
                              unsigned long long* clamp) {
  const int64_t row = blockIdx.x;
  const int64_t dst = new_row[row];
  if (dst < 0) return;
  unsigned long long nclamp = 0;
  for (int64_t p = threadIdx.x; p < n_pheno; p += blockDim.x) {
    double v = r[row * ld + p];
    if (fabs(v) > 1.0) {
      ++nclamp;
      v = v > 0.0 ? 1.0 : -1.0;
    }
    const double t = t_from_r_dev(v, df);
    if (elem_bytes == 4)
      reinterpret_cast<float*>(out)[dst * n_pheno + p] = static_cast<float>(t);
    else
      reinterpret_cast<double*>(out)[dst * n_pheno + p] = t;
  }
  if (nclamp) atomicAdd(clamp, nclamp);
}

// FULL mode beta rows: out[new_row(m), p] = beta(r[m, p]) for non-skipped markers
__global__ void full_beta_kernel(const double* __restrict__ r, int64_t m, int64_t ld, int64_t n_pheno,
                                 const int64_t* __restrict__ new_row, double df, int elem_bytes, void* out,
                                 const double* __restrict__ var_m, const double* __restrict__ sd_p) {
  const int64_t row = blockIdx.x;
  const int64_t dst = new_row[row];
  if (dst < 0) return;
  const double vm = var_m[row];
  for (int64_t p = threadIdx.x; p < n_pheno; p += blockDim.x) {
    double v = r[row * ld + p];
    if (fabs(v) > 1.0) v = v > 0.0 ? 1.0 : -1.0;
    double b, se;
    beta_se(v, t_from_r_dev(v, df), vm, sd_p[p], df, b, se);
    if (elem_bytes == 4)
      reinterpret_cast<float*>(out)[dst * n_pheno + p] = static_cast<float>(b);
    else
      reinterpret_cast<double*>(out)[dst * n_pheno + p] = b;
  }
}

__global__ void t_from_r_kernel(const double* r, int64_t n, double df, double* t) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    t[i] = t_from_r_dev(r[i], df);
}

__global__ void p_from_t_kernel(const double* t, int64_t n, double df, double* p, unsigned long long* underflow) {
  unsigned long long u = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = p_from_t_arr(t[i], df, nullptr);
    p[i] = v;
    u += (v <= kPFloor) ? 1ull : 0ull;
  }
  if (u && underflow) atomicAdd(underflow, u);
}

__global__ void reg_inc_beta_kernel(const double* a, const double* b, const double* x, int64_t n, double* out,
                                    int* err) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = reg_inc_beta_arr(a[i], b[i], x[i], err);
}

// Scalar inputs take the reference's scalar path (kernel.py:136-144, :201-204):
// which 0 -> I_x(a, b) (a, b, x); which 1 -> p_from_t (t = a, df = b).
__global__ void scalar_stat_kernel(int which, double a, double b, double x, double* out, int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  *out = which == 0 ? reg_inc_beta_scalar(a, b, x, err) : p_from_t_scalar(a, b, err);
}

__global__ void t_threshold_kernel(double p_thr, double df, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  if (p_thr >= 1.0) {
    *out = 0.0;
    return;
  }
  if (p_thr < kPFloor) {
    *out = inf;
    return;
  }
  double lo = 0.0, hi = 1.0;
  while (p_from_t_scalar(hi, df, nullptr) > p_thr) {
    hi *= 2.0;
    if (hi > 1e300) {
      *out = inf;
      return;
    }
  }
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (p_from_t_scalar(mid, df, nullptr) > p_thr)
      lo = mid;
    else
      hi = mid;
  }
  *out = hi;
}

unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

}  // namespace

int finalize_candidates(const unsigned long long* key, const double* r_in, int64_t n, double df, int64_t* rows,
                        int64_t* cols, double* r_out, double* t_out, double* p_out, unsigned long long* clamp,
                        const BetaArgs& beta, cudaStream_t s) {
  if (n <= 0) return PG_OK;
  finalize_kernel<<<grid_for(n, 256), 256, 0, s>>>(key, r_in, n, df, rows, cols, r_out, t_out, p_out, clamp,
                                                   beta);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int full_rows_to_t(const double* r, int64_t m, int64_t ld, int64_t n_pheno, const int64_t* new_row, double df,
                   int elem_bytes, void* out, unsigned long long* clamp, cudaStream_t s) {
  if (m <= 0) return PG_OK;
  full_t_kernel<<<static_cast<unsigned>(m), 256, 0, s>>>(r, m, ld, n_pheno, new_row, df, elem_bytes, out, clamp);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int full_rows_to_beta(const double* r, int64_t m, int64_t ld, int64_t n_pheno, const int64_t* new_row, double df,
                      int elem_bytes, void* out, const double* var_m, const double* sd_p, cudaStream_t s) {
  if (m <= 0) return PG_OK;
  full_beta_kernel<<<static_cast<unsigned>(m), 256, 0, s>>>(r, m, ld, n_pheno, new_row, df, elem_bytes, out, var_m,
                                                            sd_p);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int elementwise_t_from_r(const double* r, int64_t n, double df, double* t, cudaStream_t s) {
  if (n <= 0) return PG_OK;
  t_from_r_kernel<<<grid_for(n, 256), 256, 0, s>>>(r, n, df, t);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int elementwise_p_from_t(const double* t, int64_t n, double df, double* p, unsigned long long* underflow,
                         cudaStream_t s) {
  if (n <= 0) return PG_OK;
  p_from_t_kernel<<<grid_for(n, 128), 128, 0, s>>>(t, n, df, p, underflow);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int elementwise_reg_inc_beta(const double* a, const double* b, const double* x, int64_t n, double* out,
                             int* err_flag, cudaStream_t s) {
  if (n <= 0) return PG_OK;
  reg_inc_beta_kernel<<<grid_for(n, 128), 128, 0, s>>>(a, b, x, n, out, err_flag);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int scalar_stat(int which, double a, double b, double x, double* d_out, int* err_flag, cudaStream_t s) {
  scalar_stat_kernel<<<1, 32, 0, s>>>(which, a, b, x, d_out, err_flag);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int t_threshold(double p_threshold, double df, double* d_out, cudaStream_t s) {
  t_threshold_kernel<<<1, 32, 0, s>>>(p_threshold, df, d_out);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

}  // namespace pg

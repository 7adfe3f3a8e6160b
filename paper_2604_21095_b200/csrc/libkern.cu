// Library-level kernels behind the public kernel.py API (not the scan hot path,
// which fuses these steps): fp64 prepare_genotype_batch and correlate.
//
//   prepare_genotype_batch  /root/reference/pkg/src/panelgwas/kernel.py:376-421
//   correlate               kernel.py:428-457
//
// Both run in float64 with a fixed reduction order per output element, so a
// row's results do not depend on which rows share its launch
// (reference test: tests/test_kernel.py:244-257).
#include <cmath>

#include "pg_common.cuh"

struct pg_ctx;

namespace pg {
namespace {

constexpr int kPrepThreads = 256;
constexpr int kMaxRank = 256;

__device__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < kPrepThreads / 32; ++w) t += sh[w];
    sh[32] = t;
  }
  __syncthreads();
  t = sh[32];
  __syncthreads();
  return t;
}

// One block per marker row; `work` holds the row in f64 while it is transformed.
__global__ void __launch_bounds__(kPrepThreads) prepare_kernel(const double* __restrict__ in, int64_t n,
                                                               const double* __restrict__ q, int64_t rank,
                                                               double* __restrict__ work, int elem_bytes, void* out,
                                                               double* af, int64_t* miss_out, double* var_out,
                                                               int8_t* skip_out) {
  __shared__ double sh[33];
  const int64_t m = blockIdx.x;
  const double* row = in + m * n;
  double* w = work + m * n;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  double s = 0.0, cnt = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    const double x = row[k];
    if (isnan(x)) {
      cnt += 1.0;
    } else {
      s += x;
    }
  }
  const double n_miss = block_sum(cnt, sh);
  const double sum = block_sum(s, sh);
  const double n_obs = static_cast<double>(n) - n_miss;
  const bool all_missing = n_obs == 0.0;
  const double mean = all_missing ? 0.0 : sum / n_obs;
  // impute, then centre on the imputed row mean
  double s2 = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    const double x = row[k];
    const double v = isnan(x) ? mean : x;
    w[k] = v;
    s2 += v;
  }
  const double rowmean = block_sum(s2, sh) / static_cast<double>(n);
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) w[k] -= rowmean;
  __syncthreads();
  if (q != nullptr && rank > 0) {
    // d -= (d @ Q) @ Q^T: all coefficients from the centred row first, then one subtraction
    __shared__ double coef[kMaxRank];
    for (int64_t jcol = 0; jcol < rank; ++jcol) {
      double part = 0.0;
      for (int64_t k = threadIdx.x; k < n; k += blockDim.x) part += w[k] * q[k * rank + jcol];
      const double c = block_sum(part, sh);
      if (threadIdx.x == 0) coef[jcol] = c;
    }
    __syncthreads();
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
      double acc = 0.0;
      for (int64_t jcol = 0; jcol < rank; ++jcol) acc += q[k * rank + jcol] * coef[jcol];
      w[k] -= acc;
    }
    __syncthreads();
  }
  double sq = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) sq += w[k] * w[k];
  const double var = block_sum(sq, sh) / static_cast<double>(n);
  int8_t skip = 0;
  if (var <= 1e-12) skip = 1;
  if (all_missing) skip = 2;
  const double scale = skip == 0 ? sqrt(var) : 1.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    const double v = skip == 0 ? w[k] / scale : 0.0;
    if (elem_bytes == 4)
      reinterpret_cast<float*>(out)[m * n + k] = static_cast<float>(v);
    else
      reinterpret_cast<double*>(out)[m * n + k] = v;
  }
  if (threadIdx.x == 0) {
    af[m] = all_missing ? nan : mean / 2.0;
    miss_out[m] = static_cast<int64_t>(n_miss);
    var_out[m] = var;
    skip_out[m] = skip;
  }
}

// fp64 SIMT GEMM, 64x64 output tile, 16-deep K slices, 4x4 outputs per thread.
__global__ void __launch_bounds__(256) correlate_kernel(const double* __restrict__ g, int64_t m, int64_t n,
                                                        const double* __restrict__ y, int64_t p,
                                                        double* __restrict__ r, unsigned long long* clamp) {
  __shared__ double sg[16][64 + 1];
  __shared__ double sy[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t row0 = static_cast<int64_t>(blockIdx.y) * 64, col0 = static_cast<int64_t>(blockIdx.x) * 64;
  double acc[4][4] = {};
  for (int64_t k0 = 0; k0 < n; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int kk = i & 15, rr = i >> 4;
      const int64_t gr = row0 + rr, gk = k0 + kk;
      sg[kk][rr] = (gr < m && gk < n) ? g[gr * n + gk] : 0.0;
      const int cc = i & 63, kk2 = i >> 6;
      const int64_t yc = col0 + cc, yk = k0 + kk2;
      sy[kk2][cc] = (yc < p && yk < n) ? y[yk * p + yc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sg[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sy[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  unsigned long long nc = 0;
  const double fn = static_cast<double>(n);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t rr = row0 + ty * 4 + i, cc = col0 + tx * 4 + j;
      if (rr < m && cc < p) {
        double v = acc[i][j] / fn;
        if (fabs(v) > 1.0) {
          ++nc;
          v = v > 0.0 ? 1.0 : -1.0;
        }
        r[rr * p + cc] = v;
      }
    }
  }
  if (nc) atomicAdd(clamp, nc);
}

}  // namespace
}  // namespace pg

extern "C" {

int pg_prepare_batch(pg_ctx* ctx, const double* dosages, int64_t n_markers, int64_t n_samples, const double* q,
                     int64_t rank, int elem_bytes, void* out, double* af, int64_t* missing_count, double* variance,
                     int8_t* skip) {
  using namespace pg;
  (void)ctx;
  PG_REQUIRE(elem_bytes == 4 || elem_bytes == 8, PG_ERR_INVALID, "elem_bytes must be 4 or 8");
  PG_REQUIRE(n_samples >= 1, PG_ERR_INVALID, "prepare: empty rows");
  PG_REQUIRE(rank <= kMaxRank, PG_ERR_INVALID, "prepare: covariate basis rank %lld > %d", (long long)rank, kMaxRank);
  if (n_markers <= 0) return PG_OK;
  cudaStream_t s = nullptr;
  PG_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t nm = static_cast<size_t>(n_markers) * n_samples;
  double *d_in = nullptr, *d_work = nullptr, *d_q = nullptr, *d_af = nullptr, *d_var = nullptr;
  int64_t* d_miss = nullptr;
  int8_t* d_skip = nullptr;
  void* d_out = nullptr;
  int rc = PG_OK;
  auto cleanup = [&]() {
    for (void* p : {(void*)d_in, (void*)d_work, (void*)d_q, (void*)d_af, (void*)d_var, (void*)d_miss,
                    (void*)d_skip, d_out})
      if (p) cudaFree(p);
    cudaStreamDestroy(s);
  };
  do {
    if (cudaMalloc(&d_in, nm * 8) != cudaSuccess || cudaMalloc(&d_work, nm * 8) != cudaSuccess ||
        cudaMalloc(&d_out, nm * elem_bytes) != cudaSuccess || cudaMalloc(&d_af, 8 * n_markers) != cudaSuccess ||
        cudaMalloc(&d_var, 8 * n_markers) != cudaSuccess || cudaMalloc(&d_miss, 8 * n_markers) != cudaSuccess ||
        cudaMalloc(&d_skip, n_markers) != cudaSuccess) {
      cudaGetLastError();
      set_error("prepare: device allocation failed");
      rc = PG_ERR_NOMEM;
      break;
    }
    if (q != nullptr && rank > 0) {
      if (cudaMalloc(&d_q, 8 * n_samples * rank) != cudaSuccess) {
        rc = PG_ERR_NOMEM;
        break;
      }
      cudaMemcpyAsync(d_q, q, 8 * n_samples * rank, cudaMemcpyHostToDevice, s);
    }
    cudaMemcpyAsync(d_in, dosages, nm * 8, cudaMemcpyHostToDevice, s);
    prepare_kernel<<<static_cast<unsigned>(n_markers), kPrepThreads, 0, s>>>(
        d_in, n_samples, d_q, d_q ? rank : 0, d_work, elem_bytes, d_out, d_af, d_miss, d_var, d_skip);
    cudaMemcpyAsync(out, d_out, nm * elem_bytes, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(af, d_af, 8 * n_markers, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(missing_count, d_miss, 8 * n_markers, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(variance, d_var, 8 * n_markers, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(skip, d_skip, n_markers, cudaMemcpyDeviceToHost, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      set_error("prepare kernel failed: %s", cudaGetErrorString(e));
      rc = PG_ERR_CUDA;
    }
  } while (0);
  cleanup();
  return rc;
}

int pg_correlate_f64(pg_ctx* ctx, const double* gt, int64_t m, int64_t n, const double* yt, int64_t p, double* r,
                     int64_t* clamp_count) {
  using namespace pg;
  (void)ctx;
  PG_REQUIRE(m >= 0 && n >= 1 && p >= 0, PG_ERR_INVALID, "correlate: bad shape");
  if (clamp_count) *clamp_count = 0;
  if (m == 0 || p == 0) return PG_OK;
  cudaStream_t s = nullptr;
  PG_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double *d_g = nullptr, *d_y = nullptr, *d_r = nullptr;
  unsigned long long* d_c = nullptr;
  int rc = PG_OK;
  if (cudaMalloc(&d_g, 8 * m * n) != cudaSuccess || cudaMalloc(&d_y, 8 * n * p) != cudaSuccess ||
      cudaMalloc(&d_r, 8 * m * p) != cudaSuccess || cudaMalloc(&d_c, 8) != cudaSuccess) {
    cudaGetLastError();
    set_error("correlate: device allocation failed");
    rc = PG_ERR_NOMEM;
  } else {
    cudaMemcpyAsync(d_g, gt, 8 * m * n, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_y, yt, 8 * n * p, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(d_c, 0, 8, s);
    dim3 grid(static_cast<unsigned>((p + 63) / 64), static_cast<unsigned>((m + 63) / 64));
    correlate_kernel<<<grid, 256, 0, s>>>(d_g, m, n, d_y, p, d_r, d_c);
    unsigned long long hc = 0;
    cudaMemcpyAsync(r, d_r, 8 * m * p, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&hc, d_c, 8, cudaMemcpyDeviceToHost, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      set_error("correlate kernel failed: %s", cudaGetErrorString(e));
      rc = PG_ERR_CUDA;
    }
    if (clamp_count) *clamp_count = static_cast<int64_t>(hc);
  }
  for (void* ptr : {(void*)d_g, (void*)d_y, (void*)d_r, (void*)d_c})
    if (ptr) cudaFree(ptr);
  cudaStreamDestroy(s);
  return rc;
}

}  // extern "C"

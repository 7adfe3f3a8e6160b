// Panel preparation on the device: the standardized phenotype matrix
// Y~ (kernel.standardize_columns output, /root/reference/pkg/src/panelgwas/kernel.py:330-347)
// is quantized once per phenotype column and split into the three int8 limbs
// the association GEMM consumes (assoc.cuh). The quantized panel stays
// resident in HBM for the whole scan (reference: engine._Prepared.ytil,
// engine.py:154-167, shared read-only by every batch).
//
// Layout: limb planes are phenotype-major [p_pad, k_pad] int8 (K-major for
// TMA / UMMA), where k is the GENOTYPE-FILE sample index: kept sample i lands
// on column geno_row_index[i]; excluded samples and padding columns are 0, so
// the GEMM runs over all source samples without a gather
// (reference gathers instead: engine.py:348-352, 388-392).
#include <cmath>

#include "assoc.cuh"
#include "panel.cuh"

namespace pg {
namespace {

__global__ void maxabs_kernel(const double* __restrict__ y, int64_t n_rows, int64_t n_cols, int64_t ld,
                              const int64_t* __restrict__ cols, double* __restrict__ maxabs) {
  // blockDim (32, 8): 32 consecutive columns x 8 row-strands
  __shared__ double red[8][33];
  const int64_t col = blockIdx.x * 32 + threadIdx.x;
  double m = 0.0;
  if (col < n_cols) {
    const int64_t src = cols ? cols[col] : col;
    for (int64_t r = blockIdx.y * 8 + threadIdx.y; r < n_rows; r += gridDim.y * 8) {
      m = fmax(m, fabs(y[r * ld + src]));
    }
  }
  red[threadIdx.y][threadIdx.x] = m;
  __syncthreads();
  if (threadIdx.y == 0 && col < n_cols) {
    for (int i = 1; i < 8; ++i) m = fmax(m, red[i][threadIdx.x]);
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(maxabs + col), __double_as_longlong(m));
  }
}

__global__ void scale_kernel(const double* __restrict__ maxabs, int64_t n_cols, int64_t p_pad, double* scale_d,
                             float* scale_f) {
  const int64_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= p_pad) return;
  double s = 1.0;
  if (p < n_cols && maxabs[p] > 0.0) s = maxabs[p] / static_cast<double>(kQMax);
  scale_d[p] = s;
  scale_f[p] = static_cast<float>(s);
}

__device__ __forceinline__ long long floor_div(long long a, long long b) {
  long long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

// 32x32 transpose tiles: read y[i, p] coalesced along p, write limb[p][g_idx[i]].
__global__ void quantize_kernel(const double* __restrict__ y, int64_t n_rows, int64_t n_cols, int64_t ld,
                                const int64_t* __restrict__ cols, const int64_t* __restrict__ g_idx, const double* __restrict__ scale_d,
                                int64_t k_pad, int8_t* __restrict__ qh, int8_t* __restrict__ q1,
                                int8_t* __restrict__ q0, unsigned long long* __restrict__ cq, int8_t* __restrict__ qh2,
                                int8_t* __restrict__ q12, int8_t* __restrict__ q02, unsigned long long* __restrict__ cq2) {
  __shared__ int tile_h[32][33], tile_1[32][33], tile_0[32][33];
  __shared__ int tile_h2[32][33], tile_12[32][33], tile_02[32][33];
  __shared__ long long csum[32][33], csum2[32][33];
  const int64_t row0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int64_t col0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // blockDim (32, 8)
  for (int yy = ty; yy < 32; yy += 8) {
    const int64_t r = row0 + yy, c = col0 + tx;
    long long q = 0, q2 = 0;
    if (r < n_rows && c < n_cols) {
      const double v = y[r * ld + (cols ? cols[c] : c)] / scale_d[c];
      q = llrint(v);
      if (q > kQMax) q = kQMax;
      if (q < -kQMax) q = -kQMax;
      q2 = llrint((v - static_cast<double>(q)) * kLoScale);  // v - q is exact (|v - q| <= 1/2)
    }
    auto split = [](long long x, int& h, int& a, int& b) {
      const long long xH = floor_div(x + 16192, kWH);
      const long long xL = x - xH * kWH;  // [-16192, 16192]
      const long long d1 = floor_div(xL + 63, 127);
      h = static_cast<int>(xH);
      a = static_cast<int>(d1);
      b = static_cast<int>(xL - d1 * 127);  // [-63, 63]
    };
    split(q, tile_h[yy][tx], tile_1[yy][tx], tile_0[yy][tx]);
    csum[yy][tx] = q;
    if (qh2) {
      split(q2, tile_h2[yy][tx], tile_12[yy][tx], tile_02[yy][tx]);
      csum2[yy][tx] = q2;
    }
  }
  __syncthreads();
  // column sums of q (exact integers; order-independent)
  if (ty == 0) {
    long long s = 0;
    for (int i = 0; i < 32; ++i) s += csum[i][tx];
    if (col0 + tx < n_cols) atomicAdd(cq + col0 + tx, static_cast<unsigned long long>(s));
    if (qh2) {
      long long s2 = 0;
      for (int i = 0; i < 32; ++i) s2 += csum2[i][tx];
      if (col0 + tx < n_cols) atomicAdd(cq2 + col0 + tx, static_cast<unsigned long long>(s2));
    }
  }
  // transposed write: thread (tx, ty) writes phenotype col0+yy, sample row0+tx
  for (int yy = ty; yy < 32; yy += 8) {
    const int64_t c = col0 + yy, r = row0 + tx;
    if (c < n_cols && r < n_rows) {
      const int64_t k = g_idx[r];
      const int64_t o = c * k_pad + k;
      qh[o] = static_cast<int8_t>(tile_h[tx][yy]);
      q1[o] = static_cast<int8_t>(tile_1[tx][yy]);
      q0[o] = static_cast<int8_t>(tile_0[tx][yy]);
      if (qh2) {
        qh2[o] = static_cast<int8_t>(tile_h2[tx][yy]);
        q12[o] = static_cast<int8_t>(tile_12[tx][yy]);
        q02[o] = static_cast<int8_t>(tile_02[tx][yy]);
      }
    }
  }
}

__global__ void cq_float_kernel(const long long* __restrict__ cq, int64_t p_pad, float* __restrict__ cq_f) {
  const int64_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < p_pad) cq_f[p] = static_cast<float>(cq[p]);
}

}  // namespace

int panel_quantize(const double* d_y, int64_t n_rows, int64_t n_cols, int64_t ld, const int64_t* d_cols,
                   const int64_t* d_gidx, int64_t k_pad, int64_t p_pad, PanelPlanes& out, double* d_maxabs_scratch,
                   cudaStream_t st) {
  const size_t plane = static_cast<size_t>(p_pad) * k_pad;
  PG_CUDA_CHECK(cudaMemsetAsync(out.qh, 0, plane, st));
  PG_CUDA_CHECK(cudaMemsetAsync(out.q1, 0, plane, st));
  PG_CUDA_CHECK(cudaMemsetAsync(out.q0, 0, plane, st));
  PG_CUDA_CHECK(cudaMemsetAsync(out.cq, 0, sizeof(long long) * p_pad, st));
  if (out.qh_lo) {
    PG_CUDA_CHECK(cudaMemsetAsync(out.qh_lo, 0, plane, st));
    PG_CUDA_CHECK(cudaMemsetAsync(out.q1_lo, 0, plane, st));
    PG_CUDA_CHECK(cudaMemsetAsync(out.q0_lo, 0, plane, st));
    PG_CUDA_CHECK(cudaMemsetAsync(out.cq_lo, 0, sizeof(long long) * p_pad, st));
  }
  PG_CUDA_CHECK(cudaMemsetAsync(d_maxabs_scratch, 0, sizeof(double) * p_pad, st));
  {
    dim3 blk(32, 8);
    const int64_t gy = std::min<int64_t>((n_rows + 7) / 8, 256);
    dim3 grd(static_cast<unsigned>((n_cols + 31) / 32), static_cast<unsigned>(gy));
    maxabs_kernel<<<grd, blk, 0, st>>>(d_y, n_rows, n_cols, ld, d_cols, d_maxabs_scratch);
    PG_CUDA_CHECK(cudaGetLastError());
  }
  scale_kernel<<<static_cast<unsigned>((p_pad + 255) / 256), 256, 0, st>>>(d_maxabs_scratch, n_cols, p_pad,
                                                                             out.scale_d, out.scale_f);
  PG_CUDA_CHECK(cudaGetLastError());
  {
    dim3 blk(32, 8);
    dim3 grd(static_cast<unsigned>((n_cols + 31) / 32), static_cast<unsigned>((n_rows + 31) / 32));
    quantize_kernel<<<grd, blk, 0, st>>>(d_y, n_rows, n_cols, ld, d_cols, d_gidx, out.scale_d, k_pad, out.qh, out.q1, out.q0,
                                         reinterpret_cast<unsigned long long*>(out.cq), out.qh_lo, out.q1_lo,
                                         out.q0_lo, reinterpret_cast<unsigned long long*>(out.cq_lo));
    PG_CUDA_CHECK(cudaGetLastError());
  }
  cq_float_kernel<<<static_cast<unsigned>((p_pad + 255) / 256), 256, 0, st>>>(out.cq, p_pad, out.cq_f);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

}  // namespace pg

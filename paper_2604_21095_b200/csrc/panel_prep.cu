// Panel preparation on the device: the reference's
// residualize + standardize_columns
// (/root/reference/pkg/src/panelgwas/kernel.py:310-327, 330-347; driven from
// engine.py:259-279) on the kept-sample x phenotype matrix, in fp64, in place:
//
//   mean_p   = sum_n y[n,p] / N                        (kernel.py:324)
//   W[j,p]   = sum_n Q[n,j] (y[n,p] - mean_p)           (Q^T Yc, kernel.py:326)
//   res      = (y - mean) - Q W                         (kernel.py:326)
//   centre_p = sum_n res / N,  sd_p = sqrt(sum_n (res - centre)^2 / N)   (kernel.py:341-343)
//   flat_p   = sd_p <= 1e-12 max(1, |centre_p|)         (kernel.py:344)
//   y~       = flat ? 0 : (res - centre) / sd            (kernel.py:345-346)
//
// Every column reduction is two-level with a fixed order (row chunks -> partials ->
// one ordered sum per column), so the prepared panel is bitwise reproducible run to
// run. Values differ from numpy's BLAS/pairwise order only at the 1e-16 relative
// level, far below the 23-bit panel quantization that follows (panel.cu).
//
// Layout: y is [N, P] row-major (the reference's samples x phenotypes), so a warp
// reads 32 consecutive phenotypes of one sample row: fully coalesced, one pass over
// the 3.8 GB C3 panel per step (5 passes, HBM bound).
#include <cmath>

#include "panel.cuh"

namespace pg {
namespace {

constexpr int kChunkRows = 1024;  // rows per partial-sum chunk
constexpr int kJB = 16;           // basis columns per projection pass

int64_t n_chunks(int64_t n_rows) { return (n_rows + kChunkRows - 1) / kChunkRows; }

// blockDim (32, 8): 32 columns x 8 row strands over one row chunk (blockIdx.y).
// MODE 0: sum y (+ non-finite check); 1: sum (res - centre)^2.
template <int MODE>
__global__ void col_partial_kernel(const double* __restrict__ y, int64_t n_rows, int64_t n_cols,
                                   const double* __restrict__ centre, double* __restrict__ partial,
                                   int* __restrict__ bad) {
  __shared__ double red[8][33];
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kChunkRows;
  const int64_t r1 = min(r0 + kChunkRows, n_rows);
  double acc = 0.0;
  if (col < n_cols) {
    const double c = MODE == 1 ? centre[col] : 0.0;
    bool finite = true;
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      const double v = y[r * n_cols + col];
      if (MODE == 0) {
        finite &= isfinite(v);
        acc += v;
      } else {
        const double d = v - c;
        acc += d * d;
      }
    }
    if (MODE == 0 && !finite) atomicExch(bad, 1);
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && col < n_cols) {
    double s = red[0][threadIdx.x];
#pragma unroll
    for (int i = 1; i < 8; ++i) s += red[i][threadIdx.x];
    partial[static_cast<int64_t>(blockIdx.y) * n_cols + col] = s;
  }
}

// W-partials for basis columns [j0, j0 + jn): sum over the chunk of Q[r,j] (y[r,c] - mean_c).
__global__ void proj_partial_kernel(const double* __restrict__ y, int64_t n_rows, int64_t n_cols,
                                    const double* __restrict__ mean, const double* __restrict__ q, int64_t rank,
                                    int j0, int jn, double* __restrict__ partial) {
  __shared__ double red[8][kJB][33];
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kChunkRows;
  const int64_t r1 = min(r0 + kChunkRows, n_rows);
  double acc[kJB];
#pragma unroll
  for (int j = 0; j < kJB; ++j) acc[j] = 0.0;
  if (col < n_cols) {
    const double m = mean[col];
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      const double v = y[r * n_cols + col] - m;
      const double* qr = q + r * rank + j0;
#pragma unroll
      for (int j = 0; j < kJB; ++j)
        if (j < jn) acc[j] += __ldg(qr + j) * v;
    }
  }
#pragma unroll
  for (int j = 0; j < kJB; ++j) red[threadIdx.y][j][threadIdx.x] = acc[j];
  __syncthreads();
  if (col < n_cols) {
    for (int j = threadIdx.y; j < jn; j += 8) {
      double s = red[0][j][threadIdx.x];
#pragma unroll
      for (int i = 1; i < 8; ++i) s += red[i][j][threadIdx.x];
      partial[(static_cast<int64_t>(j) * gridDim.y + blockIdx.y) * n_cols + col] = s;
    }
  }
}

// out[c] = (sum over the n_part partials of column c, in chunk order) / div
// (numpy's mean is a true division of the sum, not a reciprocal product)
__global__ void col_finish_kernel(const double* __restrict__ partial, int64_t n_part, int64_t n_cols, double div,
                                  double* __restrict__ out) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  double s = 0.0;
  for (int64_t i = 0; i < n_part; ++i) s += partial[i * n_cols + c];
  out[c] = s / div;
}

// res = (y - mean) - sum_j Q[r,j] W[j,c], in place; partial column sums of res.
__global__ void residual_kernel(double* __restrict__ y, int64_t n_rows, int64_t n_cols,
                                const double* __restrict__ mean, const double* __restrict__ q, int64_t rank,
                                const double* __restrict__ w, double* __restrict__ partial) {
  __shared__ double red[8][33];
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kChunkRows;
  const int64_t r1 = min(r0 + kChunkRows, n_rows);
  double acc = 0.0;
  if (col < n_cols) {
    const double m = mean[col];
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      double proj = 0.0;
      for (int64_t j = 0; j < rank; ++j) proj += __ldg(q + r * rank + j) * w[j * n_cols + col];
      const double v = (y[r * n_cols + col] - m) - proj;
      y[r * n_cols + col] = v;
      acc += v;
    }
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && col < n_cols) {
    double s = red[0][threadIdx.x];
#pragma unroll
    for (int i = 1; i < 8; ++i) s += red[i][threadIdx.x];
    partial[static_cast<int64_t>(blockIdx.y) * n_cols + col] = s;
  }
}

__global__ void sd_kernel(const double* __restrict__ ss, const double* __restrict__ centre, int64_t n_cols,
                          double* __restrict__ sd, uint8_t* __restrict__ flat) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  const double s = sqrt(ss[c]);
  sd[c] = s;
  flat[c] = s <= 1e-12 * fmax(1.0, fabs(centre[c])) ? 1 : 0;
}

__global__ void scale_cols_kernel(double* __restrict__ y, int64_t n_rows, int64_t n_cols,
                                  const double* __restrict__ centre, const double* __restrict__ sd,
                                  const uint8_t* __restrict__ flat) {
  const int64_t total = n_rows * n_cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = i % n_cols;
    y[i] = flat[c] ? 0.0 : (y[i] - centre[c]) / sd[c];
  }
}

}  // namespace

int64_t panel_prep_scratch_doubles(int64_t n_rows, int64_t n_cols, int64_t rank) {
  const int64_t ch = n_chunks(n_rows);
  const int64_t jb = rank < kJB ? rank : kJB;
  // partials (max of 1 and jb planes) + W [rank, n_cols] + ss [n_cols]
  return ch * n_cols * (jb > 1 ? jb : 1) + rank * n_cols + n_cols;
}

int panel_prepare(double* d_y, int64_t n_rows, int64_t n_cols, const double* d_q, int64_t rank, double* d_scratch,
                  PanelPrepOut& out, cudaStream_t st) {
  const int64_t ch = n_chunks(n_rows);
  const int64_t jb_max = rank < kJB ? rank : kJB;
  double* partial = d_scratch;
  double* w = partial + ch * n_cols * (jb_max > 1 ? jb_max : 1);
  double* ss = w + rank * n_cols;
  const dim3 blk(32, 8);
  const dim3 grd(static_cast<unsigned>((n_cols + 31) / 32), static_cast<unsigned>(ch));
  const unsigned fin_blocks = static_cast<unsigned>((n_cols + 255) / 256);
  const double n = static_cast<double>(n_rows);
  PG_CUDA_CHECK(cudaMemsetAsync(out.bad, 0, sizeof(int), st));
  // 1. column means (+ finiteness)
  col_partial_kernel<0><<<grd, blk, 0, st>>>(d_y, n_rows, n_cols, nullptr, partial, out.bad);
  PG_CUDA_CHECK(cudaGetLastError());
  col_finish_kernel<<<fin_blocks, 256, 0, st>>>(partial, ch, n_cols, n, out.mean);
  PG_CUDA_CHECK(cudaGetLastError());
  // 2. W = Q^T (y - mean), kJB basis columns per pass over y
  for (int64_t j0 = 0; j0 < rank; j0 += kJB) {
    const int jn = static_cast<int>(rank - j0 < kJB ? rank - j0 : kJB);
    proj_partial_kernel<<<grd, blk, 0, st>>>(d_y, n_rows, n_cols, out.mean, d_q, rank, static_cast<int>(j0), jn,
                                             partial);
    PG_CUDA_CHECK(cudaGetLastError());
    for (int j = 0; j < jn; ++j) {
      col_finish_kernel<<<fin_blocks, 256, 0, st>>>(partial + j * ch * n_cols, ch, n_cols, 1.0,
                                                    w + (j0 + j) * n_cols);
      PG_CUDA_CHECK(cudaGetLastError());
    }
  }
  // 3. residuals in place + their column means
  residual_kernel<<<grd, blk, 0, st>>>(d_y, n_rows, n_cols, out.mean, d_q, rank, w, partial);
  PG_CUDA_CHECK(cudaGetLastError());
  col_finish_kernel<<<fin_blocks, 256, 0, st>>>(partial, ch, n_cols, n, out.centre);
  PG_CUDA_CHECK(cudaGetLastError());
  // 4. 1/N variance about the centre, zero-variance flags
  col_partial_kernel<1><<<grd, blk, 0, st>>>(d_y, n_rows, n_cols, out.centre, partial, out.bad);
  PG_CUDA_CHECK(cudaGetLastError());
  col_finish_kernel<<<fin_blocks, 256, 0, st>>>(partial, ch, n_cols, n, ss);
  PG_CUDA_CHECK(cudaGetLastError());
  sd_kernel<<<fin_blocks, 256, 0, st>>>(ss, out.centre, n_cols, out.sd, out.flat);
  PG_CUDA_CHECK(cudaGetLastError());
  // 5. standardize in place
  scale_cols_kernel<<<148 * 16, 256, 0, st>>>(d_y, n_rows, n_cols, out.centre, out.sd, out.flat);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

}  // namespace pg

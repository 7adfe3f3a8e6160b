// BGEN batches staged compressed: the host ships the raw file range of a
// batch (compressed genotype blocks + interleaved variant headers) to the device; blocks
// are inflated on the GPU (inflate.cu), validated with every check of the reference
// reader (/root/reference/pkg/src/panelgwas/genotypes/bgen.py:183-232, same order) and
// repacked into the device rows the BGEN decode kernels consume:
//     [ 2n probabilities (u8 | u16, little-endian) | n ploidy bytes ]
// Mixed 8/16-bit batches are widened exactly (x257), as in the host path (bgen_io.cu).
#include <cstdint>

#include "bgen_stage.cuh"

namespace pg {
namespace {

__device__ __forceinline__ uint32_t rd32(const uint8_t* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
         (static_cast<uint32_t>(p[3]) << 24);
}

// One block per variant. reason codes as pg_bgen_inflate (include/panelgwas_b200.h).
__global__ void validate_kernel(const uint8_t* __restrict__ blob, const int64_t* __restrict__ off,
                                const int64_t* __restrict__ size, const uint8_t* __restrict__ raw, int64_t raw_stride,
                                const int64_t* __restrict__ raw_len, const int* __restrict__ zstatus, int64_t count,
                                int64_t n, long long* __restrict__ diag /*[count][3]*/, int* __restrict__ bits_of,
                                unsigned long long* __restrict__ summary /*[0] first bad, [1] bits mask*/) {
  const int64_t v = blockIdx.x;
  if (v >= count) return;
  __shared__ int nondiploid;
  if (threadIdx.x == 0) nondiploid = 0;
  __syncthreads();
  const uint8_t* d = raw + v * raw_stride;
  const int64_t len = raw_len[v];
  long long reason = 0, a = 0, b = 0;
  int bits = 0;
  if (size[v] < 4) {
    reason = 1;
  } else if (zstatus[v] != 0) {
    reason = 2;
    a = zstatus[v];
  } else {
    const int64_t want = rd32(blob + off[v]);
    if (len != want) {
      reason = 3, a = len, b = want;
    } else if (len < 8) {
      reason = 10, a = len, b = 10 + n;
    } else {
      const int64_t nn = rd32(d), k = d[4] | (d[5] << 8), pmin = d[6], pmax = d[7];
      if (nn != n) {
        reason = 4, a = nn;
      } else if (k != 2) {
        reason = 5, a = k;
      } else if (pmin != 2 || pmax != 2) {
        reason = 6, a = pmin, b = pmax;
      } else if (len < 10 + n) {
        reason = 10, a = len, b = 10 + n;
      } else {
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
          if ((d[8 + i] & 0x3F) != 2) nondiploid = 1;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (reason == 0) {
    if (nondiploid) {
      reason = 7;
    } else if (d[8 + n] != 0) {
      reason = 8;
    } else {
      const int bb = d[9 + n];
      if (bb != 8 && bb != 16) {
        reason = 9, a = bb;
      } else {
        const int64_t expected = 10 + n + 2 * n * (bb / 8);
        if (len != expected) reason = 10, a = len, b = expected;
        else bits = bb;
      }
    }
  }
  diag[3 * v] = reason;
  diag[3 * v + 1] = a;
  diag[3 * v + 2] = b;
  bits_of[v] = bits;
  if (reason) atomicMin(summary, static_cast<unsigned long long>(v));
  else atomicOr(summary + 1, bits == 8 ? 1ull : 2ull);
}

// rows[v] = probs (widened to 16 bits when wide16 and the block is 8-bit) | ploidy
__global__ void repack_kernel(const uint8_t* __restrict__ raw, int64_t raw_stride, const int* __restrict__ bits_of,
                              int64_t n, int wide16, uint8_t* __restrict__ rows, int64_t pitch) {
  const int64_t v = blockIdx.y;
  const uint8_t* d = raw + v * raw_stride;
  uint8_t* row = rows + v * pitch;
  const int bits = bits_of[v];
  const uint8_t* probs = d + 10 + n;
  const uint8_t* ploidy = d + 8;
  const int64_t out_probs = 2 * n * (wide16 ? 2 : 1);
  const int64_t total = out_probs + n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint8_t val;
    if (i < out_probs) {
      if (wide16 && bits == 8) {
        const uint32_t w = 257u * probs[i >> 1];
        val = static_cast<uint8_t>((i & 1) ? (w >> 8) : (w & 0xFF));
      } else {
        val = probs[i];
      }
    } else {
      val = ploidy[i - out_probs];
    }
    row[i] = val;
  }
}

}  // namespace

int bgen_validate(const uint8_t* d_blob, const int64_t* d_off, const int64_t* d_size, const uint8_t* d_raw,
                  int64_t raw_stride, const int64_t* d_raw_len, const int* d_zstatus, int64_t count, int64_t n,
                  long long* d_diag, int* d_bits, unsigned long long* d_summary, cudaStream_t s) {
  if (count <= 0) return PG_OK;
  validate_kernel<<<static_cast<unsigned>(count), 128, 0, s>>>(d_blob, d_off, d_size, d_raw, raw_stride, d_raw_len,
                                                               d_zstatus, count, n, d_diag, d_bits, d_summary);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

int bgen_repack(const uint8_t* d_raw, int64_t raw_stride, const int* d_bits, int64_t count, int64_t n, bool wide16,
                uint8_t* d_rows, int64_t pitch, cudaStream_t s) {
  if (count <= 0) return PG_OK;
  const int64_t total = 2 * n * (wide16 ? 2 : 1) + n;
  const unsigned gx = static_cast<unsigned>((total + 255) / 256 < 64 ? (total + 255) / 256 : 64);
  repack_kernel<<<dim3(gx, static_cast<unsigned>(count)), 256, 0, s>>>(d_raw, raw_stride, d_bits, n, wide16 ? 1 : 0,
                                                                      d_rows, pitch);
  PG_CUDA_CHECK(cudaGetLastError());
  return PG_OK;
}

}  // namespace pg

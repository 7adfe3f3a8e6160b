// Error plumbing, TMA descriptor encoding and the single-kernel test hook.
#include <cstdarg>
#include <cstdio>
#include <vector>

#include "assoc.cuh"
#include "pg_common.cuh"

namespace pg {

namespace {
thread_local char g_err[1024] = {0};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
}  // namespace

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* get_error() { return g_err; }

int encode_tmap_2d_i8(CUtensorMap* out, const void* base, uint64_t inner_elems, uint64_t rows,
                      uint64_t row_pitch_bytes, uint32_t box_inner, uint32_t box_rows, bool swizzle64) {
  if (g_encode == nullptr) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    PG_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    PG_REQUIRE(fn != nullptr && q == cudaDriverEntryPointSuccess, PG_ERR_CUDA,
               "cuTensorMapEncodeTiled unavailable from the driver");
    g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  PG_REQUIRE(reinterpret_cast<uintptr_t>(base) % 16 == 0 && row_pitch_bytes % 16 == 0, PG_ERR_INVALID,
             "TMA operand must be 16-byte aligned");
  cuuint64_t dims[2] = {inner_elems, rows};
  cuuint64_t strides[1] = {row_pitch_bytes};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(out, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  PG_REQUIRE(r == CUDA_SUCCESS, PG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PG_OK;
}

}  // namespace pg

extern "C" {

const char* pg_last_error(void) { return pg::get_error(); }

int pg_abi_version(void) { return 1; }

int pg_host_alloc(int64_t bytes, void** out) {
  PG_REQUIRE(out != nullptr && bytes > 0, PG_ERR_INVALID, "pg_host_alloc: bad arguments");
  *out = nullptr;
  PG_CUDA_CHECK(cudaHostAlloc(out, static_cast<size_t>(bytes), cudaHostAllocPortable));
  return PG_OK;
}

int pg_host_free(void* ptr) {
  if (ptr) PG_CUDA_CHECK(cudaFreeHost(ptr));
  return PG_OK;
}

int pg_device_count(int* n) {
  int count = 0;
  *n = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return PG_OK;
  }
  int usable = 0;
  for (int d = 0; d < count; ++d) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && prop.major == 10 && prop.minor == 0) ++usable;
  }
  *n = usable;
  return PG_OK;
}

int pg_debug_assoc_gemm(const void* d_qh, const void* d_q1, const void* d_q0, int64_t p_pad, const void* d_v,
                        const void* d_v127, int64_t c_pad, int64_t k_pad, double* d_x, void* stream) {
  using namespace pg;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // neutral epilogue: mu = 0, 1/den = 1, s = 1, Cq = 0  ->  r == X exactly
  std::vector<float> ones_c(c_pad, 1.f), ones_p(p_pad, 1.f);
  std::vector<double> ones_cd(c_pad, 1.0), ones_pd(p_pad, 1.0);
  float *mu_f, *iv_f, *sc_f, *cq_f;
  double *mu_d, *iv_d, *sc_d;
  long long* cq;
  unsigned long long* cnt;
  PG_CUDA_CHECK(cudaMallocAsync(&mu_f, 4 * c_pad, st));
  PG_CUDA_CHECK(cudaMallocAsync(&iv_f, 4 * c_pad, st));
  PG_CUDA_CHECK(cudaMallocAsync(&mu_d, 8 * c_pad, st));
  PG_CUDA_CHECK(cudaMallocAsync(&iv_d, 8 * c_pad, st));
  PG_CUDA_CHECK(cudaMallocAsync(&sc_f, 4 * p_pad, st));
  PG_CUDA_CHECK(cudaMallocAsync(&cq_f, 4 * p_pad, st));
  PG_CUDA_CHECK(cudaMallocAsync(&sc_d, 8 * p_pad, st));
  PG_CUDA_CHECK(cudaMallocAsync(&cq, 8 * p_pad, st));
  PG_CUDA_CHECK(cudaMallocAsync(&cnt, 8, st));
  PG_CUDA_CHECK(cudaMemsetAsync(mu_f, 0, 4 * c_pad, st));
  PG_CUDA_CHECK(cudaMemsetAsync(mu_d, 0, 8 * c_pad, st));
  PG_CUDA_CHECK(cudaMemsetAsync(cq_f, 0, 4 * p_pad, st));
  PG_CUDA_CHECK(cudaMemsetAsync(cq, 0, 8 * p_pad, st));
  PG_CUDA_CHECK(cudaMemsetAsync(cnt, 0, 8, st));
  PG_CUDA_CHECK(cudaMemcpyAsync(iv_f, ones_c.data(), 4 * c_pad, cudaMemcpyHostToDevice, st));
  PG_CUDA_CHECK(cudaMemcpyAsync(iv_d, ones_cd.data(), 8 * c_pad, cudaMemcpyHostToDevice, st));
  PG_CUDA_CHECK(cudaMemcpyAsync(sc_f, ones_p.data(), 4 * p_pad, cudaMemcpyHostToDevice, st));
  PG_CUDA_CHECK(cudaMemcpyAsync(sc_d, ones_pd.data(), 8 * p_pad, cudaMemcpyHostToDevice, st));
  AssocEpilogue ep{};
  ep.rows_per_marker = 1;
  ep.m_valid = c_pad;
  ep.p_valid = p_pad;
  ep.mu_f = mu_f;
  ep.mu_d = mu_d;
  ep.invd_f = iv_f;
  ep.invd_d = iv_d;
  ep.scale_f = sc_f;
  ep.scale_d = sc_d;
  ep.cq_f = cq_f;
  ep.cq = cq;
  ep.rbar = nullptr;
  ep.cand_count = cnt;
  ep.full_r = d_x;
  ep.full_ld = p_pad;
  int rc = launch_assoc(static_cast<const int8_t*>(d_qh), static_cast<const int8_t*>(d_q1),
                        static_cast<const int8_t*>(d_q0), p_pad, static_cast<const int8_t*>(d_v),
                        static_cast<const int8_t*>(d_v127), c_pad, k_pad, ep, st);
  PG_CUDA_CHECK(cudaStreamSynchronize(st));
  for (void* p : {(void*)mu_f, (void*)iv_f, (void*)mu_d, (void*)iv_d, (void*)sc_f, (void*)cq_f, (void*)sc_d,
                  (void*)cq, (void*)cnt})
    cudaFreeAsync(p, st);
  PG_CUDA_CHECK(cudaStreamSynchronize(st));
  return rc;
}

}  // extern "C"

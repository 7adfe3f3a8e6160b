// Shared host/device plumbing for the panelgwas_b200 C-ABI library:
// status codes + a thread-local error message, CUDA error checking, and the
// driver entry point used to encode TMA tensor maps (no -lcuda link needed).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/panelgwas_b200.h"

namespace pg {

void set_error(const char* fmt, ...);
const char* get_error();

#define PG_CUDA_CHECK(expr)                                                                        \
  do {                                                                                             \
    cudaError_t err__ = (expr);                                                                    \
    if (err__ != cudaSuccess) {                                                                    \
      ::pg::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(err__), __FILE__, __LINE__, \
                      cudaGetErrorString(err__));                                                  \
      return PG_ERR_CUDA;                                                                          \
    }                                                                                              \
  } while (0)

#define PG_CHECK_STATUS(expr)        \
  do {                               \
    int st__ = (expr);               \
    if (st__ != PG_OK) return st__;  \
  } while (0)

#define PG_REQUIRE(cond, code, ...)    \
  do {                                 \
    if (!(cond)) {                     \
      ::pg::set_error(__VA_ARGS__);    \
      return (code);                   \
    }                                  \
  } while (0)

// cuTensorMapEncodeTiled resolved through the runtime's driver entry point.
// 2-D byte tensor map; 64-byte swizzle by default (box_inner must then be 64).
int encode_tmap_2d_i8(CUtensorMap* out, const void* base, uint64_t inner_elems, uint64_t rows,
                      uint64_t row_pitch_bytes, uint32_t box_inner, uint32_t box_rows, bool swizzle64 = true);

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace pg

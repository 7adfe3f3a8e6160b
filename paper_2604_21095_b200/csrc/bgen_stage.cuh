// Device-side BGEN block validation / repacking (bgen_stage.cu).
#pragma once
#include <cstdint>

#include "pg_common.cuh"

namespace pg {

// Per variant: diag[3v..3v+2] = (reason, a, b) with the reason codes of pg_bgen_inflate,
// bits[v] = 8 / 16 (0 on error); summary[0] = lowest failing variant (init ~0ull),
// summary[1] |= 1 for 8-bit, 2 for 16-bit blocks (init 0).
int bgen_validate(const uint8_t* d_blob, const int64_t* d_off, const int64_t* d_size, const uint8_t* d_raw,
                  int64_t raw_stride, const int64_t* d_raw_len, const int* d_zstatus, int64_t count, int64_t n,
                  long long* d_diag, int* d_bits, unsigned long long* d_summary, cudaStream_t s);

int bgen_repack(const uint8_t* d_raw, int64_t raw_stride, const int* d_bits, int64_t count, int64_t n, bool wide16,
                uint8_t* d_rows, int64_t pitch, cudaStream_t s);

}  // namespace pg

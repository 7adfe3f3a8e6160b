// GPU zlib inflate (inflate.cu) and BGEN block staging (bgen_stage.cu).
#pragma once
#include <cstdint>

#include "pg_common.cuh"

namespace pg {

// Inflate `count` zlib streams: stream i is d_blob[d_off[i] + skip, d_off[i] + d_len[i]);
// output to d_out + i * out_stride (at most out_stride bytes). Per stream: d_out_len =
// bytes produced, d_status = 0 ok, 1 malformed stream / checksum, 2 output overflow.
// Warp-per-stream decoder by default. With token scratch (d_tokens: count x
// inflate_token_stride(out_stride) u32, d_ntok: 2 x count i32) and PG_INFLATE_MODE=tokens, the
// two-phase decoder (thread-per-stream Huffman decode to LZ77 tokens, then warp-per-stream
// expansion) runs instead (A/B).
int64_t inflate_token_stride(int64_t out_stride);
int inflate_streams(const uint8_t* d_blob, const int64_t* d_off, const int64_t* d_len, int64_t count, int64_t skip,
                    uint8_t* d_out, int64_t out_stride, int64_t* d_out_len, int* d_status, cudaStream_t s,
                    uint32_t* d_tokens = nullptr, int32_t* d_ntok = nullptr);

}  // namespace pg

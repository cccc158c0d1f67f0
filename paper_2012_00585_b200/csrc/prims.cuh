// Device primitives of the symbolic phase (north-star subsystem 1: "GPU sort/unique and an
// exclusive scan"), hand-written for this library — no CUB / Thrust on the path:
//   * exclusive_sum: three-kernel tiled scan (tile sums -> recursive scan of the sums -> apply)
//   * radix_sort_pairs: stable LSD radix sort of (uint32 key, int32 value) pairs, 8-bit digits;
//     every warp owns a contiguous chunk, so stability is positional: per pass a per-(digit,
//     warp) count table, one exclusive scan over it, then each warp replays its chunk in order
//     and ranks the 32 keys of a step with match.any (peers of equal digit) + popc.
// The unique step of the symbolic phase is the warp bitonic sort + ballot in plan.cu
// (k_node_pattern). Everything here is stream-ordered; temporaries are freed on return
// (cudaFree synchronises, like the DevBuf temporaries of the callers).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace feagpu {

// out[i] = sum of in[0..i) for i in [0, n); in and out may be the same array.
void exclusive_sum(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);
void exclusive_sum(const uint32_t* in, uint32_t* out, int64_t n, cudaStream_t s);

// Stable sort of n pairs by bits [begin_bit, end_bit) of the key. Result in keys_out / vals_out;
// the inputs are left intact. n < 2^31.
void radix_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, const int32_t* vals_in,
                      int32_t* vals_out, int64_t n, int begin_bit, int end_bit, cudaStream_t s);

}  // namespace feagpu

// merge_raw.cuh -- K7 over raw uint8 planes for small selections, shared by
// the raw merges (capi.cu) and the packed flags merge (packed.cu), which
// takes this path on the device when the selection it compacted is small.
#pragma once

#include "pdm_common.cuh"

namespace pdm {

// U chunks x M maps per lap (U*M = 8 128-bit loads in flight per thread),
// packed accumulators; chunks of a lap are one grid-width apart so each warp
// access is 512 contiguous bytes of one map.
template <int U, int M, bool kAccumulate>
__device__ __forceinline__ void merge_small_k(const uint8_t *__restrict__ pdms, int64_t pitch,
                                              int64_t nvec, const int32_t *idx, int k,
                                              uint8_t *__restrict__ out) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < nvec;
         base += T * U) {
        uint4 acc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = base + u * T;
            if (kAccumulate && v < nvec)
                acc[u] = *reinterpret_cast<const uint4 *>(out + v * 16);
            else
                acc[u] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        }
        for (int m = 0; m < k; m += M) {
            uint4 r[U][M];
#pragma unroll
            for (int j = 0; j < M; ++j) {
                const uint8_t *plane = pdms + (int64_t)idx[m + j < k ? m + j : m] * pitch;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t v = base + u * T;
                    if (m + j < k && v < nvec) r[u][j] = ld_stream_u4(plane + v * 16);
                }
            }
#pragma unroll
            for (int j = 0; j < M; ++j)
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (m + j < k && base + u * T < nvec) acc[u] = vmin_u8x16(acc[u], r[u][j]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = base + u * T;
            if (v < nvec) st_stream_u4(out + v * 16, acc[u]);
        }
    }
}

// Bytes past the last full 16-byte chunk (map_bytes % 16), byte by byte.
__device__ __forceinline__ void merge_tail(const uint8_t *__restrict__ pdms, int64_t pitch,
                                           int64_t from, int64_t map_bytes, const int32_t *idx,
                                           int k, bool accumulate, uint8_t *__restrict__ out) {
    if (blockIdx.x != 0) return;
    for (int64_t c = from + threadIdx.x; c < map_bytes; c += blockDim.x) {
        uint32_t acc = accumulate ? out[c] : 255u;
        for (int m = 0; m < k; ++m) {
            uint32_t v = pdms[(int64_t)idx[m] * pitch + c];
            acc = v < acc ? v : acc;
        }
        out[c] = (uint8_t)acc;
    }
}

}  // namespace pdm

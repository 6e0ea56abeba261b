// pdm_common.cuh -- shared helpers for the sm_100a distance-map update path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/pdm_b200.h"

namespace pdm {

constexpr int kDistClamp = 255;  // acceleration.py:33 DIST_CLAMP

// ---- error plumbing (thread-local message, int status) ----------------------
void set_error(const char *fmt, ...);
int cuda_status(const char *where);  // checks cudaGetLastError after a launch

#define PDM_REQUIRE(cond, ...)             \
    do {                                   \
        if (!(cond)) {                     \
            ::pdm::set_error(__VA_ARGS__); \
            return PDM_EINVAL;             \
        }                                  \
    } while (0)

#define PDM_CUDA_TRY(expr)                                                                  \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess) {                                                            \
            ::pdm::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                             __LINE__);                                                     \
            return PDM_ECUDA;                                                               \
        }                                                                                   \
    } while (0)

inline cudaStream_t as_stream(pdm_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();  // cached SM count of the current device

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- memory access helpers ------------------------------------------------------
// Streaming 128-bit load that does not allocate in L1 (each byte is read once).
__device__ __forceinline__ uint4 ld_stream_u4(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Streaming (evict-first) 128-bit store.
__device__ __forceinline__ void st_stream_u4(void *p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ uint4 vmin_u8x16(uint4 a, uint4 b) {
    return make_uint4(__vminu4(a.x, b.x), __vminu4(a.y, b.y), __vminu4(a.z, b.z),
                      __vminu4(a.w, b.w));
}

template <int BITS>
struct VoxT;
template <>
struct VoxT<8> {
    using type = uint8_t;
};
template <>
struct VoxT<16> {
    using type = uint16_t;
};

}  // namespace pdm

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
// Resident CTAs per SM of a kernel at (threads, dynamic smem), cached per
// (kernel, threads, smem); at least 1.
int resident_ctas(const void *kernel, int threads, size_t smem);
// A zeroed device counter for one launch on stream s (capi.cu).
int work_counter(cudaStream_t s, unsigned long long **out);

// dt.cu: the three Chebyshev passes in place over one {0, 255}-seeded map
// (the tail of pdm_distance_transform, shared with the fused recompute).
int dt_from_seed(const char *fn, int64_t bx, int64_t by, int64_t bz, uint8_t *map,
                 cudaStream_t s);

// apron.cu: streaming apron min/max (+ mask) when b divides a 16-byte voxel
// chunk; returns PDM_EUNSUPPORTED without launching otherwise.  outs: bit 0 =
// write mins/maxs, bit 1 = write the partition mask.
int apron_fast_launch(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz, int b,
                      int outs, void *mins, void *maxs, const int32_t *pid, uint32_t *mask,
                      int words, cudaStream_t s);

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

// ---- programmatic dependent launch (select kernel -> merge kernel) ----------
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Warp 0 compacts flags[0..n) into a shared index list (ballot + popc).
__device__ __forceinline__ void compact_flags(const uint8_t *__restrict__ flags, int n,
                                              int32_t *s_idx, int *s_k) {
    if (threadIdx.x < 32) {
        const unsigned lane = threadIdx.x;
        int k = 0;
        for (int base = 0; base < n; base += 32) {
            const int p = base + (int)lane;
            const bool on = p < n && flags[p] != 0;
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, on);
            if (on) s_idx[k + __popc(bal & ((1u << lane) - 1u))] = p;
            k += __popc(bal);
        }
        if (lane == 0) *s_k = k;
    }
}

// 32-bit shared-window address of a shared-memory pointer (PTX operands).
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// LDGSTS (cp.async): global -> shared without register staging; completion
// is tracked per thread in commit groups.
namespace cpa {

__device__ __forceinline__ void copy16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void copy4(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace cpa


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

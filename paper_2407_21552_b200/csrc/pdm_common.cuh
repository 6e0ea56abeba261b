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

// ---- TMA bulk copies + mbarriers (sm_90+ async proxy, used on sm_100a) ------
namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

// Make the barrier initialisation visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Spin until the phase with the given parity has completed.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "PDM_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra PDM_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Bulk global -> shared copy (TMA, UBLKCP); completes `bytes` on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace tma

// LDGSTS (cp.async): global -> shared without register staging; completion
// is tracked per thread in commit groups.
namespace cpa {

__device__ __forceinline__ void copy16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tma::smem_u32(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void copy4(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tma::smem_u32(smem)),
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

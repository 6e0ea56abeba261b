// packed.cu -- nibble-packed PDM planes and the TF-change merge (K7) over them.
//
// A partition distance map is a clamped Chebyshev distance field, so along z
// (the contiguous axis) neighbouring blocks differ by at most 1: any 16
// consecutive blocks of one z row span at most 15 distance values.  Each
// plane is therefore stored a second time as
//   base[c]   = min over the 16-block chunk c            (1 byte / 16 blocks)
//   nib[c][j] = (d[16c+2j] - base) | (d[16c+2j+1] - base) << 4   (8 bytes)
// -- 4.5 bits per block instead of 8, lossless.  The merge reads k packed
// planes (0.5625 B per block each) instead of k raw ones (1 B), decodes
// nibble + base in registers and writes D' as plain uint8, bit-identical to
// the raw merge.  The raw planes stay the source of truth (DistanceMap views,
// save/load); a plane set is only packed when every chunk of every plane
// spans <= 15 values (pdm_pack_pdms reports violations, e.g. for rows that
// are not a multiple of 16 blocks or for maps loaded from elsewhere), and the
// raw merge serves everything else.
//
// Merge layout: a thread owns 2 chunks (32 blocks): one 16-byte nibble load
// and one 2-byte base load per selected plane, kPackedBatch planes in flight.
// The accumulator keeps blocks (8w+s, 8w+s+4) in the 16-bit lanes of acc[w][s]
// -- exactly the pair (W >> 4s) & 0x000F000F extracts from nibble word w --
// so folding one plane is shift, mask, add base, VIMNMX.U16x2 per lane pair,
// and 4 PRMTs per 8 blocks restore byte order once at the end.

#include <cuda_fp16.h>

#include <cstdlib>

#include "pdm_common.cuh"

namespace pdm {

constexpr int kPackedThreads = 256;
constexpr int kPackedMaxSel = 240;       // indices in kernel parameters
constexpr int kPackedMaxFlags = 4096;

struct PackedSel {
    int32_t k;
    int32_t idx[kPackedMaxSel];
};

// ---- packing ---------------------------------------------------------------
// Thread = one chunk of one plane: 16 raw bytes in, 8 nibble bytes + 1 base
// out.  Blocks past the map are padded with an in-range value (they are
// decoded but never stored).  `bad` counts chunks spanning > 15 values.
__global__ void __launch_bounds__(256)
    pack_kernel(const uint8_t *__restrict__ pdms, int64_t pitch, int64_t map_bytes, int n,
                int64_t nchunks, uint8_t *__restrict__ nib, int64_t nib_pitch,
                uint8_t *__restrict__ base, int64_t base_pitch, unsigned int *bad) {
    const int64_t total = (int64_t)n * nchunks;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned int nbad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t p = i / nchunks, c = i - p * nchunks;
        const uint8_t *src = pdms + p * pitch + c * 16;
        uint8_t v[16];
        if (c * 16 + 16 <= map_bytes) {
            const uint4 q = *reinterpret_cast<const uint4 *>(src);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
        } else {  // tail: pad with the chunk's first value (a chunk wholly past the map: 255)
            const uint8_t pad = c * 16 < map_bytes ? src[0] : 255;
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = c * 16 + j < map_bytes ? src[j] : pad;
        }
        int lo = 255, hi = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            lo = min(lo, (int)v[j]);
            hi = max(hi, (int)v[j]);
        }
        nbad += hi - lo > 15;
        uint32_t q0 = 0, q1 = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) q0 |= (uint32_t)((v[j] - lo) & 15) << (4 * j);
#pragma unroll
        for (int j = 0; j < 8; ++j) q1 |= (uint32_t)((v[8 + j] - lo) & 15) << (4 * j);
        *reinterpret_cast<uint2 *>(nib + p * nib_pitch + c * 8) = make_uint2(q0, q1);
        base[p * base_pitch + c] = (uint8_t)lo;
    }
    if (nbad) atomicAdd(bad, nbad);
}

// ---- merge -----------------------------------------------------------------
// x >> (32 - e) as the high word of x * 2^e (IMAD.HI on the FMA pipe; PTX
// keeps ptxas from turning it back into a shift on the ALU pipe).
__device__ __forceinline__ uint32_t umulhi_pow2(uint32_t x, int e) {
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(1u << e));
    return r;
}

// Byte values v in [0, 255] are kept as the fp16 numbers 1024 + v (bit
// pattern 0x6400 | v): the order is the same, and the min runs as HMNMX2 on
// the FMA pipe -- VIMNMX.U16x2 issues to the XU pipe, which ncu showed
// saturated (the fold was XU bound at ~3.9 TB/s of packed bytes).
constexpr uint32_t kHalfBias = 0x64006400u;

__device__ __forceinline__ uint32_t hmin2_bits(uint32_t a, uint32_t b) {
    __half2 r = __hmin2(*reinterpret_cast<const __half2 *>(&a),
                        *reinterpret_cast<const __half2 *>(&b));
    return *reinterpret_cast<uint32_t *>(&r);
}

struct PackedAcc {
    uint32_t a[4][4];  // [nibble word][shift]: 16-bit lanes = blocks (8w+s, 8w+s+4)

    __device__ __forceinline__ void init() {
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
            for (int s = 0; s < 4; ++s) a[w][s] = kHalfBias | 0x00FF00FFu;
    }
    // Fold one plane: 4 nibble words (2 chunks) and the chunks' bases.
    __device__ __forceinline__ void fold(uint4 q, uint32_t bases) {
        const uint32_t b0 = (bases & 0xFFu) * 0x00010001u + kHalfBias;
        const uint32_t b1 = ((bases >> 8) & 0xFFu) * 0x00010001u + kHalfBias;
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t bb = i < 2 ? b0 : b1;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                // The fold is bound by the integer ALU pipe (mask, min); the
                // right shifts go to the FMA pipe as high multiplies.
                const uint32_t sh = s == 0 ? w[i] : umulhi_pow2(w[i], 32 - 4 * s);
                a[i][s] = hmin2_bits(a[i][s], (sh & 0x000F000Fu) + bb);
            }
        }
    }
    // 32 blocks in byte order.
    __device__ __forceinline__ void result(uint4 &lo, uint4 &hi) const {
        uint32_t o[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t t01 = __byte_perm(a[i][0], a[i][1], 0x6240);  // b0 b1 b4 b5
            const uint32_t t23 = __byte_perm(a[i][2], a[i][3], 0x6240);  // b2 b3 b6 b7
            o[2 * i] = __byte_perm(t01, t23, 0x5410);
            o[2 * i + 1] = __byte_perm(t01, t23, 0x7632);
        }
        lo = make_uint4(o[0], o[1], o[2], o[3]);
        hi = make_uint4(o[4], o[5], o[6], o[7]);
    }
};

__device__ __forceinline__ uint32_t ld_stream_u16(const void *p) {
    unsigned short r;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
}

// Thread item t covers blocks [32t, 32t + 32).  Items past the last full one
// (map_bytes % 32) write byte by byte.
template <int B>  // selected planes per load batch
__device__ __forceinline__ void merge_packed(const uint8_t *__restrict__ nib, int64_t nib_pitch,
                                             const uint8_t *__restrict__ base,
                                             int64_t base_pitch, int64_t map_bytes,
                                             const int32_t *idx, int k,
                                             uint8_t *__restrict__ out) {
    const int64_t items = ceil_div(map_bytes, 32);
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < items; t += T) {
        PackedAcc acc;
        acc.init();
        for (int m = 0; m < k; m += B) {
            uint4 q[B];
            uint32_t b[B];
#pragma unroll
            for (int j = 0; j < B; ++j) {
                if (m + j < k) {
                    const int64_t p = idx[m + j];
                    q[j] = ld_stream_u4(nib + p * nib_pitch + t * 16);
                    b[j] = ld_stream_u16(base + p * base_pitch + t * 2);
                }
            }
#pragma unroll
            for (int j = 0; j < B; ++j)
                if (m + j < k) acc.fold(q[j], b[j]);
        }
        uint4 lo, hi;
        acc.result(lo, hi);
        uint8_t *dst = out + t * 32;
        if (t * 32 + 32 <= map_bytes) {
            st_stream_u4(dst, lo);
            st_stream_u4(dst + 16, hi);
        } else {
            const uint32_t o[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
            for (int i = 0; t * 32 + i < map_bytes; ++i) dst[i] = (uint8_t)(o[i >> 2] >> (8 * (i & 3)));
        }
    }
}

template <int B>
__global__ void __launch_bounds__(kPackedThreads, B >= 6 ? 4 : 5)
    combine_packed_kernel(const uint8_t *__restrict__ nib, int64_t nib_pitch,
                          const uint8_t *__restrict__ base, int64_t base_pitch, int64_t map_bytes,
                          const __grid_constant__ PackedSel sel, uint8_t *__restrict__ out) {
    merge_packed<B>(nib, nib_pitch, base, base_pitch, map_bytes, sel.idx, sel.k, out);
}

// Selection resident on the device (written by the select kernel ahead of it
// in the stream, PDL): every CTA compacts the flags, then merges.
template <int B>
__global__ void __launch_bounds__(kPackedThreads, B >= 6 ? 4 : 5)
    combine_packed_flags_kernel(const uint8_t *__restrict__ nib, int64_t nib_pitch,
                                const uint8_t *__restrict__ base, int64_t base_pitch,
                                int64_t map_bytes, int n, const uint8_t *__restrict__ flags,
                                uint8_t *__restrict__ out) {
    __shared__ int32_t s_idx[kPackedMaxFlags];
    __shared__ int s_k;
    pdl_wait();
    compact_flags(flags, n, s_idx, &s_k);
    __syncthreads();
    merge_packed<B>(nib, nib_pitch, base, base_pitch, map_bytes, s_idx, s_k, out);
}

template <class K>
static int packed_grid(K kernel, int64_t map_bytes) {
    static const void *keys[8] = {nullptr};
    static int vals[8] = {0};
    int per_sm = 0;
    for (int i = 0; i < 8; ++i) {
        if (keys[i] == (const void *)kernel) {
            per_sm = vals[i];
            break;
        }
        if (keys[i] == nullptr) {
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kPackedThreads,
                                                              0) != cudaSuccess ||
                per_sm < 1)
                per_sm = 1;
            keys[i] = (const void *)kernel;
            vals[i] = per_sm;
            break;
        }
    }
    if (per_sm < 1) per_sm = 1;
    // One wave; laps equalised so no CTA runs an extra one.
    const int64_t items = ceil_div(map_bytes, 32);
    const int64_t cap = (int64_t)sm_count() * per_sm;
    const int64_t laps = ceil_div(items, cap * kPackedThreads);
    int64_t grid = ceil_div(items, laps * kPackedThreads);
    if (grid > cap) grid = cap;
    return grid < 1 ? 1 : (int)grid;
}

// PDM_PACKED_BATCH=4|6|8: planes per load batch (A/B measurements).  Default
// 4: 48 registers, 5 CTAs per SM.  The merge is bound by bytes in flight per
// SM (Little's law at ~3 us loaded HBM latency): 4 planes x 18 B x 1280
// threads ~ 92 KB/SM gives ~3.9 TB/s of packed bytes; 6 and 8 need 63-64+
// registers, drop to 3-4 CTAs and measured no faster (k=32: 82.9 / 95.8 us
// vs 81.9 us).  One 16-block chunk per thread (8-register accumulator, 8-byte
// loads, 8 or 12 planes per batch) measured slower too (k=32: 87 us).  A
// dominance skip (read the selected planes' bases first, then only the
// nibbles of planes whose base is within 15 of the chunk minimum) is exact but
// measured slower at config c (63.4 vs 51.2 us per step): the dependent
// second round of loads costs more latency than the skipped bytes save.
static int packed_batch() {
    static int b = 0;
    if (b == 0) {
        const char *e = getenv("PDM_PACKED_BATCH");
        b = e ? atoi(e) : 4;
        if (b != 6 && b != 8) b = 4;
    }
    return b;
}

static bool packed_layout_ok(const void *nib, int64_t nib_pitch, const void *base,
                             int64_t base_pitch, const void *out) {
    return nib_pitch % 16 == 0 && base_pitch % 2 == 0 && (uintptr_t)nib % 16 == 0 &&
           (uintptr_t)base % 2 == 0 && (uintptr_t)out % 16 == 0;
}

}  // namespace pdm

using namespace pdm;

extern "C" int pdm_packed_chunks(int64_t map_bytes) {
    return map_bytes < 1 ? -1 : (int)(2 * ceil_div(map_bytes, 32));
}

extern "C" int pdm_pack_pdms(const uint8_t *pdms, int64_t plane_pitch, int64_t map_bytes,
                             int32_t n, uint8_t *nib, int64_t nib_pitch, uint8_t *base,
                             int64_t base_pitch, uint32_t *violations, pdm_stream_t stream) {
    PDM_REQUIRE(pdms && nib && base && violations, "pdm_pack_pdms: null pointer");
    PDM_REQUIRE(map_bytes >= 1 && plane_pitch >= map_bytes && n >= 1,
                "pdm_pack_pdms: bad sizes");
    const int64_t nchunks = 2 * ceil_div(map_bytes, 32);
    PDM_REQUIRE(nib_pitch >= nchunks * 8 && base_pitch >= nchunks,
                "pdm_pack_pdms: nib_pitch >= %lld and base_pitch >= %lld required",
                (long long)(nchunks * 8), (long long)nchunks);
    PDM_REQUIRE(plane_pitch % 16 == 0 && (uintptr_t)pdms % 16 == 0 && nib_pitch % 8 == 0 &&
                    (uintptr_t)nib % 8 == 0,
                "pdm_pack_pdms: needs 16-byte aligned planes");
    cudaStream_t s = as_stream(stream);
    PDM_CUDA_TRY(cudaMemsetAsync(violations, 0, sizeof(uint32_t), s));
    int64_t grid = ceil_div((int64_t)n * nchunks, 256);
    const int64_t cap = (int64_t)sm_count() * 8;
    if (grid > cap) grid = cap;
    pack_kernel<<<(unsigned)grid, 256, 0, s>>>(pdms, plane_pitch, map_bytes, n, nchunks, nib,
                                               nib_pitch, base, base_pitch, violations);
    return cuda_status("pack_kernel");
}

extern "C" int pdm_combine_packed(const uint8_t *nib, int64_t nib_pitch, const uint8_t *base,
                                  int64_t base_pitch, int64_t map_bytes, int32_t n,
                                  const int32_t *sel, int32_t k, uint8_t *out,
                                  pdm_stream_t stream) {
    PDM_REQUIRE(nib && base && out && (k == 0 || sel), "pdm_combine_packed: null pointer");
    PDM_REQUIRE(map_bytes >= 1 && n >= 1 && k >= 0 && k <= n && k <= kPackedMaxSel,
                "pdm_combine_packed: bad sizes (map_bytes=%lld n=%d k=%d, k <= %d)",
                (long long)map_bytes, n, k, kPackedMaxSel);
    PDM_REQUIRE(nib_pitch >= 16 * ceil_div(map_bytes, 32) && base_pitch >= 2 * ceil_div(map_bytes, 32),
                "pdm_combine_packed: pitches below the packed plane size");
    PDM_REQUIRE(packed_layout_ok(nib, nib_pitch, base, base_pitch, out),
                "pdm_combine_packed: needs 16-byte aligned nibble planes and output");
    PackedSel p;
    p.k = k;
    for (int i = 0; i < k; ++i) {
        PDM_REQUIRE(sel[i] >= 0 && sel[i] < n, "pdm_combine_packed: index %d outside [0, %d)",
                    sel[i], n);
        p.idx[i] = sel[i];
    }
    cudaStream_t s = as_stream(stream);
    if (packed_batch() == 4)
        combine_packed_kernel<4><<<packed_grid(combine_packed_kernel<4>, map_bytes),
                                   kPackedThreads, 0, s>>>(nib, nib_pitch, base, base_pitch,
                                                           map_bytes, p, out);
    else if (packed_batch() == 6)
        combine_packed_kernel<6><<<packed_grid(combine_packed_kernel<6>, map_bytes),
                                   kPackedThreads, 0, s>>>(nib, nib_pitch, base, base_pitch,
                                                           map_bytes, p, out);
    else
        combine_packed_kernel<8><<<packed_grid(combine_packed_kernel<8>, map_bytes),
                                   kPackedThreads, 0, s>>>(nib, nib_pitch, base, base_pitch,
                                                           map_bytes, p, out);
    return cuda_status("combine_packed_kernel");
}

extern "C" int pdm_combine_flags_packed(const uint8_t *nib, int64_t nib_pitch,
                                        const uint8_t *base, int64_t base_pitch,
                                        int64_t map_bytes, int32_t n, const uint8_t *flags,
                                        uint8_t *out, pdm_stream_t stream) {
    PDM_REQUIRE(nib && base && flags && out, "pdm_combine_flags_packed: null pointer");
    PDM_REQUIRE(map_bytes >= 1 && n >= 1 && n <= kPackedMaxFlags,
                "pdm_combine_flags_packed: bad sizes (n=%d, <= %d)", n, kPackedMaxFlags);
    PDM_REQUIRE(nib_pitch >= 16 * ceil_div(map_bytes, 32) && base_pitch >= 2 * ceil_div(map_bytes, 32),
                "pdm_combine_flags_packed: pitches below the packed plane size");
    PDM_REQUIRE(packed_layout_ok(nib, nib_pitch, base, base_pitch, out),
                "pdm_combine_flags_packed: needs 16-byte aligned nibble planes and output");
    auto kern = packed_batch() == 4 ? combine_packed_flags_kernel<4> : combine_packed_flags_kernel<8>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)packed_grid(kern, map_bytes));
    cfg.blockDim = dim3(kPackedThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PDM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, nib, nib_pitch, base,
                                    base_pitch, map_bytes, (int)n, flags, out));
    return cuda_status("combine_packed_flags_kernel");
}

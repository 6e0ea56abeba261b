// pom.cu -- block reduction of the volume into per-block partition masks
// (POM build, K1/K2) and per-block occupancy for one partition or one TF
// (K3/K4/K5).  All HBM-bound: the volume is streamed once; outputs are
// 1/num_voxels_per_block of it.
//
// Two code paths per reduction:
//  * fast path (b divides a 16-byte chunk of voxels along z and nz*bytes is a
//    multiple of 16): one thread owns one 16-byte z-chunk of one block row
//    (i, j) and loads the b x b rows of it with 128-bit loads (b*b loads in
//    flight per thread), warps cover 512 contiguous bytes of a row, and the
//    partition id of every voxel is looked up in a shared-memory copy of the
//    scheme's pid LUT;
//  * generic path (any b, any dims): one thread per block, scalar loads,
//    coalesced across the warp along z.
#include <cuda_runtime.h>

#include "pdm_common.cuh"

namespace pdm {

// ---- generic path -------------------------------------------------------------

// _kernels.py:137-149 partition_presence / _kernels.py:84-134 block_any_*:
// thread per block.  kKind 1: out[c] = OR of lut[v] (0/1); kKind 2: the same
// written as the distance transform's seed (0 occupied, 255 empty); kKind 0:
// mask bits 1 << pid[v], words > 2 via global atomics into a pre-zeroed mask.
template <int BITS, int kKind>
__global__ void block_lut_generic_kernel(const typename VoxT<BITS>::type *__restrict__ vox,
                                         int64_t nx, int64_t ny, int64_t nz, int b,
                                         int64_t bx, int64_t by, int64_t bz,
                                         const int32_t *__restrict__ pid,
                                         const uint8_t *__restrict__ lut, uint32_t *mask,
                                         int words, uint8_t *out) {
    constexpr bool kBool = kKind != 0;
    const int64_t nb = bx * by * bz;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nb; c += stride) {
        const int64_t k = c % bz, j = (c / bz) % by, i = c / (bz * by);
        const int64_t x1 = min((i + 1) * b, nx), y1 = min((j + 1) * b, ny),
                      z1 = min((k + 1) * b, nz);
        uint64_t m = 0;
        for (int64_t x = i * b; x < x1; ++x)
            for (int64_t y = j * b; y < y1; ++y) {
                const typename VoxT<BITS>::type *row = vox + (x * ny + y) * nz;
                for (int64_t z = k * b; z < z1; ++z) {
                    const uint32_t v = row[z];
                    if (kBool) {
                        m |= lut[v];
                    } else {
                        const int p = pid[v];
                        if (words <= 2)
                            m |= 1ull << p;
                        else
                            atomicOr(&mask[c * words + (p >> 5)], 1u << (p & 31));
                    }
                }
            }
        if (kBool) {
            out[c] = kKind == 2 ? (m != 0 ? 0 : kDistClamp) : (m != 0);
        } else if (words <= 2) {
            mask[c * words] = (uint32_t)m;
            if (words == 2) mask[c * words + 1] = (uint32_t)(m >> 32);
        }
    }
}

// Bits pid[lo]..pid[hi] of a block's mask (partitions are contiguous and
// covering, so (min <= hi_p) & (max >= lo_p) holds exactly for that run).
__device__ __forceinline__ void write_mask_range(uint32_t *mask, int64_t c, int words, int plo,
                                                 int phi) {
    for (int w = 0; w < words; ++w) {
        const int b0 = w * 32, b1 = b0 + 31;
        uint32_t bits = 0;
        if (plo <= b1 && phi >= b0) {
            const int lo = max(plo, b0) - b0, hi = min(phi, b1) - b0;
            const uint32_t upto = hi == 31 ? 0xFFFFFFFFu : ((1u << (hi + 1)) - 1u);
            bits = upto & ~((1u << lo) - 1u);
        }
        mask[c * words + w] = bits;
    }
}

enum ApronOut { kApronMinMax = 1, kApronMask = 2 };

// volume.py:289-300 block_min_max (apron, clipped) -- thread per block -- with
// an optional fused mask epilogue (acceleration.py:223-229).
template <int BITS>
__global__ void apron_generic_kernel(const typename VoxT<BITS>::type *__restrict__ vox,
                                     int64_t nx, int64_t ny, int64_t nz, int b, int64_t bx,
                                     int64_t by, int64_t bz, int outs,
                                     typename VoxT<BITS>::type *__restrict__ mins,
                                     typename VoxT<BITS>::type *__restrict__ maxs,
                                     const int32_t *__restrict__ pid, uint32_t *__restrict__ mask,
                                     int words) {
    const int64_t nb = bx * by * bz;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nb; c += stride) {
        const int64_t k = c % bz, j = (c / bz) % by, i = c / (bz * by);
        const int64_t x0 = max(i * b - 1, (int64_t)0), x1 = min((i + 1) * b + 1, nx);
        const int64_t y0 = max(j * b - 1, (int64_t)0), y1 = min((j + 1) * b + 1, ny);
        const int64_t z0 = max(k * b - 1, (int64_t)0), z1 = min((k + 1) * b + 1, nz);
        uint32_t mn = 0xFFFFFFFFu, mx = 0;
        for (int64_t x = x0; x < x1; ++x)
            for (int64_t y = y0; y < y1; ++y) {
                const typename VoxT<BITS>::type *row = vox + (x * ny + y) * nz;
                for (int64_t z = z0; z < z1; ++z) {
                    const uint32_t v = row[z];
                    mn = v < mn ? v : mn;
                    mx = v > mx ? v : mx;
                }
            }
        if (outs & kApronMinMax) {
            mins[c] = (typename VoxT<BITS>::type)mn;
            maxs[c] = (typename VoxT<BITS>::type)mx;
        }
        if (outs & kApronMask) write_mask_range(mask, c, words, pid[mn], pid[mx]);
    }
}

// ---- fast path: 16-byte z-chunks, shared-memory LUT ---------------------------

// Thread = (block row (i, j), 16-byte chunk q along z).  VPC voxels per chunk,
// B the block edge (B divides VPC), ZB = VPC / B z-blocks per chunk.
// kMode 0: mask words (1 or 2) from a u8 pid LUT; kMode 1: bool from a 0/1 LUT;
// kMode 2: that bool written as the distance transform's seed (0 / 255).
template <int BITS, int B, int kMode, int WORDS>
__global__ void __launch_bounds__(512)
    block_lut_fast_kernel(const typename VoxT<BITS>::type *__restrict__ vox, int64_t nx,
                          int64_t ny, int64_t nz, int64_t bx, int64_t by, int64_t bz,
                          const int32_t *__restrict__ pid, const uint8_t *__restrict__ lut01,
                          uint32_t *__restrict__ mask, uint8_t *__restrict__ out) {
    constexpr int SPAN = 1 << BITS;
    constexpr int VPC = 16 / (BITS / 8);
    constexpr int ZB = VPC / B;
    extern __shared__ __align__(16) uint8_t s_lut[];  // SPAN bytes
    // LUT fill with vector loads (64 KB per CTA at 16 bits: a byte loop here
    // was 128 dependent-latency loads per thread before the first voxel)
    if (kMode == 0) {  // int32 pid -> bytes, 4 per int4 load
        if (((uintptr_t)pid & 15) == 0) {
#pragma unroll 8
            for (int q = threadIdx.x; q < SPAN / 4; q += blockDim.x) {
                const int4 p4 = __ldg(reinterpret_cast<const int4 *>(pid) + q);
                reinterpret_cast<uint32_t *>(s_lut)[q] =
                    (uint32_t)(p4.x & 0xFF) | (uint32_t)(p4.y & 0xFF) << 8 |
                    (uint32_t)(p4.z & 0xFF) << 16 | (uint32_t)(p4.w & 0xFF) << 24;
            }
        } else {
            for (int v = threadIdx.x; v < SPAN; v += blockDim.x) s_lut[v] = (uint8_t)pid[v];
        }
    } else if (((uintptr_t)lut01 & 15) == 0 && SPAN >= 16) {
#pragma unroll 8
        for (int q = threadIdx.x; q < SPAN / 16; q += blockDim.x)
            reinterpret_cast<uint4 *>(s_lut)[q] = __ldg(reinterpret_cast<const uint4 *>(lut01) + q);
    } else {
        for (int v = threadIdx.x; v < SPAN; v += blockDim.x) s_lut[v] = lut01[v];
    }
    __syncthreads();

    const int64_t nzc = nz / VPC;
    const int64_t items = bx * by * nzc;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items; it += stride) {
        const int64_t q = it % nzc;
        const int64_t ij = it / nzc;
        const int64_t j = ij % by, i = ij / by;
        const int xr = (int)min((int64_t)B, nx - i * B);
        const int yr = (int)min((int64_t)B, ny - j * B);
        uint64_t acc[ZB];
#pragma unroll
        for (int t = 0; t < ZB; ++t) acc[t] = 0;
        const typename VoxT<BITS>::type *base = vox + ((i * B) * ny + j * B) * nz + q * VPC;
#pragma unroll
        for (int dx = 0; dx < B; ++dx) {
            if (dx < xr) {
                uint4 r[B];
#pragma unroll
                for (int dy = 0; dy < B; ++dy)
                    if (dy < yr) r[dy] = ld_stream_u4(base + ((int64_t)dx * ny + dy) * nz);
#pragma unroll
                for (int dy = 0; dy < B; ++dy) {
                    if (dy < yr) {
                        const uint32_t w[4] = {r[dy].x, r[dy].y, r[dy].z, r[dy].w};
#pragma unroll
                        for (int e = 0; e < VPC; ++e) {
                            const uint32_t v = BITS == 8 ? (w[e >> 2] >> ((e & 3) * 8)) & 0xFFu
                                                         : (w[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;
                            const uint32_t l = s_lut[v];
                            if (kMode == 0)
                                acc[e / B] |= 1ull << l;
                            else
                                acc[e / B] |= l;
                        }
                    }
                }
            }
        }
        const int64_t c0 = (i * by + j) * bz + q * ZB;
#pragma unroll
        for (int t = 0; t < ZB; ++t) {
            if (kMode == 0) {
                mask[(c0 + t) * WORDS] = (uint32_t)acc[t];
                if (WORDS == 2) mask[(c0 + t) * WORDS + 1] = (uint32_t)(acc[t] >> 32);
            } else if (kMode == 1) {
                out[c0 + t] = acc[t] != 0;
            } else {
                out[c0 + t] = acc[t] != 0 ? 0 : kDistClamp;
            }
        }
    }
}

static bool fast_ok(int bits, int64_t nz, int b, const void *vox) {
    const int vpc = bits == 8 ? 16 : 8;
    return (nz % vpc == 0) && (vpc % b == 0) && ((uintptr_t)vox % 16 == 0);
}

static int grid_for(int64_t items, int threads, int per_sm) {
    int64_t want = ceil_div(items, threads);
    int64_t cap = (int64_t)sm_count() * per_sm;
    if (want > cap) want = cap;
    return want < 1 ? 1 : (int)want;
}

template <int BITS, int B, int kMode, int WORDS>
static int launch_lut_fast(const void *vox, int64_t nx, int64_t ny, int64_t nz, int64_t bx,
                           int64_t by, int64_t bz, const int32_t *pid, const uint8_t *lut01,
                           uint32_t *mask, uint8_t *out, cudaStream_t s) {
    constexpr int SPAN = 1 << BITS;
    constexpr int VPC = 16 / (BITS / 8);
    auto kern = block_lut_fast_kernel<BITS, B, kMode, WORDS>;
    if (SPAN > 48 * 1024)
        PDM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          SPAN));
    const int threads = 512;
    // One wave of resident CTAs (2 per SM: 64 registers x 512 threads), laps
    // equalised: a fixed 3 per SM at 16 bits made 1.5 waves, the last third
    // of the volume then streamed at half occupancy (ncu: 405 us).
    const int per_sm = resident_ctas((const void *)kern, threads, SPAN);
    const int64_t items = bx * by * (nz / VPC);
    const int64_t cap = (int64_t)sm_count() * per_sm;
    const int64_t laps = ceil_div(items, cap * threads);
    const int grid = (int)min(cap, max((int64_t)1, ceil_div(items, laps * threads)));
    kern<<<grid, threads, SPAN, s>>>(
        (const typename VoxT<BITS>::type *)vox, nx, ny, nz, bx, by, bz, pid, lut01, mask, out);
    return cuda_status("block_lut_fast_kernel");
}

template <int BITS, int kMode, int WORDS>
static int dispatch_lut_fast(int b, const void *vox, int64_t nx, int64_t ny, int64_t nz,
                             int64_t bx, int64_t by, int64_t bz, const int32_t *pid,
                             const uint8_t *lut01, uint32_t *mask, uint8_t *out, cudaStream_t s) {
    switch (b) {
        case 1: return launch_lut_fast<BITS, 1, kMode, WORDS>(vox, nx, ny, nz, bx, by, bz, pid, lut01, mask, out, s);
        case 2: return launch_lut_fast<BITS, 2, kMode, WORDS>(vox, nx, ny, nz, bx, by, bz, pid, lut01, mask, out, s);
        case 4: return launch_lut_fast<BITS, 4, kMode, WORDS>(vox, nx, ny, nz, bx, by, bz, pid, lut01, mask, out, s);
        case 8: return launch_lut_fast<BITS, 8, kMode, WORDS>(vox, nx, ny, nz, bx, by, bz, pid, lut01, mask, out, s);
        default: break;
    }
    if (BITS == 8 && b == 16)
        return launch_lut_fast<BITS, (BITS == 8 ? 16 : 8), kMode, WORDS>(vox, nx, ny, nz, bx, by,
                                                                         bz, pid, lut01, mask, out,
                                                                         s);
    set_error("no fast path for b=%d", b);
    return PDM_EUNSUPPORTED;
}

// ---- occupancy from precomputed min/max -------------------------------------------

template <typename T>
__global__ void minmax_range_kernel(const T *__restrict__ mins, const T *__restrict__ maxs,
                                    int64_t nb, uint32_t lo, uint32_t hi, uint8_t *out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nb; c += stride)
        out[c] = (uint32_t)mins[c] <= hi && (uint32_t)maxs[c] >= lo;
}

// kSeed: written as the distance transform's seed (0 occupied, 255 empty).
// A thread takes 8 consecutive blocks: one vector load of their mins and one
// of their maxs (8 * sizeof(T) bytes each), 16 prefix lookups (the intensity
// range is spatially coherent, so they mostly hit L1), one 8-byte store; the
// caller guarantees 8-block alignment of the three pointers for the vector
// part, a scalar tail covers nb % 8.
template <typename T>
struct Vec8;
template <>
struct Vec8<uint8_t> {
    using type = uint2;
};
template <>
struct Vec8<uint16_t> {
    using type = uint4;
};

template <typename T, bool kSeed = false>
__global__ void minmax_prefix_kernel(const T *__restrict__ mins, const T *__restrict__ maxs,
                                     int64_t nb, const int32_t *__restrict__ prefix, uint8_t *out,
                                     bool vec) {
    using V = typename Vec8<T>::type;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nv = vec ? nb / 8 : 0;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nv; q += stride) {
        V lo = __ldcs(reinterpret_cast<const V *>(mins) + q);
        V hi = __ldcs(reinterpret_cast<const V *>(maxs) + q);
        const T *l = reinterpret_cast<const T *>(&lo), *h = reinterpret_cast<const T *>(&hi);
        uint32_t w[2];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            uint32_t word = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = half * 4 + e;
                const bool occ = __ldg(prefix + (uint32_t)h[i] + 1) - __ldg(prefix + (uint32_t)l[i]) > 0;
                const uint32_t byte = kSeed ? (occ ? 0u : (uint32_t)kDistClamp) : (uint32_t)occ;
                word |= byte << (8 * e);
            }
            w[half] = word;
        }
        __stcs(reinterpret_cast<uint2 *>(out) + q, make_uint2(w[0], w[1]));
    }
    for (int64_t c = nv * 8 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nb; c += stride) {
        const bool occ = prefix[(uint32_t)maxs[c] + 1] - prefix[(uint32_t)mins[c]] > 0;
        out[c] = kSeed ? (occ ? 0 : kDistClamp) : occ;
    }
}

template <bool kSeed>
static int launch_minmax_prefix(const void *mins, const void *maxs, int bits, int64_t nb,
                                const int32_t *prefix, uint8_t *out, cudaStream_t s) {
    const uintptr_t vb = bits == 8 ? 8 : 16;
    const bool vec = (uintptr_t)mins % vb == 0 && (uintptr_t)maxs % vb == 0 &&
                     (uintptr_t)out % 8 == 0;
    const int grid = grid_for(vec ? ceil_div(nb, 8) : nb, 256, 8);
    if (bits == 8)
        minmax_prefix_kernel<uint8_t, kSeed><<<grid, 256, 0, s>>>(
            (const uint8_t *)mins, (const uint8_t *)maxs, nb, prefix, out, vec);
    else
        minmax_prefix_kernel<uint16_t, kSeed><<<grid, 256, 0, s>>>(
            (const uint16_t *)mins, (const uint16_t *)maxs, nb, prefix, out, vec);
    return cuda_status("minmax_prefix_kernel");
}

template <typename T>
__global__ void minmax_mask_kernel(const T *__restrict__ mins, const T *__restrict__ maxs,
                                   int64_t nb, const int32_t *__restrict__ pid,
                                   uint32_t *__restrict__ mask, int words) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nb; c += stride)
        write_mask_range(mask, c, words, pid[(uint32_t)mins[c]], pid[(uint32_t)maxs[c]]);
}

// Fold a neighbour slab's apron plane into a block plane: mins = min(mins, pm),
// maxs = max(maxs, px) (slab-sharded range_apron, see sharded.py).
template <typename T>
__global__ void minmax_fold_kernel(T *__restrict__ mins, T *__restrict__ maxs,
                                   const T *__restrict__ pmins, const T *__restrict__ pmaxs,
                                   int64_t count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < count; c += stride) {
        mins[c] = pmins[c] < mins[c] ? pmins[c] : mins[c];
        maxs[c] = pmaxs[c] > maxs[c] ? pmaxs[c] : maxs[c];
    }
}

struct Dims {
    int64_t nx, ny, nz, bx, by, bz;
};

static int check_volume(const char *fn, const void *vox, int bits, int64_t nx, int64_t ny,
                        int64_t nz, int32_t b, Dims *d) {
    PDM_REQUIRE(vox, "%s: null volume", fn);
    PDM_REQUIRE(bits == 8 || bits == 16, "%s: bits must be 8 or 16, got %d", fn, bits);
    PDM_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1, "%s: dims must be positive", fn);
    PDM_REQUIRE(b >= 1, "%s: block edge must be >= 1", fn);
    d->nx = nx;
    d->ny = ny;
    d->nz = nz;
    d->bx = ceil_div(nx, b);
    d->by = ceil_div(ny, b);
    d->bz = ceil_div(nz, b);
    return PDM_OK;
}

}  // namespace pdm

using namespace pdm;

extern "C" int pdm_partition_mask_voxel(const void *vox, int bits, int64_t nx, int64_t ny,
                                        int64_t nz, int32_t b, const int32_t *pid, int32_t n,
                                        uint32_t *mask, int32_t words, pdm_stream_t stream) {
    Dims d;
    int st = check_volume("pdm_partition_mask_voxel", vox, bits, nx, ny, nz, b, &d);
    if (st) return st;
    PDM_REQUIRE(pid && mask, "pdm_partition_mask_voxel: null pointer");
    PDM_REQUIRE(n >= 1 && n <= (1 << bits) && words == (n + 31) / 32,
                "pdm_partition_mask_voxel: n=%d words=%d", n, words);
    cudaStream_t s = as_stream(stream);
    const int64_t nb = d.bx * d.by * d.bz;
    if (words <= 2 && fast_ok(bits, nz, b, vox)) {
        if (bits == 8)
            return words == 1 ? dispatch_lut_fast<8, 0, 1>(b, vox, nx, ny, nz, d.bx, d.by, d.bz, pid, nullptr, mask, nullptr, s)
                              : dispatch_lut_fast<8, 0, 2>(b, vox, nx, ny, nz, d.bx, d.by, d.bz, pid, nullptr, mask, nullptr, s);
        return words == 1 ? dispatch_lut_fast<16, 0, 1>(b, vox, nx, ny, nz, d.bx, d.by, d.bz, pid, nullptr, mask, nullptr, s)
                          : dispatch_lut_fast<16, 0, 2>(b, vox, nx, ny, nz, d.bx, d.by, d.bz, pid, nullptr, mask, nullptr, s);
    }
    if (words > 2) PDM_CUDA_TRY(cudaMemsetAsync(mask, 0, (size_t)nb * words * 4, s));
    const int threads = 256;
    const int grid = grid_for(nb, threads, 8);
    if (bits == 8)
        block_lut_generic_kernel<8, 0><<<grid, threads, 0, s>>>(
            (const uint8_t *)vox, nx, ny, nz, b, d.bx, d.by, d.bz, pid, nullptr, mask, words,
            nullptr);
    else
        block_lut_generic_kernel<16, 0><<<grid, threads, 0, s>>>(
            (const uint16_t *)vox, nx, ny, nz, b, d.bx, d.by, d.bz, pid, nullptr, mask, words,
            nullptr);
    return cuda_status("block_lut_generic_kernel");
}

extern "C" int pdm_block_any_lut(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz,
                                 int32_t b, const uint8_t *lut, uint8_t *out,
                                 pdm_stream_t stream) {
    Dims d;
    int st = check_volume("pdm_block_any_lut", vox, bits, nx, ny, nz, b, &d);
    if (st) return st;
    PDM_REQUIRE(lut && out, "pdm_block_any_lut: null pointer");
    cudaStream_t s = as_stream(stream);
    if (fast_ok(bits, nz, b, vox)) {
        if (bits == 8)
            return dispatch_lut_fast<8, 1, 1>(b, vox, nx, ny, nz, d.bx, d.by, d.bz, nullptr, lut, nullptr, out, s);
        return dispatch_lut_fast<16, 1, 1>(b, vox, nx, ny, nz, d.bx, d.by, d.bz, nullptr, lut, nullptr, out, s);
    }
    const int64_t nb = d.bx * d.by * d.bz;
    const int threads = 256;
    const int grid = grid_for(nb, threads, 8);
    if (bits == 8)
        block_lut_generic_kernel<8, 1><<<grid, threads, 0, s>>>(
            (const uint8_t *)vox, nx, ny, nz, b, d.bx, d.by, d.bz, nullptr, lut, nullptr, 0, out);
    else
        block_lut_generic_kernel<16, 1><<<grid, threads, 0, s>>>(
            (const uint16_t *)vox, nx, ny, nz, b, d.bx, d.by, d.bz, nullptr, lut, nullptr, 0, out);
    return cuda_status("block_lut_generic_kernel");
}

static int apron_launch(const void *vox, int bits, const Dims &d, int b, int outs, void *mins,
                        void *maxs, const int32_t *pid, uint32_t *mask, int words,
                        cudaStream_t s) {
    const int fast = apron_fast_launch(vox, bits, d.nx, d.ny, d.nz, b, outs, mins, maxs, pid,
                                       mask, words, s);
    if (fast != PDM_EUNSUPPORTED) return fast;
    const int64_t nb = d.bx * d.by * d.bz;
    const int threads = 256;
    const int grid = grid_for(nb, threads, 8);
    if (bits == 8)
        apron_generic_kernel<8><<<grid, threads, 0, s>>>(
            (const uint8_t *)vox, d.nx, d.ny, d.nz, b, d.bx, d.by, d.bz, outs, (uint8_t *)mins,
            (uint8_t *)maxs, pid, mask, words);
    else
        apron_generic_kernel<16><<<grid, threads, 0, s>>>(
            (const uint16_t *)vox, d.nx, d.ny, d.nz, b, d.bx, d.by, d.bz, outs, (uint16_t *)mins,
            (uint16_t *)maxs, pid, mask, words);
    return cuda_status("apron_generic_kernel");
}

extern "C" int pdm_block_min_max(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz,
                                 int32_t b, void *mins, void *maxs, pdm_stream_t stream) {
    Dims d;
    int st = check_volume("pdm_block_min_max", vox, bits, nx, ny, nz, b, &d);
    if (st) return st;
    PDM_REQUIRE(mins && maxs, "pdm_block_min_max: null output");
    return apron_launch(vox, bits, d, b, kApronMinMax, mins, maxs, nullptr, nullptr, 0,
                        as_stream(stream));
}

extern "C" int pdm_partition_mask_range_apron(const void *vox, int bits, int64_t nx, int64_t ny,
                                              int64_t nz, int32_t b, const int32_t *pid,
                                              int32_t n, uint32_t *mask, int32_t words,
                                              pdm_stream_t stream) {
    Dims d;
    int st = check_volume("pdm_partition_mask_range_apron", vox, bits, nx, ny, nz, b, &d);
    if (st) return st;
    PDM_REQUIRE(pid && mask, "pdm_partition_mask_range_apron: null pointer");
    PDM_REQUIRE(n >= 1 && n <= (1 << bits) && words == (n + 31) / 32,
                "pdm_partition_mask_range_apron: n=%d words=%d", n, words);
    return apron_launch(vox, bits, d, b, kApronMask, nullptr, nullptr, pid, mask, words,
                        as_stream(stream));
}

extern "C" int pdm_partition_mask_minmax(const void *mins, const void *maxs, int bits,
                                         int64_t nblocks, const int32_t *pid, int32_t n,
                                         uint32_t *mask, int32_t words, pdm_stream_t stream) {
    PDM_REQUIRE(mins && maxs && pid && mask, "pdm_partition_mask_minmax: null pointer");
    PDM_REQUIRE(bits == 8 || bits == 16, "pdm_partition_mask_minmax: bits");
    PDM_REQUIRE(nblocks >= 1 && n >= 1 && words == (n + 31) / 32,
                "pdm_partition_mask_minmax: bad sizes");
    cudaStream_t s = as_stream(stream);
    const int grid = grid_for(nblocks, 256, 8);
    if (bits == 8)
        minmax_mask_kernel<uint8_t><<<grid, 256, 0, s>>>((const uint8_t *)mins,
                                                         (const uint8_t *)maxs, nblocks, pid,
                                                         mask, words);
    else
        minmax_mask_kernel<uint16_t><<<grid, 256, 0, s>>>((const uint16_t *)mins,
                                                          (const uint16_t *)maxs, nblocks, pid,
                                                          mask, words);
    return cuda_status("minmax_mask_kernel");
}

extern "C" int pdm_occupancy_minmax_range(const void *mins, const void *maxs, int bits,
                                          int64_t nblocks, uint32_t lo, uint32_t hi,
                                          uint8_t *out, pdm_stream_t stream) {
    PDM_REQUIRE(mins && maxs && out, "pdm_occupancy_minmax_range: null pointer");
    PDM_REQUIRE(bits == 8 || bits == 16, "pdm_occupancy_minmax_range: bits");
    PDM_REQUIRE(nblocks >= 1, "pdm_occupancy_minmax_range: nblocks");
    cudaStream_t s = as_stream(stream);
    const int grid = grid_for(nblocks, 256, 8);
    if (bits == 8)
        minmax_range_kernel<uint8_t><<<grid, 256, 0, s>>>((const uint8_t *)mins,
                                                          (const uint8_t *)maxs, nblocks, lo, hi,
                                                          out);
    else
        minmax_range_kernel<uint16_t><<<grid, 256, 0, s>>>((const uint16_t *)mins,
                                                           (const uint16_t *)maxs, nblocks, lo,
                                                           hi, out);
    return cuda_status("minmax_range_kernel");
}

extern "C" int pdm_occupancy_minmax_prefix(const void *mins, const void *maxs, int bits,
                                           int64_t nblocks, const int32_t *prefix, uint8_t *out,
                                           pdm_stream_t stream) {
    PDM_REQUIRE(mins && maxs && prefix && out, "pdm_occupancy_minmax_prefix: null pointer");
    PDM_REQUIRE(bits == 8 || bits == 16, "pdm_occupancy_minmax_prefix: bits");
    PDM_REQUIRE(nblocks >= 1, "pdm_occupancy_minmax_prefix: nblocks");
    return launch_minmax_prefix<false>(mins, maxs, bits, nblocks, prefix, out,
                                       as_stream(stream));
}

extern "C" int pdm_minmax_fold(void *mins, void *maxs, const void *plane_mins,
                               const void *plane_maxs, int bits, int64_t count,
                               pdm_stream_t stream) {
    PDM_REQUIRE(mins && maxs && plane_mins && plane_maxs, "pdm_minmax_fold: null pointer");
    PDM_REQUIRE((bits == 8 || bits == 16) && count >= 1, "pdm_minmax_fold: bad args");
    cudaStream_t s = as_stream(stream);
    const int grid = grid_for(count, 256, 8);
    if (bits == 8)
        minmax_fold_kernel<uint8_t><<<grid, 256, 0, s>>>((uint8_t *)mins, (uint8_t *)maxs,
                                                         (const uint8_t *)plane_mins,
                                                         (const uint8_t *)plane_maxs, count);
    else
        minmax_fold_kernel<uint16_t><<<grid, 256, 0, s>>>((uint16_t *)mins, (uint16_t *)maxs,
                                                          (const uint16_t *)plane_mins,
                                                          (const uint16_t *)plane_maxs, count);
    return cuda_status("minmax_fold_kernel");
}

// acceleration.py:184-196 standard_distance_map, fused: the TF's occupancy is
// written directly as the distance transform's {0, 255} seed (no bool map, no
// expand pass), then the three passes run in place (dt.cu dt_from_seed).
extern "C" int pdm_standard_distance_map_voxel(const void *vox, int bits, int64_t nx, int64_t ny,
                                               int64_t nz, int32_t b, const uint8_t *lut,
                                               uint8_t *out, pdm_stream_t stream) {
    Dims d;
    int st = check_volume("pdm_standard_distance_map_voxel", vox, bits, nx, ny, nz, b, &d);
    if (st) return st;
    PDM_REQUIRE(lut && out, "pdm_standard_distance_map_voxel: null pointer");
    cudaStream_t s = as_stream(stream);
    if (fast_ok(bits, nz, b, vox)) {
        st = bits == 8 ? dispatch_lut_fast<8, 2, 1>(b, vox, nx, ny, nz, d.bx, d.by, d.bz, nullptr, lut, nullptr, out, s)
                       : dispatch_lut_fast<16, 2, 1>(b, vox, nx, ny, nz, d.bx, d.by, d.bz, nullptr, lut, nullptr, out, s);
    } else {
        const int grid = grid_for(d.bx * d.by * d.bz, 256, 8);
        if (bits == 8)
            block_lut_generic_kernel<8, 2><<<grid, 256, 0, s>>>(
                (const uint8_t *)vox, nx, ny, nz, b, d.bx, d.by, d.bz, nullptr, lut, nullptr, 0,
                out);
        else
            block_lut_generic_kernel<16, 2><<<grid, 256, 0, s>>>(
                (const uint16_t *)vox, nx, ny, nz, b, d.bx, d.by, d.bz, nullptr, lut, nullptr, 0,
                out);
        st = cuda_status("block_lut_generic_kernel");
    }
    if (st) return st;
    return dt_from_seed("pdm_standard_distance_map_voxel", d.bx, d.by, d.bz, out, s);
}

extern "C" int pdm_standard_distance_map_minmax(const void *mins, const void *maxs, int bits,
                                                int64_t bx, int64_t by, int64_t bz,
                                                const int32_t *prefix, uint8_t *out,
                                                pdm_stream_t stream) {
    const char *fn = "pdm_standard_distance_map_minmax";
    PDM_REQUIRE(mins && maxs && prefix && out, "%s: null pointer", fn);
    PDM_REQUIRE(bits == 8 || bits == 16, "%s: bits", fn);
    PDM_REQUIRE(bx >= 1 && by >= 1 && bz >= 1, "%s: bad sizes", fn);
    cudaStream_t s = as_stream(stream);
    int st = launch_minmax_prefix<true>(mins, maxs, bits, bx * by * bz, prefix, out, s);
    if (st) return st;
    return dt_from_seed(fn, bx, by, bz, out, s);
}

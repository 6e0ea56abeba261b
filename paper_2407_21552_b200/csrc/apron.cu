// apron.cu -- streaming apron min/max (volume.py:289-300 block_min_max) with
// the fused POM / per-TF epilogues of acceleration.py:138-141,169-173,223-229.
//
// A warp owns one y-block row j, one 32-chunk z strip (32 lanes x 16 bytes,
// i.e. 8 uint16 or 16 uint8 voxels per lane) and a run of XB block planes
// along x.  It walks the voxel planes x of the run once (plus the one apron
// plane on each side): per plane every lane loads its 16-byte chunk of the
// b+2 apron rows (clipped), reduces them per voxel, takes each z-block's
// min/max over the block's voxels plus one apron voxel on each side (lane
// neighbours through shuffles, strip edges through one extra scalar load by
// lanes 0 and 31), and folds the result into three rolling accumulators --
// the block row that just ended (its trailing apron plane), the current one
// and the next one (its leading apron plane).  A block row is emitted as soon
// as its trailing apron plane has been folded.  The volume is read once from
// HBM (y-apron rows are re-read from L2 by the neighbouring warp).
#include <cuda_runtime.h>

#include "pdm_common.cuh"

namespace pdm {

enum ApronOuts { kOutMinMax = 1, kOutMask = 2 };

template <int BITS>
__device__ __forceinline__ void unpack16(uint4 q, uint32_t (&v)[16 / (BITS / 8)]) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    if (BITS == 8) {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = (w[e >> 2] >> ((e & 3) * 8)) & 0xFFu;
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = (w[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;
    }
}

__device__ __forceinline__ void write_range_bits(uint32_t *mask, int64_t c, int words, int plo,
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

// Planes prefetched per warp (cp.async ring depth) and the ring footprint.
// Two: the kernel is ALU-bound, so resident warps matter more than depth
// (config c range_apron mask: depth 4 -> 0.666 ms, 3 -> 0.625, 2 -> 0.601,
// 1 -> 0.596; 2 keeps one plane of prefetch per warp).
template <int B>
__host__ __device__ constexpr int apron_ring() {
    return 2;
}
template <int B>
constexpr size_t apron_smem_per_warp() {
    return (size_t)apron_ring<B>() * (B + 2) * (32 * 16 + 2 * 4);
}
constexpr int kApronWarps = 4;

template <int BITS, int B, int OUTS>
__global__ void __launch_bounds__(32 * kApronWarps)
    apron_fast_kernel(const typename VoxT<BITS>::type *__restrict__ vox, int64_t nx, int64_t ny,
                      int64_t nz, int64_t bx, int64_t by, int64_t bz, int XB,
                      typename VoxT<BITS>::type *__restrict__ mins,
                      typename VoxT<BITS>::type *__restrict__ maxs,
                      const int32_t *__restrict__ pid, uint32_t *__restrict__ mask, int words) {
    using T = typename VoxT<BITS>::type;
    constexpr int VPC = 16 / (BITS / 8);
    constexpr int ZB = VPC / B;
    constexpr int kRows = B + 2;
    constexpr int kRing = apron_ring<B>();
    constexpr uint32_t kHi = 0xFFFFFFFFu;
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    extern __shared__ __align__(16) uint8_t s_apron[];
    uint4 *ring_main = reinterpret_cast<uint4 *>(s_apron) +
                       (size_t)(threadIdx.x >> 5) * kRing * kRows * 32;
    uint32_t *ring_edge = reinterpret_cast<uint32_t *>(
                              reinterpret_cast<uint4 *>(s_apron) +
                              (size_t)(blockDim.x >> 5) * kRing * kRows * 32) +
                          (size_t)(threadIdx.x >> 5) * kRing * kRows * 2;
    const int64_t strip = 32 * VPC;
    const int64_t nstrips = ceil_div(nz, strip);
    const int64_t xchunks = ceil_div(bx, XB);
    const int64_t items = by * nstrips * xchunks;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
         it += warps) {
        const int64_t s = it % nstrips;
        const int64_t rest = it / nstrips;
        const int64_t xc = rest % xchunks, j = rest / xchunks;
        const int64_t zs = s * strip;
        const int64_t zl = zs + (int64_t)lane * VPC;
        const bool active = zl < nz;
        const int64_t i0 = xc * XB, i1 = min(i0 + XB, bx);
        const int64_t y0 = max(j * B - 1, (int64_t)0), y1 = min(j * B + B, ny - 1);
        const int64_t xs = max(i0 * B - 1, (int64_t)0), xe = min(i1 * B, nx - 1);
        const bool has_left = zs > 0, has_right = zs + strip < nz;

        uint32_t pmn[ZB], pmx[ZB], cmn[ZB], cmx[ZB], nmn[ZB], nmx[ZB];
#pragma unroll
        for (int t = 0; t < ZB; ++t) {
            pmn[t] = cmn[t] = nmn[t] = kHi;
            pmx[t] = cmx[t] = nmx[t] = 0;
        }
        // plane prefetch: rows y0..y1 of plane px into ring slot `slot` (16 B
        // per lane + the strip-edge words of lanes 0/31), one commit group per
        // plane (empty past the run, so group counting stays uniform)
        const int nrows = (int)(y1 - y0 + 1);
        auto issue_plane = [&](int64_t px, int slot) {
            if (px <= xe) {
                const T *plane = vox + px * ny * nz + y0 * nz;
#pragma unroll
                for (int yy = 0; yy < kRows; ++yy) {  // unrolled, rows past nrows skipped
                    if (yy >= nrows) break;
                    const T *row = plane + (int64_t)yy * nz;
                    if (active) cpa::copy16(&ring_main[(slot * kRows + yy) * 32 + lane], row + zl);
                    if (lane == 0 && has_left)
                        cpa::copy4(&ring_edge[(slot * kRows + yy) * 2],
                                        row + zs - (BITS == 8 ? 4 : 2));
                    if (lane == 31 && has_right)
                        cpa::copy4(&ring_edge[(slot * kRows + yy) * 2 + 1], row + zs + strip);
                }
            }
            cpa::commit();
        };
        for (int d = 0; d < kRing; ++d) issue_plane(xs + d, d);

        auto emit = [&](int64_t i, const uint32_t(&mn)[ZB], const uint32_t(&mx)[ZB]) {
            if (!active) return;
            const int64_t c0 = (i * by + j) * bz + zl / B;
#pragma unroll
            for (int t = 0; t < ZB; ++t) {
                if (OUTS & kOutMinMax) {
                    mins[c0 + t] = (T)mn[t];
                    maxs[c0 + t] = (T)mx[t];
                }
                if (OUTS & kOutMask) write_range_bits(mask, c0 + t, words, pid[mn[t]], pid[mx[t]]);
            }
        };

        for (int64_t x = xs; x <= xe; ++x) {
            const int64_t i = x / B;
            const int r = (int)(x - i * B);
            if (r == 0) {  // a new block row starts: rotate the accumulators
#pragma unroll
                for (int t = 0; t < ZB; ++t) {
                    pmn[t] = cmn[t];
                    pmx[t] = cmx[t];
                    cmn[t] = nmn[t];
                    cmx[t] = nmx[t];
                    nmn[t] = kHi;
                    nmx[t] = 0;
                }
            }
            // y-apron reduction of this plane, per voxel, from the prefetched slot
            const int slot = (int)((x - xs) % kRing);
            cpa::wait<kRing - 1>();
            uint32_t vmn[VPC], vmx[VPC];
#pragma unroll
            for (int e = 0; e < VPC; ++e) {
                vmn[e] = kHi;
                vmx[e] = 0;
            }
            uint32_t lmn = kHi, lmx = 0, rmn = kHi, rmx = 0;  // strip-edge voxels
            // 16-bit voxels: reduce the rows two voxels per instruction
            // (u16x2 min/max on the packed words), unpack once per plane.
            uint32_t wmn[4] = {kHi, kHi, kHi, kHi}, wmx[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int yy = 0; yy < kRows; ++yy) {
                if (yy >= nrows) break;
                if (active) {
                    const uint4 q = ring_main[(slot * kRows + yy) * 32 + lane];
                    if (BITS == 16) {
                        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            wmn[i] = __vminu2(wmn[i], w[i]);
                            wmx[i] = __vmaxu2(wmx[i], w[i]);
                        }
                    } else {
                        uint32_t v[VPC];
                        unpack16<BITS>(q, v);
#pragma unroll
                        for (int e = 0; e < VPC; ++e) {
                            vmn[e] = min(vmn[e], v[e]);
                            vmx[e] = max(vmx[e], v[e]);
                        }
                    }
                }
                if (lane == 0 && has_left) {  // voxel zs-1: top of its aligned word
                    const uint32_t w = ring_edge[(slot * kRows + yy) * 2];
                    const uint32_t e = BITS == 8 ? w >> 24 : w >> 16;
                    lmn = min(lmn, e);
                    lmx = max(lmx, e);
                }
                if (lane == 31 && has_right) {  // voxel zs+strip: bottom of its word
                    const uint32_t w = ring_edge[(slot * kRows + yy) * 2 + 1];
                    const uint32_t e = BITS == 8 ? w & 0xFFu : w & 0xFFFFu;
                    rmn = min(rmn, e);
                    rmx = max(rmx, e);
                }
            }
            if (BITS == 16) {
#pragma unroll
                for (int i = 0; i < VPC / 2; ++i) {
                    vmn[2 * i] = wmn[i] & 0xFFFFu;
                    vmn[2 * i + 1] = wmn[i] >> 16;
                    vmx[2 * i] = wmx[i] & 0xFFFFu;
                    vmx[2 * i + 1] = wmx[i] >> 16;
                }
            }
            issue_plane(x + kRing, slot);  // refill the slot just consumed
            // neighbouring voxels across lanes (inactive lanes hold the identity)
            const uint32_t umn = __shfl_up_sync(FULL, vmn[VPC - 1], 1);
            const uint32_t umx = __shfl_up_sync(FULL, vmx[VPC - 1], 1);
            const uint32_t dmn = __shfl_down_sync(FULL, vmn[0], 1);
            const uint32_t dmx = __shfl_down_sync(FULL, vmx[0], 1);
            if (lane != 0) {
                lmn = umn;
                lmx = umx;
            }
            if (lane != 31) {
                rmn = dmn;
                rmx = dmx;
            }
#pragma unroll
            for (int t = 0; t < ZB; ++t) {
                uint32_t mn = t == 0 ? lmn : vmn[t * B - 1];
                uint32_t mx = t == 0 ? lmx : vmx[t * B - 1];
#pragma unroll
                for (int e = 0; e < B; ++e) {
                    mn = min(mn, vmn[t * B + e]);
                    mx = max(mx, vmx[t * B + e]);
                }
                mn = min(mn, t == ZB - 1 ? rmn : vmn[t * B + B]);
                mx = max(mx, t == ZB - 1 ? rmx : vmx[t * B + B]);
                cmn[t] = min(cmn[t], mn);
                cmx[t] = max(cmx[t], mx);
                if (r == 0) {
                    pmn[t] = min(pmn[t], mn);
                    pmx[t] = max(pmx[t], mx);
                }
                if (r == B - 1) {
                    nmn[t] = min(nmn[t], mn);
                    nmx[t] = max(nmx[t], mx);
                }
            }
            if (r == 0 && i - 1 >= i0) emit(i - 1, pmn, pmx);
        }
        if (xe < i1 * B) emit(i1 - 1, cmn, cmx);
        cpa::wait<0>();  // the ring is reused by the next item
    }
}

template <int BITS, int B>
static int launch_b(const void *vox, int64_t nx, int64_t ny, int64_t nz, int64_t bx, int64_t by,
                    int64_t bz, int outs, void *mins, void *maxs, const int32_t *pid,
                    uint32_t *mask, int words, cudaStream_t s) {
    using T = typename VoxT<BITS>::type;
    constexpr int VPC = 16 / (BITS / 8);
    const int XB = 32;
    const int64_t items = by * ceil_div(nz, 32 * VPC) * ceil_div(bx, XB);
    const size_t smem = kApronWarps * apron_smem_per_warp<B>();
    const int threads = 32 * kApronWarps;
    auto pick = [&]() {
        if (outs == kOutMinMax) return apron_fast_kernel<BITS, B, kOutMinMax>;
        if (outs == kOutMask) return apron_fast_kernel<BITS, B, kOutMask>;
        return apron_fast_kernel<BITS, B, kOutMinMax | kOutMask>;
    };
    auto kern = pick();
    PDM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) !=
            cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    int64_t grid = ceil_div(items, kApronWarps);
    const int64_t cap = (int64_t)sm_count() * per_sm;
    if (grid > cap) grid = cap;
    kern<<<(unsigned)grid, threads, smem, s>>>((const T *)vox, nx, ny, nz, bx, by, bz, XB,
                                              (T *)mins, (T *)maxs, pid, mask, words);
    return cuda_status("apron_fast_kernel");
}

// Fast path when b divides a 16-byte chunk of voxels and rows are 16-byte
// aligned; returns PDM_EUNSUPPORTED (nothing launched) otherwise.
int apron_fast_launch(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz, int b,
                      int outs, void *mins, void *maxs, const int32_t *pid, uint32_t *mask,
                      int words, cudaStream_t s) {
    const int vpc = bits == 8 ? 16 : 8;
    if ((nz % vpc) != 0 || (vpc % b) != 0 || ((uintptr_t)vox % 16) != 0) return PDM_EUNSUPPORTED;
    const int64_t bx = ceil_div(nx, b), by = ceil_div(ny, b), bz = ceil_div(nz, b);
    if (bits == 8) {
        switch (b) {
            case 1: return launch_b<8, 1>(vox, nx, ny, nz, bx, by, bz, outs, mins, maxs, pid, mask, words, s);
            case 2: return launch_b<8, 2>(vox, nx, ny, nz, bx, by, bz, outs, mins, maxs, pid, mask, words, s);
            case 4: return launch_b<8, 4>(vox, nx, ny, nz, bx, by, bz, outs, mins, maxs, pid, mask, words, s);
            case 8: return launch_b<8, 8>(vox, nx, ny, nz, bx, by, bz, outs, mins, maxs, pid, mask, words, s);
            case 16: return launch_b<8, 16>(vox, nx, ny, nz, bx, by, bz, outs, mins, maxs, pid, mask, words, s);
            default: return PDM_EUNSUPPORTED;
        }
    }
    switch (b) {
        case 1: return launch_b<16, 1>(vox, nx, ny, nz, bx, by, bz, outs, mins, maxs, pid, mask, words, s);
        case 2: return launch_b<16, 2>(vox, nx, ny, nz, bx, by, bz, outs, mins, maxs, pid, mask, words, s);
        case 4: return launch_b<16, 4>(vox, nx, ny, nz, bx, by, bz, outs, mins, maxs, pid, mask, words, s);
        case 8: return launch_b<16, 8>(vox, nx, ny, nz, bx, by, bz, outs, mins, maxs, pid, mask, words, s);
        default: return PDM_EUNSUPPORTED;
    }
}

}  // namespace pdm

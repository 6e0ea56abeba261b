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
// Two: resident warps matter more than depth (depth 4 -> 0.666 ms, 3 ->
// 0.625, 2 -> 0.601, 1 -> 0.596 at config c in the previous kernel).
#ifndef PDM_APRON_RING  // (overridable for A/B builds)
#define PDM_APRON_RING 2
#endif
constexpr int kApronRing = PDM_APRON_RING;
template <int B>
constexpr size_t apron_smem_per_warp() {
    return (size_t)kApronRing * (B + 2) * (32 * 16 + 2 * 4);
}
constexpr int kApronWarps = 4;

// Voxels as unsigned 16-bit lanes: a 16-byte chunk is NW = VPC / 2 words of
// two voxels (8-bit volumes are widened byte -> u16 lane with one PRMT per
// two voxels), so the row reduction is VIMNMX(3).U16x2 on whole words.
template <int BITS>
__device__ __forceinline__ void chunk_words(uint4 q, uint32_t (&w)[16 / (BITS / 8) / 2]) {
    const uint32_t v[4] = {q.x, q.y, q.z, q.w};
    if (BITS == 16) {
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = v[i];
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            w[2 * i] = __byte_perm(v[i], 0u, 0x4140);      // bytes 0, 1
            w[2 * i + 1] = __byte_perm(v[i], 0u, 0x4342);  // bytes 2, 3
        }
    }
}

// Straight-line plane walk.  Every out-of-volume row, plane or z-edge voxel is
// replaced by an in-volume voxel of the SAME block (clamped index), and a min
// or max over a set does not change when one of its members is repeated -- so
// there is no boundary branch anywhere: rows y = clamp(jB - 1 .. jB + B), planes
// x = clamp(i0 B - 1 .. i1 B), the strip's outer z voxels the strip's own end
// voxels at the volume's z ends.  Per plane and lane: 6 (B + 2) row chunks and
// the two strip-edge words are cp.async'd a plane ahead; the rows reduce with
// 3-input u16x2 min/max; the z-blocks take their apron voxels from lane
// neighbours; the plane then folds into the current block row (and into the
// previous one at r = 0, the next one at r = B - 1), all decided at compile
// time by unrolling the B planes of a block.
template <int BITS, int B, int OUTS>
__global__ void __launch_bounds__(32 * kApronWarps)
    apron_fast_kernel(const typename VoxT<BITS>::type *__restrict__ vox, int64_t nx, int64_t ny,
                      int64_t nz, int64_t bx, int64_t by, int64_t bz, int XB,
                      typename VoxT<BITS>::type *__restrict__ mins,
                      typename VoxT<BITS>::type *__restrict__ maxs,
                      const int32_t *__restrict__ pid, uint32_t *__restrict__ mask, int words) {
    using T = typename VoxT<BITS>::type;
    constexpr int VPC = 16 / (BITS / 8);  // voxels per lane chunk
    constexpr int NW = VPC / 2;           // u16x2 words per chunk
    constexpr int ZB = VPC / B;           // z-blocks per lane
    constexpr int kRows = B + 2;
    constexpr int WV = 4 / (BITS / 8);  // voxels per 4-byte edge word
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    extern __shared__ __align__(16) uint8_t s_apron[];
    uint4 *ring_main = reinterpret_cast<uint4 *>(s_apron) +
                       (size_t)(threadIdx.x >> 5) * kApronRing * kRows * 32;
    uint32_t *ring_edge = reinterpret_cast<uint32_t *>(
                              reinterpret_cast<uint4 *>(s_apron) +
                              (size_t)(blockDim.x >> 5) * kApronRing * kRows * 32) +
                          (size_t)(threadIdx.x >> 5) * kApronRing * kRows * 2;
    const int64_t strip = 32 * VPC;
    const int64_t nstrips = ceil_div(nz, strip);
    const int64_t xchunks = ceil_div(bx, XB);
    const int64_t items = by * nstrips * xchunks;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t plane_elems = ny * nz;
    for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
         it += warps) {
        const int64_t s = it % nstrips;
        const int64_t rest = it / nstrips;
        const int64_t xc = rest % xchunks, j = rest / xchunks;
        const int64_t zs = s * strip;
        const int64_t zl = zs + (int64_t)lane * VPC;
        const bool active = zl < nz;
        const bool right_in = zl + VPC < nz;  // the next lane's chunk exists
        const int64_t i0 = xc * XB, i1 = min(i0 + XB, bx);
        // element offsets inside a plane: this lane's chunk of row r, and the
        // strip-edge word (lane 0: the word ending at zs - 1, lane 31: the word
        // starting at zs + strip; at the volume's z ends the strip's own end word)
        const bool has_left = zs > 0, has_right = zs + strip < nz;
        const int64_t zcol = active ? zl : zs;
        int64_t eoff = 0;
        int esel = 0;  // voxel of the edge word to use
        if (lane == 0) {
            eoff = has_left ? zs - WV : zs;
            esel = has_left ? WV - 1 : 0;
        } else if (lane == 31) {
            const int64_t last = min(zs + strip, nz) - WV;  // word holding the strip's last voxel
            eoff = has_right ? zs + strip : last;
            esel = has_right ? 0 : WV - 1;
        }
        int64_t roff[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            const int64_t y = min(max(j * B - 1 + r, (int64_t)0), ny - 1);
            roff[r] = y * nz;
        }
        const int64_t xa = i0 * B - 1;                      // first plane of the run
        const int nplanes = (int)((i1 - i0) * B + 2);  // + leading and trailing apron planes
        // byte addresses: this lane's chunk of row r in plane 0, and the edge
        // word relative to it; a plane is one 64-bit add away
        const char *lane0 = reinterpret_cast<const char *>(vox + zcol);
        const int64_t edelta = (eoff - zcol) * (int64_t)sizeof(T);
        const int64_t plane_bytes = plane_elems * (int64_t)sizeof(T);
        int64_t roffb[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r) roffb[r] = roff[r] * (int64_t)sizeof(T);
        auto issue = [&](int q) {  // plane q of the run into ring slot q % kApronRing
            if (q < nplanes) {
                const int64_t x = min(max(xa + q, (int64_t)0), nx - 1);
                const char *plane = lane0 + x * plane_bytes;
                const int slot = q % kApronRing;
#pragma unroll
                for (int r = 0; r < kRows; ++r) {
                    const char *row = plane + roffb[r];
                    cpa::copy16(&ring_main[(slot * kRows + r) * 32 + lane], row);
                    if (lane == 0 || lane == 31)
                        cpa::copy4(&ring_edge[(slot * kRows + r) * 2 + (lane == 31)],
                                   row + edelta);
                }
            }
            cpa::commit();
        };
        // z-block min/max of plane q (after its copies landed)
        auto plane_mm = [&](int q, uint32_t (&mn)[ZB], uint32_t (&mx)[ZB]) {
            const int slot = q % kApronRing;
            uint32_t wmn[NW], wmx[NW];
            {
                uint32_t w0[NW], w1[NW];
                chunk_words<BITS>(ring_main[(slot * kRows + 0) * 32 + lane], w0);
                chunk_words<BITS>(ring_main[(slot * kRows + 1) * 32 + lane], w1);
#pragma unroll
                for (int i = 0; i < NW; ++i) {
                    wmn[i] = __vminu2(w0[i], w1[i]);
                    wmx[i] = __vmaxu2(w0[i], w1[i]);
                }
            }
#pragma unroll
            for (int r = 2; r < kRows; r += 2) {
                uint32_t wa[NW], wb[NW];
                chunk_words<BITS>(ring_main[(slot * kRows + r) * 32 + lane], wa);
                if (r + 1 < kRows) {
                    chunk_words<BITS>(ring_main[(slot * kRows + r + 1) * 32 + lane], wb);
#pragma unroll
                    for (int i = 0; i < NW; ++i) {
                        wmn[i] = __vimin3_u16x2(wmn[i], wa[i], wb[i]);
                        wmx[i] = __vimax3_u16x2(wmx[i], wa[i], wb[i]);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < NW; ++i) {
                        wmn[i] = __vminu2(wmn[i], wa[i]);
                        wmx[i] = __vmaxu2(wmx[i], wa[i]);
                    }
                }
            }
            // strip-edge voxel (lanes 0 and 31): reduce its rows
            uint32_t emn = 0xFFFFFFFFu, emx = 0;
            if (lane == 0 || lane == 31) {
#pragma unroll
                for (int r = 0; r < kRows; ++r) {
                    const uint32_t w = ring_edge[(slot * kRows + r) * 2 + (lane == 31)];
                    const uint32_t e = BITS == 8 ? (w >> (8 * esel)) & 0xFFu
                                                 : (w >> (16 * esel)) & 0xFFFFu;
                    emn = min(emn, e);
                    emx = max(emx, e);
                }
            }
            uint32_t vmn[VPC], vmx[VPC];
#pragma unroll
            for (int i = 0; i < NW; ++i) {
                vmn[2 * i] = wmn[i] & 0xFFFFu;
                vmn[2 * i + 1] = wmn[i] >> 16;
                vmx[2 * i] = wmx[i] & 0xFFFFu;
                vmx[2 * i + 1] = wmx[i] >> 16;
            }
            // apron voxels from the lane neighbours (strip edges: the edge words)
            const uint32_t umn = __shfl_up_sync(FULL, vmn[VPC - 1], 1);
            const uint32_t umx = __shfl_up_sync(FULL, vmx[VPC - 1], 1);
            const uint32_t dmn = __shfl_down_sync(FULL, vmn[0], 1);
            const uint32_t dmx = __shfl_down_sync(FULL, vmx[0], 1);
            const uint32_t lmn = lane == 0 ? emn : umn, lmx = lane == 0 ? emx : umx;
            // right neighbour: the next lane's first voxel if its chunk exists,
            // the edge word at the strip end, else (volume end) our own last voxel
            const uint32_t rmn = lane == 31 ? emn : (right_in ? dmn : vmn[VPC - 1]);
            const uint32_t rmx = lane == 31 ? emx : (right_in ? dmx : vmx[VPC - 1]);
#pragma unroll
            for (int t = 0; t < ZB; ++t) {
                uint32_t a = t == 0 ? lmn : vmn[t * B - 1];
                uint32_t b2 = t == 0 ? lmx : vmx[t * B - 1];
#pragma unroll
                for (int e = 0; e < B; ++e) {
                    a = min(a, vmn[t * B + e]);
                    b2 = max(b2, vmx[t * B + e]);
                }
                mn[t] = min(a, t == ZB - 1 ? rmn : vmn[t * B + B]);
                mx[t] = max(b2, t == ZB - 1 ? rmx : vmx[t * B + B]);
            }
        };
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
#pragma unroll
        for (int d = 0; d < kApronRing; ++d) issue(d);
        uint32_t pmn[ZB], pmx[ZB], cmn[ZB], cmx[ZB], nmn[ZB], nmx[ZB];
#pragma unroll
        for (int t = 0; t < ZB; ++t) {
            pmn[t] = nmn[t] = 0xFFFFFFFFu;
            pmx[t] = nmx[t] = 0u;
        }
        // plane 0: the leading apron plane of block i0 starts its accumulator
        cpa::wait<kApronRing - 1>();
        __syncwarp();
        plane_mm(0, cmn, cmx);
        __syncwarp();
        issue(kApronRing);
        int q = 1;
        for (int64_t i = i0; i < i1; ++i) {
#pragma unroll
            for (int r = 0; r < B; ++r, ++q) {
                cpa::wait<kApronRing - 1>();
                __syncwarp();
                uint32_t mn[ZB], mx[ZB];
                plane_mm(q, mn, mx);
                __syncwarp();
                issue(q + kApronRing);  // refill the slot just read
#pragma unroll
                for (int t = 0; t < ZB; ++t) {
                    cmn[t] = min(cmn[t], mn[t]);
                    cmx[t] = max(cmx[t], mx[t]);
                    if (r == 0) {  // trailing apron plane of block i - 1
                        pmn[t] = min(pmn[t], mn[t]);
                        pmx[t] = max(pmx[t], mx[t]);
                    }
                    if (r == B - 1) {  // leading apron plane of block i + 1
                        nmn[t] = mn[t];
                        nmx[t] = mx[t];
                    }
                }
                if (r == 0 && i > i0) emit(i - 1, pmn, pmx);
            }
#pragma unroll
            for (int t = 0; t < ZB; ++t) {
                pmn[t] = cmn[t];
                pmx[t] = cmx[t];
                cmn[t] = nmn[t];
                cmx[t] = nmx[t];
            }
        }
        // trailing apron plane of the run's last block
        cpa::wait<kApronRing - 1>();
        __syncwarp();
        {
            uint32_t mn[ZB], mx[ZB];
            plane_mm(q, mn, mx);
#pragma unroll
            for (int t = 0; t < ZB; ++t) {
                pmn[t] = min(pmn[t], mn[t]);
                pmx[t] = max(pmx[t], mx[t]);
            }
        }
        emit(i1 - 1, pmn, pmx);
        cpa::wait<0>();  // the ring is reused by the next item
        __syncwarp();
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

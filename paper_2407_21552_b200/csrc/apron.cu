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

#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "pdm_common.cuh"

namespace pdm {

// ---- TMA plane loads (16-bit volumes, b = 4) ----------------------------------------
// One warp's plane of a run is a box of the volume seen as a 3-D tensor
// (z innermost): 6 rows x 256 voxels (its strip) plus two 6 x 8 boxes holding
// the strip-edge voxels -- three cp.async.bulk.tensor issued by lane 0 onto an
// mbarrier per ring slot, instead of 6 x 32 16-byte cp.async + 12 edge words
// per plane (the cp.async version was MIO-throttle and long-scoreboard bound).
// Coordinates are chosen so every voxel the kernel uses lies inside the
// volume (TMA would fill out-of-range voxels with zeros; the kernel needs the
// clamped, replicated voxels): rows start at clamp(jB - 1, 0, ny - 6) and the
// kernel maps its clamped rows into the box.
struct ApronMaps {
    CUtensorMap main;  // box {256, 6, 1}
    CUtensorMap edge;  // box {8, 6, 1}
};
constexpr int kTmaMain = 6 * 256 * 2, kTmaEdge = 6 * 8 * 2;
constexpr int kTmaSlot = kTmaMain + 2 * 128;  // edge boxes at 128-byte offsets
constexpr uint32_t kTmaBytes = kTmaMain + 2 * kTmaEdge;

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int z, int y,
                                            int x, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(z), "r"(y), "r"(x), "r"(smem_addr(bar))
        : "memory");
}

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
template <int B, int RB>
constexpr size_t apron_smem_per_warp() {
    return (size_t)kApronRing * (RB * B + 2) * (32 * 16 + 2 * 4);
}
// Block rows per warp.  Two (16-bit volumes, b = 4: a warp reads 2b + 2 rows
// for 2b instead of 2b + 4, the two shared apron rows reduce once) measured
// 0.445 vs 0.438 ms at config c: the register cost (96 vs 72, 5 vs 6 CTAs per
// SM) outweighs the rows saved (ncu: DRAM read 2.35 vs 2.46 GB).  One is the
// default; PDM_APRON_RB=2 selects two (A/B; same results, tested).
template <int BITS, int B>
constexpr bool apron_two_rows() {
    return BITS == 16 && B == 4;
}
#ifndef PDM_APRON_MINCTAS  // (overridable for A/B builds)
#define PDM_APRON_MINCTAS 6
#endif
constexpr int kApronMinCtas = PDM_APRON_MINCTAS;  // 16-bit, b = 4, one block row
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
template <int BITS, int B, int OUTS, int RB, bool kTma = false>
__global__ void __launch_bounds__(32 * kApronWarps,
                                  (BITS == 16 && B == 4) ? (RB == 1 ? kApronMinCtas : 5) : 1)
    apron_fast_kernel(const typename VoxT<BITS>::type *__restrict__ vox, int64_t nx, int64_t ny,
                      int64_t nz, int64_t bx, int64_t by, int64_t bz, int XB,
                      typename VoxT<BITS>::type *__restrict__ mins,
                      typename VoxT<BITS>::type *__restrict__ maxs,
                      const int32_t *__restrict__ pid, uint32_t *__restrict__ mask, int words,
                      const __grid_constant__ ApronMaps maps) {
    static_assert(!kTma || (BITS == 16 && B == 4 && RB == 1), "TMA planes: 16-bit, b = 4");
    using T = typename VoxT<BITS>::type;
    constexpr int VPC = 16 / (BITS / 8);  // voxels per lane chunk
    constexpr int NW = VPC / 2;           // u16x2 words per chunk
    constexpr int ZB = VPC / B;           // z-blocks per lane
    constexpr int kRows = RB * B + 2;     // RB block rows and their two apron rows
    constexpr int WV = 4 / (BITS / 8);  // voxels per 4-byte edge word
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    extern __shared__ __align__(128) uint8_t s_apron[];
    uint4 *ring_main = reinterpret_cast<uint4 *>(s_apron) +
                       (size_t)(threadIdx.x >> 5) * kApronRing * kRows * 32;
    uint32_t *ring_edge = reinterpret_cast<uint32_t *>(
                              reinterpret_cast<uint4 *>(s_apron) +
                              (size_t)(blockDim.x >> 5) * kApronRing * kRows * 32) +
                          (size_t)(threadIdx.x >> 5) * kApronRing * kRows * 2;
    const int64_t strip = 32 * VPC;
    const int64_t nstrips = ceil_div(nz, strip);
    const int64_t xchunks = ceil_div(bx, XB);
    const int64_t groups = ceil_div(by, RB);
    const int64_t items = groups * nstrips * xchunks;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t plane_elems = ny * nz;
    // TMA ring: slot i of this warp at tma_ring + i * kTmaSlot, one mbarrier each
    __shared__ uint64_t s_bar[kTma ? kApronWarps * kApronRing : 1];
    uint8_t *tma_ring = s_apron + (size_t)(threadIdx.x >> 5) * kApronRing * kTmaSlot;
    uint64_t *bars = s_bar + (kTma ? (threadIdx.x >> 5) * kApronRing : 0);
    uint32_t phase = 0;  // bit i: parity of ring slot i's next completion
    if (kTma) {
        if (lane == 0)
            for (int i = 0; i < kApronRing; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncwarp();
    }
    for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items;
         it += warps) {
        const int64_t s = it % nstrips;
        const int64_t rest = it / nstrips;
#ifdef PDM_APRON_ROW_MAJOR  // (A/B: the round-2 order, x-chunk before block row)
        const int64_t xc = rest % xchunks, jg = rest / xchunks;
#else
        // x-chunk slowest: the warps resident at once walk the same run of
        // planes instead of one run per x-chunk (config c 0.41 -> 0.39 ms,
        // config d 5.1 -> 4.7 ms with TMA, 4.0 ms with cp.async)
        const int64_t jg = rest % groups, xc = rest / groups;
#endif
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
        // rows y = clamp(jg RB B - 1 + r); a block row past the volume (odd by
        // with RB = 2) reads clamped rows and is never emitted
        uint32_t roffb[kRows];  // (a plane is < 2 GB: apron_fast_launch checks)
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            const int64_t y = min(max(jg * RB * B - 1 + r, (int64_t)0), ny - 1);
            roffb[r] = (uint32_t)(y * nz * (int64_t)sizeof(T));
        }
        // TMA: the box's first row, the clamped row r's index inside it
        // (3 bits each), the edge boxes' z and the voxel each edge lane uses
        const int64_t y0 = min(max(jg * B - 1, (int64_t)0), ny - 6);
        uint32_t ridx = 0;
#pragma unroll
        for (int r = 0; r < kRows; ++r)
            ridx |= (uint32_t)(min(max(jg * B - 1 + r, (int64_t)0), ny - 1) - y0) << (3 * r);
        const int zleft = (int)(has_left ? zs - 8 : zs);
        const int zright = (int)(has_right ? zs + strip : min(zs + strip, nz) - 8);
        const int tsel = lane == 0 ? (has_left ? 7 : 0) : (has_right ? 0 : 7);
        const int64_t xa = i0 * B - 1;                      // first plane of the run
        const int nplanes = (int)((i1 - i0) * B + 2);  // + leading and trailing apron planes
        // byte addresses: this lane's chunk of row r in plane 0, and the edge
        // word relative to it; a plane is one 64-bit add away
        const char *lane0 = reinterpret_cast<const char *>(vox + zcol);
        const int64_t edelta = (eoff - zcol) * (int64_t)sizeof(T);
        const int64_t plane_bytes = plane_elems * (int64_t)sizeof(T);
        auto issue = [&](int q) {  // plane q of the run into ring slot q % kApronRing
            if constexpr (kTma) {
                if (q < nplanes && lane == 0) {
                    const int x = (int)min(max(xa + q, (int64_t)0), nx - 1);
                    const int slot = q % kApronRing;
                    uint8_t *dst = tma_ring + slot * kTmaSlot;
                    // the slot's previous contents were read through the generic
                    // proxy (the caller's __syncwarp orders the lanes' reads)
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&bars[slot], kTmaBytes);
                    tma_load_3d(dst, &maps.main, (int)zs, (int)y0, x, &bars[slot]);
                    tma_load_3d(dst + kTmaMain, &maps.edge, zleft, (int)y0, x, &bars[slot]);
                    tma_load_3d(dst + kTmaMain + 128, &maps.edge, zright, (int)y0, x,
                                &bars[slot]);
                }
                return;
            }
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
        // u16x2 min/max over rows [a, b) of ring slot `slot` (3-input forms)
        // row r of ring slot `slot`: this lane's 16-byte chunk
        auto row_chunk = [&](int slot, int r) -> uint4 {
            if constexpr (kTma)
                return *reinterpret_cast<const uint4 *>(tma_ring + slot * kTmaSlot +
                                                        ((ridx >> (3 * r)) & 7u) * 512 +
                                                        lane * 16);
            return ring_main[(slot * kRows + r) * 32 + lane];
        };
        auto rows_mm = [&](int slot, int a, int b, uint32_t (&wmn)[NW], uint32_t (&wmx)[NW]) {
            uint32_t w0[NW];
            chunk_words<BITS>(row_chunk(slot, a), w0);
#pragma unroll
            for (int i = 0; i < NW; ++i) wmn[i] = wmx[i] = w0[i];
#pragma unroll
            for (int r = a + 1; r < b; r += 2) {
                uint32_t wa[NW], wb[NW];
                chunk_words<BITS>(row_chunk(slot, r), wa);
                if (r + 1 < b) {
                    chunk_words<BITS>(row_chunk(slot, r + 1), wb);
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
        };
        // z-block min/max of block row k of plane q (after its copies landed),
        // given the row reduction of its B + 2 rows
        auto zblocks = [&](int slot, int k, const uint32_t (&wmn)[NW], const uint32_t (&wmx)[NW],
                           uint32_t (&mn)[ZB], uint32_t (&mx)[ZB]) {
            // strip-edge voxel (lanes 0 and 31): reduce its rows
            uint32_t emn = 0xFFFFFFFFu, emx = 0;
            if (lane == 0 || lane == 31) {
#pragma unroll
                for (int r = k * B; r < k * B + B + 2; ++r) {
                    uint32_t e;
                    if constexpr (kTma) {
                        e = reinterpret_cast<const uint16_t *>(
                            tma_ring + slot * kTmaSlot + kTmaMain + (lane == 31) * 128)
                            [((ridx >> (3 * r)) & 7u) * 8 + tsel];
                    } else {
                        const uint32_t w = ring_edge[(slot * kRows + r) * 2 + (lane == 31)];
                        e = BITS == 8 ? (w >> (8 * esel)) & 0xFFu : (w >> (16 * esel)) & 0xFFFFu;
                    }
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
        auto plane_mm = [&](int q, uint32_t (&mn)[RB][ZB], uint32_t (&mx)[RB][ZB]) {
            const int slot = q % kApronRing;
            if (RB == 1) {
                uint32_t wmn[NW], wmx[NW];
                rows_mm(slot, 0, kRows, wmn, wmx);
                zblocks(slot, 0, wmn, wmx, mn[0], mx[0]);
            } else {
                // block rows 0 and 1 share their two middle rows B, B + 1
                uint32_t smn[NW], smx[NW], amn[NW], amx[NW];
                rows_mm(slot, B, B + 2, smn, smx);
                rows_mm(slot, 0, B, amn, amx);
#pragma unroll
                for (int i = 0; i < NW; ++i) {
                    amn[i] = __vminu2(amn[i], smn[i]);
                    amx[i] = __vmaxu2(amx[i], smx[i]);
                }
                zblocks(slot, 0, amn, amx, mn[0], mx[0]);
                rows_mm(slot, B + 2, 2 * B + 2, amn, amx);
#pragma unroll
                for (int i = 0; i < NW; ++i) {
                    amn[i] = __vminu2(amn[i], smn[i]);
                    amx[i] = __vmaxu2(amx[i], smx[i]);
                }
                zblocks(slot, 1, amn, amx, mn[RB - 1], mx[RB - 1]);
            }
        };
        auto emit = [&](int64_t i, int k, const uint32_t(&mn)[ZB], const uint32_t(&mx)[ZB]) {
            const int64_t j = jg * RB + k;
            if (!active || j >= by) return;
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
        // plane q's data has landed and is visible to every lane
        auto wait_plane = [&](int q) {
            if constexpr (kTma) {
                const int slot = q % kApronRing;
                mbar_wait(&bars[slot], (phase >> slot) & 1u);
                phase ^= 1u << slot;
            } else {
                cpa::wait<kApronRing - 1>();
            }
            __syncwarp();
        };
#pragma unroll
        for (int d = 0; d < kApronRing; ++d) issue(d);
        uint32_t pmn[RB][ZB], pmx[RB][ZB], cmn[RB][ZB], cmx[RB][ZB], nmn[RB][ZB], nmx[RB][ZB];
#pragma unroll
        for (int k = 0; k < RB; ++k)
#pragma unroll
            for (int t = 0; t < ZB; ++t) {
                pmn[k][t] = nmn[k][t] = 0xFFFFFFFFu;
                pmx[k][t] = nmx[k][t] = 0u;
            }
        // plane 0: the leading apron plane of block i0 starts its accumulator
        wait_plane(0);
        plane_mm(0, cmn, cmx);
        __syncwarp();
        issue(kApronRing);
        int q = 1;
        for (int64_t i = i0; i < i1; ++i) {
#pragma unroll
            for (int r = 0; r < B; ++r, ++q) {
                wait_plane(q);
                uint32_t mn[RB][ZB], mx[RB][ZB];
                plane_mm(q, mn, mx);
                __syncwarp();
                issue(q + kApronRing);  // refill the slot just read
#pragma unroll
                for (int k = 0; k < RB; ++k)
#pragma unroll
                    for (int t = 0; t < ZB; ++t) {
                        cmn[k][t] = min(cmn[k][t], mn[k][t]);
                        cmx[k][t] = max(cmx[k][t], mx[k][t]);
                        if (r == 0) {  // trailing apron plane of block i - 1
                            pmn[k][t] = min(pmn[k][t], mn[k][t]);
                            pmx[k][t] = max(pmx[k][t], mx[k][t]);
                        }
                        if (r == B - 1) {  // leading apron plane of block i + 1
                            nmn[k][t] = mn[k][t];
                            nmx[k][t] = mx[k][t];
                        }
                    }
                if (r == 0 && i > i0)
#pragma unroll
                    for (int k = 0; k < RB; ++k) emit(i - 1, k, pmn[k], pmx[k]);
            }
#pragma unroll
            for (int k = 0; k < RB; ++k)
#pragma unroll
                for (int t = 0; t < ZB; ++t) {
                    pmn[k][t] = cmn[k][t];
                    pmx[k][t] = cmx[k][t];
                    cmn[k][t] = nmn[k][t];
                    cmx[k][t] = nmx[k][t];
                }
        }
        // trailing apron plane of the run's last block
        wait_plane(q);
        {
            uint32_t mn[RB][ZB], mx[RB][ZB];
            plane_mm(q, mn, mx);
#pragma unroll
            for (int k = 0; k < RB; ++k)
#pragma unroll
                for (int t = 0; t < ZB; ++t) {
                    pmn[k][t] = min(pmn[k][t], mn[k][t]);
                    pmx[k][t] = max(pmx[k][t], mx[k][t]);
                }
        }
#pragma unroll
        for (int k = 0; k < RB; ++k) emit(i1 - 1, k, pmn[k], pmx[k]);
        if (!kTma) cpa::wait<0>();  // the ring is reused by the next item
        __syncwarp();
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// The volume as a 3-D uint16 tensor (z innermost) with boxes of {bz_box, 6, 1}.
static bool encode_volume_map(CUtensorMap *m, const void *vox, int64_t nx, int64_t ny,
                              int64_t nz, uint32_t zbox) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)nz, (cuuint64_t)ny, (cuuint64_t)nx};
    const cuuint64_t strides[2] = {(cuuint64_t)nz * 2, (cuuint64_t)(ny * nz * 2)};
    const cuuint32_t box[3] = {zbox, 6, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void *>(vox), dims, strides, box,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BITS, int B>
static int launch_b(const void *vox, int64_t nx, int64_t ny, int64_t nz, int64_t bx, int64_t by,
                    int64_t bz, int outs, void *mins, void *maxs, const int32_t *pid,
                    uint32_t *mask, int words, cudaStream_t s) {
    using T = typename VoxT<BITS>::type;
    constexpr int VPC = 16 / (BITS / 8);
    static const int XB = getenv("PDM_APRON_XB") ? atoi(getenv("PDM_APRON_XB")) : 32;  // (A/B)
    static const bool two = getenv("PDM_APRON_RB") && getenv("PDM_APRON_RB")[0] == '2';
    constexpr int RB2 = apron_two_rows<BITS, B>() ? 2 : 1;
    const int RB = two ? RB2 : 1;
    // TMA plane loads: 16-bit, b = 4, one block row per warp, at least 6 rows,
    // volumes up to 4 GB (at config d, 17 GB with 8 MB planes, the cp.async
    // ring measured faster: 4.0 vs 4.7 ms); PDM_APRON_TMA=0 keeps the
    // cp.async ring (A/B)
    static const bool no_tma = getenv("PDM_APRON_TMA") && getenv("PDM_APRON_TMA")[0] == '0';
    ApronMaps maps;
    memset(&maps, 0, sizeof(maps));
    bool tma = false;
    if constexpr (BITS == 16 && B == 4) {
        tma = !no_tma && RB == 1 && ny >= 6 && nx * ny * nz * 2 <= ((int64_t)4 << 30) &&
              nx < ((int64_t)1 << 31) && encode_volume_map(&maps.main, vox, nx, ny, nz, 256) &&
              encode_volume_map(&maps.edge, vox, nx, ny, nz, 8);
    }
    const int64_t items = ceil_div(by, RB) * ceil_div(nz, 32 * VPC) * ceil_div(bx, XB);
    const size_t smem = tma ? (size_t)kApronWarps * kApronRing * kTmaSlot
                            : kApronWarps * (RB == 1 ? apron_smem_per_warp<B, 1>()
                                                     : apron_smem_per_warp<B, RB2>());
    const int threads = 32 * kApronWarps;
    auto pick = [&]() {
        if constexpr (BITS == 16 && B == 4) {
            if (tma) {
                if (outs == kOutMinMax) return apron_fast_kernel<BITS, B, kOutMinMax, 1, true>;
                if (outs == kOutMask) return apron_fast_kernel<BITS, B, kOutMask, 1, true>;
                return apron_fast_kernel<BITS, B, kOutMinMax | kOutMask, 1, true>;
            }
        }
        if (RB == 1) {
            if (outs == kOutMinMax) return apron_fast_kernel<BITS, B, kOutMinMax, 1>;
            if (outs == kOutMask) return apron_fast_kernel<BITS, B, kOutMask, 1>;
            return apron_fast_kernel<BITS, B, kOutMinMax | kOutMask, 1>;
        }
        if (outs == kOutMinMax) return apron_fast_kernel<BITS, B, kOutMinMax, RB2>;
        if (outs == kOutMask) return apron_fast_kernel<BITS, B, kOutMask, RB2>;
        return apron_fast_kernel<BITS, B, kOutMinMax | kOutMask, RB2>;
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
                                              (T *)mins, (T *)maxs, pid, mask, words, maps);
    return cuda_status("apron_fast_kernel");
}

// Fast path when b divides a 16-byte chunk of voxels and rows are 16-byte
// aligned; returns PDM_EUNSUPPORTED (nothing launched) otherwise.
int apron_fast_launch(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz, int b,
                      int outs, void *mins, void *maxs, const int32_t *pid, uint32_t *mask,
                      int words, cudaStream_t s) {
    const int vpc = bits == 8 ? 16 : 8;
    if ((nz % vpc) != 0 || (vpc % b) != 0 || ((uintptr_t)vox % 16) != 0 ||
        ny * nz * (bits / 8) >= ((int64_t)1 << 31))
        return PDM_EUNSUPPORTED;
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

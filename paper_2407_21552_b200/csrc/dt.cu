// dt.cu -- exact clamped Chebyshev distance transform of block occupancy (K6).
//
// Replaces _kernels.py:17-81 chamfer_chebyshev (two sequential raster passes
// over the 26-neighbourhood) + the clamp of acceleration.py:180 with separable,
// embarrassingly parallel passes over the partition-major map set
// pdms[p][x][y][z] (z contiguous), all in place:
//
//   expand:  g0 = 0 where partition p occupies the block, else 255
//   pass x:  g1[x] = 1-D distance along x to the nearest occupied block
//            (forward + backward run-length sweeps, clamped at 255);
//   pass y:  g2[y] = min_j max(|y - j|, g1[j])     (lower envelope)
//   pass z:  g3[z] = min_j max(|z - j|, g2[j])     (lower envelope)
//
// min(C, max(a, b)) = max(min(C, a), min(C, b)) makes uint8-clamped
// intermediates exact, and the chessboard metric is the max of the per-axis
// distances, so g3 == min(255, chamfer_chebyshev) cell for cell (pinned
// against the reference's golden vectors and the C oracle in tests/).
//
// Kernels, by shape (config c, 256^3 blocks, takes the first of each):
//   expand + pass x: dt_x_mask_kernel reads the partition mask itself (masks
//     of one word, lines <= 512); else dt_expand_mask_kernel + the x pass;
//   pass y / pass z: dt_tmem_kernel keeps each lane's line in tensor memory
//     (lines of 256 or 512 in full 32-line tiles); else dt_tile_kernel
//     (lines in shared memory); lines > 1024: dt_line_kernel.
// Lower envelopes of lines <= 512 use a stack-free forward/backward sweep with
// a per-line table indexed by value (sweep_forward / sweep_backward below);
// longer lines use Meijster et al.'s linear-time scan with the L-infinity
// separator (one lane per line, stack in local memory):
//   f(x, i)  = max(|x - i|, g(i))
//   Sep(i,u) = g(i) <= g(u) ? max(i + g(u), (i + u) / 2) : min(u - g(i), (i + u) / 2)
// Every pass works on warp tiles of 32 lines staged in shared memory with
// cp.async: each lane runs its line from shared memory (the per-element
// dependency chain sees shared-memory latency, not DRAM latency), and the warp
// writes the tile back.  Lines along x and y are strided in memory (a tile is
// 32 consecutive z of one line family); lines along z are contiguous rows (a
// tile is 32 consecutive rows, 16-byte chunks swizzled by row).  The x pass
// (1-D distance) of lines <= 256 runs 4 lines per lane on 128-z tiles.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "pdm_common.cuh"

namespace pdm {

// ---- per-line operations -----------------------------------------------------------

// Stack entry: s (12 bits) | t (12 bits) << 12 | g(s) (8 bits) << 24.
__device__ __forceinline__ uint32_t pack_entry(int s, int t, int g) {
    return (uint32_t)s | ((uint32_t)t << 12) | ((uint32_t)g << 24);
}
__device__ __forceinline__ int ent_s(uint32_t e) { return (int)(e & 0xFFFu); }
__device__ __forceinline__ int ent_t(uint32_t e) { return (int)((e >> 12) & 0xFFFu); }
__device__ __forceinline__ int ent_g(uint32_t e) { return (int)(e >> 24); }

// Meijster lower envelope of one line of m <= LMAX values (LMAX <= 4096):
// out[u] = min(255, min_i max(|u - i|, g[i])).  Ld/St access element u.
// The top of the envelope stack lives in a register (`top`); only entries
// below it are in the local-memory array, so an element that neither pops nor
// pushes touches no memory but its own input, and the next input is loaded
// one element ahead.
template <int LMAX, class Ld, class St>
__device__ __forceinline__ void cone_line(int m, Ld ld, St st) {
    uint32_t stk[LMAX];
    int q = 0;  // entries stored below the top
    uint32_t top = pack_entry(0, 0, ld(0));
    int gnext = m > 1 ? ld(1) : 0;
    for (int u = 1; u < m; ++u) {
        const int gu = gnext;
        if (u + 1 < m) gnext = ld(u + 1);
        bool empty = false;
        for (;;) {  // pop while the top's cone is above u's at the top's threshold
            const int t = ent_t(top);
            const int fs = max(abs(t - ent_s(top)), ent_g(top));
            const int fu = max(abs(t - u), gu);
            if (fs <= fu) break;
            if (q == 0) {
                empty = true;
                break;
            }
            top = stk[--q];
        }
        if (empty) {
            top = pack_entry(u, 0, gu);
        } else {
            const int s = ent_s(top), gs = ent_g(top);
            const int mid = (s + u) >> 1;
            const int sep = gs <= gu ? max(s + gu, mid) : min(u - gs, mid);
            const int w = 1 + sep;
            if (w < m) {
                stk[q++] = top;
                top = pack_entry(u, w, gu);
            }
        }
    }
    for (int u = m - 1; u >= 0; --u) {
        const int d = max(abs(u - ent_s(top)), ent_g(top));
        st(u, d < kDistClamp ? d : kDistClamp);
        if (u == ent_t(top) && q > 0) top = stk[--q];
    }
}

// 1-D distance of a {0 = occupied, else not} line: forward then backward
// run-length sweep, clamped at 255.
template <class Ld, class St>
__device__ __forceinline__ void dist1d_line(int m, Ld ld, St st) {
    int run = kDistClamp;
    for (int u = 0; u < m; ++u) {
        run = ld(u) == 0 ? 0 : min(run + 1, kDistClamp);
        st(u, run);
    }
    run = kDistClamp;
    for (int u = m - 1; u >= 0; --u) {
        const int fwd = ld(u);
        run = fwd == 0 ? 0 : min(run + 1, kDistClamp);
        st(u, min(fwd, run));
    }
}

// Lower envelope of a line of len <= 256 values by two running sweeps, no
// stack.  Forward: L[u] = min_{i<=u} max(u - i, g[i]).  Given m = L[u-1],
// every i in [u-m, u-1] has g[i] >= m, so
//   L[u] = g[u]                        if g[u] <= m
//        = m    if the last i < u with g[i] == m lies in [u-m, u-1]
//        = m+1  otherwise
// (= min(g[u], m + [miss]), g[u] <= m giving g[u] either way), and one
// table indexed by value decides it.  Backward: the same sweep over L
// reversed gives the full envelope (env(L) == env(g), and L is its own left
// envelope), written in place.  Values stay <= 255 (m + 1 is only taken when
// g[u] > m).  `tab` is the lane's column of a [256][32] byte table (32-bit
// shared-window address); the caller clears it before each sweep.
//
// Table entry of value v: min(255, last position of v + v).  The window test
// last[m] + m >= u is then entry >= u (u <= 255, so saturation keeps it
// exact), and a cleared entry (0) fails it for every u >= 1 -- correct, since
// m >= u implies the minimiser i* < u has g[i*] == m, i.e. a real entry.
// Table accesses are PTX with the select written out so the compiler keeps
// the loop-carried chain at load -> compare -> select (left to itself it
// re-derives the next address from min(g, m + miss): four dependent ops).
__device__ __forceinline__ int lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return (int)v;
}
__device__ __forceinline__ void sts_u8(uint32_t a, int v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int lds_u16(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return (int)v;
}
__device__ __forceinline__ void sts_u16(uint32_t a, int v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Table geometry by entry width TB (bytes): lines <= 256 use byte entries
// (positions + values saturate at 255, exact because positions <= 255);
// lines 257..512 use 16-bit entries (position + value <= 766, no saturation).
// A value row of the [256][32] table is 32 * TB bytes.
template <int TB>
struct SweepTable {
    static constexpr uint32_t kRow = 32u * TB;
    static constexpr int kShift = TB == 1 ? 5 : 6;  // log2(kRow)
    static constexpr size_t kBytes = (size_t)256 * kRow;
};

// One step in "address space": M = tab + R m is the table entry of the
// running value (R = the table's value-row bytes) and G = tab + R g; min()
// commutes with that map, so the two candidates are min(G, M) and
// min(G, M + R).  Returns R * m.
template <int TB>
__device__ __forceinline__ uint32_t step_scaled(uint32_t &M, int g, int j, uint32_t tab) {
    constexpr uint32_t R = SweepTable<TB>::kRow;
    const uint32_t G = tab + R * (uint32_t)g;
    const uint32_t a0 = min(G, M), a1 = min(G, M + R);
    const int e = TB == 1 ? lds_u8(M) : lds_u16(M);
    uint32_t nM;
    asm("{\n\t.reg .pred p;\n\t"
        "setp.lt.s32 p, %1, %2;\n\t"
        "selp.b32 %0, %3, %4, p;\n\t}"
        : "=r"(nM)
        : "r"(e), "r"(j), "r"(a1), "r"(a0));
    if (TB == 1)
        sts_u8(G, min(g + j, kDistClamp));
    else
        sts_u16(G, g + j);
    M = nM;
    return M - tab;
}

// Four steps on one word of 4 consecutive elements (one PRMT per byte).
// kRev walks the bytes high to low (backward sweep); j0 is the sweep position
// of the first element handled.
template <int TB, bool kRev>
__device__ __forceinline__ uint32_t sweep_word(uint32_t &M, uint32_t w, int j0, uint32_t tab) {
    constexpr int sh = SweepTable<TB>::kShift;
    uint32_t a[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int byte = kRev ? 3 - k : k;
        step_scaled<TB>(M, (int)__byte_perm(w, 0u, 0x4440u + byte), j0 + k, tab);
        a[byte] = M;
    }
    // a[b] = tab + (m_b << sh); the word is sum_b (a[b] - tab) << (8 b - sh), and
    // the tab terms of bytes 1..3 fold into one loop-invariant constant (three
    // shift-adds per word instead of a subtract per byte plus shifts and ors;
    // the fields do not overlap, so + is |)
    constexpr uint32_t F = (1u << (8 - sh)) + (1u << (16 - sh)) + (1u << (24 - sh));
    return ((a[0] - tab) >> sh) + a[1] * (1u << (8 - sh)) + a[2] * (1u << (16 - sh)) +
           a[3] * (1u << (24 - sh)) - tab * F;
}

template <int TB>
__device__ __forceinline__ uint4 sweep_chunk_fwd(uint32_t &M, uint4 c, int j0, uint32_t tab) {
    uint4 o;
    o.x = sweep_word<TB, false>(M, c.x, j0, tab);
    o.y = sweep_word<TB, false>(M, c.y, j0 + 4, tab);
    o.z = sweep_word<TB, false>(M, c.z, j0 + 8, tab);
    o.w = sweep_word<TB, false>(M, c.w, j0 + 12, tab);
    return o;
}
template <int TB>
__device__ __forceinline__ uint4 sweep_chunk_bwd(uint32_t &M, uint4 c, int j0, uint32_t tab) {
    uint4 o;
    o.w = sweep_word<TB, true>(M, c.w, j0, tab);
    o.z = sweep_word<TB, true>(M, c.z, j0 + 4, tab);
    o.y = sweep_word<TB, true>(M, c.y, j0 + 8, tab);
    o.x = sweep_word<TB, true>(M, c.x, j0 + 12, tab);
    return o;
}

// Line layouts in a warp's shared-memory tile:
//   kStrided: element u of lane l at tile[u * 32 + l] ([u][32] tile of lines
//             along x or y);
//   kRow:     contiguous row (sstride = 4 x odd, conflict-free 32-bit access);
//   kRowSwz:  256 B-aligned rows of L % 128 == 0, 16-byte chunk c of row r
//             stored at chunk c ^ (r & 7): each quarter-warp's 16-byte
//             accesses hit 8 distinct bank groups.
enum { kStrided = 0, kRow = 1, kRowSwz = 2 };

template <int LAYOUT>
struct TileLine {
    uint8_t *p;  // kStrided: tile + lane; rows: the lane's row
    int lane;
    __device__ __forceinline__ int ld(int u) const { return p[LAYOUT == kStrided ? u * 32 : u]; }
    __device__ __forceinline__ void st(int u, uint32_t v) const {
        p[LAYOUT == kStrided ? u * 32 : u] = (uint8_t)v;
    }
    __device__ __forceinline__ uint32_t ld4(int u) const {
        return *reinterpret_cast<const uint32_t *>(p + u);
    }
    __device__ __forceinline__ void st4(int u, uint32_t v) const {
        *reinterpret_cast<uint32_t *>(p + u) = v;
    }
    __device__ __forceinline__ uint4 *chunk(int c) const {
        return reinterpret_cast<uint4 *>(p) + (c ^ (lane & 7));
    }
};

// Forward sweep in place.  Every layout loads the next group of elements
// before the current group's results are stored (the table accesses are
// ordered PTX, so the compiler cannot hoist loads across them by itself).
template <int TB, int LAYOUT>
__device__ __forceinline__ void sweep_forward(int len, TileLine<LAYOUT> line, uint32_t tab) {
    constexpr int sh = SweepTable<TB>::kShift;
    uint32_t M = tab + SweepTable<TB>::kRow * kDistClamp;
    if (LAYOUT == kRowSwz) {
        const int nc = len >> 4;
        uint4 c = *line.chunk(0);
        for (int cc = 0; cc < nc; ++cc) {
            const uint4 nx = cc + 1 < nc ? *line.chunk(cc + 1) : make_uint4(0u, 0u, 0u, 0u);
            *line.chunk(cc) = sweep_chunk_fwd<TB>(M, c, 16 * cc, tab);
            c = nx;
        }
        return;
    }
    if (LAYOUT == kRow && (len & 3) == 0) {
        uint32_t w = line.ld4(0);
        for (int u = 0; u < len; u += 4) {
            const uint32_t wn = u + 4 < len ? line.ld4(u + 4) : 0u;
            line.st4(u, sweep_word<TB, false>(M, w, u, tab));
            w = wn;
        }
        return;
    }
    if (LAYOUT == kStrided && (len & 3) == 0) {
        int q0 = line.ld(0), q1 = line.ld(1), q2 = line.ld(2), q3 = line.ld(3);
        for (int u = 0; u < len; u += 4) {
            int n0 = 0, n1 = 0, n2 = 0, n3 = 0;
            if (u + 4 < len) {
                n0 = line.ld(u + 4), n1 = line.ld(u + 5), n2 = line.ld(u + 6), n3 = line.ld(u + 7);
            }
            line.st(u, step_scaled<TB>(M, q0, u, tab) >> sh);
            line.st(u + 1, step_scaled<TB>(M, q1, u + 1, tab) >> sh);
            line.st(u + 2, step_scaled<TB>(M, q2, u + 2, tab) >> sh);
            line.st(u + 3, step_scaled<TB>(M, q3, u + 3, tab) >> sh);
            q0 = n0, q1 = n1, q2 = n2, q3 = n3;
        }
        return;
    }
    for (int u = 0; u < len; ++u) line.st(u, step_scaled<TB>(M, line.ld(u), u, tab) >> sh);
}

// Backward sweep in place: sweep position j = len - 1 - u.
template <int TB, int LAYOUT>
__device__ __forceinline__ void sweep_backward(int len, TileLine<LAYOUT> line, uint32_t tab) {
    constexpr int sh = SweepTable<TB>::kShift;
    uint32_t M = tab + SweepTable<TB>::kRow * kDistClamp;
    if (LAYOUT == kRowSwz) {
        const int nc = len >> 4;
        uint4 c = *line.chunk(nc - 1);
        for (int cc = nc - 1, j = 0; cc >= 0; --cc, j += 16) {
            const uint4 nx = cc > 0 ? *line.chunk(cc - 1) : make_uint4(0u, 0u, 0u, 0u);
            *line.chunk(cc) = sweep_chunk_bwd<TB>(M, c, j, tab);
            c = nx;
        }
        return;
    }
    if (LAYOUT == kRow && (len & 3) == 0) {
        uint32_t w = line.ld4(len - 4);
        for (int u0 = len - 4, j = 0; u0 >= 0; u0 -= 4, j += 4) {
            const uint32_t wn = u0 >= 4 ? line.ld4(u0 - 4) : 0u;
            line.st4(u0, sweep_word<TB, true>(M, w, j, tab));
            w = wn;
        }
        return;
    }
    if (LAYOUT == kStrided && (len & 3) == 0) {
        int q0 = line.ld(len - 1), q1 = line.ld(len - 2), q2 = line.ld(len - 3),
            q3 = line.ld(len - 4);
        for (int u = len - 1, j = 0; u >= 0; u -= 4, j += 4) {
            int n0 = 0, n1 = 0, n2 = 0, n3 = 0;
            if (u >= 4) {
                n0 = line.ld(u - 4), n1 = line.ld(u - 5), n2 = line.ld(u - 6), n3 = line.ld(u - 7);
            }
            line.st(u, step_scaled<TB>(M, q0, j, tab) >> sh);
            line.st(u - 1, step_scaled<TB>(M, q1, j + 1, tab) >> sh);
            line.st(u - 2, step_scaled<TB>(M, q2, j + 2, tab) >> sh);
            line.st(u - 3, step_scaled<TB>(M, q3, j + 3, tab) >> sh);
            q0 = n0, q1 = n1, q2 = n2, q3 = n3;
        }
        return;
    }
    for (int j = 0; j < len; ++j) {
        const int u = len - 1 - j;
        line.st(u, step_scaled<TB>(M, line.ld(u), j, tab) >> sh);
    }
}

// Warp-collective clear of a [256][32] table (16 B per lane per store).
template <int TB>
__device__ __forceinline__ void clear_table(uint8_t *tab_warp, int lane) {
    uint4 *t = reinterpret_cast<uint4 *>(tab_warp);
#pragma unroll
    for (int i = 0; i < 16 * TB; ++i) t[i * 32 + lane] = make_uint4(0u, 0u, 0u, 0u);
}

// ---- expand: partition occupancy -> {0, 255} planes ---------------------------------
// Thread = 16 consecutive blocks: it reads their mask words once and writes a
// 16-byte vector to every partition plane (coalesced 512 B per warp store).
struct MaskSrc {
    const uint32_t *mask;
    int words;
};

__global__ void __launch_bounds__(256)
    dt_expand_mask_kernel(MaskSrc src, int n, int64_t nb, uint8_t *__restrict__ pdms,
                          int64_t pitch) {
    const int64_t nchunks = ceil_div(nb, 16);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ch < nchunks; ch += stride) {
        const int64_t c0 = ch * 16;
        const int cnt = (int)min((int64_t)16, nb - c0);
        for (int w = 0; w < src.words; ++w) {
            uint32_t m[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) m[i] = i < cnt ? src.mask[(c0 + i) * src.words + w] : 0u;
            const int pend = min(32, n - w * 32);
            for (int pp = 0; pp < pend; ++pp) {
                uint32_t q[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    uint32_t v = 0;
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        v |= (((m[4 * k + b] >> pp) & 1u) ? 0u : 0xFFu) << (8 * b);
                    q[k] = v;
                }
                uint8_t *dst = pdms + (int64_t)(w * 32 + pp) * pitch + c0;
                if (cnt == 16) {
                    *reinterpret_cast<uint4 *>(dst) = make_uint4(q[0], q[1], q[2], q[3]);
                } else {
                    for (int i = 0; i < cnt; ++i) dst[i] = (uint8_t)(q[i >> 2] >> (8 * (i & 3)));
                }
            }
        }
    }
}

// Single map from a uint8 occupancy: byte == 0 -> 255, nonzero -> 0.
__global__ void __launch_bounds__(256)
    dt_expand_occ_kernel(const uint8_t *__restrict__ occ, int64_t nb, uint8_t *__restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nb; c += stride)
        out[c] = occ[c] ? 0 : 255;
}

// ---- warp-tile passes ----------------------------------------------------------------

// Is the warp's shared-memory tile (bytes [0, bytes), 16-byte aligned, bytes %
// 16 == 0) constant at 0 or at 255?  Every pass here maps such a tile to
// itself (no occupied block within reach / every block occupied), so the warp
// skips its sweeps and its write-back.  On config c's PDM build 45 % of the x
// pass's tiles and 20 % of the y pass's are (tools/exp/dt_tile_stats.py).
__device__ __forceinline__ bool tile_is_flat(const uint8_t *tile, int bytes, int lane) {
    uint32_t a = 0xFFFFFFFFu, o = 0;
    for (int i = lane * 16; i < bytes; i += 32 * 16) {
        const uint4 q = *reinterpret_cast<const uint4 *>(tile + i);
        a &= q.x & q.y & q.z & q.w;
        o |= q.x | q.y | q.z | q.w;
    }
    return __all_sync(0xFFFFFFFFu, a == 0xFFFFFFFFu) || __all_sync(0xFFFFFFFFu, o == 0u);
}

enum { kAxisX = 0, kAxisY = 1, kAxisZ = 2 };

// Optional fused epilogue of the last pass (z rows): the packed copy of the
// finished rows (csrc/packed.cu encoding: per 16-block chunk its min + 4-bit
// offsets), written while the rows are still in shared memory so no separate
// pass re-reads the PDMs.  nib == nullptr: off.
struct PackDst {
    uint8_t *nib;
    int64_t nib_pitch;
    uint8_t *base;
    int64_t base_pitch;
    unsigned int *bad;  // chunks spanning > 15 values (none for distance fields)
    uint16_t *tb;       // the merge's per-tile plane bounds [tiles][n] (may be null)
    int n;
};

__device__ __forceinline__ uint32_t hmin2_u(uint32_t a, uint32_t b) {
    __half2 r = __hmin2(*reinterpret_cast<const __half2 *>(&a),
                        *reinterpret_cast<const __half2 *>(&b));
    return *reinterpret_cast<uint32_t *>(&r);
}
__device__ __forceinline__ uint32_t hmax2_u(uint32_t a, uint32_t b) {
    __half2 r = __hmax2(*reinterpret_cast<const __half2 *>(&a),
                        *reinterpret_cast<const __half2 *>(&b));
    return *reinterpret_cast<uint32_t *>(&r);
}

// Pack one 16-byte chunk: bytes as fp16 1024 + v in 16-bit lanes (HMNMX2 on
// the FMA pipe) for min/max, offsets v - min (< 16, no borrow between bytes),
// then two nibble bytes per byte pair via shift/or and one PRMT per 8 blocks.
__device__ __forceinline__ uint2 pack_chunk(uint4 q, uint32_t &mn, uint32_t &mx,
                                            unsigned int &nbad) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    uint32_t lo = 0x64FF64FFu, hi = 0x64006400u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t e = __byte_perm(w[i], 0x64646464u, 0x4240);
        const uint32_t o = __byte_perm(w[i], 0x64646464u, 0x4341);
        lo = hmin2_u(lo, hmin2_u(e, o));
        hi = hmax2_u(hi, hmax2_u(e, o));
    }
    lo = hmin2_u(lo, __byte_perm(lo, 0u, 0x1032));
    hi = hmax2_u(hi, __byte_perm(hi, 0u, 0x1032));
    mn = lo & 0xFFu;
    mx = hi & 0xFFu;
    nbad += mx - mn > 15u;
    const uint32_t mb = mn * 0x01010101u;
    uint32_t t[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t d = w[i] - mb;  // bytes v - min, each < 16 for a valid chunk
        t[i] = d | (d >> 4);           // byte 0: b0 | b1 << 4, byte 2: b2 | b3 << 4
    }
    return make_uint2(__byte_perm(t[0], t[1], 0x6420), __byte_perm(t[2], t[3], 0x6420));
}

template <int LMAX, int AXIS, bool kDist1D, bool kSweep>
__global__ void __launch_bounds__(256)
    dt_tile_kernel(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *__restrict__ pdms,
                   int64_t pitch, int sstride, int64_t tiles, PackDst pk) {
    static_assert(!kSweep || (LMAX <= 512 && !kDist1D), "sweep envelope: lines <= 512");
    constexpr int TB = LMAX > 256 ? 2 : 1;  // sweep table entry bytes
    extern __shared__ __align__(16) uint8_t s_tiles[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wpc = blockDim.x >> 5;
    constexpr bool kRows = AXIS == kAxisZ;  // contiguous lines
    const int L = (int)(AXIS == kAxisX ? bx : (AXIS == kAxisY ? by : bz));
    const int64_t S = AXIS == kAxisX ? by * bz : bz;  // element stride of strided lines
    const size_t tile_bytes = kRows ? 32 * (size_t)sstride : 32 * (size_t)L;
    uint8_t *s = s_tiles + (size_t)warp * tile_bytes;
    // Per-warp scratch after all tiles: the sweep's [256][32] table.
    uint8_t *tab_warp = s_tiles + (size_t)wpc * tile_bytes + (size_t)warp * SweepTable<TB>::kBytes;
    const int64_t zblocks = ceil_div(bz, 32);
    const bool vec = (bz & 3) == 0;
    // Swizzled 16-byte row tiles (the host sets sstride == L only when L is
    // 128, 256 or 512 and rows are 16-byte aligned).
    const bool swz = kSweep && kRows && sstride == L && (L & 127) == 0 && (L & (L - 1)) == 0;
    const int cpr = L >> 4, csh = __ffs(cpr) - 1;  // chunks per row (power of 2 if swz)
    // Tile t: rows -> 32 consecutive (x, y) rows of partition p; strided ->
    // 32 consecutive z of one line family (p, outer).
    auto tile_at = [&](int64_t tt, int &nl) -> uint8_t * {
        if (kRows) {
            const int64_t rows = bx * by, per_p = ceil_div(rows, 32);
            const int64_t r0 = (tt % per_p) * 32;
            nl = (int)min((int64_t)32, rows - r0);
            return pdms + (tt / per_p) * pitch + r0 * bz;
        }
        const int64_t outer_n = AXIS == kAxisX ? by : bx;
        const int64_t po = tt / zblocks, z0 = (tt % zblocks) * 32;
        const int64_t o = po % outer_n;
        nl = (int)min((int64_t)32, bz - z0);
        return pdms + (po / outer_n) * pitch + (AXIS == kAxisX ? o * bz : o * by * bz) + z0;
    };
    for (int64_t t = (int64_t)blockIdx.x * wpc + warp; t < tiles; t += (int64_t)gridDim.x * wpc) {
        int nlines;
        uint8_t *g = tile_at(t, nlines);
        if (kRows) {
            if (swz) {
                for (int i = lane; i < nlines << csh; i += 32) {
                    const int r = i >> csh, c = i & (cpr - 1);
                    cpa::copy16(s + r * L + ((c ^ (r & 7)) << 4), g + (int64_t)r * bz + 16 * c);
                }
            } else if (vec) {
                const int words = L >> 2;  // rows outer: no division per word
                for (int r = 0; r < nlines; ++r)
                    for (int w = lane; w < words; w += 32)
                        cpa::copy4(s + r * sstride + 4 * w, g + (int64_t)r * bz + 4 * w);
            } else {
                for (int i = lane; i < nlines * L; i += 32) {
                    const int r = i / L, u = i - r * L;
                    s[r * sstride + u] = g[(int64_t)r * bz + u];
                }
            }
        } else {
            if (nlines == 32 && (bz & 15) == 0) {  // 2 lanes per 32-byte row
                for (int i = lane; i < L * 2; i += 32) {
                    const int u = i >> 1, w = i & 1;
                    cpa::copy16(s + u * 32 + 16 * w, g + (int64_t)u * S + 16 * w);
                }
            } else if (nlines == 32 && vec) {  // 8 lanes per 32-byte row
                for (int i = lane; i < L * 8; i += 32) {
                    const int u = i >> 3, w = i & 7;
                    cpa::copy4(s + u * 32 + 4 * w, g + (int64_t)u * S + 4 * w);
                }
            } else {
                for (int u = 0; u < L; ++u)
                    if (lane < nlines) s[u * 32 + lane] = g[(int64_t)u * S + lane];
            }
        }
        // Tile loads are cp.async (no register staging), so every load of the
        // tile is in flight at once instead of a few per dependent wait.
        cpa::commit();
        cpa::wait<0>();
        __syncwarp();
        uint8_t *line = kRows ? s + lane * sstride : s + lane;
        const int es = kRows ? 1 : 32;
        auto ld = [&](int u) -> int { return line[u * es]; };
        auto st = [&](int u, int v) { line[u * es] = (uint8_t)v; };
        // a flat tile (all 0 / all 255) is its own result: no sweep, no write-back
        // (the z pass still packs it)
        const bool flat = kSweep && nlines == 32 && (!kRows || swz) &&
                          tile_is_flat(s, (int)tile_bytes, lane);
        if (kSweep && !flat) {
            const uint32_t tab = smem_addr(tab_warp + TB * lane);  // lane column
            for (int dir = 0; dir < 2; ++dir) {
                clear_table<TB>(tab_warp, lane);
                __syncwarp();
                if (lane < nlines) {
                    if (!kRows) {
                        const TileLine<kStrided> tl{line, lane};
                        dir == 0 ? sweep_forward<TB>(L, tl, tab) : sweep_backward<TB>(L, tl, tab);
                    } else if (swz) {
                        const TileLine<kRowSwz> tl{line, lane};
                        dir == 0 ? sweep_forward<TB>(L, tl, tab) : sweep_backward<TB>(L, tl, tab);
                    } else {
                        const TileLine<kRow> tl{line, lane};
                        dir == 0 ? sweep_forward<TB>(L, tl, tab) : sweep_backward<TB>(L, tl, tab);
                    }
                }
                __syncwarp();
            }
        } else if (!kSweep && lane < nlines) {
            if (kDist1D)
                dist1d_line(L, ld, st);
            else
                cone_line<LMAX>(L, ld, st);
        }
        __syncwarp();
        if (kRows) {
            if (flat) {
                // unchanged rows: nothing to write back
            } else if (swz) {
                for (int i = lane; i < nlines << csh; i += 32) {
                    const int r = i >> csh, c = i & (cpr - 1);
                    *reinterpret_cast<uint4 *>(g + (int64_t)r * bz + 16 * c) =
                        *reinterpret_cast<const uint4 *>(s + r * L + ((c ^ (r & 7)) << 4));
                }
            } else if (vec) {
                const int words = L >> 2;
                for (int r = 0; r < nlines; ++r)
                    for (int w = lane; w < words; w += 32)
                        *reinterpret_cast<uint32_t *>(g + (int64_t)r * bz + 4 * w) =
                            *reinterpret_cast<const uint32_t *>(s + r * sstride + 4 * w);
            } else {
                for (int i = lane; i < nlines * L; i += 32) {
                    const int r = i / L, u = i - r * L;
                    g[(int64_t)r * bz + u] = s[r * sstride + u];
                }
            }
            if (kSweep && swz && pk.nib != nullptr) {
                // The rows are final: pack them.  Staging reuses the sweep's
                // table area (nibbles [32][L/2 + 8], bases [32][L/16 + 4]).
                const int nst = L / 2 + 8, bst = L / 16 + 4;
                uint8_t *sn = tab_warp, *sb = tab_warp + 32 * nst;
                unsigned int nbad = 0;
                uint32_t rlo = 255, rhi = 0;  // the row's min / max
                if (lane < nlines) {
                    const TileLine<kRowSwz> tl{line, lane};
                    for (int c = 0; c < cpr; ++c) {
                        uint32_t mn, mx;
                        const uint2 pw = pack_chunk(*tl.chunk(c), mn, mx, nbad);
                        *reinterpret_cast<uint2 *>(sn + lane * nst + 8 * c) = pw;
                        sb[lane * bst + c] = (uint8_t)mn;
                        rlo = min(rlo, mn);
                        rhi = max(rhi, mx);
                    }
                }
                if (nbad) atomicAdd(pk.bad, nbad);
                __syncwarp();
                // rows r0.. of plane p are contiguous in the packed planes too
                const int64_t rows = bx * by, per_p = ceil_div(rows, 32);
                const int64_t p = t / per_p, r0 = (t % per_p) * 32;
                if (pk.tb != nullptr) {
                    // the merge's tile bounds: a 1024-block tile is rpt = 1024 / L
                    // whole rows (r0 is a multiple of 32 >= rpt), reduced over lanes
                    const int rpt = 1024 / L;
                    for (int o = 1; o < rpt; o <<= 1) {
                        rlo = min(rlo, __shfl_xor_sync(0xFFFFFFFFu, rlo, o));
                        rhi = max(rhi, __shfl_xor_sync(0xFFFFFFFFu, rhi, o));
                    }
                    if ((lane & (rpt - 1)) == 0 && lane < nlines)
                        pk.tb[((r0 + lane) / rpt) * pk.n + p] = (uint16_t)(rlo | (rhi << 8));
                }
                uint8_t *gn = pk.nib + p * pk.nib_pitch + r0 * (L / 2);
                uint8_t *gb = pk.base + p * pk.base_pitch + r0 * (L / 16);
                const int nu = L / 16;  // 8-byte nibble units (= chunks) per row
                for (int i = lane; i < nlines * nu; i += 32) {
                    const int r = i / nu, c = i - r * nu;
                    *reinterpret_cast<uint2 *>(gn + 8 * (int64_t)i) =
                        *reinterpret_cast<const uint2 *>(sn + r * nst + 8 * c);
                }
                const int bu = L / 64;  // 4-byte base units per row
                for (int i = lane; i < nlines * bu; i += 32) {
                    const int r = i / bu, c = i - r * bu;
                    *reinterpret_cast<uint32_t *>(gb + 4 * (int64_t)i) =
                        *reinterpret_cast<const uint32_t *>(sb + r * bst + 4 * c);
                }
            }
        } else if (!flat) {
            if (nlines == 32 && (bz & 15) == 0) {
                for (int i = lane; i < L * 2; i += 32) {
                    const int u = i >> 1, w = i & 1;
                    *reinterpret_cast<uint4 *>(g + (int64_t)u * S + 16 * w) =
                        *reinterpret_cast<const uint4 *>(s + u * 32 + 16 * w);
                }
            } else if (nlines == 32 && vec) {
                for (int i = lane; i < L * 8; i += 32) {
                    const int u = i >> 3, w = i & 7;
                    *reinterpret_cast<uint32_t *>(g + (int64_t)u * S + 4 * w) =
                        *reinterpret_cast<const uint32_t *>(s + u * 32 + 4 * w);
                }
            } else {
                for (int u = 0; u < L; ++u)
                    if (lane < nlines) g[(int64_t)u * S + lane] = s[u * 32 + lane];
            }
        }
        __syncwarp();
    }
}

// ---- sweep passes with the lines held in tensor memory -------------------------
// dt_tile_kernel keeps every warp's tile (8 KB) AND its sweep table (8 KB) in
// shared memory, so an SM holds 14 sweeping warps -- and the sweep is bound
// by the latency of its table lookup chain (ncu: 54-66 % issue active,
// short-scoreboard and wait stalls).  Here a warp's 32 lines live in TMEM
// (the tensor cores' 256 KB per SM, idle in this pass): each lane's line is
// 64 private 32-bit columns of its TMEM lane (tcgen05.st / tcgen05.ld of 16
// columns = 64 elements at a time), so the warp needs only one 8 KB
// shared-memory buffer -- the cp.async staging of its tile, then the table
// of each sweep, then the staging of the write-back -- and 24 to 28 warps
// sweep per SM.  Lines of 256 or 512 blocks in full 32-line tiles (config c's
// 256^3 and config d's 512^3 block grids); everything else runs
// dt_tile_kernel.
namespace tmem {

__device__ __forceinline__ void alloc(uint32_t *dst, uint32_t cols) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(dst)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t cols) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
                 : "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 16 consecutive columns of the thread's lane <- w[0..16)
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&w)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
        "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]),
        "r"(w[15])
        : "memory");
}
// w[0..16) <- 16 consecutive columns; waits for this thread's earlier stores
// first and for the load itself before returning (one asm block, so no use
// of w can be scheduled ahead of the wait).
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&w)[16]) {
    asm volatile(
        "tcgen05.wait::st.sync.aligned;\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
          "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]),
          "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

}  // namespace tmem

// Warps per CTA of the TMEM sweep (warp w uses TMEM lane quarter w % 4 and
// column group w / 4).  Two shapes: 4 warps per CTA, 6 CTAs per SM (3 for
// L = 512) -- 24 (12) warps; or one CTA per SM filling the shared memory
// with 28 (14) warps' tables, used for jobs that give every warp several
// tiles (a PDM set build: config c y + z 0.964 -> 0.946 ms, config d 9.47 ->
// 8.67 ms).  The one-CTA shape slowed single-map passes (the fused
// recompute, 0.56 -> 0.62 ms), which keep the small CTAs.
template <int L>
constexpr int tmem_big_warps() {
    return L == 256 ? 28 : 14;
}
// TMEM columns a CTA allocates: a lane's line is L / 4 columns, one column
// group per 4 warps, rounded up to a power of two (>= 32).
template <int L, int W>
constexpr int tmem_cols() {
    constexpr int need = ((W + 3) / 4) * (L / 4);
    int c = 32;
    while (c < need) c *= 2;
    return c;
}
// CTAs per SM from shared memory (one 32 L-byte buffer per warp + the 1 KB
// per-CTA reserve, 228 KB per SM) and the 512 TMEM columns.
template <int L, int W>
constexpr int tmem_ctas() {
    constexpr int by_smem = (228 * 1024) / (W * 32 * L + 1024);
    constexpr int by_tmem = 512 / tmem_cols<L, W>();
    return by_smem < by_tmem ? by_smem : by_tmem;
}

// 4 x 4 byte transpose inside each quad of lanes: lane 4g + j holds row j
// (bytes = columns 0..3) on entry and column j (bytes = rows 0..3) on exit.
__device__ __forceinline__ uint32_t quad_transpose(uint32_t a, int lane) {
    const uint32_t p = __shfl_xor_sync(0xFFFFFFFFu, a, 1);
    // even lanes: [a.b0, p.b0, a.b2, p.b2]; odd: [p.b1, a.b1, p.b3, a.b3]
    const uint32_t t = __byte_perm(a, p, (lane & 1) ? 0x3715u : 0x6240u);
    const uint32_t q = __shfl_xor_sync(0xFFFFFFFFu, t, 2);
    // lanes 0, 1 of the quad: [t.b0, t.b1, q.b0, q.b1]; lanes 2, 3: [q.b2, q.b3, t.b2, t.b3]
    return __byte_perm(t, q, (lane & 2) ? 0x3276u : 0x5410u);
}

template <int AXIS, int L, int W>
__global__ void __launch_bounds__(32 * W, tmem_ctas<L, W>())
    dt_tmem_kernel(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *__restrict__ pdms,
                   int64_t pitch, int64_t tiles, PackDst pk, unsigned long long *next) {
    static_assert(L == 256 || L == 512, "TMEM sweep: lines of 256 or 512");
    constexpr int NC = L / 64;            // TMEM chunks of 16 columns
    constexpr int kCols = L / 4;          // a lane's line: L bytes
    constexpr int TB = L > 256 ? 2 : 1;   // sweep table entry bytes
    constexpr int CPR = L / 16, CSH = L == 256 ? 4 : 5;  // 16-byte chunks per row
    constexpr bool kRows = AXIS == kAxisZ;
    static_assert(SweepTable<TB>::kBytes == 32 * L, "table and tile share the buffer");
    extern __shared__ __align__(16) uint8_t s_dyn[];
    __shared__ uint32_t s_taddr;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) tmem::alloc(&s_taddr, tmem_cols<L, W>());
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const uint32_t tbase = s_taddr;
    const uint32_t taddr =
        tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * kCols);
    uint8_t *s = s_dyn + (size_t)warp * 32 * L;
    const uint32_t tab = smem_addr(s + TB * lane);  // the sweep table's lane column
    const int64_t S = bz;                      // y lines: element stride
    const int64_t zblocks = bz / 32;
    // Tiles are handed out by an atomic counter, claimed one tile ahead: a
    // tile is ~16k chain steps per lane and flat tiles are skipped, so a
    // static split left a warp's CTA-mates idle at the end (ncu: barrier
    // stalls at the dealloc sync).
    auto claim = [&]() -> int64_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(next, 1ull);
        return (int64_t)__shfl_sync(0xFFFFFFFFu, v, 0);
    };
    int64_t t_next = claim();
    for (;;) {
        const int64_t t = t_next;
        if (t >= tiles) break;
        t_next = claim();
        uint8_t *g;
        if (kRows) {
            const int64_t per_p = bx * by / 32;
            g = pdms + (t / per_p) * pitch + (t % per_p) * 32 * bz;
        } else {
            const int64_t po = t / zblocks, z0 = (t % zblocks) * 32;
            g = pdms + (po / bx) * pitch + (po % bx) * by * bz + z0;
        }
        // stage the tile (rows: 16-byte chunks swizzled by row; y lines: [u][32])
        if (kRows) {
            for (int i = lane; i < 32 * CPR; i += 32) {
                const int r = i >> CSH, c = i & (CPR - 1);
                cpa::copy16(s + r * L + ((c ^ (r & 7)) << 4), g + (int64_t)r * bz + 16 * c);
            }
        } else {
            for (int i = lane; i < L * 2; i += 32) {
                const int u = i >> 1, w = i & 1;
                cpa::copy16(s + u * 32 + 16 * w, g + (int64_t)u * S + 16 * w);
            }
        }
        cpa::commit();
        cpa::wait<0>();
        __syncwarp();
        const bool flat = tile_is_flat(s, 32 * L, lane);
        if (!kRows && flat) {  // no change, nothing to pack
            __syncwarp();
            continue;
        }
        // the lane's line -> TMEM (words of 4 consecutive elements)
#pragma unroll 1
        for (int cc = 0; cc < NC; ++cc) {
            uint32_t w[16];
            if (kRows) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int c = 4 * cc + q;
                    const uint4 v = *reinterpret_cast<const uint4 *>(
                        s + lane * L + ((c ^ (lane & 7)) << 4));
                    w[4 * q] = v.x, w[4 * q + 1] = v.y, w[4 * q + 2] = v.z, w[4 * q + 3] = v.w;
                }
            } else {
                // [u][32] tile -> the lane's column: each lane loads the word of
                // row u + (lane & 3) holding columns 4 (lane >> 2) .. +3, and a
                // 4 x 4 byte transpose inside each lane quad (two shuffles, two
                // byte permutes) hands lane l column l of the 4 rows
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int u = 64 * cc + 4 * i;
                    const uint32_t a = *reinterpret_cast<const uint32_t *>(
                        s + (u + (lane & 3)) * 32 + 4 * (lane >> 2));
                    w[i] = quad_transpose(a, lane);
                }
            }
            tmem::st16(taddr + 16 * cc, w);
        }
        tmem::wait_st();
        __syncwarp();  // the staged tile is consumed: the buffer becomes the table
        if (!flat) {
            // forward sweep: L[u] = min_{i<=u} max(u - i, g[i])
            clear_table<TB>(s, lane);
            __syncwarp();
            {
                uint32_t M = tab + SweepTable<TB>::kRow * kDistClamp;
#pragma unroll 1
                for (int cc = 0; cc < NC; ++cc) {
                    uint32_t w[16];
                    tmem::ld16(taddr + 16 * cc, w);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        w[i] = sweep_word<TB, false>(M, w[i], 64 * cc + 4 * i, tab);
                    tmem::st16(taddr + 16 * cc, w);
                }
            }
            __syncwarp();
            clear_table<TB>(s, lane);
            __syncwarp();
            {   // backward sweep over L gives the envelope, in place
                uint32_t M = tab + SweepTable<TB>::kRow * kDistClamp;
#pragma unroll 1
                for (int cc = NC - 1; cc >= 0; --cc) {
                    uint32_t w[16];
                    tmem::ld16(taddr + 16 * cc, w);
#pragma unroll
                    for (int i = 15; i >= 0; --i)
                        w[i] = sweep_word<TB, true>(M, w[i], L - 4 - (64 * cc + 4 * i), tab);
                    tmem::st16(taddr + 16 * cc, w);
                }
            }
            __syncwarp();
        }
        if (!kRows) {
            // transpose back through the buffer, then coalesced 16-byte stores
#pragma unroll 1
            for (int cc = 0; cc < NC; ++cc) {
                uint32_t w[16];
                tmem::ld16(taddr + 16 * cc, w);
#pragma unroll
                for (int i = 0; i < 16; ++i) {  // the same transpose, back to rows
                    const int u = 64 * cc + 4 * i;
                    *reinterpret_cast<uint32_t *>(s + (u + (lane & 3)) * 32 + 4 * (lane >> 2)) =
                        quad_transpose(w[i], lane);
                }
            }
            __syncwarp();
            for (int i = lane; i < L * 2; i += 32) {
                const int u = i >> 1, w = i & 1;
                *reinterpret_cast<uint4 *>(g + (int64_t)u * S + 16 * w) =
                    *reinterpret_cast<const uint4 *>(s + u * 32 + 16 * w);
            }
            __syncwarp();
            continue;
        }
        // rows: write back (unless flat) through the buffer, swizzled like the
        // load, so the tile's 32 contiguous rows leave as 512-byte warp stores
        // (lane-per-row 16-byte stores kept L1 80 % busy), then pack (staging
        // in the buffer too)
        if (!flat) {
#pragma unroll 1
            for (int cc = 0; cc < NC; ++cc) {
                uint32_t w[16];
                tmem::ld16(taddr + 16 * cc, w);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int c = 4 * cc + q;
                    *reinterpret_cast<uint4 *>(s + lane * L + ((c ^ (lane & 7)) << 4)) =
                        make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
                }
            }
            __syncwarp();
            for (int i = lane; i < 32 * CPR; i += 32) {
                const int r = i >> CSH, c = i & (CPR - 1);
                *reinterpret_cast<uint4 *>(g + (int64_t)r * bz + 16 * c) =
                    *reinterpret_cast<const uint4 *>(s + r * L + ((c ^ (r & 7)) << 4));
            }
            __syncwarp();
        }
        const int nst = L / 2 + 8, bst = L / 16 + 4;
        uint8_t *sn = s, *sb = s + 32 * nst;
        unsigned int nbad = 0;
        uint32_t rlo = 255, rhi = 0;
#pragma unroll 1
        for (int cc = 0; cc < NC && pk.nib != nullptr; ++cc) {
            uint32_t w[16];
            tmem::ld16(taddr + 16 * cc, w);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
                const int c = 4 * cc + q;
                {
                    uint32_t mn, mx;
                    const uint2 pw = pack_chunk(v, mn, mx, nbad);
                    *reinterpret_cast<uint2 *>(sn + lane * nst + 8 * c) = pw;
                    sb[lane * bst + c] = (uint8_t)mn;
                    rlo = min(rlo, mn);
                    rhi = max(rhi, mx);
                }
            }
        }
        if (pk.nib != nullptr) {
            if (nbad) atomicAdd(pk.bad, nbad);
            __syncwarp();
            const int64_t rows = bx * by, per_p = rows / 32;
            const int64_t p = t / per_p, r0 = (t % per_p) * 32;
            if (pk.tb != nullptr) {  // 1024-block tile = 4 rows of 256
                constexpr int rpt = 1024 / L;
#pragma unroll
                for (int o = 1; o < rpt; o <<= 1) {
                    rlo = min(rlo, __shfl_xor_sync(0xFFFFFFFFu, rlo, o));
                    rhi = max(rhi, __shfl_xor_sync(0xFFFFFFFFu, rhi, o));
                }
                if ((lane & (rpt - 1)) == 0)
                    pk.tb[((r0 + lane) / rpt) * pk.n + p] = (uint16_t)(rlo | (rhi << 8));
            }
            uint8_t *gn = pk.nib + p * pk.nib_pitch + r0 * (L / 2);
            uint8_t *gb = pk.base + p * pk.base_pitch + r0 * (L / 16);
            constexpr int nu = L / 16;
            for (int i = lane; i < 32 * nu; i += 32) {
                const int r = i / nu, c = i - r * nu;
                *reinterpret_cast<uint2 *>(gn + 8 * (int64_t)i) =
                    *reinterpret_cast<const uint2 *>(sn + r * nst + 8 * c);
            }
            constexpr int bu = L / 64;
            for (int i = lane; i < 32 * bu; i += 32) {
                const int r = i / bu, c = i - r * bu;
                *reinterpret_cast<uint32_t *>(gb + 4 * (int64_t)i) =
                    *reinterpret_cast<const uint32_t *>(sb + r * bst + 4 * c);
            }
        }
        __syncwarp();
    }
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    if (warp == 0) tmem::dealloc(tbase, tmem_cols<L, W>());
}

// Lines longer than 1024 blocks: one thread per line straight from global
// memory (correct for any length up to 4095, slower).
template <int AXIS, bool kDist1D>
__global__ void __launch_bounds__(128)
    dt_line_kernel(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *__restrict__ pdms,
                   int64_t pitch) {
    const int L = (int)(AXIS == kAxisX ? bx : (AXIS == kAxisY ? by : bz));
    const int64_t S = AXIS == kAxisX ? by * bz : (AXIS == kAxisY ? bz : 1);
    const int64_t per_p = bx * by * bz / L;
    const int64_t lines = (int64_t)n * per_p;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < lines; l += stride) {
        const int p = (int)(l / per_p);
        const int64_t r = l % per_p;
        int64_t base;
        if (AXIS == kAxisX)
            base = r;  // r = y * bz + z
        else if (AXIS == kAxisY)
            base = (r / bz) * by * bz + (r % bz);  // r = x * bz + z
        else
            base = r * bz;  // r = x * by + y
        uint8_t *line = pdms + (int64_t)p * pitch + base;
        auto ld = [&](int u) -> int { return line[(int64_t)u * S]; };
        auto st = [&](int u, int v) { line[(int64_t)u * S] = (uint8_t)v; };
        if (kDist1D)
            dist1d_line(L, ld, st);
        else
            cone_line<4096>(L, ld, st);
    }
}

// ---- x pass, wide tiles: 1-D distance of 2 lines per lane in 16-bit lanes -------
// The 1-D distance has no lookup in its chain (run = nonzero ? run + 1 : 0),
// so it is instruction bound; each lane runs 2 adjacent z lines at once in
// one u16x2 register.  Runs are not clamped while sweeping (they stay <= 255
// + L <= 511, inside the 9-bit lane mask) and are clamped with one
// VIMNMX.U16x2 on output.  Lines <= 256.  (4 lines per lane on 128-z tiles
// measured 0.49 vs 0.46 ms for expand + pass x at config c: half the
// resident warps.)
__device__ __forceinline__ uint32_t nonzero16(uint32_t x) {  // u16x2 lanes <= 255
    return (((x + 0x00FF00FFu) >> 8) & 0x00010001u) * 0x1FFu;  // 0x1FF where x != 0
}

// Tile: [u][64 z] bytes per warp (16 KB for L = 256), lane l owns z0 + 2l,
// z0 + 2l + 1.  The forward sweep relies on its input being the expand
// kernels' {0, 255} planes (mask = byte * 0x101); the backward sweep tests its
// general input.
__global__ void __launch_bounds__(256)
    dt_dist1d_wide_kernel(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *__restrict__ pdms,
                           int64_t pitch, int64_t tiles) {
    extern __shared__ __align__(16) uint8_t s_wide[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpc = blockDim.x >> 5;
    const int L = (int)bx;
    const int64_t S = by * bz;
    uint8_t *s = s_wide + (size_t)warp * 64 * L;
    uint16_t *col = reinterpret_cast<uint16_t *>(s) + lane;  // element pair u at col[32 u]
    const int64_t zq = ceil_div(bz, 64);
    for (int64_t t = (int64_t)blockIdx.x * wpc + warp; t < tiles; t += (int64_t)gridDim.x * wpc) {
        const int64_t py = t / zq, z0 = (t % zq) * 64;
        const int nz = (int)min((int64_t)64, bz - z0);  // multiple of 16 (bz % 16 == 0)
        uint8_t *g = pdms + (py / by) * pitch + (py % by) * bz + z0;
        for (int i = lane; i < L * 4; i += 32) {
            const int u = i >> 2, c = i & 3;
            if (16 * c < nz) cpa::copy16(s + u * 64 + 16 * c, g + (int64_t)u * S + 16 * c);
        }
        cpa::commit();
        cpa::wait<0>();
        __syncwarp();
        if (nz == 64 && tile_is_flat(s, 64 * L, lane)) continue;  // all 0 or all 255
        if (2 * lane < nz) {
            uint32_t r = 0x00FF00FFu;  // "no occupied block yet" = 255
            uint32_t w = col[0];
            for (int u = 0; u < L; ++u) {
                const uint32_t wn = u + 1 < L ? col[32 * (u + 1)] : 0u;
                const uint32_t x = __byte_perm(w, 0u, 0x4140);  // bytes -> u16x2 lanes
                r = (r + 0x00010001u) & (x * 0x101u);          // {0, 255} -> {0, 0xFFFF}
                col[32 * u] = (uint16_t)__byte_perm(__vminu2(r, 0x00FF00FFu), 0u, 0x0020);
                w = wn;
            }
            r = 0x00FF00FFu;
            w = col[32 * (L - 1)];
            for (int u = L - 1; u >= 0; --u) {
                const uint32_t wn = u > 0 ? col[32 * (u - 1)] : 0u;
                const uint32_t f = __byte_perm(w, 0u, 0x4140);
                r = (r + 0x00010001u) & nonzero16(f);
                col[32 * u] = (uint16_t)__byte_perm(__vminu2(r, f), 0u, 0x0020);
                w = wn;
            }
        }
        __syncwarp();
        for (int i = lane; i < L * 4; i += 32) {
            const int u = i >> 2, c = i & 3;
            if (16 * c < nz)
                *reinterpret_cast<uint4 *>(g + (int64_t)u * S + 16 * c) =
                    *reinterpret_cast<const uint4 *>(s + u * 64 + 16 * c);
        }
        __syncwarp();
    }
}

// ---- expand + x pass in one kernel, from the partition mask --------------------
// dt_expand_mask_kernel writes every {0, 255} plane (n B bytes) and the x pass
// reads them back: ~1 GB of DRAM traffic at config c for what is a function
// of the 4 B mask word per block.  Here a CTA stages the mask words of one
// (y, 32-z) column of x lines, [x][32 z] (32 KB, every partition's bits),
// ORs/ANDs them to find the partitions whose lines are all empty / all
// occupied (written as constant rows by the whole CTA, no sweep), and its 8
// warps claim the other partitions one at a time (a shared counter: a static
// split left warps waiting at the column barrier) and run their lines' 1-D
// distance from the mask bits: lane l line z0 + l, forward run into a [x][32]
// byte tile, backward run min'ed into it, then 16-byte row stores.  Config c:
// 0.29 / 0.37 ms (voxel / range_apron masks) vs 0.30 / 0.45 ms for expand +
// pass x, 0.58 instead of ~1.6 GB of DRAM traffic.  Masks of one word per
// block (n <= 32), lines <= 512, bz % 32 == 0; PDM_DT_XMASK=0: expand + x.
// Measured and rejected: the forward runs parked in TMEM instead of the byte
// tile, backward results stored straight to HBM (one 32-byte sector per warp
// store), 24-32 warps per SM: 0.34 / 0.47 ms -- the byte-wide global stores
// cost more than the occupancy bought.
constexpr int kXMaskWarps = 8;

__global__ void __launch_bounds__(32 * kXMaskWarps, 2)
    dt_x_mask_kernel(const uint32_t *__restrict__ mask, int n, int64_t bx, int64_t by,
                     int64_t bz, uint8_t *__restrict__ pdms, int64_t pitch, int64_t tiles,
                     unsigned long long *next) {
    extern __shared__ __align__(16) uint8_t s_xm[];
    const int L = (int)bx;
    uint32_t *sm = reinterpret_cast<uint32_t *>(s_xm);                 // [L][32] mask words
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t *so = s_xm + (size_t)L * 128 + (size_t)warp * L * 32;     // [L][32] this warp's lines
    __shared__ uint32_t s_red[2][kXMaskWarps];
    __shared__ int s_next;  // next mixed partition of the column to claim
    const int64_t zq = bz / 32, S = by * bz;
    // columns claimed from a counter (the mixed partitions per column vary, so
    // a static split left CTAs idle at the end); next == nullptr: static
    __shared__ long long s_col;
    auto claim = [&](int64_t cur) {
        __syncthreads();
        if (threadIdx.x == 0)
            s_col = next ? (long long)atomicAdd(next, 1ull) : (long long)(cur + gridDim.x);
        __syncthreads();
        return (int64_t)s_col;
    };
    for (int64_t t = claim((int64_t)blockIdx.x - gridDim.x); t < tiles; t = claim(t)) {
        const int64_t y = t / zq, z0 = (t % zq) * 32;
        const uint32_t *src = mask + y * bz + z0;
        for (int i = threadIdx.x; i < L * 8; i += blockDim.x) {
            const int x = i >> 3, c = i & 7;
            cpa::copy16(sm + x * 32 + 4 * c, src + (int64_t)x * S + 4 * c);
        }
        cpa::commit();
        if (threadIdx.x == 0) s_next = 0;
        cpa::wait<0>();
        __syncthreads();
        uint32_t any = 0, all = 0xFFFFFFFFu;
        for (int i = threadIdx.x; i < L * 32; i += blockDim.x) {
            any |= sm[i];
            all &= sm[i];
        }
        any = __reduce_or_sync(0xFFFFFFFFu, any);
        all = __reduce_and_sync(0xFFFFFFFFu, all);
        if (lane == 0) s_red[0][warp] = any, s_red[1][warp] = all;
        __syncthreads();
        any = 0, all = 0xFFFFFFFFu;
#pragma unroll
        for (int w = 0; w < kXMaskWarps; ++w) any |= s_red[0][w], all &= s_red[1][w];
        const uint32_t nmask = n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1u);
        const uint32_t mixed = any & ~all & nmask;  // partitions whose lines need the sweep
        // constant partitions (every line 255 / 0): row stores split over the warps
        const uint32_t flat = nmask & ~mixed;
        for (int i = threadIdx.x; i < __popc(flat) * L * 2; i += blockDim.x) {
            const int q = i / (L * 2), rr = i - q * L * 2;
            uint32_t fm = flat;
            for (int j = 0; j < q; ++j) fm &= fm - 1;
            const int p = __ffs(fm) - 1;
            const uint32_t v = ((any >> p) & 1u) ? 0u : 0xFFFFFFFFu;
            *reinterpret_cast<uint4 *>(pdms + (int64_t)p * pitch + y * bz + z0 +
                                       (int64_t)(rr >> 1) * S + 16 * (rr & 1)) =
                make_uint4(v, v, v, v);
        }
        // mixed partitions: claimed by the warps one at a time
        for (;;) {
            int j = 0;
            if (lane == 0) j = atomicAdd(&s_next, 1);
            j = __shfl_sync(0xFFFFFFFFu, j, 0);
            if (j >= __popc(mixed)) break;
            uint32_t mm = mixed;
            for (int i = 0; i < j; ++i) mm &= mm - 1;
            const int p = __ffs(mm) - 1;
            uint8_t *dst = pdms + (int64_t)p * pitch + y * bz + z0;
            const uint32_t *col = sm + lane;
            uint8_t *oc = so + lane;
            const uint32_t bit = 1u << p;
            // batches of 8 rows: the shared loads of a batch are issued before
            // its stores (the compiler cannot tell the two tiles apart)
            constexpr int kB = 8;
            const int L8 = L & ~(kB - 1);
            uint32_t r = kDistClamp;  // "no occupied block yet"
            for (int x0 = 0; x0 < L8; x0 += kB) {
                uint32_t w[kB];
#pragma unroll
                for (int j = 0; j < kB; ++j) w[j] = col[32 * (x0 + j)];
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    r = (w[j] & bit) ? 0u : min(r + 1u, (uint32_t)kDistClamp);
                    w[j] = r;
                }
#pragma unroll
                for (int j = 0; j < kB; ++j) oc[32 * (x0 + j)] = (uint8_t)w[j];
            }
            for (int x = L8; x < L; ++x) {
                r = (col[32 * x] & bit) ? 0u : min(r + 1u, (uint32_t)kDistClamp);
                oc[32 * x] = (uint8_t)r;
            }
            r = kDistClamp;
            for (int x = L - 1; x >= L8; --x) {
                r = (col[32 * x] & bit) ? 0u : min(r + 1u, (uint32_t)kDistClamp);
                oc[32 * x] = (uint8_t)min(r, (uint32_t)oc[32 * x]);
            }
            for (int x0 = L8 - kB; x0 >= 0; x0 -= kB) {
                uint32_t w[kB], f[kB];
#pragma unroll
                for (int j = 0; j < kB; ++j) {
                    w[j] = col[32 * (x0 + j)];
                    f[j] = oc[32 * (x0 + j)];
                }
#pragma unroll
                for (int j = kB - 1; j >= 0; --j) {
                    r = (w[j] & bit) ? 0u : min(r + 1u, (uint32_t)kDistClamp);
                    f[j] = min(r, f[j]);
                }
#pragma unroll
                for (int j = 0; j < kB; ++j) oc[32 * (x0 + j)] = (uint8_t)f[j];
            }
            __syncwarp();
            for (int i = lane; i < L * 2; i += 32)
                *reinterpret_cast<uint4 *>(dst + (int64_t)(i >> 1) * S + 16 * (i & 1)) =
                    *reinterpret_cast<const uint4 *>(so + (i >> 1) * 32 + 16 * (i & 1));
            __syncwarp();
        }
        __syncthreads();  // the mask tile is restaged for the next column
    }
}

// ---- slab pieces --------------------------------------------------------------------
__global__ void slab_edges_kernel(const uint8_t *__restrict__ pdms, int64_t pitch, int n,
                                  int64_t bx, int64_t plane, uint8_t *__restrict__ edges) {
    const int64_t total = (int64_t)n * plane;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < total; l += stride) {
        const int p = (int)(l / plane);
        const int64_t yz = l % plane;
        const uint8_t *src = pdms + (int64_t)p * pitch + yz;
        edges[l] = src[0];
        edges[total + l] = src[(bx - 1) * plane];
    }
}

constexpr int kMaxWorld = 64;
struct SlabBounds {
    int64_t x0[kMaxWorld + 1];
};

__global__ void slab_fold_kernel(uint8_t *__restrict__ pdms, int64_t pitch, int n, int64_t bx,
                                 int64_t plane, const uint8_t *__restrict__ edges_all, int world,
                                 int rank, const __grid_constant__ SlabBounds sb) {
    const int64_t total = (int64_t)n * plane;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t my0 = sb.x0[rank], my1 = sb.x0[rank + 1];
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < total; l += stride) {
        int below = 1 << 20, above = 1 << 20;
        for (int j = 0; j < world; ++j) {
            if (j == rank) continue;
            const uint8_t *e = edges_all + (int64_t)j * 2 * total;
            if (j < rank) {  // nearest occupied in slab j, seen from our first plane
                const int hi = e[total + l];
                if (hi < kDistClamp) below = min(below, (int)(hi + my0 - sb.x0[j + 1] + 1));
            } else {
                const int lo = e[l];
                if (lo < kDistClamp) above = min(above, (int)(lo + sb.x0[j] - my1 + 1));
            }
        }
        if (below >= kDistClamp && above >= kDistClamp) continue;
        const int p = (int)(l / plane);
        uint8_t *dst = pdms + (int64_t)p * pitch + (l % plane);
        for (int64_t x = 0; x < bx; ++x) {
            int v = dst[x * plane];
            v = min(v, (int)min((int64_t)below + x, (int64_t)kDistClamp));
            v = min(v, (int)min((int64_t)above + (bx - 1 - x), (int64_t)kDistClamp));
            dst[x * plane] = (uint8_t)v;
        }
    }
}

// ---- host launchers ---------------------------------------------------------------------

static int grid_for(int64_t items, int threads, int per_sm) {
    int64_t want = ceil_div(items, threads);
    int64_t cap = (int64_t)sm_count() * per_sm;
    if (want > cap) want = cap;
    return want < 1 ? 1 : (int)want;
}

template <int LMAX, int AXIS, bool kDist1D, bool kSweep = false>
static int tile_pass(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *pdms, int64_t pitch,
                     cudaStream_t s, PackDst pk = PackDst{}) {
    const int64_t L = AXIS == kAxisX ? bx : (AXIS == kAxisY ? by : bz);
    int sw = (int)ceil_div(L, 4);
    if (sw % 2 == 0) sw += 1;
    // Row tiles for the sweep with L % 128 == 0 and 16-byte aligned rows use
    // unpadded 16-byte-swizzled rows (sstride == L); otherwise rows are
    // padded to 4 x odd bytes.
    const bool swz = kSweep && AXIS == kAxisZ && L % 128 == 0 && (L & (L - 1)) == 0 &&
                     bz % 16 == 0;  // 128, 256 or 512: chunk index math uses shifts
    const int sstride = swz ? (int)L : 4 * sw;
    const size_t per_warp = (AXIS == kAxisZ ? (size_t)32 * sstride : (size_t)32 * L) +
                            (kSweep ? SweepTable<(LMAX > 256 ? 2 : 1)>::kBytes : 0);
    // Sweep tiles: as many warps per SM as shared memory holds -- 2 CTAs of up
    // to 7 warps (<= 113 KB each) for lines <= 256 (14 warps instead of 12),
    // one CTA of up to 7 warps for 512-long lines (32 KB per warp).  Other
    // passes: up to 4 warps / 64 KB per CTA.
    const bool big = kSweep && LMAX > 256;
    const size_t budget = big ? 227 * 1024 : (kSweep ? 113 * 1024 : 65536);
    const int wmax = kSweep ? 7 : 4;
    int wpc = (int)(budget / per_warp);
    wpc = wpc < 1 ? 1 : (wpc > wmax ? wmax : wpc);
    const size_t smem = per_warp * wpc;
    auto kern = dt_tile_kernel<LMAX, AXIS, kDist1D, kSweep>;
    PDM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    const int64_t tiles = AXIS == kAxisZ ? (int64_t)n * ceil_div(bx * by, 32)
                                         : (int64_t)n * (AXIS == kAxisX ? by : bx) *
                                               ceil_div(bz, 32);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpc, smem) !=
            cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    int64_t grid = ceil_div(tiles, wpc);
    const int64_t cap = (int64_t)sm_count() * per_sm;
    if (grid > cap) grid = cap;
    kern<<<(unsigned)grid, 32 * wpc, smem, s>>>(n, bx, by, bz, pdms, pitch, sstride, tiles, pk);
    return cuda_status("dt_tile_kernel");
}

// x pass (1-D distance along x) on 64-z tiles, 2 lines per lane.
static int wide_x_pass(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *pdms, int64_t pitch,
                       cudaStream_t s) {
    constexpr int zw = 64;
    auto kern = dt_dist1d_wide_kernel;
    const size_t per_warp = (size_t)zw * bx;
    const size_t budget = 113 * 1024;  // 2 CTAs per SM
    int wpc = (int)(budget / per_warp);
    wpc = wpc < 1 ? 1 : (wpc > 8 ? 8 : wpc);
    const size_t smem = per_warp * wpc;
    PDM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t tiles = (int64_t)n * by * ceil_div(bz, zw);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpc, smem) !=
            cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    int64_t grid = ceil_div(tiles, wpc);
    const int64_t cap = (int64_t)sm_count() * per_sm;
    if (grid > cap) grid = cap;
    kern<<<(unsigned)grid, 32 * wpc, smem, s>>>(n, bx, by, bz, pdms, pitch, tiles);
    return cuda_status("dt_dist1d_wide_kernel");
}

// The TMEM sweep serves lines of 256 or 512 blocks in full 32-line tiles
// with 16-byte aligned rows; PDM_DT_TMEM=0 keeps dt_tile_kernel (A/B).
template <int AXIS>
static bool tmem_pass_ok(int64_t bx, int64_t by, int64_t bz) {
    static const bool off = getenv("PDM_DT_TMEM") && getenv("PDM_DT_TMEM")[0] == '0';
    if (off || AXIS == kAxisX) return false;
    if (AXIS == kAxisY) return (by == 256 || by == 512) && bz % 32 == 0;
    return (bz == 256 || bz == 512) && (bx * by) % 32 == 0;
}

template <int AXIS, int L, int W>
static int tmem_pass_l(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *pdms,
                       int64_t pitch, cudaStream_t s, PackDst pk, int64_t tiles) {
    auto kern = dt_tmem_kernel<AXIS, L, W>;
    const size_t smem = (size_t)W * 32 * L;
    static bool attr_set = false;  // (per instantiation)
    if (!attr_set) {
        PDM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        PDM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          (int)cudaSharedmemCarveoutMaxShared));
        attr_set = true;
    }
    // (the occupancy API answers 1 for a kernel that allocates TMEM; the
    // limits are shared memory, 80 registers and the TMEM columns: tmem_ctas)
    const int per_sm = tmem_ctas<L, W>();
    int64_t grid = ceil_div(tiles, W);
    const int64_t cap = (int64_t)sm_count() * per_sm;
    if (grid > cap) grid = cap;
    unsigned long long *ctr = nullptr;
    int st = work_counter(s, &ctr);
    if (st) return st;
    kern<<<(unsigned)grid, 32 * W, smem, s>>>(n, bx, by, bz, pdms, pitch, tiles, pk, ctr);
    return cuda_status("dt_tmem_kernel");
}

template <int AXIS>
static int tmem_pass(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *pdms, int64_t pitch,
                     cudaStream_t s, PackDst pk) {
    const int64_t L = AXIS == kAxisY ? by : bz;
    const int64_t tiles = AXIS == kAxisZ ? (int64_t)n * (bx * by / 32)
                                         : (int64_t)n * bx * (bz / 32);
    // the one-CTA shape once every warp of the grid gets >= 8 tiles
    // (PDM_DT_TMEM_BIG=0 / 1 forces the choice, A/B)
    static const int force = getenv("PDM_DT_TMEM_BIG") ? atoi(getenv("PDM_DT_TMEM_BIG")) : -1;
    const int64_t big_w = L == 256 ? tmem_big_warps<256>() : tmem_big_warps<512>();
    const bool big = force >= 0 ? force != 0 : tiles >= 8 * sm_count() * big_w;
    if (L == 256)
        return big ? tmem_pass_l<AXIS, 256, tmem_big_warps<256>()>(n, bx, by, bz, pdms, pitch, s,
                                                                   pk, tiles)
                   : tmem_pass_l<AXIS, 256, 4>(n, bx, by, bz, pdms, pitch, s, pk, tiles);
    return big ? tmem_pass_l<AXIS, 512, tmem_big_warps<512>()>(n, bx, by, bz, pdms, pitch, s, pk,
                                                               tiles)
               : tmem_pass_l<AXIS, 512, 4>(n, bx, by, bz, pdms, pitch, s, pk, tiles);
}

// pk (z pass only): fused packing epilogue; honoured when the z pass runs the
// swizzled sweep (dt_fused_pack_ok), ignored otherwise.
template <int AXIS, bool kDist1D>
static int axis_pass(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *pdms, int64_t pitch,
                     cudaStream_t s, PackDst pk = PackDst{}) {
    const int64_t L = AXIS == kAxisX ? bx : (AXIS == kAxisY ? by : bz);
    if (L <= 1) return PDM_OK;  // a 1-long line is already final
    if constexpr (kDist1D) {
        if (AXIS == kAxisX && L <= 256 && bz % 16 == 0)
            return wide_x_pass(n, bx, by, bz, pdms, pitch, s);
        if (L <= 1024) return tile_pass<64, AXIS, true>(n, bx, by, bz, pdms, pitch, s);
    } else {
        // lines <= 512: stack-free sweep envelope; longer: Meijster's scan
        if (tmem_pass_ok<AXIS>(bx, by, bz))
            return tmem_pass<AXIS>(n, bx, by, bz, pdms, pitch, s, pk);
        if (L <= 256) return tile_pass<256, AXIS, false, true>(n, bx, by, bz, pdms, pitch, s, pk);
        if (L <= 512) return tile_pass<512, AXIS, false, true>(n, bx, by, bz, pdms, pitch, s, pk);
        if (L <= 1024) return tile_pass<1024, AXIS, false>(n, bx, by, bz, pdms, pitch, s);
    }
    const int64_t lines = (int64_t)n * bx * by * bz / L;
    dt_line_kernel<AXIS, kDist1D><<<grid_for(lines, 128, 16), 128, 0, s>>>(n, bx, by, bz, pdms,
                                                                           pitch);
    return cuda_status("dt_line_kernel");
}

static bool x_mask_ok(int words, int64_t bx, int64_t bz, const uint32_t *mask) {
    static const bool off = getenv("PDM_DT_XMASK") && getenv("PDM_DT_XMASK")[0] == '0';
    return !off && words == 1 && bx >= 2 && bx <= 512 && bz % 32 == 0 &&
           (uintptr_t)mask % 16 == 0;
}

static int pass_x_mask(const uint32_t *mask, int words, int n, int64_t bx, int64_t by,
                       int64_t bz, uint8_t *pdms, int64_t pitch, cudaStream_t s) {
    const int64_t nb = bx * by * bz;
    if (x_mask_ok(words, bx, bz, mask) && pitch % 16 == 0 && (uintptr_t)pdms % 16 == 0) {
        auto kern = dt_x_mask_kernel;
        const size_t smem = (size_t)bx * 128 + (size_t)kXMaskWarps * bx * 32;
        PDM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        const int64_t tiles = by * (bz / 32);
        // 2 CTAs per SM for lines <= 256 (96 KB each), 1 for longer ones
        int64_t grid = (int64_t)sm_count() * (smem <= 113 * 1024 ? 2 : 1);
        if (grid > tiles) grid = tiles;
        static const bool dyn = !(getenv("PDM_XMASK_STATIC") && getenv("PDM_XMASK_STATIC")[0] == '1');
        unsigned long long *ctr = nullptr;
        if (dyn) {
            const int st = work_counter(s, &ctr);
            if (st) return st;
        }
        kern<<<(unsigned)grid, 32 * kXMaskWarps, smem, s>>>(mask, n, bx, by, bz, pdms, pitch,
                                                            tiles, ctr);
        return cuda_status("dt_x_mask_kernel");
    }
    dt_expand_mask_kernel<<<grid_for(ceil_div(nb, 16), 256, 8), 256, 0, s>>>(
        MaskSrc{mask, words}, n, nb, pdms, pitch);
    int st = cuda_status("dt_expand_mask_kernel");
    if (st) return st;
    return axis_pass<kAxisX, true>(n, bx, by, bz, pdms, pitch, s);
}

static int pass_yz(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *pdms, int64_t pitch,
                   cudaStream_t s, PackDst pk = PackDst{}) {
    int st = axis_pass<kAxisY, false>(n, bx, by, bz, pdms, pitch, s);
    if (st) return st;
    return axis_pass<kAxisZ, false>(n, bx, by, bz, pdms, pitch, s, pk);
}

// The z pass packs its rows itself when it runs the swizzled sweep tiles.
static bool dt_fused_pack_ok(int64_t bz) { return bz == 128 || bz == 256 || bz == 512; }

static int check_grid(const char *fn, int n, int64_t bx, int64_t by, int64_t bz, int64_t pitch) {
    PDM_REQUIRE(n >= 1 && bx >= 1 && by >= 1 && bz >= 1, "%s: bad sizes", fn);
    PDM_REQUIRE(pitch >= bx * by * bz, "%s: plane_pitch below bx*by*bz", fn);
    if (by > 4095 || bz > 4095) {
        set_error("%s: block dims (%lld, %lld) exceed 4095 along y or z", fn, (long long)by,
                  (long long)bz);
        return PDM_EUNSUPPORTED;
    }
    return PDM_OK;
}

}  // namespace pdm

using namespace pdm;

int pdm::dt_from_seed(const char *fn, int64_t bx, int64_t by, int64_t bz, uint8_t *map,
                      cudaStream_t s) {
    const int64_t nb = bx * by * bz;
    int st = check_grid(fn, 1, bx, by, bz, nb);
    if (st) return st;
    st = axis_pass<kAxisX, true>(1, bx, by, bz, map, nb, s);
    if (st) return st;
    return pass_yz(1, bx, by, bz, map, nb, s);
}

extern "C" int pdm_distance_transform(const uint8_t *occ, int64_t bx, int64_t by, int64_t bz,
                                      uint8_t *out, pdm_stream_t stream) {
    PDM_REQUIRE(occ && out, "pdm_distance_transform: null pointer");
    const int64_t nb = bx * by * bz;
    int st = check_grid("pdm_distance_transform", 1, bx, by, bz, nb);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    dt_expand_occ_kernel<<<grid_for(nb, 256, 8), 256, 0, s>>>(occ, nb, out);
    st = cuda_status("dt_expand_occ_kernel");
    if (st) return st;
    return dt_from_seed("pdm_distance_transform", bx, by, bz, out, s);
}

extern "C" int pdm_distance_transform_mask(const uint32_t *mask, int32_t words, int32_t n,
                                           int64_t bx, int64_t by, int64_t bz, uint8_t *pdms,
                                           int64_t plane_pitch, pdm_stream_t stream) {
    PDM_REQUIRE(mask && pdms, "pdm_distance_transform_mask: null pointer");
    PDM_REQUIRE(words == (n + 31) / 32, "pdm_distance_transform_mask: words");
    int st = check_grid("pdm_distance_transform_mask", n, bx, by, bz, plane_pitch);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    st = pass_x_mask(mask, words, n, bx, by, bz, pdms, plane_pitch, s);
    if (st) return st;
    return pass_yz(n, bx, by, bz, pdms, plane_pitch, s);
}

extern "C" int pdm_distance_transform_mask_packed(const uint32_t *mask, int32_t words, int32_t n,
                                                  int64_t bx, int64_t by, int64_t bz,
                                                  uint8_t *pdms, int64_t plane_pitch,
                                                  uint8_t *nib, int64_t nib_pitch, uint8_t *base,
                                                  int64_t base_pitch, uint32_t *violations,
                                                  uint16_t *tile_bounds, pdm_stream_t stream) {
    const char *fn = "pdm_distance_transform_mask_packed";
    PDM_REQUIRE(mask && pdms && nib && base && violations, "%s: null pointer", fn);
    PDM_REQUIRE(words == (n + 31) / 32, "%s: words", fn);
    int st = check_grid(fn, n, bx, by, bz, plane_pitch);
    if (st) return st;
    const int64_t nb = bx * by * bz, nchunks = 2 * ceil_div(nb, 32);
    PDM_REQUIRE(nib_pitch >= nchunks * 8 && base_pitch >= nchunks && nib_pitch % 16 == 0 &&
                    base_pitch % 4 == 0 && (uintptr_t)nib % 16 == 0 && (uintptr_t)base % 4 == 0,
                "%s: packed planes too small or misaligned", fn);
    cudaStream_t s = as_stream(stream);
    if (!dt_fused_pack_ok(bz)) {  // separate packing pass
        st = pdm_distance_transform_mask(mask, words, n, bx, by, bz, pdms, plane_pitch, stream);
        if (st) return st;
        st = pdm_pack_pdms(pdms, plane_pitch, nb, n, nib, nib_pitch, base, base_pitch,
                           violations, stream);
        if (st || !tile_bounds) return st;
        return pdm_packed_tile_bounds(nib, nib_pitch, base, base_pitch, nb, n, tile_bounds,
                                      stream);
    }
    PDM_CUDA_TRY(cudaMemsetAsync(violations, 0, sizeof(uint32_t), s));
    st = pass_x_mask(mask, words, n, bx, by, bz, pdms, plane_pitch, s);
    if (st) return st;
    // (the last tile of a plane whose rows do not fill it: its missing rows
    // are simply absent from the reduction; a partial last warp tile of 32
    // rows likewise)
    st = pass_yz(n, bx, by, bz, pdms, plane_pitch, s,
                 PackDst{nib, nib_pitch, base, base_pitch, violations, tile_bounds, n});
    if (st) return st;
    if (nchunks * 16 > nb) {  // the even-count padding chunk: all 255
        PDM_CUDA_TRY(cudaMemset2DAsync(nib + (nchunks - 1) * 8, nib_pitch, 0, 8, n, s));
        PDM_CUDA_TRY(cudaMemset2DAsync(base + nchunks - 1, base_pitch, 255, 1, n, s));
    }
    return PDM_OK;
}

extern "C" int pdm_dt_pass_x_mask(const uint32_t *mask, int32_t words, int32_t n, int64_t bx,
                                  int64_t by, int64_t bz, uint8_t *pdms, int64_t plane_pitch,
                                  pdm_stream_t stream) {
    PDM_REQUIRE(mask && pdms, "pdm_dt_pass_x_mask: null pointer");
    PDM_REQUIRE(words == (n + 31) / 32, "pdm_dt_pass_x_mask: words");
    int st = check_grid("pdm_dt_pass_x_mask", n, bx, by, bz, plane_pitch);
    if (st) return st;
    return pass_x_mask(mask, words, n, bx, by, bz, pdms, plane_pitch, as_stream(stream));
}

extern "C" int pdm_dt_slab_edges(const uint8_t *pdms, int64_t plane_pitch, int32_t n, int64_t bx,
                                 int64_t by, int64_t bz, uint8_t *edges, pdm_stream_t stream) {
    PDM_REQUIRE(pdms && edges, "pdm_dt_slab_edges: null pointer");
    int st = check_grid("pdm_dt_slab_edges", n, bx, by, bz, plane_pitch);
    if (st) return st;
    const int64_t plane = by * bz;
    slab_edges_kernel<<<grid_for((int64_t)n * plane, 256, 8), 256, 0, as_stream(stream)>>>(
        pdms, plane_pitch, n, bx, plane, edges);
    return cuda_status("slab_edges_kernel");
}

extern "C" int pdm_dt_slab_fold(uint8_t *pdms, int64_t plane_pitch, int32_t n, int64_t bx,
                                int64_t by, int64_t bz, const uint8_t *edges_all, int32_t world,
                                int32_t rank, const int64_t *slab_x0, pdm_stream_t stream) {
    PDM_REQUIRE(pdms && edges_all && slab_x0, "pdm_dt_slab_fold: null pointer");
    PDM_REQUIRE(world >= 1 && world <= kMaxWorld && rank >= 0 && rank < world,
                "pdm_dt_slab_fold: world=%d rank=%d", world, rank);
    int st = check_grid("pdm_dt_slab_fold", n, bx, by, bz, plane_pitch);
    if (st) return st;
    PDM_REQUIRE(slab_x0[rank + 1] - slab_x0[rank] == bx, "pdm_dt_slab_fold: slab width != bx");
    SlabBounds sb;
    for (int r = 0; r <= world; ++r) sb.x0[r] = slab_x0[r];
    const int64_t plane = by * bz;
    slab_fold_kernel<<<grid_for((int64_t)n * plane, 256, 8), 256, 0, as_stream(stream)>>>(
        pdms, plane_pitch, n, bx, plane, edges_all, world, rank, sb);
    return cuda_status("slab_fold_kernel");
}

extern "C" int pdm_dt_pass_yz(uint8_t *pdms, int64_t plane_pitch, int32_t n, int64_t bx,
                              int64_t by, int64_t bz, pdm_stream_t stream) {
    PDM_REQUIRE(pdms, "pdm_dt_pass_yz: null pointer");
    int st = check_grid("pdm_dt_pass_yz", n, bx, by, bz, plane_pitch);
    if (st) return st;
    return pass_yz(n, bx, by, bz, pdms, plane_pitch, as_stream(stream));
}

// dt.cu -- exact clamped Chebyshev distance transform of block occupancy (K6).
//
// Replaces _kernels.py:17-81 chamfer_chebyshev (two sequential raster passes
// over the 26-neighbourhood) + the clamp of acceleration.py:180 with three
// separable, embarrassingly parallel passes over the partition-major map set
// pdms[p][x][y][z] (z contiguous), all in place:
//
//   pass x:  g1[x] = 1-D distance along x to the nearest occupied block
//            (forward + backward run-length sweeps, clamped at 255);
//   pass y:  g2[y] = min_j max(|y - j|, g1[j])     (lower envelope)
//   pass z:  g3[z] = min_j max(|z - j|, g2[j])     (lower envelope)
//
// min(C, max(a, b)) = max(min(C, a), min(C, b)) makes uint8-clamped
// intermediates exact, and the chessboard metric is the max of the per-axis
// distances, so g3 == min(255, chamfer_chebyshev) cell for cell (verified
// against the reference in tests/test_gpu_parity.py and the golden vectors).
//
// The lower-envelope passes use Meijster et al.'s linear-time scan with the
// L-infinity separator (one thread per line, stack in local memory):
//   f(x, i)  = max(|x - i|, g(i))
//   Sep(i,u) = g(i) <= g(u) ? max(i + g(u), (i + u) / 2) : min(u - g(i), (i + u) / 2)
// Pass x and pass y read lines whose elements are bz bytes apart; consecutive
// threads take consecutive z so every step is a coalesced warp access.  Pass z
// runs along the contiguous axis, so a CTA stages a tile of rows in shared
// memory (coalesced in, Meijster from shared memory, coalesced out).
#include <cuda_runtime.h>

#include "pdm_common.cuh"

namespace pdm {

// Stack entry: s (12 bits) | t (12 bits) << 12 | g(s) (8 bits) << 24.
__device__ __forceinline__ uint32_t pack_entry(int s, int t, int g) {
    return (uint32_t)s | ((uint32_t)t << 12) | ((uint32_t)g << 24);
}
__device__ __forceinline__ int ent_s(uint32_t e) { return (int)(e & 0xFFFu); }
__device__ __forceinline__ int ent_t(uint32_t e) { return (int)((e >> 12) & 0xFFFu); }
__device__ __forceinline__ int ent_g(uint32_t e) { return (int)(e >> 24); }

// Meijster lower envelope of one line of m <= LMAX values (LMAX <= 4096):
// out[u] = min(255, min_i max(|u - i|, g[i])).  Ld/St access element u.
template <int LMAX, class Ld, class St>
__device__ __forceinline__ void cone_line(int m, Ld ld, St st) {
    uint32_t stk[LMAX];
    int q = 0;
    stk[0] = pack_entry(0, 0, ld(0));
    for (int u = 1; u < m; ++u) {
        const int gu = ld(u);
        while (q >= 0) {
            const uint32_t e = stk[q];
            const int t = ent_t(e), s = ent_s(e);
            const int fs = max(abs(t - s), ent_g(e));
            const int fu = max(abs(t - u), gu);
            if (fs > fu)
                --q;
            else
                break;
        }
        if (q < 0) {
            q = 0;
            stk[0] = pack_entry(u, 0, gu);
        } else {
            const uint32_t e = stk[q];
            const int s = ent_s(e), gs = ent_g(e);
            const int mid = (s + u) >> 1;
            const int sep = gs <= gu ? max(s + gu, mid) : min(u - gs, mid);
            const int w = 1 + sep;
            if (w < m) {
                ++q;
                stk[q] = pack_entry(u, w, gu);
            }
        }
    }
    for (int u = m - 1; u >= 0; --u) {
        const uint32_t e = stk[q];
        const int d = max(abs(u - ent_s(e)), ent_g(e));
        st(u, d < kDistClamp ? d : kDistClamp);
        if (u == ent_t(e)) --q;
    }
}

// ---- pass x -----------------------------------------------------------------------
// Source of occupancy: a mask (bit p of words) or a plain uint8 map (n == 1).
struct MaskSrc {
    const uint32_t *mask;
    int words;
    __device__ __forceinline__ bool occ(int64_t c, int p) const {
        return (mask[c * words + (p >> 5)] >> (p & 31)) & 1u;
    }
};
struct OccSrc {
    const uint8_t *occ8;
    __device__ __forceinline__ bool occ(int64_t c, int) const { return occ8[c] != 0; }
};

// Thread = (p, y, z); sweeps x forward then backward.  Writes pdms[p][x][y][z].
template <class Src>
__global__ void dt_pass_x_kernel(Src src, int n, int64_t bx, int64_t by, int64_t bz,
                                 uint8_t *__restrict__ pdms, int64_t pitch) {
    const int64_t plane = by * bz;
    const int64_t lines = (int64_t)n * plane;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < lines; l += stride) {
        const int p = (int)(l / plane);
        const int64_t yz = l % plane;
        uint8_t *dst = pdms + (int64_t)p * pitch + yz;
        int run = kDistClamp;
        for (int64_t x = 0; x < bx; ++x) {
            run = src.occ(x * plane + yz, p) ? 0 : min(run + 1, kDistClamp);
            dst[x * plane] = (uint8_t)run;
        }
        run = kDistClamp;
        for (int64_t x = bx - 1; x >= 0; --x) {
            run = src.occ(x * plane + yz, p) ? 0 : min(run + 1, kDistClamp);
            const int fwd = dst[x * plane];
            dst[x * plane] = (uint8_t)min(fwd, run);
        }
    }
}

// ---- pass y: strided lines ---------------------------------------------------------
// Line = (p, x, z): elements pdms[p][x][u][z], u in [0, by).
template <int LMAX>
__global__ void __launch_bounds__(128) dt_cone_y_kernel(int n, int64_t bx, int64_t by, int64_t bz,
                                                        uint8_t *__restrict__ pdms,
                                                        int64_t pitch) {
    const int64_t lines = (int64_t)n * bx * bz;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < lines; l += stride) {
        const int64_t z = l % bz;
        const int64_t px = l / bz;
        const int64_t x = px % bx;
        const int p = (int)(px / bx);
        uint8_t *base = pdms + (int64_t)p * pitch + x * by * bz + z;
        cone_line<LMAX>(
            (int)by, [&](int u) -> int { return base[(int64_t)u * bz]; },
            [&](int u, int v) { base[(int64_t)u * bz] = (uint8_t)v; });
    }
}

// ---- pass z: contiguous rows through shared memory --------------------------------
// Row = (p, x, y): pdms[p][x][y][0..bz).  A CTA of R threads owns R consecutive
// rows of one partition; row stride in shared memory is an odd number of
// 32-bit words so the R threads reading element u hit distinct banks.
template <int LMAX>
__global__ void __launch_bounds__(64) dt_cone_z_kernel(int n, int64_t rows_per_p, int64_t bz,
                                                       uint8_t *__restrict__ pdms, int64_t pitch,
                                                       int sstride) {
    extern __shared__ uint8_t s_tile[];
    const int R = blockDim.x;
    const int64_t tiles_per_p = ceil_div(rows_per_p, R);
    const int64_t tiles = tiles_per_p * n;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int p = (int)(tile / tiles_per_p);
        const int64_t r0 = (tile % tiles_per_p) * R;
        const int rows = (int)min((int64_t)R, rows_per_p - r0);
        uint8_t *g = pdms + (int64_t)p * pitch + r0 * bz;
        __syncthreads();
        for (int r = 0; r < rows; ++r)
            for (int64_t z = threadIdx.x; z < bz; z += R) s_tile[r * sstride + z] = g[r * bz + z];
        __syncthreads();
        if ((int)threadIdx.x < rows) {
            uint8_t *row = s_tile + threadIdx.x * sstride;
            cone_line<LMAX>(
                (int)bz, [&](int u) -> int { return row[u]; },
                [&](int u, int v) { row[u] = (uint8_t)v; });
        }
        __syncthreads();
        for (int r = 0; r < rows; ++r)
            for (int64_t z = threadIdx.x; z < bz; z += R) g[r * bz + z] = s_tile[r * sstride + z];
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

static int grid_lines(int64_t lines, int threads, int per_sm) {
    int64_t want = ceil_div(lines, threads);
    int64_t cap = (int64_t)sm_count() * per_sm;
    if (want > cap) want = cap;
    return want < 1 ? 1 : (int)want;
}

template <class Src>
static int pass_x(Src src, int n, int64_t bx, int64_t by, int64_t bz, uint8_t *pdms,
                  int64_t pitch, cudaStream_t s) {
    const int64_t lines = (int64_t)n * by * bz;
    dt_pass_x_kernel<Src><<<grid_lines(lines, 256, 8), 256, 0, s>>>(src, n, bx, by, bz, pdms,
                                                                    pitch);
    return cuda_status("dt_pass_x_kernel");
}

template <int LMAX>
static int cone_y(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *pdms, int64_t pitch,
                  cudaStream_t s) {
    const int64_t lines = (int64_t)n * bx * bz;
    dt_cone_y_kernel<LMAX><<<grid_lines(lines, 128, 16), 128, 0, s>>>(n, bx, by, bz, pdms, pitch);
    return cuda_status("dt_cone_y_kernel");
}

template <int LMAX>
static int cone_z(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *pdms, int64_t pitch,
                  cudaStream_t s) {
    const int R = 64;
    int sw = (int)ceil_div(bz, 4);
    if (sw % 2 == 0) sw += 1;
    const int sstride = 4 * sw;
    const size_t smem = (size_t)R * sstride;
    auto kern = dt_cone_z_kernel<LMAX>;
    if (smem > 48 * 1024)
        PDM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    const int64_t rows_per_p = bx * by;
    const int64_t tiles = ceil_div(rows_per_p, R) * n;
    kern<<<grid_lines(tiles, 1, 16), R, smem, s>>>(n, rows_per_p, bz, pdms, pitch, sstride);
    return cuda_status("dt_cone_z_kernel");
}

static int pass_yz(int n, int64_t bx, int64_t by, int64_t bz, uint8_t *pdms, int64_t pitch,
                   cudaStream_t s) {
    int st;
    if (by > 1) {
        if (by <= 64)
            st = cone_y<64>(n, bx, by, bz, pdms, pitch, s);
        else if (by <= 256)
            st = cone_y<256>(n, bx, by, bz, pdms, pitch, s);
        else if (by <= 512)
            st = cone_y<512>(n, bx, by, bz, pdms, pitch, s);
        else if (by <= 1024)
            st = cone_y<1024>(n, bx, by, bz, pdms, pitch, s);
        else
            st = cone_y<4096>(n, bx, by, bz, pdms, pitch, s);
        if (st) return st;
    }
    if (bz > 1) {
        if (bz <= 64)
            st = cone_z<64>(n, bx, by, bz, pdms, pitch, s);
        else if (bz <= 256)
            st = cone_z<256>(n, bx, by, bz, pdms, pitch, s);
        else if (bz <= 512)
            st = cone_z<512>(n, bx, by, bz, pdms, pitch, s);
        else if (bz <= 1024)
            st = cone_z<1024>(n, bx, by, bz, pdms, pitch, s);
        else
            st = cone_z<4096>(n, bx, by, bz, pdms, pitch, s);
        if (st) return st;
    }
    return PDM_OK;
}

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

extern "C" int pdm_distance_transform(const uint8_t *occ, int64_t bx, int64_t by, int64_t bz,
                                      uint8_t *out, pdm_stream_t stream) {
    PDM_REQUIRE(occ && out, "pdm_distance_transform: null pointer");
    const int64_t nb = bx * by * bz;
    int st = check_grid("pdm_distance_transform", 1, bx, by, bz, nb);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    st = pass_x(OccSrc{occ}, 1, bx, by, bz, out, nb, s);
    if (st) return st;
    return pass_yz(1, bx, by, bz, out, nb, s);
}

extern "C" int pdm_distance_transform_mask(const uint32_t *mask, int32_t words, int32_t n,
                                           int64_t bx, int64_t by, int64_t bz, uint8_t *pdms,
                                           int64_t plane_pitch, pdm_stream_t stream) {
    PDM_REQUIRE(mask && pdms, "pdm_distance_transform_mask: null pointer");
    PDM_REQUIRE(words == (n + 31) / 32, "pdm_distance_transform_mask: words");
    int st = check_grid("pdm_distance_transform_mask", n, bx, by, bz, plane_pitch);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    st = pass_x(MaskSrc{mask, words}, n, bx, by, bz, pdms, plane_pitch, s);
    if (st) return st;
    return pass_yz(n, bx, by, bz, pdms, plane_pitch, s);
}

extern "C" int pdm_dt_pass_x_mask(const uint32_t *mask, int32_t words, int32_t n, int64_t bx,
                                  int64_t by, int64_t bz, uint8_t *pdms, int64_t plane_pitch,
                                  pdm_stream_t stream) {
    PDM_REQUIRE(mask && pdms, "pdm_dt_pass_x_mask: null pointer");
    PDM_REQUIRE(words == (n + 31) / 32, "pdm_dt_pass_x_mask: words");
    int st = check_grid("pdm_dt_pass_x_mask", n, bx, by, bz, plane_pitch);
    if (st) return st;
    return pass_x(MaskSrc{mask, words}, n, bx, by, bz, pdms, plane_pitch, as_stream(stream));
}

extern "C" int pdm_dt_slab_edges(const uint8_t *pdms, int64_t plane_pitch, int32_t n, int64_t bx,
                                 int64_t by, int64_t bz, uint8_t *edges, pdm_stream_t stream) {
    PDM_REQUIRE(pdms && edges, "pdm_dt_slab_edges: null pointer");
    int st = check_grid("pdm_dt_slab_edges", n, bx, by, bz, plane_pitch);
    if (st) return st;
    const int64_t plane = by * bz;
    slab_edges_kernel<<<grid_lines((int64_t)n * plane, 256, 8), 256, 0, as_stream(stream)>>>(
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
    slab_fold_kernel<<<grid_lines((int64_t)n * plane, 256, 8), 256, 0, as_stream(stream)>>>(
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

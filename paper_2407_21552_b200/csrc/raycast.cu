// raycast.cu -- the GPU consumer of D': camera rays
// and the fixed-grid front-to-back ray marcher that skips empty space with a
// per-block Chebyshev distance field resident in HBM.
//
// Reference: pdmrender/raycast.py:163-200 (camera_rays), :232-283 (render),
// _kernels.py:152-203 (safe_box_exit), :206-365 (march_rays).  The reference
// composites in float64; so does this file, with the same operation order
// and NO fused multiply-adds (the file is compiled with -fmad=false, see
// __graft_entry__.py), so every ray's rgba and work counters are bit-identical
// to the numba marcher (tests/test_render.py against reference goldens).
//
// One thread per ray.  Each evaluated sample reads 8 voxels (trilinear) and
// one LUT row; skipped stretches cost one D' byte and a box exit.  Rays are
// row-major pixels, so a warp is 32 neighbouring pixels of one scanline and
// its samples hit nearby voxels (L1/L2 reuse).
#include "pdm_common.cuh"

namespace pdm {

namespace {

constexpr double kBig = 1e30;
constexpr double kEps = 1e-12;

// _kernels.py:152-203: ray parameter where the ray leaves the blocks
// [B - halo, B + halo] (voxel coordinates, clipped to the hull [0, h]).
__device__ __forceinline__ double safe_box_exit(double ox, double oy, double oz, double dx,
                                                double dy, double dz, int64_t bi, int64_t bj,
                                                int64_t bk, int64_t halo, int64_t b, double hx,
                                                double hy, double hz) {
    const double lox = fmax((double)((bi - halo) * b), 0.0);
    const double loy = fmax((double)((bj - halo) * b), 0.0);
    const double loz = fmax((double)((bk - halo) * b), 0.0);
    const double hix = fmin((double)((bi + halo + 1) * b), hx);
    const double hiy = fmin((double)((bj + halo + 1) * b), hy);
    const double hiz = fmin((double)((bk + halo + 1) * b), hz);
    double t = kBig;
    if (dx > kEps) t = fmin(t, (hix - ox) / dx);
    else if (dx < -kEps) t = fmin(t, (lox - ox) / dx);
    if (dy > kEps) t = fmin(t, (hiy - oy) / dy);
    else if (dy < -kEps) t = fmin(t, (loy - oy) / dy);
    if (dz > kEps) t = fmin(t, (hiz - oz) / dz);
    else if (dz < -kEps) t = fmin(t, (loz - oz) / dz);
    return t;
}

__device__ __forceinline__ double clampd(double v, double hi) {
    return v < 0.0 ? 0.0 : (v > hi ? hi : v);
}

// raycast.py:187-198: per-pixel direction from the camera frame, divided by
// the spacing and normalised (numpy's order: (f + x r) + y u; |d| summed
// left to right).
__global__ void __launch_bounds__(256)
    camera_dirs_kernel(double3 fwd, double3 right, double3 up, double tan_half, double aspect,
                       double3 sp, int width, int height, double *__restrict__ dirs) {
    const int64_t n = (int64_t)width * height;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = r % width, j = r / width;
        const double xs = (2.0 * ((double)i + 0.5) / width - 1.0) * tan_half * aspect;
        const double ys = (1.0 - 2.0 * ((double)j + 0.5) / height) * tan_half;
        double dx = fwd.x + xs * right.x + ys * up.x;
        double dy = fwd.y + xs * right.y + ys * up.y;
        double dz = fwd.z + xs * right.z + ys * up.z;
        dx = dx / sp.x;
        dy = dy / sp.y;
        dz = dz / sp.z;
        const double nrm = sqrt(dx * dx + dy * dy + dz * dz);
        dirs[3 * r] = dx / nrm;
        dirs[3 * r + 1] = dy / nrm;
        dirs[3 * r + 2] = dz / nrm;
    }
}

struct MarchArgs {
    int64_t nx, ny, nz, bx, by, bz, lut_len, n_rays;
    int b;
    double step, ert_thr, ox, oy, oz;
    int ert_on;
};

// _kernels.py:206-365, one thread per ray.  I: index type (int32 when the
// volume has < 2^31 voxels -- cheaper conversions and address math; the
// values are the same).
template <class V, class I>
__global__ void __launch_bounds__(128)
    march_rays_kernel(const V *__restrict__ vox, const double *__restrict__ lut,
                      const uint8_t *__restrict__ dist, const double *__restrict__ dirs,
                      const MarchArgs a, double *__restrict__ rgba_out,
                      int64_t *__restrict__ counters, uint8_t *__restrict__ pixels,
                      unsigned long long *__restrict__ totals) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = 0, evaluated = 0, skips = 0, ert_fired = 0;
    double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_a = 0.0;
    if (r < a.n_rays) {
        const double hx = a.nx - 1.0, hy = a.ny - 1.0, hz = a.nz - 1.0;
        const I x_hi = a.nx >= 2 ? (I)(a.nx - 2) : 0;
        const I y_hi = a.ny >= 2 ? (I)(a.ny - 2) : 0;
        const I z_hi = a.nz >= 2 ? (I)(a.nz - 2) : 0;
        const double dx = dirs[3 * r], dy = dirs[3 * r + 1], dz = dirs[3 * r + 2];
        // slab intersection with the voxel-centre hull [0, n-1]^3
        double tmin = -kBig, tmax = kBig;
        bool hit = true;
        const double o3[3] = {a.ox, a.oy, a.oz}, d3[3] = {dx, dy, dz}, h3[3] = {hx, hy, hz};
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            if (!hit) break;
            const double o = o3[ax], d = d3[ax], h = h3[ax];
            if (d > kEps || d < -kEps) {
                double t0 = (0.0 - o) / d, t1 = (h - o) / d;
                if (t0 > t1) {
                    const double tt = t0;
                    t0 = t1;
                    t1 = tt;
                }
                if (t0 > tmin) tmin = t0;
                if (t1 < tmax) tmax = t1;
            } else if (o < 0.0 || o > h) {
                hit = false;
            }
        }
        if (hit && !(tmax < tmin) && !(tmax < 0.0)) {
            const double t_entry = tmin > 0.0 ? tmin : 0.0;
            total = (int64_t)((tmax - t_entry) / a.step) + 1;
            const I plane = (I)(a.ny * a.nz), nzi = (I)a.nz;
            const I bb = (I)a.b, byi = (I)a.by, bzi = (I)a.bz;
            const int bshift = (a.b & (a.b - 1)) == 0 ? __ffs(a.b) - 1 : -1;
            // One sample's loads, issued together: its D' byte AND its 8
            // voxels (clamped indices, always inside the volume) -- the voxels
            // are needed for every sample except the ~1 in 600 that starts a
            // skip, so fetching them speculatively removes a dependent round
            // trip; the next sample's loads are issued before the current
            // one is composited.  Arithmetic and its order are unchanged.
            struct Sample {
                double px, py, pz;
                I bi, bj, bk, x0, y0, z0;
                int dval;
                V c[8];
            };
            // `prev`: the sample before (its block and cell, when valid): a
            // sample in the same block reuses its D' byte, one in the same
            // trilinear cell its 8 voxels (step 0.5: about every other
            // sample), so those lanes issue no loads.
            auto load = [&](int64_t kk, Sample &S, const Sample &prev, bool prev_ok) {
                const double t = t_entry + kk * a.step;
                S.px = clampd(a.ox + t * dx, hx);
                S.py = clampd(a.oy + t * dy, hy);
                S.pz = clampd(a.oz + t * dz, hz);
                const I vx = (I)S.px, vy = (I)S.py, vz = (I)S.pz;
                // block coordinates: a shift for power-of-two edges (b = 4, 8, ...)
                S.bi = bshift >= 0 ? vx >> bshift : vx / bb;
                S.bj = bshift >= 0 ? vy >> bshift : vy / bb;
                S.bk = bshift >= 0 ? vz >> bshift : vz / bb;
                if (prev_ok && S.bi == prev.bi && S.bj == prev.bj && S.bk == prev.bk)
                    S.dval = prev.dval;
                else
                    S.dval = dist[(S.bi * byi + S.bj) * bzi + S.bk];
                S.x0 = vx < x_hi ? vx : x_hi;
                S.y0 = vy < y_hi ? vy : y_hi;
                S.z0 = vz < z_hi ? vz : z_hi;
                if (prev_ok && S.x0 == prev.x0 && S.y0 == prev.y0 && S.z0 == prev.z0) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) S.c[i] = prev.c[i];
                    return;
                }
                const I x1 = a.nx >= 2 ? S.x0 + 1 : S.x0;
                const I y1 = a.ny >= 2 ? S.y0 + 1 : S.y0;
                const I z1 = a.nz >= 2 ? S.z0 + 1 : S.z0;
                S.c[0] = vox[S.x0 * plane + S.y0 * nzi + S.z0];
                S.c[1] = vox[x1 * plane + S.y0 * nzi + S.z0];
                S.c[2] = vox[S.x0 * plane + y1 * nzi + S.z0];
                S.c[3] = vox[x1 * plane + y1 * nzi + S.z0];
                S.c[4] = vox[S.x0 * plane + S.y0 * nzi + z1];
                S.c[5] = vox[x1 * plane + S.y0 * nzi + z1];
                S.c[6] = vox[S.x0 * plane + y1 * nzi + z1];
                S.c[7] = vox[x1 * plane + y1 * nzi + z1];
            };
            int64_t k = 0;
            Sample cur, nxt;
            load(0, cur, cur, false);
            while (k < total) {
                const bool more = k + 1 < total;
                if (more) load(k + 1, nxt, cur, true);
                if (cur.dval == 0) {
                    const double fx = cur.px - cur.x0, fy = cur.py - cur.y0, fz = cur.pz - cur.z0;
                    const double c000 = cur.c[0], c100 = cur.c[1], c010 = cur.c[2],
                                 c110 = cur.c[3], c001 = cur.c[4], c101 = cur.c[5],
                                 c011 = cur.c[6], c111 = cur.c[7];
                    const double gx = 1.0 - fx, gy = 1.0 - fy, gz = 1.0 - fz;
                    const double value =
                        gz * (gy * (gx * c000 + fx * c100) + fy * (gx * c010 + fx * c110)) +
                        fz * (gy * (gx * c001 + fx * c101) + fy * (gx * c011 + fx * c111));
                    int64_t li = (int64_t)(value + 0.5);
                    if (li >= a.lut_len) li = a.lut_len - 1;
                    const double alpha = lut[4 * li + 3];
                    if (alpha > 0.0) {
                        const double w = (1.0 - acc_a) * alpha;
                        acc_r += w * lut[4 * li];
                        acc_g += w * lut[4 * li + 1];
                        acc_b += w * lut[4 * li + 2];
                        acc_a += w;
                    }
                    ++evaluated;
                    if (a.ert_on && acc_a >= a.ert_thr) {
                        ert_fired = 1;
                        break;
                    }
                    ++k;
                    cur = nxt;
                } else {
                    const double t_exit =
                        safe_box_exit(a.ox, a.oy, a.oz, dx, dy, dz, cur.bi, cur.bj, cur.bk,
                                      cur.dval - 1, a.b, hx, hy, hz);
                    int64_t k_next = (int64_t)ceil((t_exit - t_entry) / a.step - 1e-9);
                    if (k_next <= k) k_next = k + 1;
                    ++skips;
                    if (k_next == k + 1) {
                        cur = nxt;
                    } else if (k_next < total) {
                        load(k_next, cur, cur, false);
                    }
                    k = k_next;
                }
            }
        }
        const double c4[4] = {acc_r, acc_g, acc_b, acc_a};
        if (rgba_out)
            for (int c = 0; c < 4; ++c) rgba_out[4 * r + c] = c4[c];
        if (counters) {
            counters[4 * r] = total;
            counters[4 * r + 1] = evaluated;
            counters[4 * r + 2] = skips;
            counters[4 * r + 3] = ert_fired;
        }
        if (pixels) {  // raycast.py:263-268: clip, * 255, round half to even
            uint32_t px4 = 0;
            for (int c = 0; c < 4; ++c)
                px4 |= (uint32_t)rint(fmin(fmax(c4[c], 0.0), 1.0) * 255.0) << (8 * c);
            reinterpret_cast<uint32_t *>(pixels)[r] = px4;
        }
    }
    if (totals) {  // stats = column sums of the counters (raycast.py:270-278)
        unsigned long long v[4] = {(unsigned long long)total, (unsigned long long)evaluated,
                                   (unsigned long long)skips, (unsigned long long)ert_fired};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v[c] += __shfl_down_sync(0xFFFFFFFFu, v[c], off);
            if ((threadIdx.x & 31) == 0 && v[c]) atomicAdd(totals + c, v[c]);
        }
    }
}

}  // namespace
}  // namespace pdm

using namespace pdm;

extern "C" int pdm_camera_rays(const double *frame, double tan_half, double aspect,
                               const double *spacing, int32_t width, int32_t height,
                               double *dirs, pdm_stream_t stream) {
    PDM_REQUIRE(frame && spacing && dirs, "pdm_camera_rays: null pointer");
    PDM_REQUIRE(width >= 1 && height >= 1, "pdm_camera_rays: viewport %dx%d", width, height);
    const int64_t n = (int64_t)width * height;
    int64_t grid = ceil_div(n, 256);
    if (grid > (int64_t)sm_count() * 16) grid = (int64_t)sm_count() * 16;
    camera_dirs_kernel<<<(unsigned)grid, 256, 0, as_stream(stream)>>>(
        make_double3(frame[0], frame[1], frame[2]), make_double3(frame[3], frame[4], frame[5]),
        make_double3(frame[6], frame[7], frame[8]), tan_half, aspect,
        make_double3(spacing[0], spacing[1], spacing[2]), width, height, dirs);
    return cuda_status("camera_dirs_kernel");
}

extern "C" int pdm_march_rays(const void *vox, int32_t bits, int64_t nx, int64_t ny, int64_t nz,
                              const double *lut, int64_t lut_len, const uint8_t *dist, int32_t b,
                              double step, int32_t ert_enabled, double ert_threshold,
                              const double *origin, const double *dirs, int64_t n_rays,
                              double *rgba, int64_t *counters, uint8_t *pixels,
                              unsigned long long *totals, pdm_stream_t stream) {
    PDM_REQUIRE(vox && lut && dist && origin && dirs, "pdm_march_rays: null pointer");
    PDM_REQUIRE(bits == 8 || bits == 16, "pdm_march_rays: bits must be 8 or 16, got %d", bits);
    PDM_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && b >= 1 && lut_len >= 1 && n_rays >= 0,
                "pdm_march_rays: bad sizes");
    PDM_REQUIRE(step > 0.0, "pdm_march_rays: step must be positive");
    if (n_rays == 0) return PDM_OK;
    MarchArgs a;
    a.nx = nx;
    a.ny = ny;
    a.nz = nz;
    a.bx = ceil_div(nx, b);
    a.by = ceil_div(ny, b);
    a.bz = ceil_div(nz, b);
    a.lut_len = lut_len;
    a.n_rays = n_rays;
    a.b = b;
    a.step = step;
    a.ert_thr = ert_threshold;
    a.ert_on = ert_enabled != 0;
    a.ox = origin[0];
    a.oy = origin[1];
    a.oz = origin[2];
    cudaStream_t s = as_stream(stream);
    if (totals) PDM_CUDA_TRY(cudaMemsetAsync(totals, 0, 4 * sizeof(unsigned long long), s));
    const unsigned grid = (unsigned)ceil_div(n_rays, 128);
    const bool small = nx * ny * nz < ((int64_t)1 << 31);
    if (bits == 8 && small)
        march_rays_kernel<uint8_t, int32_t><<<grid, 128, 0, s>>>(
            static_cast<const uint8_t *>(vox), lut, dist, dirs, a, rgba, counters, pixels, totals);
    else if (bits == 8)
        march_rays_kernel<uint8_t, int64_t><<<grid, 128, 0, s>>>(
            static_cast<const uint8_t *>(vox), lut, dist, dirs, a, rgba, counters, pixels, totals);
    else if (small)
        march_rays_kernel<uint16_t, int32_t><<<grid, 128, 0, s>>>(
            static_cast<const uint16_t *>(vox), lut, dist, dirs, a, rgba, counters, pixels,
            totals);
    else
        march_rays_kernel<uint16_t, int64_t><<<grid, 128, 0, s>>>(
            static_cast<const uint16_t *>(vox), lut, dist, dirs, a, rgba, counters, pixels,
            totals);
    return cuda_status("march_rays_kernel");
}

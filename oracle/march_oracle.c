/*
 * march_oracle.c -- CPU restatement of the reference's ray marcher.
 *
 * TEST INFRASTRUCTURE ONLY (see pdm_oracle.c): the parity checker for
 * paper_2407_21552_b200/csrc/raycast.cu and the CPU baseline timed by
 * tools/render_bench.py.  Reference (/root/reference/pkg/src/pdmrender):
 * _kernels.py:152-203 safe_box_exit, _kernels.py:206-365 march_rays.
 *
 * float64 throughout, in the reference's operation order; built with
 * -std=c11 (ISO mode: -ffp-contract=off) for x86-64-v2 (no FMA), so every
 * result is bit-identical to the numba marcher (tests/test_render.py pins it
 * against goldens made by the reference).  Rays are split across threads
 * with OpenMP; each ray is independent.
 */
#include <math.h>
#include <stdint.h>

int oracle_threads(void); /* pdm_oracle.c */

/* _kernels.py:152-203 */
static double box_exit(double ox, double oy, double oz, double dx, double dy, double dz,
                       int64_t bi, int64_t bj, int64_t bk, int64_t halo, int64_t b, double hx,
                       double hy, double hz) {
    double lo[3], hi[3];
    const int64_t c[3] = {bi, bj, bk};
    const double h[3] = {hx, hy, hz}, o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
    double t_exit = 1e30;
    for (int a = 0; a < 3; ++a) {
        lo[a] = (double)((c[a] - halo) * b);
        if (lo[a] < 0.0) lo[a] = 0.0;
        hi[a] = (double)((c[a] + halo + 1) * b);
        if (hi[a] > h[a]) hi[a] = h[a];
        double te = t_exit;
        if (d[a] > 1e-12) te = (hi[a] - o[a]) / d[a];
        else if (d[a] < -1e-12) te = (lo[a] - o[a]) / d[a];
        if (te < t_exit) t_exit = te;
    }
    return t_exit;
}

static inline double vox_f(const void *vox, int bits, int64_t i) {
    return bits == 8 ? (double)((const uint8_t *)vox)[i] : (double)((const uint16_t *)vox)[i];
}

static inline double clamp_hull(double v, double h) { return v < 0.0 ? 0.0 : (v > h ? h : v); }

/* _kernels.py:206-365: one ray per iteration; rgba[n][4], counters[n][4]. */
void oracle_march_rays(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz,
                       const double *lut, int64_t lut_len, const uint8_t *dist, int64_t b,
                       double step, int ert_on, double ert_thr, const double *origin,
                       const double *dirs, int64_t n_rays, double *rgba, int64_t *counters) {
    const double hx = nx - 1.0, hy = ny - 1.0, hz = nz - 1.0;
    const int64_t x_hi = nx >= 2 ? nx - 2 : 0, y_hi = ny >= 2 ? ny - 2 : 0;
    const int64_t z_hi = nz >= 2 ? nz - 2 : 0;
    const int64_t by = (ny + b - 1) / b, bz = (nz + b - 1) / b;
    const double ox = origin[0], oy = origin[1], oz = origin[2];
#pragma omp parallel for schedule(dynamic, 64) num_threads(oracle_threads())
    for (int64_t r = 0; r < n_rays; ++r) {
        const double dx = dirs[3 * r], dy = dirs[3 * r + 1], dz = dirs[3 * r + 2];
        const double o3[3] = {ox, oy, oz}, d3[3] = {dx, dy, dz}, h3[3] = {hx, hy, hz};
        double tmin = -1e30, tmax = 1e30;
        int hit = 1;
        for (int a = 0; a < 3 && hit; ++a) {
            if (d3[a] > 1e-12 || d3[a] < -1e-12) {
                double t0 = (0.0 - o3[a]) / d3[a], t1 = (h3[a] - o3[a]) / d3[a];
                if (t0 > t1) { const double t = t0; t0 = t1; t1 = t; }
                if (t0 > tmin) tmin = t0;
                if (t1 < tmax) tmax = t1;
            } else if (o3[a] < 0.0 || o3[a] > h3[a]) {
                hit = 0;
            }
        }
        double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_a = 0.0;
        int64_t total = 0, evaluated = 0, skips = 0, ert = 0;
        if (hit && !(tmax < tmin) && !(tmax < 0.0)) {
            const double t_entry = tmin > 0.0 ? tmin : 0.0;
            total = (int64_t)((tmax - t_entry) / step) + 1;
            int64_t k = 0;
            while (k < total) {
                const double t = t_entry + k * step;
                const double px = clamp_hull(ox + t * dx, hx);
                const double py = clamp_hull(oy + t * dy, hy);
                const double pz = clamp_hull(oz + t * dz, hz);
                const int64_t vx = (int64_t)px, vy = (int64_t)py, vz = (int64_t)pz;
                const int64_t bi = vx / b, bj = vy / b, bk = vz / b;
                const int dval = dist[(bi * by + bj) * bz + bk];
                if (dval == 0) {
                    const int64_t x0 = vx < x_hi ? vx : x_hi, y0 = vy < y_hi ? vy : y_hi;
                    const int64_t z0 = vz < z_hi ? vz : z_hi;
                    const double fx = px - x0, fy = py - y0, fz = pz - z0;
                    const int64_t x1 = nx >= 2 ? x0 + 1 : x0, y1 = ny >= 2 ? y0 + 1 : y0;
                    const int64_t z1 = nz >= 2 ? z0 + 1 : z0;
#define V(x, y, z) vox_f(vox, bits, ((x) * ny + (y)) * nz + (z))
                    const double c000 = V(x0, y0, z0), c100 = V(x1, y0, z0);
                    const double c010 = V(x0, y1, z0), c110 = V(x1, y1, z0);
                    const double c001 = V(x0, y0, z1), c101 = V(x1, y0, z1);
                    const double c011 = V(x0, y1, z1), c111 = V(x1, y1, z1);
#undef V
                    const double gx = 1.0 - fx, gy = 1.0 - fy, gz = 1.0 - fz;
                    const double value =
                        gz * (gy * (gx * c000 + fx * c100) + fy * (gx * c010 + fx * c110)) +
                        fz * (gy * (gx * c001 + fx * c101) + fy * (gx * c011 + fx * c111));
                    int64_t li = (int64_t)(value + 0.5);
                    if (li >= lut_len) li = lut_len - 1;
                    const double alpha = lut[4 * li + 3];
                    if (alpha > 0.0) {
                        const double w = (1.0 - acc_a) * alpha;
                        acc_r += w * lut[4 * li];
                        acc_g += w * lut[4 * li + 1];
                        acc_b += w * lut[4 * li + 2];
                        acc_a += w;
                    }
                    ++evaluated;
                    if (ert_on && acc_a >= ert_thr) {
                        ert = 1;
                        break;
                    }
                    ++k;
                } else {
                    const double t_exit =
                        box_exit(ox, oy, oz, dx, dy, dz, bi, bj, bk, dval - 1, b, hx, hy, hz);
                    int64_t k_next = (int64_t)ceil((t_exit - t_entry) / step - 1e-9);
                    if (k_next <= k) k_next = k + 1;
                    ++skips;
                    k = k_next;
                }
            }
        }
        rgba[4 * r] = acc_r;
        rgba[4 * r + 1] = acc_g;
        rgba[4 * r + 2] = acc_b;
        rgba[4 * r + 3] = acc_a;
        counters[4 * r] = total;
        counters[4 * r + 1] = evaluated;
        counters[4 * r + 2] = skips;
        counters[4 * r + 3] = ert;
    }
}

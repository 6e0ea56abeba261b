/*
 * pdm_oracle.c -- CPU restatement of the reference's distance-map update path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_2407_21552_b200/csrc and the CPU baseline timed by bench.py
 * (cpu_baseline leg and `--impl reference`).  Nothing in the product package
 * links, imports or executes it.  Only tests/, __graft_entry__.smoke() and
 * bench.py may load it (via oracle/__init__.py).
 *
 * Every function restates one reference function over plain arrays; the
 * reference file:line it follows is cited above it (paths are relative to
 * /root/reference/pkg/src/pdmrender).  It is pinned against golden vectors
 * produced by running the reference itself (tests/golden/make_golden.py).
 *
 * Layout conventions (identical to the reference, volume.py:3-4,157-160):
 * volumes and block maps are C-order [x][y][z]; z is the contiguous axis.
 * 8-bit volumes are uint8, 16-bit volumes are uint16 (host endianness).
 *
 * Threading: loops whose iterations write disjoint outputs are split with
 * OpenMP; results never depend on the thread count (checked by tests).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define INF32 (1 << 20) /* _kernels.py:14 */
#define DIST_CLAMP 255  /* acceleration.py:33 */

static int g_threads = 1;

void oracle_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
int oracle_threads(void) { return g_threads; }

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_num_procs();
#else
    return 1;
#endif
}

static inline uint32_t vox_at(const void *vox, int bits, int64_t idx) {
    return bits == 8 ? ((const uint8_t *)vox)[idx] : ((const uint16_t *)vox)[idx];
}

static inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
static inline int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

/*
 * _kernels.py:17-81 chamfer_chebyshev: exact chessboard distance by two raster
 * passes over the 26-neighbourhood with unit weights.  Cells stay at INF32 when
 * nothing is occupied.  occ is uint8 0/1, d is int32, both [nx][ny][nz].
 */
void oracle_chamfer_chebyshev(const uint8_t *occ, int64_t nx, int64_t ny, int64_t nz,
                              int32_t *d) {
    int any_occ = 0;
    const int64_t syz = ny * nz;
    for (int64_t i = 0; i < nx * syz; ++i) {
        if (occ[i]) {
            d[i] = 0;
            any_occ = 1;
        } else {
            d[i] = INF32;
        }
    }
    if (!any_occ) return;
    for (int64_t x = 0; x < nx; ++x)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t z = 0; z < nz; ++z) {
                int64_t c = x * syz + y * nz + z;
                int32_t best = d[c];
                if (best == 0) continue;
                if (x > 0)
                    for (int64_t yy = imax64(y - 1, 0); yy < imin64(y + 2, ny); ++yy)
                        for (int64_t zz = imax64(z - 1, 0); zz < imin64(z + 2, nz); ++zz) {
                            int32_t w = d[(x - 1) * syz + yy * nz + zz] + 1;
                            if (w < best) best = w;
                        }
                if (y > 0)
                    for (int64_t zz = imax64(z - 1, 0); zz < imin64(z + 2, nz); ++zz) {
                        int32_t w = d[x * syz + (y - 1) * nz + zz] + 1;
                        if (w < best) best = w;
                    }
                if (z > 0) {
                    int32_t w = d[c - 1] + 1;
                    if (w < best) best = w;
                }
                d[c] = best;
            }
    for (int64_t x = nx - 1; x >= 0; --x)
        for (int64_t y = ny - 1; y >= 0; --y)
            for (int64_t z = nz - 1; z >= 0; --z) {
                int64_t c = x * syz + y * nz + z;
                int32_t best = d[c];
                if (best == 0) continue;
                if (x < nx - 1)
                    for (int64_t yy = imax64(y - 1, 0); yy < imin64(y + 2, ny); ++yy)
                        for (int64_t zz = imax64(z - 1, 0); zz < imin64(z + 2, nz); ++zz) {
                            int32_t w = d[(x + 1) * syz + yy * nz + zz] + 1;
                            if (w < best) best = w;
                        }
                if (y < ny - 1)
                    for (int64_t zz = imax64(z - 1, 0); zz < imin64(z + 2, nz); ++zz) {
                        int32_t w = d[x * syz + (y + 1) * nz + zz] + 1;
                        if (w < best) best = w;
                    }
                if (z < nz - 1) {
                    int32_t w = d[c + 1] + 1;
                    if (w < best) best = w;
                }
                d[c] = best;
            }
}

/* acceleration.py:177-181 distance_transform: chamfer, then min(raw, 255) as uint8. */
int oracle_distance_transform(const uint8_t *occ, int64_t nx, int64_t ny, int64_t nz,
                              uint8_t *out) {
    int64_t cells = nx * ny * nz;
    int32_t *d = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cells > 0 ? cells : 1));
    if (!d) return 1;
    oracle_chamfer_chebyshev(occ, nx, ny, nz, d);
    for (int64_t i = 0; i < cells; ++i) out[i] = (uint8_t)(d[i] < DIST_CLAMP ? d[i] : DIST_CLAMP);
    free(d);
    return 0;
}

/*
 * acceleration.py:230-233 -- the per-partition distance transforms of
 * build_pdm_set.  occs is [n][cells]; out is [n][cells].  Partitions are
 * independent, so they are spread over threads.
 */
int oracle_distance_transform_batch(const uint8_t *occs, int64_t n, int64_t nx, int64_t ny,
                                    int64_t nz, uint8_t *out) {
    int64_t cells = nx * ny * nz;
    int err = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads) reduction(| : err)
    for (int64_t p = 0; p < n; ++p)
        err |= oracle_distance_transform(occs + p * cells, nx, ny, nz, out + p * cells);
    return err;
}

/*
 * _kernels.py:137-149 partition_presence: out[pid[v], x/b, y/b, z/b] = 1 for
 * every voxel.  out is uint8 [n][bx][by][bz] and must arrive zeroed.  Threads
 * own disjoint block rows i so writes never collide.
 */
void oracle_partition_presence(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz,
                               int64_t b, const int32_t *pid, int64_t n, uint8_t *out) {
    (void)n;
    int64_t bx = (nx + b - 1) / b, by = (ny + b - 1) / b, bz = (nz + b - 1) / b;
    int64_t nb = bx * by * bz;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int64_t i = 0; i < bx; ++i)
        for (int64_t x = i * b; x < imin64((i + 1) * b, nx); ++x)
            for (int64_t y = 0; y < ny; ++y) {
                int64_t j = y / b;
                const int64_t row = (x * ny + y) * nz;
                for (int64_t z = 0; z < nz; ++z) {
                    int32_t p = pid[vox_at(vox, bits, row + z)];
                    out[(int64_t)p * nb + (i * by + j) * bz + z / b] = 1;
                }
            }
}

/*
 * _kernels.py:84-110 block_any_in_range (mode="voxel" of
 * occupancy_for_partition, acceleration.py:131-136): out[blk] = 1 when any
 * in-bounds voxel of the block lies in [lo, hi].
 */
void oracle_block_any_in_range(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz,
                               int64_t b, uint32_t lo, uint32_t hi, uint8_t *out) {
    int64_t bx = (nx + b - 1) / b, by = (ny + b - 1) / b, bz = (nz + b - 1) / b;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int64_t i = 0; i < bx; ++i) {
        int64_t x1 = imin64((i + 1) * b, nx);
        for (int64_t j = 0; j < by; ++j) {
            int64_t y1 = imin64((j + 1) * b, ny);
            for (int64_t k = 0; k < bz; ++k) {
                int64_t z1 = imin64((k + 1) * b, nz);
                uint8_t occ = 0;
                for (int64_t x = i * b; x < x1 && !occ; ++x)
                    for (int64_t y = j * b; y < y1 && !occ; ++y)
                        for (int64_t z = k * b; z < z1; ++z) {
                            uint32_t v = vox_at(vox, bits, (x * ny + y) * nz + z);
                            if (v >= lo && v <= hi) {
                                occ = 1;
                                break;
                            }
                        }
                out[(i * by + j) * bz + k] = occ;
            }
        }
    }
}

/*
 * _kernels.py:113-134 block_any_nonzero (mode="voxel" of occupancy_for_tf,
 * acceleration.py:165-168): out[blk] = 1 when nz_lut[v] != 0 for some voxel.
 */
void oracle_block_any_nonzero(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz,
                              int64_t b, const uint8_t *nz_lut, uint8_t *out) {
    int64_t bx = (nx + b - 1) / b, by = (ny + b - 1) / b, bz = (nz + b - 1) / b;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int64_t i = 0; i < bx; ++i) {
        int64_t x1 = imin64((i + 1) * b, nx);
        for (int64_t j = 0; j < by; ++j) {
            int64_t y1 = imin64((j + 1) * b, ny);
            for (int64_t k = 0; k < bz; ++k) {
                int64_t z1 = imin64((k + 1) * b, nz);
                uint8_t occ = 0;
                for (int64_t x = i * b; x < x1 && !occ; ++x)
                    for (int64_t y = j * b; y < y1 && !occ; ++y)
                        for (int64_t z = k * b; z < z1; ++z)
                            if (nz_lut[vox_at(vox, bits, (x * ny + y) * nz + z)]) {
                                occ = 1;
                                break;
                            }
                out[(i * by + j) * bz + k] = occ;
            }
        }
    }
}

/*
 * volume.py:262-300 block_min_max: _erode3/_dilate3 take the 3x3x3 min/max
 * around each voxel (clipped at the bounds) and _block_reduce folds those over
 * each block; composed, that is the min/max over the block grown by a 1-voxel
 * apron clipped to the volume (the reference's own oracle,
 * tests/test_volume.py:32-47, states it that way and so does this loop).
 * mins/maxs have the volume's dtype and shape bdims.
 */
void oracle_block_min_max(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz,
                          int64_t b, void *mins, void *maxs) {
    int64_t bx = (nx + b - 1) / b, by = (ny + b - 1) / b, bz = (nz + b - 1) / b;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int64_t i = 0; i < bx; ++i) {
        int64_t x0 = imax64(i * b - 1, 0), x1 = imin64((i + 1) * b + 1, nx);
        for (int64_t j = 0; j < by; ++j) {
            int64_t y0 = imax64(j * b - 1, 0), y1 = imin64((j + 1) * b + 1, ny);
            for (int64_t k = 0; k < bz; ++k) {
                int64_t z0 = imax64(k * b - 1, 0), z1 = imin64((k + 1) * b + 1, nz);
                uint32_t mn = 0xFFFFFFFFu, mx = 0;
                for (int64_t x = x0; x < x1; ++x)
                    for (int64_t y = y0; y < y1; ++y) {
                        const int64_t row = (x * ny + y) * nz;
                        for (int64_t z = z0; z < z1; ++z) {
                            uint32_t v = vox_at(vox, bits, row + z);
                            if (v < mn) mn = v;
                            if (v > mx) mx = v;
                        }
                    }
                int64_t o = (i * by + j) * bz + k;
                if (bits == 8) {
                    ((uint8_t *)mins)[o] = (uint8_t)mn;
                    ((uint8_t *)maxs)[o] = (uint8_t)mx;
                } else {
                    ((uint16_t *)mins)[o] = (uint16_t)mn;
                    ((uint16_t *)maxs)[o] = (uint16_t)mx;
                }
            }
        }
    }
}

/*
 * acceleration.py:223-229 -- build_pdm_set's range_apron occupancy:
 * occ_p = (min <= hi_p) & (max >= lo_p) for every partition p.  Also serves
 * occupancy_for_partition(mode="range_apron"), acceleration.py:138-141
 * (n == 1).  out is uint8 [n][nblocks].
 */
void oracle_range_apron_presence(const void *mins, const void *maxs, int bits, int64_t nblocks,
                                 const uint32_t *lo, const uint32_t *hi, int64_t n,
                                 uint8_t *out) {
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t p = 0; p < n; ++p)
        for (int64_t c = 0; c < nblocks; ++c) {
            uint32_t mn = vox_at(mins, bits, c), mx = vox_at(maxs, bits, c);
            out[p * nblocks + c] = (uint8_t)(mn <= hi[p] && mx >= lo[p]);
        }
}

/*
 * acceleration.py:169-173 -- occupancy_for_tf(mode="range_apron"): prefix
 * count of alpha > 0 over [min, max] of the block's apron.  alpha is the f64
 * LUT alpha column (length span, stride alpha_stride doubles).
 */
int oracle_range_apron_tf(const void *mins, const void *maxs, int bits, int64_t nblocks,
                          const double *alpha, int64_t span, int64_t alpha_stride,
                          uint8_t *out) {
    int64_t *nz = (int64_t *)malloc(sizeof(int64_t) * (size_t)(span + 1));
    if (!nz) return 1;
    nz[0] = 0;
    for (int64_t v = 0; v < span; ++v) nz[v + 1] = nz[v] + (alpha[v * alpha_stride] > 0.0);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t c = 0; c < nblocks; ++c) {
        uint32_t mn = vox_at(mins, bits, c), mx = vox_at(maxs, bits, c);
        out[c] = (uint8_t)(nz[mx + 1] - nz[mn] > 0);
    }
    free(nz);
    return 0;
}

/*
 * transfer.py:250-259 select_partitions: flags[pid[v]] = 1 for every
 * intensity v with alpha[v] > 0.0 (an f64 compare: NaN is transparent,
 * denormals are visible).  flags is uint8 [n] and is cleared here.
 */
void oracle_select(const double *alpha, int64_t span, int64_t alpha_stride, const int32_t *pid,
                   int64_t n, uint8_t *flags) {
    memset(flags, 0, (size_t)n);
    for (int64_t v = 0; v < span; ++v)
        if (alpha[v * alpha_stride] > 0.0) flags[pid[v]] = 1;
}

/*
 * acceleration.py:244-276 combine: element-wise minimum of the selected
 * partitions' maps; an empty selection gives the all-255 map.  pdms is the
 * contiguous [n][map_bytes] set, sel holds 0-based partition indices.
 */
void oracle_combine(const uint8_t *pdms, int64_t map_bytes, const int32_t *sel, int64_t k,
                    uint8_t *out) {
    const int64_t chunk = 1 << 16;
    int64_t nchunks = (map_bytes + chunk - 1) / chunk;
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t c = 0; c < nchunks; ++c) {
        int64_t lo = c * chunk, hi = imin64(lo + chunk, map_bytes);
        memset(out + lo, DIST_CLAMP, (size_t)(hi - lo));
        for (int64_t m = 0; m < k; ++m) {
            const uint8_t *src = pdms + (int64_t)sel[m] * map_bytes;
            for (int64_t i = lo; i < hi; ++i) out[i] = src[i] < out[i] ? src[i] : out[i];
        }
    }
}

/*
 * Shared synthetic-volume generator (not a reference function): background 0
 * plus axis-aligned boxes, each filled with hashed intensities inside its band;
 * later boxes overwrite earlier ones.  The CUDA kernel pdm_synth_volume in
 * paper_2407_21552_b200/csrc/synth.cu evaluates the identical formula, so the
 * CPU and GPU arms see the same bytes.  boxes is int64 [nbox][8]:
 * x0 x1 y0 y1 z0 z1 band_lo band_hi (half-open spatial ranges).
 * Only the x-slab [xs0, xs1) is produced (out holds (xs1-xs0)*ny*nz voxels).
 */
static inline uint64_t synth_mix(uint64_t h) {
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdULL;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ULL;
    h ^= h >> 33;
    return h;
}

void oracle_synth_volume(int bits, int64_t nx, int64_t ny, int64_t nz, int64_t xs0, int64_t xs1,
                         const int64_t *boxes, int64_t nbox, uint64_t seed, void *out) {
    (void)nx;
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t x = xs0; x < xs1; ++x)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t z = 0; z < nz; ++z) {
                uint32_t v = 0;
                for (int64_t q = 0; q < nbox; ++q) {
                    const int64_t *bx = boxes + q * 8;
                    if (x >= bx[0] && x < bx[1] && y >= bx[2] && y < bx[3] && z >= bx[4] &&
                        z < bx[5]) {
                        uint64_t idx = ((uint64_t)x * (uint64_t)ny + (uint64_t)y) * (uint64_t)nz +
                                       (uint64_t)z;
                        uint64_t h = synth_mix(idx ^ (seed * 0x9E3779B97F4A7C15ULL) ^
                                               ((uint64_t)q << 56));
                        uint64_t width = (uint64_t)(bx[7] - bx[6] + 1);
                        v = (uint32_t)(bx[6] + (int64_t)(h % width));
                    }
                }
                int64_t o = ((x - xs0) * ny + y) * nz + z;
                if (bits == 8)
                    ((uint8_t *)out)[o] = (uint8_t)v;
                else
                    ((uint16_t *)out)[o] = (uint16_t)v;
            }
}

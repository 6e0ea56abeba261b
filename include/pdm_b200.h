/*
 * pdm_b200.h -- C ABI of the B200-native distance-map update path
 * (arXiv 2407.21552: partitioned occupancy / distance maps).
 *
 * Every entry point:
 *   - takes caller-owned DEVICE pointers (plus plain sizes) and a CUDA stream
 *     (`pdm_stream_t` is a cudaStream_t; NULL means the legacy default stream),
 *   - enqueues its kernels on that stream and returns without synchronising,
 *   - allocates nothing on the update path (scratch comes from the caller),
 *   - returns PDM_OK (0) or an error code; pdm_last_error() then holds a
 *     message for the calling thread.
 *
 * Layouts (same as the reference, volume.py:3-4,157-160): a volume is C-order
 * [nx][ny][nz] (z contiguous) of uint8 (bits=8) or uint16 (bits=16); a block
 * map is C-order [bx][by][bz] with bd = ceil(d / b).  A partitioned distance
 * map set is partition-major [n][plane_pitch] uint8: map p starts at byte
 * p * plane_pitch and holds bx*by*bz bytes; plane_pitch >= bx*by*bz.  A
 * partition mask is [bx*by*bz][words] uint32, bit p of block c at
 * mask[c*words + p/32] >> (p%32).
 *
 * Each function cites the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/pdmrender).  The reference "FFI" is numba functions
 * over numpy arrays (_kernels.py) plus numpy ufunc loops.
 */
#ifndef PDM_B200_H
#define PDM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *pdm_stream_t;

enum pdm_status {
    PDM_OK = 0,
    PDM_EINVAL = 1,      /* bad argument (maps to ValueError / reference error classes) */
    PDM_ECUDA = 2,       /* CUDA launch or runtime failure (RuntimeError) */
    PDM_EUNSUPPORTED = 3 /* shape outside what a kernel supports (RuntimeError) */
};

/* ---- library ------------------------------------------------------------ */
int pdm_version(void);              /* ABI version, currently 1 */
const char *pdm_last_error(void);   /* message of the last failing call (thread-local) */
int pdm_device_sm_count(int device);
/* Wait for all work enqueued on `stream` (the public API's completion point:
 * the reference's functions return finished results). */
int pdm_stream_synchronize(pdm_stream_t stream);
/* dst[0..bytes) = value, stream-ordered (a constant map: the all-255 D of an
 * empty TF support, the all-0 D of a full one). */
int pdm_fill_u8(uint8_t *dst, int64_t bytes, int32_t value, pdm_stream_t stream);

/* volume.py:86-90 intensity_range of a device-resident volume: out[0] = min,
 * out[1] = max over count voxels (out: device uint32[2]). */
int pdm_volume_range(const void *vox, int bits, int64_t count, uint32_t *out,
                     pdm_stream_t stream);

/* acceleration.py:77-79 DistanceMap.occupied_fraction on the device:
 * *count = number of bytes of data[0..bytes) equal to value (device
 * unsigned long long, cleared first). */
int pdm_count_value(const uint8_t *data, int64_t bytes, uint32_t value,
                    unsigned long long *count, pdm_stream_t stream);

/* ---- selection (K8) -------------------------------------------------------
 * transfer.py:250-259 select_partitions: flags[p] = 1 iff some intensity v of
 * partition p has alpha[v * alpha_stride] > 0.0 (f64 compare: NaN transparent,
 * denormals visible), else 0 -- every flag is written.  starts: device
 * int32[n+1], partition p = [starts[p], starts[p+1]) (contiguous, covering,
 * starts[n] = span, transfer.py:124-148), or NULL for the uniform scheme
 * (scheme_uniform, transfer.py:201-203: span / n wide, the first span % n
 * partitions one wider); max_width = widest partition (picks
 * a CTA or a warp per partition).  flags: device uint8[n]. */
int pdm_select(const double *alpha, int64_t span, int64_t alpha_stride, const int32_t *starts,
               int32_t n, int32_t max_width, uint8_t *flags, pdm_stream_t stream);

/* select_partitions(tf, scheme) end to end (transfer.py:250-259): gathers
 * alpha = lut_alpha[i * lut_stride] (host memory, e.g. &lut[0][3] with
 * lut_stride 4) into pinned stage_host, runs pdm_select on it with the kernel
 * reading stage_host and writing pinned flags_host (uint8[n]) directly
 * (zero-copy over PCIe: one launch, one wait), and synchronises `stream`:
 * returns with the finished selection on the host.  stage_dev (f64[span]) and
 * flags_dev (uint8[n]) are only used, and then required, with
 * PDM_SELECT_DMA=1 (H2D alpha, select in HBM, D2H flags). */
int pdm_select_tf(const double *lut_alpha, int64_t span, int64_t lut_stride, double *stage_host,
                  double *stage_dev, const int32_t *starts, int32_t n, int32_t max_width,
                  uint8_t *flags_dev, uint8_t *flags_host, pdm_stream_t stream);

/* transfer.py:250-259 on the LUT alone: nz[v] = alpha[v] > 0.0 and, when
 * prefix != NULL, prefix[v+1] = #{u <= v : alpha[u] > 0} with prefix[0] = 0
 * (the np.cumsum of acceleration.py:171).  prefix needs span+1 int32 and
 * then nz must be 16-byte aligned. */
int pdm_alpha_support(const double *alpha, int64_t span, int64_t alpha_stride, uint8_t *nz,
                      int32_t *prefix, pdm_stream_t stream);

/* ---- TF-change merge (K7) -------------------------------------------------
 * acceleration.py:244-276 combine: out[c] = min over the k selected maps of
 * pdms[sel[i]][c] (sel = HOST array of 0-based partition indices, passed by
 * value in kernel parameters); k == 0 writes the all-255 map. */
int pdm_combine(const uint8_t *pdms, int64_t plane_pitch, int64_t map_bytes, int32_t n,
                const int32_t *sel, int32_t k, uint8_t *out, pdm_stream_t stream);

/* Same merge with the selection resident in device memory (flags from
 * pdm_select): select + merge with no host round trip, graph-capturable. */
int pdm_combine_flags(const uint8_t *pdms, int64_t plane_pitch, int64_t map_bytes, int32_t n,
                      const uint8_t *flags, uint8_t *out, pdm_stream_t stream);

/* ---- nibble-packed planes (B200 storage for the merge) --------------------
 * Each map is a clamped Chebyshev distance field, so 16 consecutive blocks of
 * a z row span <= 15 values: chunk c (blocks 16c..16c+15) is stored as
 * base[c] = its min plus 8 bytes of 4-bit offsets (nib[c], block 16c+2j in
 * the low nibble of byte j).  No reference counterpart: an internal encoding
 * of acceleration.py:89-99 PdmSet.pdms; the merge over it is bit-identical to
 * pdm_combine.  pdm_packed_chunks(map_bytes) = chunks per plane (even, padded
 * with 255); nib_pitch >= 8 * chunks, base_pitch >= chunks.  *violations
 * (device) receives the number of chunks spanning > 15 values; the packed
 * planes are valid only when it is 0. */
int pdm_packed_chunks(int64_t map_bytes);
int pdm_pack_pdms(const uint8_t *pdms, int64_t plane_pitch, int64_t map_bytes, int32_t n,
                  uint8_t *nib, int64_t nib_pitch, uint8_t *base, int64_t base_pitch,
                  uint32_t *violations, pdm_stream_t stream);

/* *count = number of 16-block chunks (linear order, per plane; the last one
 * partial) of planes pdms[p * plane_pitch ..][0..map_bytes) whose
 * consecutive bytes differ by more than 1 -- 0 means the D' of any selection
 * may cross PCIe in the delta forms (a set loaded from a dump,
 * acceleration.py:279-354, is checked before they are used). */
int pdm_count_nonlipschitz_chunks(const uint8_t *pdms, int64_t plane_pitch, int64_t map_bytes,
                                  int32_t n, uint32_t *count, pdm_stream_t stream);

/* pdm_distance_transform_mask followed by pdm_pack_pdms, with the packing
 * fused into the last (z) pass when bz is 128, 256 or 512 (the rows are
 * packed while still in shared memory); base_pitch % 4 == 0.  tile_bounds
 * (may be NULL): also the merge's per-tile plane bounds (as
 * pdm_packed_tile_bounds), taken from the same rows in the fused case. */
int pdm_distance_transform_mask_packed(const uint32_t *mask, int32_t words, int32_t n, int64_t bx,
                                       int64_t by, int64_t bz, uint8_t *pdms,
                                       int64_t plane_pitch, uint8_t *nib, int64_t nib_pitch,
                                       uint8_t *base, int64_t base_pitch, uint32_t *violations,
                                       uint16_t *tile_bounds, pdm_stream_t stream);

/* Per-tile plane bounds of a packed set, for the merges' tile skip:
 * tile_bounds[tile][p] = min | max << 8 of plane p over blocks
 * [1024 tile, 1024 tile + 1024) (uint16 [ceil(map_bytes / 1024)][n]).  With
 * them a merge reads, per tile, only the selected planes whose minimum is
 * below the smallest maximum among the selected planes (the others cannot
 * lower any block of the tile) -- exact.  Recompute after the planes change. */
int pdm_packed_tile_bounds(const uint8_t *nib, int64_t nib_pitch, const uint8_t *base,
                           int64_t base_pitch, int64_t map_bytes, int32_t n,
                           uint16_t *tile_bounds, pdm_stream_t stream);

/* Measurement hook: while planes_read != NULL every packed merge adds the
 * number of (1024-block tile, selected plane) pairs it read to *planes_read
 * (device uint64); NULL turns it off. */
int pdm_merge_stats(unsigned long long *planes_read);

/* pdm_combine over packed planes (k <= 240), and pdm_combine_flags over them
 * (n <= 4096, PDL behind pdm_select).  Output: plain uint8 D'.  zero_count
 * (device uint64, may be NULL): set to the number of D' blocks equal to 0 --
 * DistanceMap.occupied_fraction (acceleration.py:77-79) fused into the merge.
 * tile_bounds (from pdm_packed_tile_bounds, may be NULL): per-tile plane skip
 * for selections of up to 64 planes. */
int pdm_combine_packed(const uint8_t *nib, int64_t nib_pitch, const uint8_t *base,
                       int64_t base_pitch, const uint16_t *tile_bounds, int64_t map_bytes,
                       int32_t n, const int32_t *sel, int32_t k, uint8_t *out,
                       unsigned long long *zero_count, pdm_stream_t stream);
int pdm_combine_flags_packed(const uint8_t *nib, int64_t nib_pitch, const uint8_t *base,
                             int64_t base_pitch, const uint16_t *tile_bounds, int64_t map_bytes,
                             int32_t n, const uint8_t *flags, uint8_t *out,
                             unsigned long long *zero_count, pdm_stream_t stream);

/* pdm_combine_flags_packed with the set's raw planes beside the packed ones
 * (pdms[n][plane_pitch], the pdm_combine_flags layout): the kernel compacts
 * the flags on the device and, for selections of up to 4 planes (the
 * latency-bound end of the packed merge; PDM_RAW_MAX_K overrides, 0 = never)
 * and no zero count, merges the raw planes instead.  Same D' either way.
 * Replaces acceleration.py:244-276 combine for a device-resident selection. */
int pdm_combine_flags_auto(const uint8_t *pdms, int64_t plane_pitch, const uint8_t *nib,
                           int64_t nib_pitch, const uint8_t *base, int64_t base_pitch,
                           const uint16_t *tile_bounds, int64_t map_bytes, int32_t n,
                           const uint8_t *flags, uint8_t *out, unsigned long long *zero_count,
                           pdm_stream_t stream);
/* The largest selection pdm_combine_flags_auto merges from the raw planes. */
int pdm_combine_raw_max_k(void);

/* The same two merges writing D' itself in the packed encoding (out_nib: 8 *
 * chunks bytes, out_base: chunks bytes, 16/2-byte aligned) -- 9/16 of the
 * bytes, for a D' headed to host memory over PCIe (combine(...).dist), where
 * pdm_unpack_packed_host expands it into map_bytes plain bytes (host
 * function, SSE2 + OpenMP; no device work). */
int pdm_combine_packed_to_packed(const uint8_t *nib, int64_t nib_pitch, const uint8_t *base,
                                 int64_t base_pitch, int64_t map_bytes, int32_t n,
                                 const int32_t *sel, int32_t k, uint8_t *out_nib,
                                 uint8_t *out_base, pdm_stream_t stream);
int pdm_combine_flags_packed_to_packed(const uint8_t *nib, int64_t nib_pitch,
                                       const uint8_t *base, int64_t base_pitch,
                                       int64_t map_bytes, int32_t n, const uint8_t *flags,
                                       uint8_t *out_nib, uint8_t *out_base,
                                       pdm_stream_t stream);
int pdm_unpack_packed_host(const uint8_t *nib, const uint8_t *base, int64_t map_bytes,
                           uint8_t *out);

/* Host expansion of D' in the delta form: per 16-block chunk c, base[c] is
 * block 16c and code word c (little-endian u32 at codes + 4c) holds, for
 * blocks 1..15, (step from the previous block + 1) in 2 bits each.  Valid
 * for maps that change by at most 1 per block inside each chunk.  Host
 * function (AVX-512 VBMI when present, else SSE2; OpenMP). */
int pdm_unpack_delta_host(const uint8_t *codes, const uint8_t *base, int64_t map_bytes,
                          uint8_t *out);

/* Host expansion of D' in the sparse delta form (format 3): per 32 items (64
 * chunks) one 336-byte region -- u64 nz, u64 dd (bit c: chunk c is not
 * all-zero / is not flat), the bases of the non-zero chunks, then
 * from the next 4-byte boundary the delta code words (as in
 * pdm_unpack_delta_host) of the non-flat chunks, both compacted in chunk
 * order.  Host function. */
int pdm_unpack_sparse_host(const uint8_t *regions, int64_t map_bytes, uint8_t *out);

/* combine(...).dist in one call: the merge writes D' in a compact form in
 * `pieces` launches (an event after each) straight into pinned host staging
 * (stage_nib: 8 (format 1, nibbles) or 4 (format 2, deltas) bytes per chunk;
 * stage_base: 1 byte per chunk; format 3, sparse deltas: stage_nib holds
 * ceil(items / 32) regions of 336 bytes, stage_base is unused), and the host
 * expands piece i into `out` (map_bytes) while later pieces cross PCIe.
 * Formats 2 and 3 require every selected map to be 1-Lipschitz along z
 * within chunks (true for sets built by the distance transform with
 * bz % 16 == 0).  Selection: device flags[n]
 * when flags != NULL (PDL behind pdm_select), else host sel[0..k).  Returns
 * once `out` is complete. */
int pdm_merge_packed_to_host(const uint8_t *nib, int64_t nib_pitch, const uint8_t *base,
                             int64_t base_pitch, const uint16_t *tile_bounds, int64_t map_bytes,
                             int32_t n, const uint8_t *flags, const int32_t *sel, int32_t k,
                             uint8_t *stage_nib, uint8_t *stage_base, uint8_t *out,
                             int32_t pieces, int32_t format, pdm_stream_t stream);

/* combine() for a caller that reads the host view (acceleration.py:244-276 +
 * DistanceMap.dist, :65-75), in one pass: the packed merge writes D' as plain
 * bytes into dprime_dev (HBM, map_bytes, 16-byte aligned) AND in the sparse
 * delta form (format 3 of pdm_merge_packed_to_host) into pinned `stage`; the
 * host expands piece i into `out` while later pieces are merged.  Returns
 * once both D' copies are complete.  Same selection and Lipschitz
 * requirements as pdm_merge_packed_to_host format 3. */
int pdm_combine_packed_host(const uint8_t *nib, int64_t nib_pitch, const uint8_t *base,
                            int64_t base_pitch, const uint16_t *tile_bounds, int64_t map_bytes,
                            int32_t n, const uint8_t *flags, const int32_t *sel, int32_t k,
                            uint8_t *dprime_dev, uint8_t *stage, uint8_t *out, int32_t pieces,
                            pdm_stream_t stream);

/* DistanceMap.dist for a finished D' in HBM (acceleration.py:71-79 host view;
 * combine() itself completes D' on the device, acceleration.py:244-276): D'
 * (map_bytes plain bytes, 16-byte aligned) is re-encoded in `pieces` launches
 * in compact form `format` (1 nibbles, 2 deltas, 3 sparse deltas; staging as
 * in pdm_merge_packed_to_host) straight into pinned host staging, and the
 * host expands piece i into `out` while later pieces cross PCIe.  Formats 2
 * and 3 require D' to be 1-Lipschitz along z within 16-block chunks (a min of
 * distance fields with bz % 16 == 0).  Returns once `out` is complete. */
int pdm_dprime_to_host(const uint8_t *d, int64_t map_bytes, uint8_t *stage, uint8_t *stage_base,
                       uint8_t *out, int32_t pieces, int32_t format, pdm_stream_t stream);

/* Host function: dst[i] = src[i * stride] for i < n (OpenMP) -- stages a
 * TF's alpha column lut[:, 3] (transfer.py:44-70) into pinned memory for the
 * select upload (transfer.py:250-259 reads tf.lut on every call). */
int pdm_gather_f64_host(const double *src, int64_t n, int64_t stride, double *dst);

/* ---- block reduction / occupancy (K1-K5) --------------------------------- */

/* volume.py:289-300 block_min_max: per-block min/max over the block grown by a
 * 1-voxel apron clipped to the volume; mins/maxs have the volume's dtype. */
int pdm_block_min_max(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz, int32_t b,
                      void *mins, void *maxs, pdm_stream_t stream);

/* _kernels.py:137-149 partition_presence (build_pdm_set voxel branch,
 * acceleration.py:219-222): bit p of block c set iff some in-bounds voxel v of
 * the block has pid[v] == p.  mask is overwritten. */
int pdm_partition_mask_voxel(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz,
                             int32_t b, const int32_t *pid, int32_t n, uint32_t *mask,
                             int32_t words, pdm_stream_t stream);

/* acceleration.py:223-229 (build_pdm_set range_apron branch): bit p set iff
 * pid[min] <= p <= pid[max] for the block's apron min/max -- equivalent to
 * (min <= hi_p) & (max >= lo_p) for contiguous covering partitions.  Reads the
 * volume directly (fused block_min_max).  mask is overwritten. */
int pdm_partition_mask_range_apron(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz,
                                   int32_t b, const int32_t *pid, int32_t n, uint32_t *mask,
                                   int32_t words, pdm_stream_t stream);

/* Same from precomputed min/max (the minmax= argument of the reference API). */
int pdm_partition_mask_minmax(const void *mins, const void *maxs, int bits, int64_t nblocks,
                              const int32_t *pid, int32_t n, uint32_t *mask, int32_t words,
                              pdm_stream_t stream);

/* _kernels.py:84-110 block_any_in_range and _kernels.py:113-134
 * block_any_nonzero (voxel-mode occupancy_for_partition / occupancy_for_tf,
 * acceleration.py:131-136,165-168): out[c] = 1 iff lut[v] != 0 for some
 * in-bounds voxel v of block c.  lut: device uint8[2^bits]. */
int pdm_block_any_lut(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz, int32_t b,
                      const uint8_t *lut, uint8_t *out, pdm_stream_t stream);

/* Slab-sharded range_apron: fold the apron min/max of a neighbour slab's
 * boundary voxel plane (pdm_block_min_max of a 1 x ny x nz volume) into the
 * slab's first/last block plane: mins = min(mins, plane_mins), maxs = max(...).
 * count = by * bz. */
int pdm_minmax_fold(void *mins, void *maxs, const void *plane_mins, const void *plane_maxs,
                    int bits, int64_t count, pdm_stream_t stream);

/* acceleration.py:138-141 (range_apron occupancy_for_partition):
 * out[c] = (mins[c] <= hi) & (maxs[c] >= lo). */
int pdm_occupancy_minmax_range(const void *mins, const void *maxs, int bits, int64_t nblocks,
                               uint32_t lo, uint32_t hi, uint8_t *out, pdm_stream_t stream);

/* acceleration.py:169-173 (range_apron occupancy_for_tf):
 * out[c] = prefix[maxs[c]+1] - prefix[mins[c]] > 0. */
int pdm_occupancy_minmax_prefix(const void *mins, const void *maxs, int bits, int64_t nblocks,
                                const int32_t *prefix, uint8_t *out, pdm_stream_t stream);

/* ---- Chebyshev distance transform (K6) ------------------------------------
 * _kernels.py:17-81 chamfer_chebyshev + acceleration.py:177-181 clamp: exact
 * chessboard distance (in blocks) to the nearest occupied block, clamped at
 * 255, 255 everywhere when nothing is occupied.  Computed as three separable
 * passes (1-D distance along x, then lower-envelope min-max passes along y and
 * z), bit-identical to the reference's two raster passes. */

/* One map from a uint8 occupancy [bx][by][bz] (nonzero = occupied). */
int pdm_distance_transform(const uint8_t *occ, int64_t bx, int64_t by, int64_t bz, uint8_t *out,
                           pdm_stream_t stream);

/* Full recompute for one TF, fused (acceleration.py:184-196
 * standard_distance_map = occupancy_for_tf :145-174 + distance_transform
 * :177-181): the block occupancy is written straight into out as the
 * transform's seed (0 occupied, 255 empty) and the passes run in place, so no
 * bool map is materialised.  out = uint8 [bx][by][bz], identical to
 * pdm_block_any_lut / pdm_occupancy_minmax_prefix followed by
 * pdm_distance_transform.
 * voxel: lut = the TF's nz LUT (pdm_alpha_support), voxel-exact occupancy.
 * minmax: range_apron occupancy from apron mins/maxs (pdm_block_min_max) and
 *   the TF's prefix count (pdm_alpha_support). */
int pdm_standard_distance_map_voxel(const void *vox, int bits, int64_t nx, int64_t ny, int64_t nz,
                                    int32_t b, const uint8_t *lut, uint8_t *out,
                                    pdm_stream_t stream);
int pdm_standard_distance_map_minmax(const void *mins, const void *maxs, int bits, int64_t bx,
                                     int64_t by, int64_t bz, const int32_t *prefix, uint8_t *out,
                                     pdm_stream_t stream);

/* All n partition maps of a mask (acceleration.py:230-233, the batched
 * transforms of build_pdm_set) into pdms [n][plane_pitch]. */
int pdm_distance_transform_mask(const uint32_t *mask, int32_t words, int32_t n, int64_t bx,
                                int64_t by, int64_t bz, uint8_t *pdms, int64_t plane_pitch,
                                pdm_stream_t stream);

/* Slab-sharded pieces (multi-GPU, x split into contiguous slabs of block planes).
 * pass_x: local 1-D distance along x of each partition inside the slab.
 * slab_edges: edges[0][p][y][z] = g[p][0][y][z], edges[1][p][y][z] = g[p][bx-1][y][z].
 * slab_fold: edges_all is the all-gathered [world][2][n][by][bz] edge planes
 *   of every slab (its own included); slab_x0 is a HOST int64 [world+1] array of
 *   slab start planes (slab r spans [slab_x0[r], slab_x0[r+1])).  For this
 *   rank's slab it folds in the nearest occupied block of every other slab:
 *   g[p][x] = min(g, below + x, above + bx-1-x) clamped at 255, with
 *   below = min_{j<rank} hi_j + x0 - x1_j + 1 and
 *   above = min_{j>rank} lo_j + x0_j - x1 + 1 (x0/x1 = this slab's bounds).
 * pass_yz: the two min-max passes (y, then z). */
int pdm_dt_pass_x_mask(const uint32_t *mask, int32_t words, int32_t n, int64_t bx, int64_t by,
                       int64_t bz, uint8_t *pdms, int64_t plane_pitch, pdm_stream_t stream);
int pdm_dt_slab_edges(const uint8_t *pdms, int64_t plane_pitch, int32_t n, int64_t bx,
                      int64_t by, int64_t bz, uint8_t *edges, pdm_stream_t stream);
int pdm_dt_slab_fold(uint8_t *pdms, int64_t plane_pitch, int32_t n, int64_t bx, int64_t by,
                     int64_t bz, const uint8_t *edges_all, int32_t world, int32_t rank,
                     const int64_t *slab_x0, pdm_stream_t stream);
int pdm_dt_pass_yz(uint8_t *pdms, int64_t plane_pitch, int32_t n, int64_t bx, int64_t by,
                   int64_t bz, pdm_stream_t stream);

/* ---- multi-GPU precompute over NCCL -----------
 * NCCL is loaded at run time (libnccl.so.2; inside a torch process that is
 * torch's own, so ProcessGroupNCCL._comm_ptr() communicators work).
 * `comm` is an ncclComm_t passed as void*. */
int pdm_nccl_available(void); /* 1 if NCCL could be loaded */
int pdm_nccl_unique_id(uint8_t *id_out /* 128 bytes */);
int pdm_nccl_comm_init(void **comm_out, int32_t world, const uint8_t *id, int32_t rank);
int pdm_nccl_comm_destroy(void *comm);
int pdm_nccl_comm_count(void *comm); /* ranks of the communicator, -1 on error */
/* Workspace bytes pdm_build_pdm_set_slab_nccl needs (-1 on bad sizes). */
int64_t pdm_build_pdm_set_slab_nccl_workspace(int32_t world, int bits, int64_t nx, int64_t ny,
                                              int64_t nz, int32_t b, int32_t n);
/* acceleration.py:199-241 build_pdm_set over this rank's x-slab (nx voxel
 * planes; every slab but the last a whole number of blocks) of a volume split
 * across the communicator's ranks in rank order: the slab table is
 * all-gathered and validated identically on every rank (bx0_expected >= 0
 * also checks this rank's start block plane); range_apron (mode 1) swaps one
 * boundary voxel plane with each neighbour (ncclSend/Recv); the distance
 * transform all-gathers 2*n*by*bz edge bytes per rank and folds them in
 * (bit-exact with the single-device transform).  Writes this rank's slab of
 * every plane (pdms [n][plane_pitch]) and, when nib != NULL, the merge's
 * packed planes; slab_out (host int64[3]) = start, end, total block planes.
 * Stream-ordered on `stream` (NCCL included); synchronises once, after the
 * slab table. */
int pdm_build_pdm_set_slab_nccl(void *comm, const void *vox, int bits, int64_t nx, int64_t ny,
                                int64_t nz, int32_t b, const int32_t *pid, int32_t n,
                                int32_t mode, int64_t bx0_expected, uint8_t *pdms,
                                int64_t plane_pitch, uint8_t *nib, int64_t nib_pitch,
                                uint8_t *base, int64_t base_pitch, uint32_t *violations,
                                void *workspace, int64_t workspace_bytes, int64_t *slab_out,
                                pdm_stream_t stream);

/* ---- synthetic volumes (bench / test inputs, not a reference function) ----
 * Background 0 plus hashed-intensity boxes; boxes = HOST int64 [nbox][8]
 * (x0 x1 y0 y1 z0 z1 band_lo band_hi).  Writes the x-slab [xs0, xs1).
 * Bit-identical to oracle_synth_volume in oracle/pdm_oracle.c. */
int pdm_synth_volume(int bits, int64_t nx, int64_t ny, int64_t nz, int64_t xs0, int64_t xs1,
                     const int64_t *boxes, int32_t nbox, uint64_t seed, void *out,
                     pdm_stream_t stream);

/* ---- GPU consumer of D': ray casting --------------- */

/* raycast.py:163-200 camera_rays, per-pixel part: dirs[width*height][3]
 * (device, float64, row-major pixels) from the camera frame
 * frame = {forward, right, up} (host, 9 doubles, voxel-space unit vectors),
 * tan(fov/2), aspect = width/height and spacing (host, 3 doubles). */
int pdm_camera_rays(const double *frame, double tan_half, double aspect, const double *spacing,
                    int32_t width, int32_t height, double *dirs, pdm_stream_t stream);

/* _kernels.py:206-365 march_rays (raycast.py:232-283 render): front-to-back
 * float64 compositing of n_rays rays from origin (host, 3 doubles) along
 * dirs (device) over the fixed sample grid t_entry + k*step, skipping with
 * the per-block distance field dist[ceil(n/b)^3] (device; all zeros = no
 * skipping).  vox: device [nx][ny][nz] uint8/uint16; lut: device float64
 * [lut_len][4].  Outputs (device, each optional): rgba[n][4] float64,
 * counters[n][4] int64 (total, evaluated, skip events, ert), pixels[n][4]
 * uint8 (clip, *255, round half to even), totals[4] (column sums).
 * Bit-identical to the reference marcher (no FMA contraction). */
int pdm_march_rays(const void *vox, int32_t bits, int64_t nx, int64_t ny, int64_t nz,
                   const double *lut, int64_t lut_len, const uint8_t *dist, int32_t b,
                   double step, int32_t ert_enabled, double ert_threshold, const double *origin,
                   const double *dirs, int64_t n_rays, double *rgba, int64_t *counters,
                   uint8_t *pixels, unsigned long long *totals, pdm_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* PDM_B200_H */

// capi.cu -- library plumbing plus the TF-change update: selection (K8) and
// the min-merge over the selected partition distance maps (K7).
//
// K7 over the raw planes is HBM-bound: it reads k uint8 maps and writes one,
// (k+1) * B bytes for B blocks.  Each thread owns 16-byte chunks of the map;
// it keeps 8 128-bit loads of the selected maps in flight and folds them with
// a byte-wise min (fp16-biased 16-bit lanes, HMNMX2).  Loads bypass L1 (read
// once), the store is evict-first.  The device-side default merges the
// nibble-packed copy instead (packed.cu); this one serves unpackable sets and
// host destinations of them.  TMA-bulk and cp.async ring variants were
// measured slower and removed (merge section).
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <string>

#include <cuda_fp16.h>

#include "merge_raw.cuh"
#include "pdm_common.cuh"

namespace pdm {

static thread_local char g_last_error[1024] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

int cuda_status(const char *where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", where, cudaGetErrorString(e));
        return PDM_ECUDA;
    }
    return PDM_OK;
}

int sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    static int cached[64] = {0};
    if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        n = 148;
    if (dev >= 0 && dev < 64) cached[dev] = n;
    return n;
}

// A zeroed work counter for one launch on stream s (kernels that hand out
// tiles or items with atomicAdd): a ring of 64 per device, never freed,
// zeroed in stream order, so launches in flight on different streams do not
// share one.
int work_counter(cudaStream_t s, unsigned long long **out) {
    constexpr int kSlots = 64;
    static std::mutex mu;
    static unsigned long long *ring[64] = {nullptr};
    static unsigned next_slot[64] = {0};
    int dev = 0;
    PDM_CUDA_TRY(cudaGetDevice(&dev));
    PDM_REQUIRE(dev >= 0 && dev < 64, "work_counter: device %d", dev);
    unsigned long long *p;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (ring[dev] == nullptr)
            PDM_CUDA_TRY(cudaMalloc(&ring[dev], kSlots * sizeof(unsigned long long)));
        p = ring[dev] + (next_slot[dev]++ % kSlots);
    }
    PDM_CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(unsigned long long), s));
    *out = p;
    return PDM_OK;
}

int resident_ctas(const void *kernel, int threads, size_t smem) {
    struct Slot {
        const void *k;
        int threads;
        size_t smem;
        int dev, per_sm;
    };
    static std::mutex mu;  // ctypes callers may come from several host threads
    static Slot slots[64];
    static int used = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < used; ++i)
        if (slots[i].k == kernel && slots[i].threads == threads && slots[i].smem == smem &&
            slots[i].dev == dev)
            return slots[i].per_sm;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) !=
            cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    if (used < 64) slots[used++] = Slot{kernel, threads, smem, dev, per_sm};
    return per_sm;
}

// ---------------------------------------------------------------------------
// K8: selection.  transfer.py:250-259 -- flags[p] = any(alpha[v] > 0.0) over
// partition p's contiguous intensity range [starts[p], starts[p+1]).  Every
// flag is written (0 or 1), so no clearing pass is needed.  kTPP threads per
// partition: a whole CTA (256) for wide partitions, a warp for narrow ones.
// With PDL the dependent merge launches while this runs and waits on
// griddepcontrol before it reads the flags.
// starts == nullptr: the uniform scheme (transfer.py:201-203 widths: span/n,
// the first span % n partitions one wider), bounds computed in the kernel --
// no dependent fetch of a starts table before the alpha loads (the merge
// waits on this kernel every TF change).
template <int kTPP>
__global__ void __launch_bounds__(256)
    select_kernel(const double *__restrict__ alpha, int64_t stride,
                  const int32_t *__restrict__ starts, int n, int span,
                  uint8_t *__restrict__ flags) {
    pdl_launch_dependents();
    const int group = threadIdx.x / kTPP, lane = threadIdx.x % kTPP;
    const int p = blockIdx.x * (256 / kTPP) + group;
    bool any = false;
    if (p < n) {
        int lo, hi;
        if (starts != nullptr) {
            lo = starts[p];
            hi = starts[p + 1];
        } else {
            const int q = span / n, r = span % n;
            lo = p * q + min(p, r);
            hi = lo + q + (p < r ? 1 : 0);
        }
#pragma unroll 8
        for (int v = lo + lane; v < hi; v += kTPP) any |= alpha[(int64_t)v * stride] > 0.0;
    }
    if (kTPP == 256) {
        any = __syncthreads_or(any);
    } else {
        any = __any_sync(0xFFFFFFFFu, any);  // kTPP == 32: one partition per warp
    }
    if (lane == 0 && p < n) flags[p] = any;  // NaN compares false: transparent
}

// acceleration.py:166,171 -- nz = alpha > 0 and its exclusive prefix count.
// Two launches over tiles of 1024 intensities (CTA i = tile i, coalesced):
// alpha_nz_kernel writes nz; alpha_prefix_kernel gives CTA i its carry by
// summing the 0/1 bytes of nz[0, 1024 i) (at most 64 KB, L2-resident), then
// ranks its own tile with warp ballots and a shuffle scan of the 32 warp
// counts.  No workspace, no serial walk over the span.
constexpr int kAlphaTile = 1024;

__global__ void __launch_bounds__(256)
    alpha_nz_kernel(const double *__restrict__ alpha, int64_t span, int64_t stride,
                    uint8_t *__restrict__ nz) {
    const int64_t base = (int64_t)blockIdx.x * kAlphaTile + threadIdx.x;
    bool on[kAlphaTile / 256];
#pragma unroll
    for (int j = 0; j < kAlphaTile / 256; ++j) {
        const int64_t v = base + j * 256;
        on[j] = v < span && alpha[v * stride] > 0.0;  // NaN compares false
    }
#pragma unroll
    for (int j = 0; j < kAlphaTile / 256; ++j) {
        const int64_t v = base + j * 256;
        if (v < span) nz[v] = on[j];
    }
}

__global__ void __launch_bounds__(kAlphaTile)
    alpha_prefix_kernel(const uint8_t *__restrict__ nz, int64_t span,
                        int32_t *__restrict__ prefix) {
    __shared__ int32_t s_warp[32];
    __shared__ int32_t s_carry;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t tile0 = (int64_t)blockIdx.x * kAlphaTile;
    // carry: bytes of nz before this tile (tile0 is a multiple of 16)
    int32_t cnt = 0;
    for (int64_t q = t; q < tile0 / 16; q += kAlphaTile) {
        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(nz) + q);
        cnt += (int32_t)(((w.x * 0x01010101u) >> 24) + ((w.y * 0x01010101u) >> 24) +
                         ((w.z * 0x01010101u) >> 24) + ((w.w * 0x01010101u) >> 24));
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, off);
    if (lane == 0) s_warp[warp] = cnt;
    __syncthreads();
    if (warp == 0) {
        int32_t c = s_warp[lane];
#pragma unroll
        for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, off);
        if (lane == 0) s_carry = c;
    }
    __syncthreads();  // s_warp is reused below
    const int64_t v = tile0 + t;
    const bool on = v < span && nz[v];
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, on);
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 32 warp counts
        const int32_t c = s_warp[lane];
        int32_t inc = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, off);
            if (lane >= off) inc += y;
        }
        s_warp[lane] = inc - c;
    }
    __syncthreads();
    if (v < span)
        prefix[v + 1] = s_carry + s_warp[warp] + __popc(bal & ((1u << lane) - 1u)) + on;
    if (v == 0) prefix[0] = 0;
}

// ---------------------------------------------------------------------------
// K7: merge.
constexpr int kMaxSelParam = 240;  // indices carried in kernel parameters per launch
constexpr int kMaxFlagsSmem = 4096;
constexpr int kMergeThreads = 256;


struct SelParam {
    int32_t k;
    int32_t idx[kMaxSelParam];
};

// Byte-wise min of 16-byte chunks.  sm_100a has no native 4x8-bit min
// (__vminu4 lowers to ~7 integer ops), but VIMNMX.U16x2 is one instruction:
// the accumulator keeps the even and the odd bytes of each word in separate
// 16-bit lanes (PRMT splits an input word), so folding one 16-byte chunk costs
// 8 PRMT + 8 VIMNMX instead of 28 ops.
// The 16-bit lanes hold byte v as the fp16 number 1024 + v (PRMT fills the
// high byte with 0x64): same order, and the min is HMNMX2 on the FMA pipe
// instead of VIMNMX.U16x2, which issues to the narrower XU pipe.
struct ByteMin16 {
    uint32_t lo[4], hi[4];  // lanes hold bytes {0,2} / {1,3} of each word

    __device__ __forceinline__ static uint32_t hmin2_bits(uint32_t a, uint32_t b) {
        __half2 r = __hmin2(*reinterpret_cast<const __half2 *>(&a),
                            *reinterpret_cast<const __half2 *>(&b));
        return *reinterpret_cast<uint32_t *>(&r);
    }
    __device__ __forceinline__ void init_ff() {
#pragma unroll
        for (int w = 0; w < 4; ++w) lo[w] = hi[w] = 0x64FF64FFu;
    }
    __device__ __forceinline__ void fold(uint4 v) {
        const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            lo[w] = hmin2_bits(lo[w], __byte_perm(x[w], 0x64646464u, 0x4240));
            hi[w] = hmin2_bits(hi[w], __byte_perm(x[w], 0x64646464u, 0x4341));
        }
    }
    __device__ __forceinline__ uint4 result() const {
        return make_uint4(__byte_perm(lo[0], hi[0], 0x6240), __byte_perm(lo[1], hi[1], 0x6240),
                          __byte_perm(lo[2], hi[2], 0x6240), __byte_perm(lo[3], hi[3], 0x6240));
    }
};

// Register budget: 4 CTAs x 256 threads per SM (<= 64 registers) with 8
// 128-bit loads in flight per thread = 128 KB in flight per SM.  (A deeper
// per-thread pipeline needs > 64 registers and halves the resident threads,
// which measured no faster.)  Two shapes share that budget:
//  * k <= 4: U chunks x M maps per lap (U*M = 8 loads), packed accumulators;
//  * k >  4: one chunk per lap, the selected maps in batches of 8, the
//    accumulator split into 16-bit lanes (ByteMin16) to halve ALU work.
// Chunks of a lap are one grid-width apart so each warp access is 512
// contiguous bytes of one map.
constexpr int kMergeBatch = 8;

template <bool kAccumulate>
__device__ __forceinline__ void merge_large_k(const uint8_t *__restrict__ pdms, int64_t pitch,
                                              int64_t nvec, const int32_t *idx, int k,
                                              uint8_t *__restrict__ out) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += T) {
        const int64_t off = v * 16;
        ByteMin16 acc;
        acc.init_ff();
        if (kAccumulate) acc.fold(*reinterpret_cast<const uint4 *>(out + off));
        for (int m = 0; m < k; m += kMergeBatch) {
            uint4 r[kMergeBatch];
#pragma unroll
            for (int j = 0; j < kMergeBatch; ++j)
                if (m + j < k) r[j] = ld_stream_u4(pdms + (int64_t)idx[m + j] * pitch + off);
#pragma unroll
            for (int j = 0; j < kMergeBatch; ++j)
                if (m + j < k) acc.fold(r[j]);
        }
        st_stream_u4(out + off, acc.result());
    }
}

// shape != 0 forces one loop shape (PDM_MERGE_SHAPE, measurements only):
// 1 = <1,8> packed, 2 = <2,4>, 3 = <4,2>, 4 = <8,1>, 5 = split-lane large-k.
template <bool kAccumulate>
__device__ __forceinline__ void merge_chunks(const uint8_t *__restrict__ pdms, int64_t pitch,
                                             int64_t nvec, const int32_t *idx, int k,
                                             uint8_t *__restrict__ out, int shape = 0) {
    if (shape == 1)
        merge_small_k<1, 8, kAccumulate>(pdms, pitch, nvec, idx, k, out);
    else if (shape == 2)
        merge_small_k<2, 4, kAccumulate>(pdms, pitch, nvec, idx, k, out);
    else if (shape == 3)
        merge_small_k<4, 2, kAccumulate>(pdms, pitch, nvec, idx, k, out);
    else if (shape == 4)
        merge_small_k<8, 1, kAccumulate>(pdms, pitch, nvec, idx, k, out);
    else if (shape == 5)
        merge_large_k<kAccumulate>(pdms, pitch, nvec, idx, k, out);
    else if (k <= 2)
        merge_small_k<4, 2, kAccumulate>(pdms, pitch, nvec, idx, k, out);
    else if (k <= 4)
        merge_small_k<2, 4, kAccumulate>(pdms, pitch, nvec, idx, k, out);
    else
        merge_large_k<kAccumulate>(pdms, pitch, nvec, idx, k, out);
}

__global__ void __launch_bounds__(kMergeThreads, 4)
    combine_kernel(const uint8_t *__restrict__ pdms, int64_t pitch, int64_t map_bytes,
                   const __grid_constant__ SelParam sel, uint8_t *__restrict__ out,
                   int accumulate, int shape) {
    const int64_t nvec = map_bytes / 16;
    if (accumulate)
        merge_chunks<true>(pdms, pitch, nvec, sel.idx, sel.k, out, shape);
    else
        merge_chunks<false>(pdms, pitch, nvec, sel.idx, sel.k, out, shape);
    merge_tail(pdms, pitch, nvec * 16, map_bytes, sel.idx, sel.k, accumulate != 0, out);
}

// Misaligned layouts (pitch or pointers not 16-byte aligned): byte-wise.
__global__ void combine_bytes_kernel(const uint8_t *__restrict__ pdms, int64_t pitch,
                                     int64_t map_bytes, const __grid_constant__ SelParam sel,
                                     uint8_t *__restrict__ out, int accumulate) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < map_bytes; c += stride) {
        uint32_t acc = accumulate ? out[c] : 255u;
        for (int m = 0; m < sel.k; ++m) {
            uint32_t v = pdms[(int64_t)sel.idx[m] * pitch + c];
            acc = v < acc ? v : acc;
        }
        out[c] = (uint8_t)acc;
    }
}

// Selection resident on the device: every CTA compacts the flags, then merges
// like combine_kernel.
__global__ void __launch_bounds__(kMergeThreads, 4)
    combine_flags_kernel(const uint8_t *__restrict__ pdms, int64_t pitch, int64_t map_bytes,
                         int n, const uint8_t *__restrict__ flags, uint8_t *__restrict__ out) {
    __shared__ int32_t s_idx[kMaxFlagsSmem];
    __shared__ int s_k;
    pdl_wait();  // flags come from the preceding select kernel (PDL)
    compact_flags(flags, n, s_idx, &s_k);
    __syncthreads();
    const int k = s_k;
    const int64_t nvec = map_bytes / 16;
    merge_chunks<false>(pdms, pitch, nvec, s_idx, k, out);
    merge_tail(pdms, pitch, nvec * 16, map_bytes, s_idx, k, false, out);
}

// Volume.intensity_range for device-born volumes (volume.py:86-90): out[0] =
// min, out[1] = max over all voxels.  Grid-stride, warp shuffle, one atomic
// per warp into out (pre-set to [UINT_MAX, 0] by the wrapper).
template <typename T>
__global__ void volume_range_kernel(const T *__restrict__ vox, int64_t count,
                                    uint32_t *__restrict__ out) {
    uint32_t mn = 0xFFFFFFFFu, mx = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // 16-byte loads, 4 in flight per thread (a scalar loop ran at 3.9 TB/s);
    // the vector part needs a 16-byte aligned base, the tail is scalar
    constexpr int kPer = 16 / sizeof(T);
    const int64_t nvec = ((uintptr_t)vox % 16 == 0) ? count / kPer : 0;
    const uint4 *v4 = reinterpret_cast<const uint4 *>(vox);
    // packed lane-wise accumulators (4 u8 or 2 u16 lanes per word)
    uint32_t pmn = 0xFFFFFFFFu, pmx = 0;
    auto fold = [&](uint4 q) {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            pmn = sizeof(T) == 1 ? __vminu4(pmn, w[k]) : __vminu2(pmn, w[k]);
            pmx = sizeof(T) == 1 ? __vmaxu4(pmx, w[k]) : __vmaxu2(pmx, w[k]);
        }
    };
    int64_t q = t0;
    for (; q + 3 * stride < nvec; q += 4 * stride) {
        const uint4 a = __ldcs(v4 + q), b = __ldcs(v4 + q + stride), c = __ldcs(v4 + q + 2 * stride),
                    d = __ldcs(v4 + q + 3 * stride);
        fold(a), fold(b), fold(c), fold(d);
    }
    for (; q < nvec; q += stride) fold(__ldcs(v4 + q));
    if (sizeof(T) == 1) {
        pmn = __vminu4(pmn, pmn >> 16), pmx = __vmaxu4(pmx, pmx >> 16);
        mn = min(pmn & 0xFFu, (pmn >> 8) & 0xFFu);
        mx = max(pmx & 0xFFu, (pmx >> 8) & 0xFFu);
    } else {
        mn = min(pmn & 0xFFFFu, pmn >> 16);
        mx = max(pmx & 0xFFFFu, pmx >> 16);
    }
    for (int64_t i = nvec * kPer + t0; i < count; i += stride) {
        const uint32_t v = vox[i];
        mn = v < mn ? v : mn;
        mx = v > mx ? v : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&out[0], mn);
        atomicMax(&out[1], mx);
    }
}

// DistanceMap.occupied_fraction (acceleration.py:77-79) on the device:
// count[0] += #bytes == value.  16-byte loads, __vcmpeq4 + popc, one atomic
// per warp.  count must be zeroed by the caller.
__global__ void count_value_kernel(const uint8_t *__restrict__ data, int64_t bytes,
                                   uint32_t value, unsigned long long *__restrict__ count) {
    const uint32_t rep = value * 0x01010101u;
    unsigned long long c = 0;
    const int64_t nvec = bytes / 16;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool aligned = ((uintptr_t)data & 15) == 0;
    if (aligned) {
        for (int64_t v = t0; v < nvec; v += stride) {
            const uint4 q = ld_stream_u4(data + v * 16);
            c += __popc(__vcmpeq4(q.x, rep) & 0x01010101u) + __popc(__vcmpeq4(q.y, rep) & 0x01010101u) +
                 __popc(__vcmpeq4(q.z, rep) & 0x01010101u) + __popc(__vcmpeq4(q.w, rep) & 0x01010101u);
        }
    }
    for (int64_t i = (aligned ? nvec * 16 : 0) + t0; i < bytes; i += stride) c += data[i] == value;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

__global__ void range_init_kernel(uint32_t *out) {
    out[0] = 0xFFFFFFFFu;
    out[1] = 0;
}

// One wave of resident CTAs; when the work does not fill it, just enough
// CTAs, and when it does, the per-thread iteration count is equalised so no
// CTA runs an extra lap (work_items in 16-byte chunks, U chunks per lap).
static int merge_grid(int64_t work_items, int per_sm, int U) {
    const int64_t cap = (int64_t)sm_count() * per_sm;
    const int64_t per_cta = (int64_t)kMergeThreads * U;
    const int64_t laps = ceil_div(work_items, cap * per_cta);
    int64_t grid = ceil_div(work_items, laps * per_cta);
    if (grid > cap) grid = cap;
    return grid < 1 ? 1 : (int)grid;
}

static int merge_shape() {
    static int shape = -1;
    if (shape < 0) {
        const char *e = getenv("PDM_MERGE_SHAPE");
        shape = e ? atoi(e) : 0;
    }
    return shape;
}
}  // namespace pdm

using namespace pdm;

extern "C" int pdm_version(void) { return 1; }

extern "C" const char *pdm_last_error(void) { return g_last_error; }

extern "C" int pdm_fill_u8(uint8_t *dst, int64_t bytes, int32_t value, pdm_stream_t stream) {
    PDM_REQUIRE(dst && bytes >= 0 && value >= 0 && value <= 255, "pdm_fill_u8: bad arguments");
    PDM_CUDA_TRY(cudaMemsetAsync(dst, value, (size_t)bytes, as_stream(stream)));
    return PDM_OK;
}

extern "C" int pdm_stream_synchronize(pdm_stream_t stream) {
    PDM_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
    return PDM_OK;
}

extern "C" int pdm_device_sm_count(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        set_error("cudaDeviceGetAttribute failed for device %d", device);
        return -1;
    }
    return n;
}

extern "C" int pdm_volume_range(const void *vox, int bits, int64_t count, uint32_t *out,
                                pdm_stream_t stream) {
    PDM_REQUIRE(vox && out, "pdm_volume_range: null pointer");
    PDM_REQUIRE((bits == 8 || bits == 16) && count >= 1, "pdm_volume_range: bad args");
    cudaStream_t s = as_stream(stream);
    range_init_kernel<<<1, 1, 0, s>>>(out);
    // one wave of resident CTAs, vector items (16 bytes) per thread
    int64_t grid = ceil_div(ceil_div(count * (bits / 8), 16), 256);
    const int64_t cap =
        (int64_t)sm_count() *
        resident_ctas(bits == 8 ? (const void *)volume_range_kernel<uint8_t>
                                : (const void *)volume_range_kernel<uint16_t>,
                      256, 0);
    if (grid > cap) grid = cap;
    if (bits == 8)
        volume_range_kernel<uint8_t><<<(unsigned)grid, 256, 0, s>>>((const uint8_t *)vox, count, out);
    else
        volume_range_kernel<uint16_t><<<(unsigned)grid, 256, 0, s>>>((const uint16_t *)vox, count,
                                                                       out);
    return cuda_status("volume_range_kernel");
}

extern "C" int pdm_count_value(const uint8_t *data, int64_t bytes, uint32_t value,
                               unsigned long long *count, pdm_stream_t stream) {
    PDM_REQUIRE(data && count, "pdm_count_value: null pointer");
    PDM_REQUIRE(bytes >= 1 && value <= 255, "pdm_count_value: bad args");
    cudaStream_t s = as_stream(stream);
    PDM_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(unsigned long long), s));
    int64_t grid = ceil_div(ceil_div(bytes, 16), 256);
    const int64_t cap = (int64_t)sm_count() * 8;
    if (grid > cap) grid = cap;
    count_value_kernel<<<(unsigned)(grid < 1 ? 1 : grid), 256, 0, s>>>(data, bytes, value, count);
    return cuda_status("count_value_kernel");
}

extern "C" int pdm_select(const double *alpha, int64_t span, int64_t alpha_stride,
                          const int32_t *starts, int32_t n, int32_t max_width, uint8_t *flags,
                          pdm_stream_t stream) {
    PDM_REQUIRE(alpha && flags, "pdm_select: null pointer");
    PDM_REQUIRE(span >= 1 && span <= (1 << 16) && n >= 1 && n <= span && alpha_stride >= 1,
                "pdm_select: bad sizes (span=%lld n=%d)", (long long)span, n);
    cudaStream_t s = as_stream(stream);
    if (max_width >= 512) {
        select_kernel<256><<<n, 256, 0, s>>>(alpha, alpha_stride, starts, n, (int)span, flags);
    } else {
        select_kernel<32><<<(unsigned)ceil_div(n, 8), 256, 0, s>>>(alpha, alpha_stride, starts, n,
                                                                    (int)span, flags);
    }
    return cuda_status("select_kernel");
}

// select_partitions(tf, scheme) in one call (transfer.py:250-259): gather the
// TF's alpha column from host memory into pinned staging, DMA it into HBM,
// run the f64 `> 0.0` selection on it (zero-copy, below), store the n flags
// into pinned host memory and wait -- the
// reference returns a finished host selection, and so does this.  One C call
// instead of a chain of framework calls keeps the per-TF-change host cost at
// a few microseconds.
extern "C" int pdm_select_tf(const double *lut_alpha, int64_t span, int64_t lut_stride,
                             double *stage_host, double *stage_dev, const int32_t *starts,
                             int32_t n, int32_t max_width, uint8_t *flags_dev, uint8_t *flags_host,
                             pdm_stream_t stream) {
    PDM_REQUIRE(lut_alpha && stage_host && flags_host, "pdm_select_tf: null pointer");
    cudaStream_t s = as_stream(stream);
    int st = pdm_gather_f64_host(lut_alpha, span, lut_stride, stage_host);
    if (st) return st;
    // Zero-copy (default): the select kernel reads the gathered alpha straight
    // from pinned host memory over PCIe and stores the n flags into pinned
    // host memory, so the call is one launch and one wait -- the two DMA
    // round trips (H2D alpha, D2H flags) each added a copy-engine latency.
    // PDM_SELECT_DMA=1 keeps the DMA chain (A/B).  Measured and rejected for
    // 8-bit TFs: alpha in the kernel parameters (2 KB), read from the
    // parameter bank -- 18.6 vs 16.0 us per call (the larger launch costs more
    // than the one PCIe round trip it saves).
    static const bool dma = getenv("PDM_SELECT_DMA") && getenv("PDM_SELECT_DMA")[0] == '1';
    if (dma) {
        PDM_REQUIRE(stage_dev && flags_dev, "pdm_select_tf: null device staging");
        PDM_CUDA_TRY(cudaMemcpyAsync(stage_dev, stage_host, (size_t)span * sizeof(double),
                                     cudaMemcpyHostToDevice, s));
        if ((st = pdm_select(stage_dev, span, 1, starts, n, max_width, flags_dev, stream)))
            return st;
        PDM_CUDA_TRY(
            cudaMemcpyAsync(flags_host, flags_dev, (size_t)n, cudaMemcpyDeviceToHost, s));
    } else if ((st = pdm_select(stage_host, span, 1, starts, n, max_width, flags_host, stream))) {
        return st;
    }
    PDM_CUDA_TRY(cudaStreamSynchronize(s));
    return PDM_OK;
}

extern "C" int pdm_alpha_support(const double *alpha, int64_t span, int64_t alpha_stride,
                                 uint8_t *nz, int32_t *prefix, pdm_stream_t stream) {
    PDM_REQUIRE(alpha && nz, "pdm_alpha_support: null pointer");
    PDM_REQUIRE(span >= 1 && span <= (1 << 16) && alpha_stride >= 1,
                "pdm_alpha_support: span must be in [1, 65536]");
    PDM_REQUIRE(!prefix || (uintptr_t)nz % 16 == 0,
                "pdm_alpha_support: nz must be 16-byte aligned when prefix is requested");
    cudaStream_t s = as_stream(stream);
    const int tiles = (int)ceil_div(span, kAlphaTile);
    alpha_nz_kernel<<<tiles, 256, 0, s>>>(alpha, span, alpha_stride, nz);
    int st = cuda_status("alpha_nz_kernel");
    if (st || !prefix) return st;
    alpha_prefix_kernel<<<tiles, kAlphaTile, 0, s>>>(nz, span, prefix);
    return cuda_status("alpha_prefix_kernel");
}

extern "C" int pdm_combine(const uint8_t *pdms, int64_t plane_pitch, int64_t map_bytes,
                           int32_t n, const int32_t *sel, int32_t k, uint8_t *out,
                           pdm_stream_t stream) {
    PDM_REQUIRE(out && (k == 0 || (pdms && sel)), "pdm_combine: null pointer");
    PDM_REQUIRE(map_bytes >= 1 && plane_pitch >= map_bytes && n >= 1 && k >= 0 && k <= n,
                "pdm_combine: bad sizes (map_bytes=%lld pitch=%lld n=%d k=%d)",
                (long long)map_bytes, (long long)plane_pitch, n, k);
    for (int i = 0; i < k; ++i)
        PDM_REQUIRE(sel[i] >= 0 && sel[i] < n, "pdm_combine: index %d outside [0, %d)", sel[i],
                    n);
    cudaStream_t s = as_stream(stream);
    // k == 0 (acceleration.py:261-263, the all-255 map) runs the merge kernel
    // with an empty selection: it also works when `out` is mapped host memory.
    const bool vec = (plane_pitch % 16 == 0) && ((uintptr_t)pdms % 16 == 0) &&
                     ((uintptr_t)out % 16 == 0);
    SelParam p;
    for (int base = 0; base == 0 || base < k; base += kMaxSelParam) {  // >240: passes
        p.k = k - base < kMaxSelParam ? k - base : kMaxSelParam;
        memcpy(p.idx, sel + base, sizeof(int32_t) * p.k);
        const int acc = base > 0;
        if (vec) {
            const int per_sm = resident_ctas((const void *)combine_kernel, kMergeThreads, 0);
            combine_kernel<<<merge_grid(map_bytes / 16 > 0 ? map_bytes / 16 : 1, per_sm,
                                        1),
                             kMergeThreads, 0, s>>>(pdms, plane_pitch, map_bytes, p, out, acc,
                                                    merge_shape());
        } else {
            combine_bytes_kernel<<<merge_grid(ceil_div(map_bytes, 16), 8, 1), kMergeThreads, 0,
                                   s>>>(pdms, plane_pitch, map_bytes, p, out, acc);
        }
        int st = cuda_status("combine_kernel");
        if (st) return st;
    }
    return PDM_OK;
}

extern "C" int pdm_combine_flags(const uint8_t *pdms, int64_t plane_pitch, int64_t map_bytes,
                                 int32_t n, const uint8_t *flags, uint8_t *out,
                                 pdm_stream_t stream) {
    PDM_REQUIRE(pdms && flags && out, "pdm_combine_flags: null pointer");
    PDM_REQUIRE(map_bytes >= 1 && plane_pitch >= map_bytes && n >= 1,
                "pdm_combine_flags: bad sizes");
    PDM_REQUIRE(n <= kMaxFlagsSmem, "pdm_combine_flags: n=%d above %d", n, kMaxFlagsSmem);
    PDM_REQUIRE(plane_pitch % 16 == 0 && (uintptr_t)pdms % 16 == 0 && (uintptr_t)out % 16 == 0,
                "pdm_combine_flags: needs 16-byte aligned planes");
    // Programmatic dependent launch: the merge CTAs are scheduled while the
    // preceding select kernel finishes; they wait on griddepcontrol.wait.
    const int per_sm = resident_ctas((const void *)combine_flags_kernel, kMergeThreads, 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)merge_grid(map_bytes / 16 > 0 ? map_bytes / 16 : 1, per_sm, 1));
    cfg.blockDim = dim3(kMergeThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PDM_CUDA_TRY(cudaLaunchKernelEx(&cfg, combine_flags_kernel, pdms, plane_pitch, map_bytes,
                                    (int)n, flags, out));
    return cuda_status("combine_flags_kernel");
}

// host_unpack.cpp -- host-side expansion of a compact D' that crossed PCIe
// (csrc/packed.cu writes it): plain C++ (g++), SSE2 / AVX-512 intrinsics and
// OpenMP; no device code, so it also runs (and is tested) without a GPU.
#include <immintrin.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cstdlib>

#include "../../include/pdm_b200.h"
#include "host_pool.h"

namespace pdm {
void set_error(const char *fmt, ...);  // capi.cu: pdm_last_error's buffer
}

#define REQUIRE(cond, msg)              \
    do {                                \
        if (!(cond)) {                  \
            ::pdm::set_error("%s", msg); \
            return PDM_EINVAL;          \
        }                               \
    } while (0)

// Host side: expand a packed map (pdm_combine_*_to_packed output, in host
// memory) into map_bytes plain bytes.  SSE2 per chunk (unpack low/high
// nibbles, interleave, add the base), OpenMP across chunks: 0.12 ms for a
// 16.8 MB map on 16 cores (non-temporal stores measured slower: 0.14 ms).
extern "C" int pdm_unpack_packed_host(const uint8_t *nib, const uint8_t *base, int64_t map_bytes,
                                      uint8_t *out) {
    REQUIRE(nib && base && out && map_bytes >= 1, "pdm_unpack_packed_host: bad arguments");
    const int64_t full = map_bytes / 16;
    const __m128i lo4 = _mm_set1_epi8(0x0F);
    constexpr int64_t kU = 4096;  // chunks per pool unit
    pdm::host::parallel_for((full + kU - 1) / kU, [&](int64_t u) {
        for (int64_t c = u * kU, e = std::min(full, c + kU); c < e; ++c) {
            const __m128i q = _mm_loadl_epi64(reinterpret_cast<const __m128i *>(nib + 8 * c));
            const __m128i even = _mm_and_si128(q, lo4);
            const __m128i odd = _mm_and_si128(_mm_srli_epi16(q, 4), lo4);
            __m128i v = _mm_unpacklo_epi8(even, odd);
            v = _mm_add_epi8(v, _mm_set1_epi8((char)base[c]));
            _mm_storeu_si128(reinterpret_cast<__m128i *>(out + 16 * c), v);
        }
    });
    for (int64_t i = full * 16; i < map_bytes; ++i) {
        const int64_t c = i / 16, j = i % 16;
        out[i] = (uint8_t)(base[c] + ((nib[8 * c + j / 2] >> (4 * (j & 1))) & 15));
    }
    return PDM_OK;
}

// Host side: expand the delta form (format 2) into map_bytes plain bytes.
// Block 16c takes base[c]; block 16c+i (i >= 1) adds the step coded in bits
// 2(i-1)..2i-1 of the little-endian u32 code word c (step + 1 in {0,1,2}).
// A byte prefix sum per 16-byte chunk (mod 256, exact as every value lies in
// [0, 255]) rebuilds the values.  AVX-512 VBMI when the CPU has it (4 chunks
// per 64-byte vector: VPMULTISHIFTQB pulls each block's 2-bit field), SSE2
// otherwise; OpenMP across chunks.
namespace {
static inline __m128i delta_chunk_sse(uint32_t code, uint8_t base) {
    alignas(16) uint8_t v[16];
    const uint64_t c = (uint64_t)code << 2;  // block i's field at bits 2i (block 0: none)
    for (int i = 0; i < 16; ++i) v[i] = (uint8_t)(((c >> (2 * i)) & 3u) - 1u);
    v[0] = base;
    __m128i x = _mm_load_si128(reinterpret_cast<const __m128i *>(v));
    x = _mm_add_epi8(x, _mm_slli_si128(x, 1));
    x = _mm_add_epi8(x, _mm_slli_si128(x, 2));
    x = _mm_add_epi8(x, _mm_slli_si128(x, 4));
    return _mm_add_epi8(x, _mm_slli_si128(x, 8));
}

__attribute__((target("avx2,avx512f,avx512bw,avx512vl,avx512vbmi"))) static void delta_avx512_range(
    const uint32_t *codes, const uint8_t *base, int64_t q0, int64_t q1, uint8_t *out) {
    // control: block i of a 16-byte lane reads bits 2(i mod 8).. of qword i/8
    alignas(64) uint8_t ctl[64];
    alignas(64) uint8_t bidx[64];
    for (int l = 0; l < 4; ++l)
        for (int i = 0; i < 16; ++i) {
            ctl[16 * l + i] = (uint8_t)(2 * (i & 7));  // qword 1 holds the code >> 16
            bidx[16 * l + i] = (uint8_t)l;
        }
    const __m512i vctl = _mm512_load_si512(ctl);
    const __m512i vbidx = _mm512_load_si512(bidx);
    const __m256i dup = _mm256_setr_epi32(0, 0, 1, 1, 2, 2, 3, 3);
    const __m512i three = _mm512_set1_epi8(3), one = _mm512_set1_epi8(1);
    const __mmask64 first = 0x0001000100010001ull;
    for (int64_t q = q0; q < q1; ++q) {
        const __m128i c4 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(codes + 4 * q));
        // qwords [c0, c0, c1, c1, c2, c2, c3, c3] << 2, each code zero-extended
        __m512i src = _mm512_cvtepu32_epi64(
            _mm256_permutexvar_epi32(dup, _mm256_castsi128_si256(c4)));
        src = _mm512_slli_epi64(src, 2);
        // the second qword of each lane starts at block 8: shift it by 16 bits
        src = _mm512_mask_srli_epi64(src, 0xAA, src, 16);
        __m512i x = _mm512_multishift_epi64_epi8(vctl, src);
        x = _mm512_sub_epi8(_mm512_and_si512(x, three), one);
        uint32_t b4;
        memcpy(&b4, base + 4 * q, 4);
        const __m512i bv = _mm512_permutexvar_epi8(vbidx, _mm512_set1_epi32((int)b4));
        x = _mm512_mask_blend_epi8(first, x, bv);
        x = _mm512_add_epi8(x, _mm512_bslli_epi128(x, 1));
        x = _mm512_add_epi8(x, _mm512_bslli_epi128(x, 2));
        x = _mm512_add_epi8(x, _mm512_bslli_epi128(x, 4));
        x = _mm512_add_epi8(x, _mm512_bslli_epi128(x, 8));
        _mm512_storeu_si512(reinterpret_cast<void *>(out + 64 * q), x);
    }
}

static void delta_avx512(const uint32_t *codes, const uint8_t *base, int64_t chunks4,
                         uint8_t *out) {
    constexpr int64_t kU = 1024;  // 4-chunk groups per pool unit
    pdm::host::parallel_for((chunks4 + kU - 1) / kU, [&](int64_t u) {
        delta_avx512_range(codes, base, u * kU, std::min(chunks4, u * kU + kU), out);
    });
}

static bool have_avx512vbmi() {
    static const bool ok = __builtin_cpu_supports("avx512f") &&
                           __builtin_cpu_supports("avx512bw") &&
                           __builtin_cpu_supports("avx512vl") &&
                           __builtin_cpu_supports("avx512vbmi");
    return ok;
}
}  // namespace

extern "C" int pdm_unpack_delta_host(const uint8_t *codes, const uint8_t *base, int64_t map_bytes,
                                     uint8_t *out) {
    REQUIRE(codes && base && out && map_bytes >= 1, "pdm_unpack_delta_host: bad arguments");
    const uint32_t *cw = reinterpret_cast<const uint32_t *>(codes);
    const int64_t full = map_bytes / 16;
    int64_t done = 0;
    if (have_avx512vbmi() && getenv("PDM_NO_AVX512") == nullptr) {
        const int64_t q = full / 4;
        delta_avx512(cw, base, q, out);
        done = 4 * q;
    }
    constexpr int64_t kU = 4096;
    pdm::host::parallel_for((full - done + kU - 1) / kU, [&](int64_t u) {
        for (int64_t c = done + u * kU, e = std::min(full, c + kU); c < e; ++c)
            _mm_storeu_si128(reinterpret_cast<__m128i *>(out + 16 * c),
                             delta_chunk_sse(cw[c], base[c]));
    });
    if (full * 16 < map_bytes) {
        alignas(16) uint8_t tmp[16];
        _mm_store_si128(reinterpret_cast<__m128i *>(tmp), delta_chunk_sse(cw[full], base[full]));
        for (int64_t i = full * 16; i < map_bytes; ++i) out[i] = tmp[i - full * 16];
    }
    return PDM_OK;
}


// Host side: expand the sparse delta form (format 3, packed.cu store_sparse).
// Region w (kRegion bytes) covers chunks 64w .. 64w+63.  AVX-512 VBMI2 path:
// VPEXPANDB spreads the compacted bases over the 64 chunks (0 for all-zero
// chunks), VPEXPANDD the code words (the flat code elsewhere), then the
// 4-chunks-per-vector delta expansion writes the region's 1 KB contiguously;
// no per-chunk branches.  Scalar-per-chunk SSE path otherwise.
namespace {
constexpr int64_t kRegion = 336;
constexpr uint32_t kFlatCode = 0x15555555u;

struct RegionHead {
    uint64_t nz, dd;
    const uint8_t *bases, *codes;
    explicit RegionHead(const uint8_t *r) {
        memcpy(&nz, r, 8);
        memcpy(&dd, r + 8, 8);
        bases = r + 16;
        codes = r + 16 + ((__builtin_popcountll(nz) + 3) & ~3);
    }
};

static void sparse_region_sse(const uint8_t *r, int64_t chunks, uint8_t *out, int64_t tail) {
    const RegionHead h(r);
    int bi = 0, ci = 0;
    for (int64_t c = 0; c < chunks; ++c) {
        __m128i v = _mm_setzero_si128();
        if ((h.nz >> c) & 1u) {
            const uint8_t b = h.bases[bi++];
            if ((h.dd >> c) & 1u) {
                uint32_t code;
                memcpy(&code, h.codes + 4 * ci++, 4);
                v = delta_chunk_sse(code, b);
            } else {
                v = _mm_set1_epi8((char)b);
            }
        }
        if (c + 1 < chunks || tail == 16) {
            _mm_storeu_si128(reinterpret_cast<__m128i *>(out + 16 * c), v);
        } else {
            alignas(16) uint8_t tmp[16];
            _mm_store_si128(reinterpret_cast<__m128i *>(tmp), v);
            memcpy(out + 16 * c, tmp, (size_t)tail);
        }
    }
}

// kNT: non-temporal 64-byte stores (out 64-byte aligned): no read-for-
// ownership of the 16.8 MB destination, which the plain stores pay.
template <bool kNT>
__attribute__((target("avx2,avx512f,avx512bw,avx512vl,avx512vbmi,avx512vbmi2"))) static inline void
store64(uint8_t *p, __m512i v) {
    if (kNT)
        _mm512_stream_si512(reinterpret_cast<__m512i *>(p), v);
    else
        _mm512_storeu_si512(reinterpret_cast<void *>(p), v);
}

template <bool kNT>
__attribute__((target("avx2,avx512f,avx512bw,avx512vl,avx512vbmi,avx512vbmi2"))) static void
sparse_region_vbmi2(const uint8_t *r, uint8_t *out) {
    const RegionHead h(r);
    if (h.nz == 0) {  // all-zero region (occupied space)
        const __m512i z = _mm512_setzero_si512();
        for (int i = 0; i < 16; ++i) store64<kNT>(out + 64 * i, z);
        return;
    }
    alignas(64) uint8_t ctl[64];
    for (int l = 0; l < 4; ++l)
        for (int i = 0; i < 16; ++i) ctl[16 * l + i] = (uint8_t)(2 * (i & 7));
    const __m512i vctl = _mm512_load_si512(ctl);
    const __m256i dup = _mm256_setr_epi32(0, 0, 1, 1, 2, 2, 3, 3);
    const __m512i three = _mm512_set1_epi8(3), one = _mm512_set1_epi8(1);
    const __mmask64 first = 0x0001000100010001ull;
    // byte 16j of lane j <- base of chunk 4q + j
    const __m512i bsel = _mm512_set_epi8(3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3, 3,
                                         2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2,
                                         1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1,
                                         0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0);
    const __m512i bases = _mm512_maskz_expandloadu_epi8(h.nz, h.bases);
    const uint8_t *cp = h.codes;
    for (int g = 0; g < 4; ++g) {  // 16 chunks
        const __mmask16 m = (__mmask16)(h.dd >> (16 * g));
        const __m512i codes =
            _mm512_mask_expandloadu_epi32(_mm512_set1_epi32((int)kFlatCode), m, cp);
        cp += 4 * __builtin_popcount(m);
        for (int q = 0; q < 4; ++q) {  // 4 chunks per vector
            const int c0 = 16 * g + 4 * q;  // first chunk of this vector
            const __m512i bv = _mm512_permutexvar_epi8(
                _mm512_add_epi8(bsel, _mm512_set1_epi8((char)c0)), bases);
            if (((m >> (4 * q)) & 0xFu) == 0) {  // 4 flat / zero chunks: their bases
                store64<kNT>(out + 16 * c0, bv);
                continue;
            }
            __m128i c4q;
            switch (q) {
                case 0: c4q = _mm512_extracti32x4_epi32(codes, 0); break;
                case 1: c4q = _mm512_extracti32x4_epi32(codes, 1); break;
                case 2: c4q = _mm512_extracti32x4_epi32(codes, 2); break;
                default: c4q = _mm512_extracti32x4_epi32(codes, 3); break;
            }
            __m512i src = _mm512_cvtepu32_epi64(
                _mm256_permutexvar_epi32(dup, _mm256_castsi128_si256(c4q)));
            src = _mm512_slli_epi64(src, 2);
            src = _mm512_mask_srli_epi64(src, 0xAA, src, 16);
            __m512i x = _mm512_multishift_epi64_epi8(vctl, src);
            x = _mm512_sub_epi8(_mm512_and_si512(x, three), one);
            x = _mm512_mask_blend_epi8(first, x, bv);
            x = _mm512_add_epi8(x, _mm512_bslli_epi128(x, 1));
            x = _mm512_add_epi8(x, _mm512_bslli_epi128(x, 2));
            x = _mm512_add_epi8(x, _mm512_bslli_epi128(x, 4));
            x = _mm512_add_epi8(x, _mm512_bslli_epi128(x, 8));
            store64<kNT>(out + 16 * c0, x);
        }
    }
}

static bool have_avx512vbmi2() {
    static const bool ok = have_avx512vbmi() && __builtin_cpu_supports("avx512vbmi2");
    return ok;
}
}  // namespace

namespace {
// One region of the sparse form into out + 1024 w (the last region may be
// partial: SSE path with the tail length).
struct SparseExpand {
    const uint8_t *regions;
    uint8_t *out;
    int64_t map_bytes, chunks, nreg, tail;
    bool vec, nt;
    SparseExpand(const uint8_t *r, int64_t bytes, uint8_t *o) : regions(r), out(o), map_bytes(bytes) {
        chunks = (map_bytes + 15) / 16;
        nreg = (chunks + 63) / 64;
        tail = map_bytes - 16 * (chunks - 1);  // bytes of the last chunk
        vec = have_avx512vbmi2() && getenv("PDM_NO_AVX512") == nullptr;
        static const bool nt_env = [] {
            const char *e = getenv("PDM_UNPACK_NT");
            return e == nullptr || e[0] != '0';
        }();
        nt = vec && nt_env && ((uintptr_t)out & 63) == 0;
    }
    void operator()(int64_t w) const {
        const bool full = 1024 * (w + 1) <= map_bytes;
        if (vec && full) {
            if (nt)
                sparse_region_vbmi2<true>(regions + kRegion * w, out + 1024 * w);
            else
                sparse_region_vbmi2<false>(regions + kRegion * w, out + 1024 * w);
        } else {
            sparse_region_sse(regions + kRegion * w, w + 1 < nreg ? 64 : chunks - 64 * w,
                              out + 1024 * w, w + 1 < nreg ? 16 : tail);
        }
    }
};
}  // namespace

extern "C" int pdm_unpack_sparse_host(const uint8_t *regions, int64_t map_bytes, uint8_t *out) {
    REQUIRE(regions && out && map_bytes >= 1, "pdm_unpack_sparse_host: bad arguments");
    const SparseExpand ex(regions, map_bytes, out);
    // dynamic units: coded regions cluster in space (surfaces), zero ones in bulk;
    // the pool fences each unit's streaming stores before the call returns
    constexpr int64_t kU = 16;  // regions (16 KB of output) per unit
    pdm::host::parallel_for((ex.nreg + kU - 1) / kU, [&](int64_t u) {
        for (int64_t w = u * kU, e = std::min(ex.nreg, w + kU); w < e; ++w) ex(w);
    });
    return PDM_OK;
}

// Host side: gather a strided f64 column into a contiguous (pinned) buffer --
// the alpha channel lut[:, 3] of a TransferFunction (transfer.py:44-70,
// 250-259) staged for its upload on every select_partitions call (the
// reference re-reads tf.lut each call, so no copy is cached).  A 65,536-entry
// LUT is 2 MB of strided reads: the caller starts at once and the host pool's
// helpers join as they wake (host_pool.h).
namespace {
// dst[i] = src[4 i] for i in [i0, i1) with whole 64-byte loads: 8 outputs
// from 4 loads and two 2-source permutes (the LUT rows are (r, g, b, a)).
// The last load of a group reads 3 doubles past element 4 (i + 7): the loop
// stops one group early at the end of the column (i + 9 <= n).
__attribute__((target("avx512f"))) static void gather_stride4_avx512(const double *src,
                                                                     int64_t i0, int64_t i1,
                                                                     int64_t n, double *dst) {
    const __m512i lo = _mm512_setr_epi64(0, 4, 8, 12, 0, 0, 0, 0);
    int64_t i = i0;
    for (; i + 8 <= i1 && i + 9 <= n; i += 8) {
        const double *p = src + 4 * i;
        const __m512d a = _mm512_loadu_pd(p), b = _mm512_loadu_pd(p + 8);
        const __m512d c = _mm512_loadu_pd(p + 16), d = _mm512_loadu_pd(p + 24);
        const __m512d ab = _mm512_permutex2var_pd(a, lo, b);  // a0 a4 b0 b4
        const __m512d cd = _mm512_permutex2var_pd(c, lo, d);
        _mm512_storeu_pd(dst + i, _mm512_shuffle_f64x2(ab, cd, 0x44));
    }
    for (; i < i1; ++i) dst[i] = src[4 * i];
}

static bool have_avx512f() {
    static const bool ok = __builtin_cpu_supports("avx512f") && getenv("PDM_NO_AVX512") == nullptr;
    return ok;
}
}  // namespace

extern "C" int pdm_gather_f64_host(const double *src, int64_t n, int64_t stride, double *dst) {
    REQUIRE(src && dst && n >= 0 && stride >= 1, "pdm_gather_f64_host: bad arguments");
    constexpr int64_t kU = 4096;  // entries per pool unit (128 KB of LUT rows)
    const bool vec = stride == 4 && have_avx512f();
    auto unit = [&](int64_t i0, int64_t i1) {
        if (vec)
            gather_stride4_avx512(src, i0, i1, n, dst);
        else
            for (int64_t i = i0; i < i1; ++i) dst[i] = src[i * stride];
    };
    if (n <= kU) {
        unit(0, n);
        return PDM_OK;
    }
    pdm::host::parallel_for((n + kU - 1) / kU,
                            [&](int64_t u) { unit(u * kU, std::min(n, u * kU + kU)); });
    return PDM_OK;
}

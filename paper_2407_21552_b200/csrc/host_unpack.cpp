// host_unpack.cpp -- host-side expansion of a compact D' that crossed PCIe
// (csrc/packed.cu writes it): plain C++ (g++), SSE2 / AVX-512 intrinsics and
// OpenMP; no device code, so it also runs (and is tested) without a GPU.
#include <immintrin.h>
#include <stdint.h>
#include <string.h>

#include <cstdlib>

#include "../../include/pdm_b200.h"

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
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < full; ++c) {
        const __m128i q = _mm_loadl_epi64(reinterpret_cast<const __m128i *>(nib + 8 * c));
        const __m128i even = _mm_and_si128(q, lo4);
        const __m128i odd = _mm_and_si128(_mm_srli_epi16(q, 4), lo4);
        __m128i v = _mm_unpacklo_epi8(even, odd);
        v = _mm_add_epi8(v, _mm_set1_epi8((char)base[c]));
        _mm_storeu_si128(reinterpret_cast<__m128i *>(out + 16 * c), v);
    }
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

__attribute__((target("avx2,avx512f,avx512bw,avx512vl,avx512vbmi"))) static void delta_avx512(
    const uint32_t *codes, const uint8_t *base, int64_t chunks4, uint8_t *out) {
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
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < chunks4; ++q) {
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
#pragma omp parallel for schedule(static)
    for (int64_t c = done; c < full; ++c)
        _mm_storeu_si128(reinterpret_cast<__m128i *>(out + 16 * c), delta_chunk_sse(cw[c], base[c]));
    if (full * 16 < map_bytes) {
        alignas(16) uint8_t tmp[16];
        _mm_store_si128(reinterpret_cast<__m128i *>(tmp), delta_chunk_sse(cw[full], base[full]));
        for (int64_t i = full * 16; i < map_bytes; ++i) out[i] = tmp[i - full * 16];
    }
    return PDM_OK;
}


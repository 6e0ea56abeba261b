// synth.cu -- device-born synthetic volumes for benches and tests (not a
// reference function).  Background 0 plus axis-aligned boxes filled with
// hashed intensities inside each box's band; later boxes win.  Evaluates the
// exact formula of oracle_synth_volume (oracle/pdm_oracle.c) so the CPU and
// GPU arms see identical bytes.  Thread per 16-byte chunk when aligned.
#include <cuda_runtime.h>

#include "pdm_common.cuh"

namespace pdm {

constexpr int kMaxBoxes = 64;
struct Boxes {
    int nbox;
    int64_t b[kMaxBoxes][8];  // x0 x1 y0 y1 z0 z1 band_lo band_hi
};

__device__ __forceinline__ uint64_t synth_mix(uint64_t h) {
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdULL;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ULL;
    h ^= h >> 33;
    return h;
}

__device__ __forceinline__ uint32_t synth_value(const Boxes &bx, int64_t ny, int64_t nz, int64_t x,
                                                int64_t y, int64_t z, uint64_t seed) {
    uint32_t v = 0;
    for (int q = 0; q < bx.nbox; ++q) {
        const int64_t *b = bx.b[q];
        if (x >= b[0] && x < b[1] && y >= b[2] && y < b[3] && z >= b[4] && z < b[5]) {
            const uint64_t idx = ((uint64_t)x * (uint64_t)ny + (uint64_t)y) * (uint64_t)nz + (uint64_t)z;
            const uint64_t h = synth_mix(idx ^ (seed * 0x9E3779B97F4A7C15ULL) ^ ((uint64_t)q << 56));
            const uint64_t width = (uint64_t)(b[7] - b[6] + 1);
            v = (uint32_t)(b[6] + (int64_t)(h % width));
        }
    }
    return v;
}

template <typename T>
__global__ void synth_kernel(int64_t ny, int64_t nz, int64_t xs0, int64_t xs1, uint64_t seed,
                             const __grid_constant__ Boxes boxes, T *__restrict__ out) {
    const int64_t total = (xs1 - xs0) * ny * nz;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += stride) {
        const int64_t z = o % nz, y = (o / nz) % ny, x = xs0 + o / (nz * ny);
        out[o] = (T)synth_value(boxes, ny, nz, x, y, z, seed);
    }
}

}  // namespace pdm

using namespace pdm;

extern "C" int pdm_synth_volume(int bits, int64_t nx, int64_t ny, int64_t nz, int64_t xs0,
                                int64_t xs1, const int64_t *boxes, int32_t nbox, uint64_t seed,
                                void *out, pdm_stream_t stream) {
    PDM_REQUIRE(out, "pdm_synth_volume: null output");
    PDM_REQUIRE(bits == 8 || bits == 16, "pdm_synth_volume: bits");
    PDM_REQUIRE(nx >= 1 && ny >= 1 && nz >= 1 && xs0 >= 0 && xs1 <= nx && xs0 < xs1,
                "pdm_synth_volume: bad dims/slab");
    PDM_REQUIRE(nbox >= 0 && nbox <= kMaxBoxes && (nbox == 0 || boxes),
                "pdm_synth_volume: nbox=%d (max %d)", nbox, kMaxBoxes);
    Boxes bx;
    bx.nbox = nbox;
    for (int q = 0; q < nbox; ++q)
        for (int i = 0; i < 8; ++i) bx.b[q][i] = boxes[q * 8 + i];
    const int64_t total = (xs1 - xs0) * ny * nz;
    int64_t grid = ceil_div(total, 256);
    const int64_t cap = (int64_t)sm_count() * 8;
    if (grid > cap) grid = cap;
    cudaStream_t s = as_stream(stream);
    if (bits == 8)
        synth_kernel<uint8_t><<<(unsigned)grid, 256, 0, s>>>(ny, nz, xs0, xs1, seed, bx,
                                                              (uint8_t *)out);
    else
        synth_kernel<uint16_t><<<(unsigned)grid, 256, 0, s>>>(ny, nz, xs0, xs1, seed, bx,
                                                               (uint16_t *)out);
    return cuda_status("synth_kernel");
}

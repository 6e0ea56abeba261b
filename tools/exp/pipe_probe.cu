// Throughput of the min/max instruction forms on sm_100a (which pipe each
// issues to decides the apron / DT / merge kernels' inner loops):
// VIMNMX.U32, VIMNMX.U16x2, VIMNMX3.U16x2, FMNMX, HMNMX2, ISETP+SEL, PRMT.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kAcc = 8;

#define KERNEL(NAME, OP)                                                              \
    __global__ void NAME(uint32_t *out, uint32_t seed) {                             \
        uint32_t a[kAcc];                                                             \
        for (int i = 0; i < kAcc; ++i) a[i] = seed * (threadIdx.x + 7 * i + 1);      \
        uint32_t b = seed ^ threadIdx.x, c = seed + blockIdx.x;                       \
        for (int it = 0; it < kIters; ++it) {                                         \
            _Pragma("unroll") for (int i = 0; i < kAcc; ++i) { OP; }                  \
            b += 0x10001u;                                                            \
        }                                                                             \
        uint32_t r = 0;                                                               \
        for (int i = 0; i < kAcc; ++i) r ^= a[i];                                     \
        if (r == 0x12345678u) out[threadIdx.x] = r;                                   \
    }

__device__ __forceinline__ uint32_t hmin2u(uint32_t x, uint32_t y) {
    __half2 r = __hmin2(*reinterpret_cast<__half2 *>(&x), *reinterpret_cast<__half2 *>(&y));
    return *reinterpret_cast<uint32_t *>(&r);
}
__device__ __forceinline__ uint32_t fminu(uint32_t x, uint32_t y) {
    return __float_as_uint(fminf(__uint_as_float(x), __uint_as_float(y)));
}
__device__ __forceinline__ uint32_t selmin(uint32_t x, uint32_t y) {
    uint32_t r;
    asm("{.reg .pred p; setp.lt.u32 p, %1, %2; selp.b32 %0, %1, %2, p;}" : "=r"(r) : "r"(x), "r"(y));
    return r;
}

KERNEL(k_vimnmx_u32, a[i] = min(a[i], b ^ i))
KERNEL(k_vimnmx_u16x2, a[i] = __vminu2(a[i], b ^ i))
KERNEL(k_vimnmx3_u16x2, a[i] = __vimin3_u16x2(a[i], b ^ i, c))
KERNEL(k_fmnmx, a[i] = fminu(a[i], (b ^ i) & 0x3FFFFFFFu))
KERNEL(k_hmnmx2, a[i] = hmin2u(a[i], (b ^ i) & 0x3BFF3BFFu))
KERNEL(k_setp_selp, a[i] = selmin(a[i], b ^ i))
KERNEL(k_prmt, a[i] = __byte_perm(a[i], b, 0x5140 + i))
KERNEL(k_lop3, a[i] = (a[i] & (b ^ i)) | c)
KERNEL(k_iadd, a[i] = a[i] + (b ^ i))
// forms that cannot be fused into 3-input ops: each result is xor-ed (LOP3,
// measured alone above) before the next min
KERNEL(k_vimnmx_u32_x, a[i] = min(a[i], b) ^ (i + 1))
KERNEL(k_vimnmx_u16x2_x, a[i] = __vminu2(a[i], b) ^ (i + 1))
KERNEL(k_fmnmx_x, a[i] = fminu(a[i], b & 0x3FFFFFFFu) ^ (i + 1))
KERNEL(k_hmnmx2_x, a[i] = hmin2u(a[i], b & 0x3BFF3BFFu) ^ (i + 1))
KERNEL(k_viaddmin_x, a[i] = __viaddmin_u32(a[i], b, c) ^ (i + 1))
KERNEL(k_sel_x, a[i] = selmin(a[i], b) ^ (i + 1))
KERNEL(k_lop3_x, a[i] = (a[i] & b) ^ (i + 1))

int main() {
    uint32_t *out;
    cudaMalloc(&out, 4096);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256;
    struct K { const char *name; void (*f)(uint32_t *, uint32_t); } ks[] = {
        {"VIMNMX.U32", k_vimnmx_u32}, {"VIMNMX.U16x2", k_vimnmx_u16x2},
        {"VIMNMX3.U16x2", k_vimnmx3_u16x2}, {"FMNMX", k_fmnmx}, {"HMNMX2", k_hmnmx2},
        {"ISETP+SEL", k_setp_selp}, {"PRMT", k_prmt}, {"LOP3", k_lop3}, {"IADD", k_iadd},
        {"x:VIMNMX.U32+LOP3", k_vimnmx_u32_x}, {"x:VIMNMX.U16x2+LOP3", k_vimnmx_u16x2_x},
        {"x:FMNMX+LOP3", k_fmnmx_x}, {"x:HMNMX2+LOP3", k_hmnmx2_x},
        {"x:VIADDMNMX+LOP3", k_viaddmin_x}, {"x:ISETP+SEL+LOP3", k_sel_x},
        {"x:LOP3+LOP3", k_lop3_x}};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto &k : ks) {
        k.f<<<blocks, threads>>>(out, 3);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) k.f<<<blocks, threads>>>(out, 3 + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 5.0 * blocks * threads * (double)kIters * kAcc;
        // lanes per clock per SM at the attribute's clock (kHz)
        const double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
        printf("{\"op\": \"%s\", \"ms\": %.3f, \"lane_ops_per_clk_per_sm\": %.1f}\n", k.name, ms,
               per_clk_sm);
    }
    return 0;
}

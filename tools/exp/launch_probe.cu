// Launch/completion latency floor on the box: what one eager API call can cost.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_probe launch_probe.cu
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
#include <atomic>

__global__ void empty_kernel() {}
__global__ void token_kernel(volatile unsigned *tok, unsigned v) {
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) { __threadfence_system(); *tok = v; }
}
// grid-wide: last CTA writes the token
__global__ void grid_token_kernel(unsigned *cnt, volatile unsigned *tok, unsigned v) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned prev = atomicAdd(cnt, 1u);
        if (prev == gridDim.x - 1) { *cnt = 0; __threadfence_system(); *tok = v; }
    }
}

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char **argv) {
    unsigned flags = argc > 1 ? atoi(argv[1]) : 0;
    if (flags == 1) cudaSetDeviceFlags(cudaDeviceScheduleSpin);
    if (flags == 2) cudaSetDeviceFlags(cudaDeviceScheduleYield);
    if (flags == 3) cudaSetDeviceFlags(cudaDeviceScheduleBlockingSync);
    cudaFree(0);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    unsigned *tok; cudaHostAlloc(&tok, 64, cudaHostAllocMapped); *tok = 0;
    unsigned *dtok; cudaHostGetDevicePointer(&dtok, tok, 0);
    unsigned *cnt; cudaMalloc(&cnt, 4); cudaMemset(cnt, 0, 4);
    const int N = 2000;
    for (int grid : {1, 148, 410}) {
        for (int i = 0; i < 100; ++i) { empty_kernel<<<grid, 256, 0, s>>>(); cudaStreamSynchronize(s); }
        double t0 = now_us();
        for (int i = 0; i < N; ++i) { empty_kernel<<<grid, 256, 0, s>>>(); cudaStreamSynchronize(s); }
        double t1 = now_us();
        printf("{\"flags\":%u,\"grid\":%d,\"what\":\"launch+streamsync\",\"us\":%.2f}\n", flags, grid, (t1 - t0) / N);
        t0 = now_us();
        for (int i = 0; i < N; ++i) { empty_kernel<<<grid, 256, 0, s>>>(); }
        cudaStreamSynchronize(s);
        t1 = now_us();
        printf("{\"flags\":%u,\"grid\":%d,\"what\":\"launch only (queued)\",\"us\":%.2f}\n", flags, grid, (t1 - t0) / N);
        unsigned v = 1;
        t0 = now_us();
        for (int i = 0; i < N; ++i, ++v) {
            grid_token_kernel<<<grid, 256, 0, s>>>(cnt, dtok, v);
            while (*(volatile unsigned *)tok != v) {}
        }
        t1 = now_us();
        cudaStreamSynchronize(s);
        printf("{\"flags\":%u,\"grid\":%d,\"what\":\"launch+host spin on token\",\"us\":%.2f}\n", flags, grid, (t1 - t0) / N);
        cudaEvent_t ev; cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        t0 = now_us();
        for (int i = 0; i < N; ++i) { empty_kernel<<<grid, 256, 0, s>>>(); cudaEventRecord(ev, s); while (cudaEventQuery(ev) != cudaSuccess) {} }
        t1 = now_us();
        printf("{\"flags\":%u,\"grid\":%d,\"what\":\"launch+event query spin\",\"us\":%.2f}\n", flags, grid, (t1 - t0) / N);
    }
    // two launches then one sync
    double t0 = now_us();
    for (int i = 0; i < N; ++i) { empty_kernel<<<1, 256, 0, s>>>(); empty_kernel<<<410, 256, 0, s>>>(); cudaStreamSynchronize(s); }
    double t1 = now_us();
    printf("{\"flags\":%u,\"what\":\"2 launches + 1 sync\",\"us\":%.2f}\n", flags, (t1 - t0) / N);
    return 0;
}

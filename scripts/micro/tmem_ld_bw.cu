// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM on sm_100a.
// One CTA per SM, W warps; each warp reads its TMEM lane quadrant (32 lanes x
// 32 fp32 columns = 4 KB per ld) `iters` times. Prints bytes/cycle per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2201_12854_b200/csrc/tc_common.cuh"
using namespace mca_tc;

template <int kW>
__global__ void __launch_bounds__(kW * 32, 1) tmem_bw(int iters, unsigned long long* cycles, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32) % 512;
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t v[32];
        tmem_ld32(base + ((i * 64) & 511 & ~31), v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) acc ^= v[e];
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// two loads in flight before the wait
template <int kW>
__global__ void __launch_bounds__(kW * 32, 1) tmem_bw2(int iters, unsigned long long* cycles, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t v[32], u[32];
        tmem_ld32(base + ((i * 64) & 511), v);
        tmem_ld32(base + ((i * 64 + 32) & 511), u);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) acc ^= v[e] + u[e];
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <class K>
void run(const char* name, K kern, int warps, int lds_per_iter) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, sms * 8);
    cudaMalloc(&sink, 4);
    const int iters = 4096;
    kern<<<sms, warps * 32>>>(iters, cyc, sink);
    kern<<<sms, warps * 32>>>(iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    unsigned long long* h = new unsigned long long[sms];
    cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)h[i] / sms;
    const double bytes = (double)warps * iters * lds_per_iter * 32 * 32 * 4;
    printf("%-10s warps %2d: %.1f cycles/iter, %.1f B/cycle/SM\n", name, warps, mean / iters, bytes / mean);
    cudaFree(cyc);
    cudaFree(sink);
    delete[] h;
}

int main() {
    run("ld32", tmem_bw<4>, 4, 1);
    run("ld32", tmem_bw<8>, 8, 1);
    run("ld32", tmem_bw<16>, 16, 1);
    run("ld32x2", tmem_bw2<4>, 4, 2);
    run("ld32x2", tmem_bw2<8>, 8, 2);
    run("ld32x2", tmem_bw2<16>, 16, 2);
    return 0;
}

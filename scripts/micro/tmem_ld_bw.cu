// TMEM read throughput on one B200: every SM runs warps that issue
// tcgen05.ld.sync.aligned.32x32b.x32 (4 KB per warp instruction) back to back
// and report the aggregate bytes per SM-clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2201_12854_b200/csrc tmem_ld_bw.cu -o tmem_ld_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace mca_tc;

template <int kWarps>
__global__ void __launch_bounds__(kWarps * 32, 1) tmem_read(int iters, unsigned* sink, long long* clocks) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    unsigned acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t v[32];
        tmem_ld32(base + (uint32_t)(((it + warp) & 15) * 32), v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) acc ^= v[e];
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) clocks[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int kWarps>
void run(int sms) {
    const int iters = 4096;
    unsigned* sink;
    long long* clocks;
    cudaMalloc(&sink, 4);
    cudaMalloc(&clocks, sms * sizeof(long long));
    tmem_read<kWarps><<<sms, kWarps * 32>>>(iters, sink, clocks);   // warm-up
    tmem_read<kWarps><<<sms, kWarps * 32>>>(iters, sink, clocks);
    cudaDeviceSynchronize();
    long long* h = new long long[sms];
    cudaMemcpy(h, clocks, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)h[i] / sms;
    const double bytes = (double)kWarps * iters * 4096.0;
    printf("warps/SM %2d: %.1f bytes per SM-clock (%.0f clocks for %.1f MB per SM)  err=%s\n", kWarps, bytes / mean, mean,
           bytes / 1e6, cudaGetErrorString(cudaGetLastError()));
    delete[] h;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<4>(sms);
    run<8>(sms);
    run<16>(sms);
    return 0;
}

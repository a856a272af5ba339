// tcgen05.mma issue-to-completion rate for M = 128, cta_group::1, kind::f16 (bf16),
// SS operands (128B-swizzled, K = 64 per tile): cycles per 128 x N x 64 block for
// N in {64, 128, 256}, one CTA per SM on every SM (as k12 runs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2201_12854_b200/csrc -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "mca_common.cuh"
#include "tc_common.cuh"
using namespace mca_tc;

template <int N>
__global__ void k_umma(int blocks, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < (128 + 256) * 64 * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t idesc = idesc_f16(1, 0, 128, N);
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 128 * 128);
        long long t0 = clock64();
        for (int u = 0; u < blocks; ++u) {
            const uint32_t d = tmem + (uint32_t)((u & 1) * 256);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                umma_f16(d, sw128_desc(a + kk * 32, 16, 1024), sw128_desc(b + kk * 32, 16, 1024), idesc, kk > 0);
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N>
void run(int sms, long long* d_out) {
    const int blocks = 2048;
    cudaFuncSetAttribute(k_umma<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    k_umma<N><<<sms, 128, 100 * 1024>>>(blocks, d_out);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, d_out, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    const double cyc = (double)h[0] / blocks;
    printf("N=%3d: %.1f cycles per 128x%dx64 block  (%.0f MAC/clk/SM)  %s\n", N, cyc, N, 128.0 * N * 64 / cyc,
           cudaGetErrorString(e));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d_out;
    cudaMalloc(&d_out, sizeof(long long) * 256);
    run<64>(sms, d_out);
    run<128>(sms, d_out);
    run<256>(sms, d_out);
    return 0;
}

// MUFU throughput probe: ex2.approx.ftz.f32 per SM per clock, with W warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_bw mufu_bw.cu && ./mufu_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ex2(float* out, int iters, long long* clk) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float r;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v[i]));
            v[i] = r - 1.0f;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* clk;
    cudaMalloc(&out, sizeof(float) * sms * 1024);
    cudaMalloc(&clk, sizeof(long long) * sms);
    const int iters = 4096;
    for (int threads : {128, 256, 512, 1024}) {
        k_ex2<<<sms, threads>>>(out, iters, clk);
        cudaDeviceSynchronize();
        long long c[1024];
        cudaMemcpy(c, clk, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        double ops = (double)threads * iters * 8;   // ex2 per SM
        printf("threads/SM %4d: ex2.approx.f32 %.2f per clk per SM (2 FADD per 2 ex2 interleaved)\n", threads,
               ops / (double)c[0]);
    }
    return 0;
}

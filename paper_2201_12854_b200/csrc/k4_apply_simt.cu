// k4_apply_simt.cu — K4 (CUDA-core variant): y = attn . H~ (SPEC.md:309,
// matrix.hpp:33-34) for one (b, h, 32-query tile) per CTA.
//
// The attention matrix is never materialised: scores are recomputed per key
// tile and normalised with the row log-sum-exp K1 saved,
//   P[i, j] = exp(scale * q_i.k_j - lse_i) = A[i, j],
// then accumulated against the H~ tile. fp32 arithmetic (Y tolerance contract,
// DESIGN.md §4). The tensor-core variant for bf16 is k4_apply_tc.cu.
#include "mca_common.cuh"

namespace mca_dev {

constexpr int kQT4 = 32;
constexpr int kKT4 = 32;
constexpr int kT4 = 256;

template <class T>
__global__ void __launch_bounds__(kT4) k4_apply_simt(const T* __restrict__ q, const T* __restrict__ k,
                                                     const typename HType<T>::type* __restrict__ hmat,
                                                     const float* __restrict__ lse,
                                                     int n, int heads, float scale, T* __restrict__ y) {
    __shared__ float qs[kQT4][kDh + 1];
    __shared__ float ks[kKT4][kDh + 1];
    __shared__ float hs[kKT4][kDh];
    __shared__ float ps[kQT4][kKT4 + 1];
    __shared__ float lse_s[kQT4];

    const int b = blockIdx.z, h = blockIdx.y, i0 = blockIdx.x * kQT4;
    const int tid = threadIdx.x;
    const int r = tid >> 3, cg = tid & 7;
    const size_t HD = (size_t)heads * kDh;
    const T* qb = q + (size_t)b * n * HD + (size_t)h * kDh;
    const T* kb = k + (size_t)b * n * HD + (size_t)h * kDh;
    const typename HType<T>::type* hb = hmat + (size_t)b * n * HD + (size_t)h * kDh;

    for (int e = tid; e < kQT4 * kDh; e += kT4) {
        const int rr = e / kDh, c = e % kDh;
        qs[rr][c] = (i0 + rr < n) ? to_f32(qb[(size_t)(i0 + rr) * HD + c]) : 0.0f;
    }
    if (tid < kQT4) lse_s[tid] = (i0 + tid < n) ? lse[((size_t)b * heads + h) * n + i0 + tid] : 0.0f;

    float o[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) o[u] = 0.0f;

    for (int j0 = 0; j0 < n; j0 += kKT4) {
        __syncthreads();
        for (int e = tid; e < kKT4 * kDh; e += kT4) {
            const int rr = e / kDh, c = e % kDh;
            const bool ok = j0 + rr < n;
            ks[rr][c] = ok ? to_f32(kb[(size_t)(j0 + rr) * HD + c]) : 0.0f;
            hs[rr][c] = ok ? to_f32(hb[(size_t)(j0 + rr) * HD + c]) : 0.0f;
        }
        __syncthreads();
        const float lr = lse_s[r];
#pragma unroll 2
        for (int u = 0; u < kKT4 / 8; ++u) {
            const int jj = cg + 8 * u;
            float s = 0.0f;
#pragma unroll 16
            for (int d = 0; d < kDh; ++d) s += qs[r][d] * ks[jj][d];
            ps[r][jj] = (j0 + jj < n) ? expf(s * scale - lr) : 0.0f;
        }
        __syncthreads();
#pragma unroll 4
        for (int jj = 0; jj < kKT4; ++jj) {
            const float p = ps[r][jj];
#pragma unroll
            for (int u = 0; u < 8; ++u) o[u] += p * hs[jj][cg * 8 + u];
        }
    }
    if (i0 + r < n) store8(y + ((size_t)b * n + i0 + r) * HD + (size_t)h * kDh + cg * 8, o);
}

template __global__ void k4_apply_simt<float>(const float*, const float*, const float*, const float*, int, int, float,
                                              float*);
template __global__ void k4_apply_simt<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, const __half*,
                                                      const float*, int, int, float, __nv_bfloat16*);

}  // namespace mca_dev

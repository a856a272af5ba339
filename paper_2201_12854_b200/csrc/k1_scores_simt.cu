// k1_scores_simt.cu — K1 (CUDA-core variant): score pass of attention_matrix
// + col_max (matrix.hpp:46-53) for one (b, h, 32-query
// tile) per CTA.
//
// Per row i (sweep 1, online): m_i = max_j t_ij, l_i = sum_j exp(t_ij - m_i),
// t = scale * q_i . k_j. Written as fp64 row statistics plus lse_i (fp32, for K4).
//
// Per column j (sweep 2), two column-key formats:
//   kValue  (fp32 inputs, fp64 arithmetic — the parity-precision path):
//           A_ij = exp(t_ij - m_i) / l_i, exactly the oracle's softmax_rows
//           formula (matrix.hpp:46-50); key = order-preserving u64 of A_ij;
//           atomicMax over query tiles gives max_i A_ij directly.
//   kArgmax (bf16 inputs, fp32 arithmetic): v_ij = t_ij - m_i - log l_i; key =
//           (ordered32(v) << 32) | ~i, so atomicMax keeps the row index of the
//           column maximum (smallest i on ties: order-independent). K2 then
//           re-evaluates that single winning entry in fp64 with the oracle's
//           formula, so special cases (uniform attention: cmax = 1/n exactly,
//           SPEC.md:302) come out exact and the score pass never exponentiates
//           twice per element.
#include "mca_common.cuh"

namespace mca_dev {

__device__ __forceinline__ unsigned long long double_to_ordered(double d) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(d);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ unsigned long long argmax_key(float v, int i) {
    return ((unsigned long long)float_to_ordered(v) << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)i);
}

__device__ __forceinline__ double ex(double v) { return ::exp(v); }
__device__ __forceinline__ float ex(float v) { return ::expf(v); }
__device__ __forceinline__ double lg(double v) { return ::log(v); }
__device__ __forceinline__ float lg(float v) { return ::logf(v); }

constexpr int kQT = 32;   // query rows per CTA
template <class Acc>
constexpr int kKTof = 256 / sizeof(Acc);  // keys per tile: 64 (float) / 32 (double), keeps smem < 48 KB
constexpr int kThreads = 256;

template <class T, class Acc>
__global__ void __launch_bounds__(kThreads) k1_scores_simt(const T* __restrict__ q, const T* __restrict__ k, int n,
                                                           int heads, double scale, double* __restrict__ row_m,
                                                           double* __restrict__ row_l, float* __restrict__ lse_out,
                                                           unsigned long long* __restrict__ colkey) {
    constexpr int kKT = kKTof<Acc>;
    constexpr bool kValue = sizeof(Acc) == 8;
    __shared__ Acc qs[kQT][kDh + 1];
    __shared__ Acc ks[kKT][kDh + 1];
    __shared__ unsigned long long red[kThreads / 32][kKT];
    __shared__ Acc m_s[kQT], l_s[kQT];

    const int b = blockIdx.z, h = blockIdx.y, i0 = blockIdx.x * kQT;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r = tid >> 3;        // query row within the tile (0..31)
    const int cg = tid & 7;        // column group: keys cg, cg+8, ...
    const size_t HD = (size_t)heads * kDh;
    const T* qb = q + (size_t)b * n * HD + (size_t)h * kDh;
    const T* kb = k + (size_t)b * n * HD + (size_t)h * kDh;

    for (int e = tid; e < kQT * kDh; e += kThreads) {
        const int rr = e / kDh, c = e % kDh;
        qs[rr][c] = (i0 + rr < n) ? (Acc)to_f32(qb[(size_t)(i0 + rr) * HD + c]) : (Acc)0;
    }
    const Acc sc = (Acc)scale;
    const bool row_ok = (i0 + r) < n;

    // ---- sweep 1: online row max / sum
    Acc m = -INFINITY, l = 0;
    for (int j0 = 0; j0 < n; j0 += kKT) {
        __syncthreads();
        for (int e = tid; e < kKT * kDh; e += kThreads) {
            const int rr = e / kDh, c = e % kDh;
            ks[rr][c] = (j0 + rr < n) ? (Acc)to_f32(kb[(size_t)(j0 + rr) * HD + c]) : (Acc)0;
        }
        __syncthreads();
#pragma unroll 2
        for (int u = 0; u < kKT / 8; ++u) {
            const int jj = cg + 8 * u;
            if (j0 + jj >= n) continue;
            Acc s = 0;
#pragma unroll 16
            for (int d = 0; d < kDh; ++d) s += qs[r][d] * ks[jj][d];
            const Acc t = s * sc;
            if (t > m) {
                l = l * ex(m - t) + (Acc)1;
                m = t;
            } else {
                l += ex(t - m);
            }
        }
    }
    // combine the 8 column groups of each row (lanes differ in bits 0..2)
#pragma unroll
    for (int off = 1; off < 8; off <<= 1) {
        const Acc m2 = __shfl_xor_sync(0xffffffffu, m, off);
        const Acc l2 = __shfl_xor_sync(0xffffffffu, l, off);
        const Acc mn = m > m2 ? m : m2;
        l = (m == -INFINITY ? (Acc)0 : l * ex(m - mn)) + (m2 == -INFINITY ? (Acc)0 : l2 * ex(m2 - mn));
        m = mn;
    }
    if (cg == 0) {
        m_s[r] = m;
        l_s[r] = l;
        if (row_ok) {
            const size_t t = ((size_t)b * heads + h) * n + i0 + r;
            row_m[t] = (double)m;
            row_l[t] = (double)l;
            lse_out[t] = (float)(m + lg(l));
        }
    }

    // ---- sweep 2: column maxima
    for (int j0 = 0; j0 < n; j0 += kKT) {
        __syncthreads();
        for (int e = tid; e < kKT * kDh; e += kThreads) {
            const int rr = e / kDh, c = e % kDh;
            ks[rr][c] = (j0 + rr < n) ? (Acc)to_f32(kb[(size_t)(j0 + rr) * HD + c]) : (Acc)0;
        }
        __syncthreads();
        const Acc mr = m_s[r], lr = l_s[r];
        const Acc log_l = lg(lr);
#pragma unroll 2
        for (int u = 0; u < kKT / 8; ++u) {
            const int jj = cg + 8 * u;
            Acc s = 0;
#pragma unroll 16
            for (int d = 0; d < kDh; ++d) s += qs[r][d] * ks[jj][d];
            unsigned long long key = 0;  // below every real key
            if (row_ok) {
                if constexpr (kValue) key = double_to_ordered((double)(ex(s * sc - mr) / lr));
                else key = argmax_key((float)(s * sc - mr - log_l), i0 + r);
            }
            // reduce over the 4 rows of this warp (lanes differ in bits 3, 4)
            unsigned long long o = __shfl_xor_sync(0xffffffffu, key, 8);
            key = o > key ? o : key;
            o = __shfl_xor_sync(0xffffffffu, key, 16);
            key = o > key ? o : key;
            if (lane < 8) red[warp][jj] = key;
        }
        __syncthreads();
        if (tid < kKT && j0 + tid < n) {
            unsigned long long v = red[0][tid];
#pragma unroll
            for (int w = 1; w < kThreads / 32; ++w) v = red[w][tid] > v ? red[w][tid] : v;
            atomicMax(colkey + ((size_t)b * heads + h) * n + j0 + tid, v);
        }
    }
}

template __global__ void k1_scores_simt<float, double>(const float*, const float*, int, int, double, double*, double*,
                                                       float*, unsigned long long*);
template __global__ void k1_scores_simt<__nv_bfloat16, float>(const __nv_bfloat16*, const __nv_bfloat16*, int, int,
                                                              double, double*, double*, float*,
                                                              unsigned long long*);

}  // namespace mca_dev

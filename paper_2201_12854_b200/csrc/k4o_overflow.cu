// k4o_overflow.cu — K4o: the fp16 range guard's fix-up after the aggregation.
//
// On the bf16 path H~ is stored in fp16 (K4's P.H~ operand). The encoders
// (K3, K3b) queue every token-head j whose fp32 encoding leaves fp16's range
// (mca_common.cuh OvfSink) and store zeros for it, so K4 computes
// y_i = sum_{j not queued} P_ij H~_j. This kernel adds the missing terms,
//   y[b, i, h] += P_ij H~_j   for every query i of the sequence,
// with P_ij = exp(a q_i.k_j - lse_i) recomputed from the score pass's row
// statistics (the forward), or the given attention entry (mca_forward_attn).
// The queue is empty unless the weights or inputs are extreme (a row of W_V
// with a tiny p(s) drawn for an outlier x). On the
// forward the fix-up runs at the end of K4 itself, in the last CTA to finish
// (k4_apply_tc: no extra launch); the given-attention path launches
// k4o_overflow after ka_aggregate.
#pragma once

#include "mca_common.cuh"

namespace mca_dev {

struct K4oArgs {
    OvfSink ovf;
    const void* q;                   // [B, n, H*64] bf16 (forward)
    const void* k;
    const float* lse;                // [B, H, n]
    const double* attn;              // [B, H, n, n] (given attention)
    double scale;
    int n, heads;
    __nv_bfloat16* y;                // [B, n, H*64]
};

// The fix-up for queue entries e0, e0 + step, ... by the calling CTA (every
// thread of it; s_h, s_k: 64 floats each of shared memory).
template <bool kGiven>
__device__ __forceinline__ void ovf_fixup(const K4oArgs& a, unsigned long long cnt, unsigned long long e0,
                                          unsigned long long step, float* s_h, float* s_k) {
    const int tid = threadIdx.x;
    const size_t HD = (size_t)a.heads * kDh;
    for (unsigned long long e = e0; e < cnt; e += step) {
        const long long t = a.ovf.list[e] >> 3;
        const int chunk = (int)(a.ovf.list[e] & 7);   // columns [8 chunk, 8 chunk + 8)
        const long bh = (long)(t / a.n);
        const int j = (int)(t - (long long)bh * a.n);
        const int b = (int)(bh / a.heads), h = (int)(bh - (long)b * a.heads);
        __syncthreads();
        if (tid < kDh) {
            s_h[tid] = (tid >> 3) == chunk ? a.ovf.rows[e * 8 + (tid & 7)] : 0.f;
            if (!kGiven)
                s_k[tid] = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.k)[((size_t)b * a.n + j) * HD +
                                                                                     (size_t)h * kDh + tid]);
        }
        __syncthreads();
        for (int i = tid; i < a.n; i += blockDim.x) {
            float p;
            if constexpr (kGiven) {
                p = (float)a.attn[((size_t)bh * a.n + i) * a.n + j];
            } else {
                float qv[kDh];
                const __nv_bfloat16* qi = reinterpret_cast<const __nv_bfloat16*>(a.q) + ((size_t)b * a.n + i) * HD +
                                          (size_t)h * kDh;
#pragma unroll
                for (int c = 0; c < kDh; c += 8) load8(qi + c, qv + c);
                float d0 = 0.f, d1 = 0.f;
#pragma unroll
                for (int c = 0; c < kDh; c += 2) {
                    d0 = fmaf(qv[c], s_k[c], d0);
                    d1 = fmaf(qv[c + 1], s_k[c + 1], d1);
                }
                p = expf((float)a.scale * (d0 + d1) - a.lse[(size_t)bh * a.n + i]);
            }
            __nv_bfloat162* yr = reinterpret_cast<__nv_bfloat162*>(a.y + ((size_t)b * a.n + i) * HD + (size_t)h * kDh +
                                                                  8 * chunk);
#pragma unroll
            for (int c = 0; c < 8; c += 2)
                atomicAdd(yr + c / 2, __floats2bfloat162_rn(p * s_h[8 * chunk + c], p * s_h[8 * chunk + c + 1]));
        }
    }
}

// Standalone launch (the given-attention path): one CTA per queue entry stride.
template <bool kGiven>
__global__ void __launch_bounds__(256) k4o_overflow(K4oArgs a) {
    __shared__ float s_h[kDh], s_k[kDh];
    griddep_trigger();
    griddep_wait();                  // the aggregation's y and the encoders' queue
    const unsigned long long cnt = *(volatile const unsigned long long*)a.ovf.count;
    if (cnt == 0) return;
    if (cnt > (unsigned long long)a.ovf.cap) __trap();   // more out-of-range encodings than the queue holds
    ovf_fixup<kGiven>(a, cnt, blockIdx.x, gridDim.x, s_h, s_k);
}

}  // namespace mca_dev

// k0_weights.cu — K0: one-time per-head sampling tables (device, fp64).
//
// Implements weight_probs + make_distribution
// for every head slice W_h = W_V[:, h*64:(h+1)*64], with the
// accumulation order the oracle fixes (oracle/sampling.cpp, oracle/amm.cpp):
//   sq[i]  = sum_c w[i,c]^2 left to right          (one thread per row)
//   total  = sum_i sq[i] top to bottom              (one thread)
//   p[i]   = sq[i] / total, < 1e-15 -> 0, renormalised only if something clamped
//   cdf[i] = min(prefix sum, 1), = 1 from the last positive entry on
// Every op is an explicit correctly rounded binary64 op (__dadd_rn etc.), so
// p and cdf are bitwise equal to the oracle's. Then, for the sampler:
//   thr[i]   = ceil(cdf[i] * 2^53)   (u64; exact: power-of-two scaling)
//   invp[i]  = (float)(1 / p[i])     (0 where p = 0; never drawn)
//   guide[g] = first i with thr[i] > g * 2^39, | 0x8000 when thr[i] >= (g + 1) * 2^39
//   (one row covers the bucket), else | 0x4000 when thr[i + 1] >= (g + 1) * 2^39 (one boundary)
//              (the whole bucket draws row i: no compare needed)
// One-time cost; it runs once per weight matrix ("embedded in the model or
// cached").
#include "mca_common.cuh"

#ifndef MCA_GUIDE_ONE
#define MCA_GUIDE_ONE 1
#endif

namespace mca_dev {

template <class T>
__global__ void k0_row_sq(const T* __restrict__ w, int d_in, int heads, double* __restrict__ sq) {
    const int h = blockIdx.y;
    const int HD = heads * kDh;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d_in; i += gridDim.x * blockDim.x) {
        const T* row = w + (size_t)i * HD + (size_t)h * kDh;
        double s = 0.0;
        for (int c = 0; c < kDh; ++c) {
            const double v = (double)to_f32(row[c]);
            s = __dadd_rn(s, __dmul_rn(v, v));
        }
        sq[(size_t)h * d_in + i] = s;
    }
}

// One block per head; thread 0 runs the sequential parts.
__global__ void k0_dist(const double* __restrict__ sq, int d_in, double* __restrict__ probs, double* __restrict__ cdf,
                        uint64_t* __restrict__ thr, float* __restrict__ invp, uint16_t* __restrict__ guide,
                        int* __restrict__ status) {
    const int h = blockIdx.x;
    const double* s = sq + (size_t)h * d_in;
    double* p = probs + (size_t)h * d_in;
    double* c = cdf + (size_t)h * d_in;
    uint64_t* t = thr + (size_t)h * d_in;
    if (threadIdx.x == 0) {
        double total = 0.0;
        for (int i = 0; i < d_in; ++i) total = __dadd_rn(total, s[i]);
        if (!(total > 0.0) || !isfinite(total)) {
            status[h] = 1;  // degenerate head (zero or non-finite W_h)
            for (int i = 0; i < d_in; ++i) { p[i] = 0.0; c[i] = 1.0; }
        } else {
            status[h] = 0;
            bool clamped = false;
            for (int i = 0; i < d_in; ++i) {
                double v = __ddiv_rn(s[i], total);
                if (v < 1e-15) {
                    if (v != 0.0) clamped = true;
                    v = 0.0;
                }
                p[i] = v;
            }
            if (clamped) {
                double z = 0.0;
                for (int i = 0; i < d_in; ++i) z = __dadd_rn(z, p[i]);
                for (int i = 0; i < d_in; ++i) p[i] = __ddiv_rn(p[i], z);
            }
            double acc = 0.0;
            int last = 0;
            for (int i = 0; i < d_in; ++i) {
                acc = __dadd_rn(acc, p[i]);
                c[i] = acc < 1.0 ? acc : 1.0;
                if (p[i] > 0.0) last = i;
            }
            for (int i = last; i < d_in; ++i) c[i] = 1.0;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < d_in; i += blockDim.x) {
        t[i] = (uint64_t)ceil(c[i] * 9007199254740992.0);  // 2^53, exact scaling
        invp[(size_t)h * d_in + i] = p[i] > 0.0 ? (float)__drcp_rn(p[i]) : 0.0f;
    }
    __syncthreads();
    for (int g = threadIdx.x; g < kGuide; g += blockDim.x) {
        const uint64_t key = (uint64_t)g << (53 - kGuideBits);
        int lo = 0, hi = d_in - 1;  // thr[d_in-1] = 2^53 > key always
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (t[mid] > key) hi = mid; else lo = mid + 1;
        }
        const uint64_t upper = (uint64_t)(g + 1) << (53 - kGuideBits);   // bucket = [key, upper)
        const uint16_t flag = t[lo] >= upper ? kGuideClean : (MCA_GUIDE_ONE && t[lo + 1] >= upper ? kGuideOne : 0u);
        guide[(size_t)h * kGuide + g] = (uint16_t)(lo | flag);
    }
}

template __global__ void k0_row_sq<float>(const float*, int, int, double*);
template __global__ void k0_row_sq<__nv_bfloat16>(const __nv_bfloat16*, int, int, double*);

}  // namespace mca_dev

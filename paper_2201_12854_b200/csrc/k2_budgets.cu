// k2_budgets.cu — K2: column maxima -> Eq. 9 sample budgets + FLOP accounting.
//
// sample_budgets:
//   t = (n * cmax) / alpha;  raw = t * t;  c = ceil(raw)
//   exact = c >= d;  r = clamp(c, min_samples, d)
// evaluated with explicitly rounded binary64 ops (__dmul_rn/__ddiv_rn: no FMA
// contraction), so a given cmax yields bitwise the oracle's budget
// (oracle/attention.cpp budget_for).
//
// cmax comes from K1's column key (k1_scores_*.cu):
//   kKeyValue:  the key is the fp64 column maximum itself.
//   kKeyArgmax: the key holds the winning row i*; the score t = scale q_i*.k_j is
//               recomputed here in fp64 from the (bf16) inputs — products of
//               bf16 values are exact in fp64 — and cmax = exp(t - m_i*) / l_i*,
//               the oracle's softmax formula, with K1's row statistics.
// The kernel also reduces flops_for_plan: approx cost, the
// number of sampled draws and exact token-heads.
#include "mca_common.cuh"

namespace mca_dev {

enum K2Source { kKeyValue = 0, kKeyArgmax = 1, kGivenCmax = 2 };

__device__ __forceinline__ double ordered_to_double(unsigned long long u) {
    const unsigned long long b = (u & 0x8000000000000000ull) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
    return __longlong_as_double((long long)b);
}

__device__ __forceinline__ void budget_for(double cmax, int n, double alpha, int min_samples, int d, int* r,
                                           bool* exact) {
    const double t = __ddiv_rn(__dmul_rn((double)n, cmax), alpha);
    const double raw = __dmul_rn(t, t);
    const double c = ceil(raw);
    const bool ex = c >= (double)d;
    int rr = ex ? d : (int)c;
    if (rr < min_samples) rr = min_samples;
    if (rr > d) rr = d;
    *r = rr;
    *exact = ex;
}

struct K2Args {
    const unsigned long long* colkey;  // [B, H, n]
    const double* cmax_in;             // kGivenCmax
    const double* row_m;               // [B, H, n] (kKeyArgmax)
    const double* row_l;
    const void* q;                     // [B, n, H*64] (kKeyArgmax)
    const void* k;
    double scale;
    long count;                        // B*H*n
    int n, heads, d, dh, min_samples;
    double alpha;
    bool force_exact;
    const int32_t* budgets_override;
    const uint8_t* exact_override;
    int32_t* budgets;
    uint8_t* exact;
    double* cmax_out;
    unsigned long long* counters;      // [0] approx cost, [1] sampled draws, [2] exact token-heads
};

template <int kSrc, class T>
__global__ void k2_budgets(K2Args a) {
    unsigned long long cost = 0, samples = 0, nexact = 0;
    const unsigned long long exact_cost = 2ull * (unsigned long long)a.d * (unsigned long long)a.dh;
    for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < a.count; t += (long)gridDim.x * blockDim.x) {
        int r;
        bool ex;
        if (a.force_exact) {
            r = a.d;
            ex = true;
        } else if (a.budgets_override) {
            r = a.budgets_override[t];
            ex = a.exact_override[t] != 0;
        } else {
            double cm;
            if constexpr (kSrc == kGivenCmax) {
                cm = a.cmax_in[t];
            } else if constexpr (kSrc == kKeyValue) {
                cm = ordered_to_double(a.colkey[t]);
            } else {
                const unsigned long long key = a.colkey[t];
                const int i = (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull));
                const long bh = t / a.n;                 // b * H + h
                const int j = (int)(t - bh * a.n);
                const int b = (int)(bh / a.heads), h = (int)(bh - (long)b * a.heads);
                const size_t HD = (size_t)a.heads * kDh;
                const T* qi = reinterpret_cast<const T*>(a.q) + ((size_t)b * a.n + i) * HD + (size_t)h * kDh;
                const T* kj = reinterpret_cast<const T*>(a.k) + ((size_t)b * a.n + j) * HD + (size_t)h * kDh;
                double s = 0.0;
                for (int c = 0; c < kDh; ++c) s = __dadd_rn(s, __dmul_rn((double)to_f32(qi[c]), (double)to_f32(kj[c])));
                const size_t ri = (size_t)bh * a.n + i;
                cm = __ddiv_rn(exp(__dsub_rn(__dmul_rn(a.scale, s), a.row_m[ri])), a.row_l[ri]);
            }
            if (a.cmax_out) a.cmax_out[t] = cm;
            budget_for(cm, a.n, a.alpha, a.min_samples, a.d, &r, &ex);
        }
        a.budgets[t] = r;
        a.exact[t] = ex ? 1 : 0;
        if (ex) {
            cost += exact_cost;
            nexact += 1;
        } else {
            cost += (unsigned long long)r * (2ull * a.dh + 3ull);
            samples += (unsigned long long)r;
        }
    }
    if (!a.counters) return;
    for (int off = 16; off; off >>= 1) {  // warp reduce, one atomic per warp
        cost += __shfl_xor_sync(0xffffffffu, cost, off);
        samples += __shfl_xor_sync(0xffffffffu, samples, off);
        nexact += __shfl_xor_sync(0xffffffffu, nexact, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (cost) atomicAdd(a.counters + 0, cost);
        if (samples) atomicAdd(a.counters + 1, samples);
        if (nexact) atomicAdd(a.counters + 2, nexact);
    }
}

template __global__ void k2_budgets<kKeyValue, float>(K2Args);
template __global__ void k2_budgets<kKeyArgmax, __nv_bfloat16>(K2Args);
template __global__ void k2_budgets<kKeyArgmax, float>(K2Args);
template __global__ void k2_budgets<kGivenCmax, float>(K2Args);

}  // namespace mca_dev

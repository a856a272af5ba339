// k2c_certify.cu — K2c: certified Eq. 9 budgets at integer boundaries.
//
// The bf16 score passes (K12, K1a/K1b + K2) form a column maximum
//   cmax_j = max_i A_ij,   A_ij = exp(t_ij - m_i) / l_i,   t_ij = a q_i.k_j
// (softmax_rows + col_max, matrix.hpp:46-53) from tensor-core scores with fp32
// accumulation and ex2.approx row sums: within ~2e-6 relative of the fp64
// value (measured <= 1.9e-6 over C1-C4, tests/test_gpu_configs.py). Eq. 9
// (sample_budgets) is discontinuous: ceil((n cmax / alpha)^2)
// jumps at every integer, so a token-head whose raw value lies within that
// error of an integer could get a budget one off the fp64 reference's.
//
// The budget pass therefore flags every token-head whose raw value is within
// kCertTau (relative) of an integer boundary that changes (r, exact) and
// defers it here (eq9_ambiguous / cert_push). For each flagged key j this
// kernel re-derives cmax_j in binary64 the way the oracle does
// (oracle/tensor.cpp softmax_rows, col_max):
//   1. every query's t_ij in fp64 (bf16 products and their sums are exact in
//      binary64, so t_ij is the oracle's t_ij bit for bit), and
//      v_i = t_ij - lse_i with the score pass's fp32 lse;
//   2. the candidate rows: v_i within the lse error of max_i v_i;
//   3. each candidate's exact row statistics m_i = max_j' t_ij',
//      l_i = sum_j' exp(t_ij' - m_i) (cached per row for the forward: the
//      budget pass clears row_done[], the first warp to need a row fills it);
//   4. cmax_j = max over the candidates of exp(t_ij - m_i) / l_i, then Eq. 9,
//      the FLOP counters and the budget histogram the work lists are built from.
// What remains between device and oracle is the order of the l_i summation
// and exp's last ulp: ~1e-15 relative, so budgets equal the fp64 oracle's
// end to end (tests/test_gpu_configs.py, tests/test_gpu_parity.py).
//
// One warp per flagged key; the grid is persistent and reads the flag count
// after griddep_wait (the count is only known on the device).
#pragma once

#include "mca_common.cuh"

namespace mca_dev {

constexpr double kCertTau = 1e-5;   // relative distance of raw to an integer that is re-derived in fp64

// Flag sink of the budget passes (K12 group B, k2_budgets): null list = off.
struct CertSink {
    long long* list;                 // [B*H*n] flagged token-head indices t = (b*H + h)*n + j
    unsigned long long* count;       // number of flagged entries (zeroed per forward)
    uint8_t* row_done;               // [B*H*n] exact row statistics cached (cleared by the budget pass)
};

// (r, exact) of Eq. 9 could change under a relative perturbation of cmax of
// up to ~kCertTau / 2: raw lies within kCertTau of an integer m whose two sides
// give different outcomes (m >= min_samples: below it both clamp to
// min_samples; m <= d - 1: at or above d both are exact).
__device__ __forceinline__ bool eq9_ambiguous(double cm, int n, double alpha, int min_samples, int d) {
    const double t = __ddiv_rn(__dmul_rn((double)n, cm), alpha);
    const double raw = __dmul_rn(t, t);
    const double m = rint(raw);
    return m >= (double)min_samples && m <= (double)(d - 1) && fabs(raw - m) <= kCertTau * fmax(raw, 1.0);
}

__device__ __forceinline__ void cert_push(const CertSink& c, long long t) {
    const unsigned long long pos = atomicAdd(c.count, 1ull);
    c.list[pos] = t;
}

struct K2cArgs {
    const void* q;                   // [B, n, H*64]
    const void* k;
    const float* lse;                // [B, H, n] natural-log lse of the scaled score rows (score pass)
    double scale;
    int n, heads, d, dh, min_samples;
    double alpha;
    CertSink cert;
    double* row_m;                   // [B, H, n] exact row max (filled on demand)
    double* row_l;                   // [B, H, n] exact row sum
    int32_t* budgets;
    uint8_t* exact;
    double* cmax_out;                // nullable
    unsigned long long* counters;    // [0] approx cost, [1] sampled draws, [2] exact token-heads
    unsigned int* hist;              // [H, d + 1] (nullable)
};

// 64-term dot in binary64 against a warp-private fp64 copy of the other row.
template <class T>
__device__ __forceinline__ double dot64_sm(const T* __restrict__ a, const double* __restrict__ b) {
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
    for (int c = 0; c < kDh; c += 8) {
        float va[8];
        load8(a + c, va);
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
            acc0 = fma((double)va[e], b[c + e], acc0);
            acc1 = fma((double)va[e + 1], b[c + e + 1], acc1);
        }
    }
    return acc0 + acc1;
}

__device__ __forceinline__ double warp_max_d(double v) {
    for (int off = 16; off; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

constexpr int kCertWarps = 8;

template <class T>
__global__ void __launch_bounds__(kCertWarps * 32) k2c_certify(K2cArgs a) {
    __shared__ double s_row[kCertWarps][2][kDh];   // [warp][key j | candidate query i][64]
    griddep_trigger();
    griddep_wait();                                 // flags, provisional budgets, lse of the budget pass
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long nflag = (long long)*(volatile const unsigned long long*)a.cert.count;
    const long long gw = (long long)blockIdx.x * kCertWarps + wid, nw = (long long)gridDim.x * kCertWarps;
    const size_t HD = (size_t)a.heads * kDh;
    const T* Q = reinterpret_cast<const T*>(a.q);
    const T* K = reinterpret_cast<const T*>(a.k);
    double* kj = s_row[wid][0];
    double* qi = s_row[wid][1];
    for (long long f = gw; f < nflag; f += nw) {
        const long long t = a.cert.list[f];
        const long bh = (long)(t / a.n);
        const int j = (int)(t - (long long)bh * a.n);
        const int b = (int)(bh / a.heads), h = (int)(bh - (long)b * a.heads);
        const T* Qb = Q + (size_t)b * a.n * HD + (size_t)h * kDh;   // row i at Qb + i * HD
        const T* Kb = K + (size_t)b * a.n * HD + (size_t)h * kDh;
        const float* lse = a.lse + (size_t)bh * a.n;
        __syncwarp();
        kj[lane] = (double)to_f32(Kb[(size_t)j * HD + lane]);
        kj[lane + 32] = (double)to_f32(Kb[(size_t)j * HD + lane + 32]);
        __syncwarp();
        // 1. v_i = t_ij - lse_i over the queries; its maximum and the lse scale
        double vmax = -INFINITY, lmax = 0.0;
        for (int i = lane; i < a.n; i += 32) {
            const double ti = a.scale * dot64_sm(Qb + (size_t)i * HD, kj);
            const double l = (double)lse[i];
            vmax = fmax(vmax, ti - l);
            lmax = fmax(lmax, fabs(l));
        }
        vmax = warp_max_d(vmax);
        lmax = warp_max_d(lmax);
        // 2. candidates: within the fp32 lse error (~1e-6 absolute, ulp-scaled) of the maximum
        const double thr = vmax - (2e-4 + 4e-6 * lmax);
        double best = 0.0;
        // the 32-query blocks in a key-dependent rotation: when many keys share
        // tied candidates (near-uniform rows), warps fill different rows' cache
        // entries first instead of all computing the same row
        const int nblk = (a.n + 31) >> 5;
        for (int it = 0; it < nblk; ++it) {
            const int base = (int)((it + j) % nblk) << 5;
            const int i = base + lane;
            double ti = 0.0;
            bool cand = false;
            if (i < a.n) {
                ti = a.scale * dot64_sm(Qb + (size_t)i * HD, kj);
                cand = ti - (double)lse[i] >= thr;
            }
            unsigned ballot = __ballot_sync(0xffffffffu, cand);
            while (ballot) {
                const int src = __ffs(ballot) - 1;
                ballot &= ballot - 1;
                const int ci = base + src;
                const double tc = __shfl_sync(0xffffffffu, ti, src);
                // 3. the candidate row's exact statistics (cached for this forward)
                const size_t ri = (size_t)bh * a.n + ci;
                double m, l;
                if (*(volatile uint8_t*)(a.cert.row_done + ri)) {
                    m = *(volatile double*)(a.row_m + ri);
                    l = *(volatile double*)(a.row_l + ri);
                } else {
                    __syncwarp();
                    qi[lane] = (double)to_f32(Qb[(size_t)ci * HD + lane]);
                    qi[lane + 32] = (double)to_f32(Qb[(size_t)ci * HD + lane + 32]);
                    __syncwarp();
                    m = -INFINITY;
                    for (int jj = lane; jj < a.n; jj += 32)
                        m = fmax(m, a.scale * dot64_sm(Kb + (size_t)jj * HD, qi));
                    m = warp_max_d(m);
                    l = 0.0;
                    for (int jj = lane; jj < a.n; jj += 32) l += exp(a.scale * dot64_sm(Kb + (size_t)jj * HD, qi) - m);
                    l = warp_sum_d(l);
                    if (lane == 0) {
                        a.row_m[ri] = m;
                        a.row_l[ri] = l;
                        __threadfence();
                        a.cert.row_done[ri] = 1;
                    }
                }
                // 4. the candidate's A_ij in the oracle's form
                best = fmax(best, exp(tc - m) / l);
            }
        }
        if (lane == 0) {
            const double cm = best;
            int r;
            bool ex;
            const double tt = __ddiv_rn(__dmul_rn((double)a.n, cm), a.alpha);
            const double raw = __dmul_rn(tt, tt);
            const double c = ceil(raw);
            ex = c >= (double)a.d;
            r = ex ? a.d : (int)c;
            if (r < a.min_samples) r = a.min_samples;
            if (r > a.d) r = a.d;
            a.budgets[t] = r;
            a.exact[t] = ex ? 1 : 0;
            if (a.cmax_out) a.cmax_out[t] = cm;
            if (a.counters) {
                if (ex) {
                    atomicAdd(a.counters + 0, 2ull * (unsigned long long)a.d * (unsigned long long)a.dh);
                    atomicAdd(a.counters + 2, 1ull);
                } else {
                    atomicAdd(a.counters + 0, (unsigned long long)r * (2ull * a.dh + 3ull));
                    atomicAdd(a.counters + 1, (unsigned long long)r);
                }
            }
            if (a.hist) atomicAdd(&a.hist[(size_t)h * (a.d + 1) + (ex ? a.d : min(r, a.d - 1))], 1u);
        }
    }
}

}  // namespace mca_dev

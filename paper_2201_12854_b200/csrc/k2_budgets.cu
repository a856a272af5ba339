// k2_budgets.cu — K2: column maxima -> Eq. 9 sample budgets, FLOP accounting,
// and the per-head work lists the encoding kernels consume.
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
//   kKeyArgmax: the key holds the winning row i*; cmax = exp(scale S - m_i*) / l_i*,
//               the oracle's softmax formula, in fp64 with K1's row statistics.
//               S is the winner's tensor-core score from K1b (exact bf16
//               products, fp32 sum), or, for the CUDA-core score pass,
//               q_i*.k_j recomputed here in fp64.
//
// Bucketing ("tokens bucketed by sample count"): a block covers
// 256 tokens of ONE (b, h) row, so it histograms budgets per head in shared
// memory; k2_scan turns the histograms into descending-budget offsets and
// k2_scatter writes each head's sampled-token list sorted by budget (largest
// first: LPT order for K3) and its exact-token list (for K3b).
#include "k2c_certify.cu"
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
    const void* q;                     // [B, n, H*64] (kKeyArgmax without colscore)
    const void* k;
    const float* colscore;             // [B, H, n] raw winning score (kKeyArgmax; nullable)
    double scale;
    long count;                        // B*H*n
    int row_len;                       // tokens per block row (= n in the forward)
    int n, heads, d, dh, min_samples;
    double alpha;
    bool force_exact;
    const int32_t* budgets_override;
    const uint8_t* exact_override;
    int32_t* budgets;
    uint8_t* exact;
    double* cmax_out;
    unsigned long long* counters;      // [0] approx cost, [1] sampled draws, [2] exact token-heads
    unsigned int* hist;                // [H, d + 1]: bins 1..d-1 sampled budgets, bin d = exact (nullable)
    CertSink cert;                     // Eq. 9 values at an integer boundary: deferred to k2c_certify
};

template <class T>
__device__ __forceinline__ double dot64_f64(const T* a, const T* b) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < kDh; c += 8) {
        float va[8], vb[8];
        load8(a + c, va);
        load8(b + c, vb);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e & 3] = fma((double)va[e], (double)vb[e], acc[e & 3]);
    }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// grid = (ceil(row_len / 256), B * H); block = 256 tokens of one (b, h).
template <int kSrc, class T>
__global__ void __launch_bounds__(256) k2_budgets(K2Args a) {
    __shared__ unsigned int s_hist[1025];
    const bool use_hist = a.hist != nullptr && a.d <= 1024;
    if (use_hist)
        for (int i = threadIdx.x; i <= a.d; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const long bh = grid_bh();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long cost = 0, samples = 0, nexact = 0;
    if (j < a.row_len && bh * a.row_len < a.count) {
        const long t = bh * a.row_len + j;
        if (a.cert.row_done) a.cert.row_done[t] = 0;   // k2c's row-statistics cache
        int r;
        bool ex;
        bool deferred = false;
        double cert_mag = 1.0;
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
                double s;
                if (a.colscore) {
                    s = (double)a.colscore[t];   // tensor-core score (bf16: exact products, fp32 sum; fp32: 3xTF32)
                } else {
                    const int b = (int)(bh / a.heads), h = (int)(bh - (long)b * a.heads);
                    const size_t HD = (size_t)a.heads * kDh;
                    const T* qi = reinterpret_cast<const T*>(a.q) + ((size_t)b * a.n + i) * HD + (size_t)h * kDh;
                    const T* kj = reinterpret_cast<const T*>(a.k) + ((size_t)b * a.n + j) * HD + (size_t)h * kDh;
                    s = dot64_f64(qi, kj);
                }
                const size_t ri = (size_t)bh * a.n + i;
                cm = __ddiv_rn(exp(__dsub_rn(__dmul_rn(a.scale, s), a.row_m[ri])), a.row_l[ri]);
                // certification scale: the winner's |t| and |lse| (k2c_certify.cu error model)
                cert_mag = 1.0 + fabs(a.scale * s) + 2.0 * fabs(a.row_m[ri] + log(a.row_l[ri]));
            }
            if (a.cmax_out) a.cmax_out[t] = cm;
            budget_for(cm, a.n, a.alpha, a.min_samples, a.d, &r, &ex);
            if (a.cert.list && eq9_ambiguous(cm, a.n, a.alpha, a.min_samples, a.d, (double)a.cert.tau_rel * cert_mag)) {
                cert_push(a.cert, (long long)t, cm, a.n);   // k2c re-derives it in fp64 and accounts it
                deferred = true;
            }
        }
        if (!deferred) {
            a.budgets[t] = r;
            a.exact[t] = ex ? 1 : 0;
            if (ex) {
                cost = 2ull * (unsigned long long)a.d * (unsigned long long)a.dh;
                nexact = 1;
            } else {
                cost = (unsigned long long)r * (2ull * a.dh + 3ull);
                samples = (unsigned long long)r;
            }
            // sort bin: budgets above d - 1 only occur through budgets_override (tests)
            const int bin = ex ? a.d : min(r, a.d - 1);
            // warp-aggregated: lanes with the same bin add once (small budgets are common)
            const unsigned peers = __match_any_sync(__activemask(), bin);
            if ((threadIdx.x & 31) == __ffs(peers) - 1) {
                if (use_hist) atomicAdd(&s_hist[bin], (unsigned)__popc(peers));
                else if (a.hist)
                    atomicAdd(&a.hist[(size_t)(bh % a.heads) * (a.d + 1) + bin], (unsigned)__popc(peers));
            }
        }
    }
    if (a.counters) {
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
    if (use_hist) {
        __syncthreads();
        const int h = (int)(bh % a.heads);
        for (int i = threadIdx.x; i <= a.d; i += blockDim.x)
            if (s_hist[i]) atomicAdd(&a.hist[(size_t)h * (a.d + 1) + i], s_hist[i]);
    }
}

// One block per head: cursor[h][bin] = start of `bin` in the head's sampled
// list, bins in DESCENDING budget order; cursor[h][d] = 0 for the exact list.
// counts[h] = {number of sampled tokens, number of exact tokens}.
__global__ void __launch_bounds__(1024) k2_scan(const unsigned int* __restrict__ hist, int d,
                                                unsigned int* __restrict__ cursor, int* __restrict__ counts) {
    __shared__ unsigned int s[1024];
    __shared__ unsigned int carry;
    griddep_trigger();
    griddep_wait();      // the histograms of the budget pass
    const int h = blockIdx.x;
    const unsigned int* hh = hist + (size_t)h * (d + 1);
    unsigned int* cc = cursor + (size_t)h * (d + 1);
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    // bins r = d-1, d-2, ..., 1 (descending), processed 1024 at a time
    for (int base = 0; base < d - 1; base += 1024) {
        const int idx = base + threadIdx.x;           // position in descending order
        const int r = d - 1 - idx;
        const unsigned int v = (idx < d - 1) ? hh[r] : 0u;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int off = 1; off < 1024; off <<= 1) {    // Hillis-Steele inclusive scan
            const unsigned int add = threadIdx.x >= off ? s[threadIdx.x - off] : 0u;
            __syncthreads();
            s[threadIdx.x] += add;
            __syncthreads();
        }
        if (idx < d - 1) cc[r] = carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += s[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        cc[d] = 0;
        counts[2 * h + 0] = (int)carry;
        counts[2 * h + 1] = (int)hh[d];
    }
}

// Scatter token ids ((b << 16) | j) into the per-head lists. Order inside a bin is
// whatever the atomics give: it only changes which warp encodes a token, never
// the token's result.
__global__ void __launch_bounds__(256) k2_scatter(const int32_t* __restrict__ budgets,
                                                  const uint8_t* __restrict__ exact, int n, int heads, int d,
                                                  long tokens, unsigned int* __restrict__ cursor,
                                                  int32_t* __restrict__ samp_list, int32_t* __restrict__ exact_list) {
    const long bh = grid_bh();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    griddep_trigger();
    griddep_wait();      // the scan's cursors
    if (j >= n || bh * n >= tokens * heads) return;
    const long t = bh * n + j;
    const int b = (int)(bh / heads), h = (int)(bh - (long)b * heads);
    const int tok = (b << 16) | j;   // list entry: (b << 16) | j (n, B <= 65535, checked by the host)
    const bool ex = exact[t] != 0;
    const int bin = ex ? d : min(budgets[t], d - 1);
    // warp-aggregated cursor bump: one atomic per distinct bin in the warp
    const unsigned peers = __match_any_sync(__activemask(), bin);
    const int leader = __ffs(peers) - 1;
    const int lane = threadIdx.x & 31;
    unsigned int base = 0;
    if (lane == leader) base = atomicAdd(&cursor[(size_t)h * (d + 1) + bin], (unsigned)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    const unsigned int pos = base + (unsigned)__popc(peers & ((1u << lane) - 1u));
    (ex ? exact_list : samp_list)[(size_t)h * tokens + pos] = tok;
}

// Scan and scatter in one kernel: every CTA (2048 tokens of one head) recomputes its head's bin bases
// from the (complete) histogram in shared memory (a 1 K-bin exclusive scan is
// cheaper than a separate kernel and its dependency hop), then places its
// tokens at base[bin] + a bump of the zero-initialised fill counter.
// Same lists as k2_scan + k2_scatter: bins in descending budget order.
constexpr int kScatterThreads = 1024, kScatterPerThread = 2;   // 2048 tokens of one head per CTA
__global__ void __launch_bounds__(kScatterThreads) k2_scan_scatter(const int32_t* __restrict__ budgets,
                                                                   const uint8_t* __restrict__ exact,
                                                                   const unsigned int* __restrict__ hist, int n,
                                                                   int heads, int d, long tokens,
                                                                   unsigned int* __restrict__ fill,
                                                                   int* __restrict__ counts,
                                                                   int32_t* __restrict__ samp_list,
                                                                   int32_t* __restrict__ exact_list) {
    extern __shared__ unsigned int s_base[];   // [d + 1] bin bases, then [d + 1] this CTA's per-bin counts / offsets
    unsigned int* s_cnt = s_base + (d + 1);
    __shared__ unsigned int s_warp[kScatterThreads / 32];
    const int h = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    griddep_trigger();
    for (int i = tid; i <= d; i += kScatterThreads) s_cnt[i] = 0;
    __syncthreads();     // zeroed before any thread ranks its tokens (ahead of the scan's barrier)
    griddep_wait();      // the histograms and budgets of the budget pass
    // this CTA's tokens (positions g of the head's B*n, sequence-major): their
    // budget loads go out first (overlapping the histogram loads and the scan),
    // rank within their bin in shared memory, then one global reservation per
    // non-empty bin after the scan
    int bin[kScatterPerThread];
    unsigned int rank[kScatterPerThread];
#pragma unroll
    for (int u = 0; u < kScatterPerThread; ++u) {
        const long g = ((long)blockIdx.x * kScatterPerThread + u) * kScatterThreads + tid;
        bin[u] = -1;
        if (g < tokens) {
            const long b = g / n, j = g - b * n;
            const long t = (b * heads + h) * n + j;
            bin[u] = exact[t] ? d : min(budgets[t], d - 1);
        }
    }
    const unsigned int* hh = hist + (size_t)h * (d + 1);
    // thread tid owns descending positions [tid * per, +per): bins r = d - 1 - position
    const int nb = d - 1, per = (nb + kScatterThreads - 1) / kScatterThreads;
    unsigned int loc = 0;
    for (int k = 0; k < per; ++k) {
        const int idx = tid * per + k;
        if (idx < nb) loc += hh[d - 1 - idx];
    }
    unsigned int inc = loc;                     // block-wide exclusive scan of loc
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned int v = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += v;
    }
    if (lane == 31) s_warp[wid] = inc;
#pragma unroll
    for (int u = 0; u < kScatterPerThread; ++u)
        if (bin[u] >= 0) rank[u] = atomicAdd(&s_cnt[bin[u]], 1u);
    __syncthreads();
    unsigned int woff = 0;
    for (int w2 = 0; w2 < wid; ++w2) woff += s_warp[w2];
    unsigned int run = woff + inc - loc;
    for (int k = 0; k < per; ++k) {
        const int idx = tid * per + k;
        if (idx < nb) {
            const int r = d - 1 - idx;
            s_base[r] = run;
            run += hh[r];
        }
    }
    if (tid == 0) s_base[d] = 0;
    if (blockIdx.x == 0 && tid == kScatterThreads - 1) {
        counts[2 * h + 0] = (int)run;           // the last thread's running total: all sampled tokens
        counts[2 * h + 1] = (int)hh[d];
    }
    __syncthreads();
    for (int i = tid; i <= d; i += kScatterThreads) {
        const unsigned int c = s_cnt[i];
        if (c) s_cnt[i] = atomicAdd(&fill[(size_t)h * (d + 1) + i], c);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kScatterPerThread; ++u) {
        if (bin[u] < 0) continue;
        const long g = ((long)blockIdx.x * kScatterPerThread + u) * kScatterThreads + tid;
        const int b = (int)(g / n), j = (int)(g - (long)b * n);
        const unsigned int pos = s_base[bin[u]] + s_cnt[bin[u]] + rank[u];
        (bin[u] == d ? exact_list : samp_list)[(size_t)h * tokens + pos] = (b << 16) | j;   // (n, B <= 65535)
    }
}

template __global__ void k2_budgets<kKeyValue, float>(K2Args);
template __global__ void k2_budgets<kKeyArgmax, __nv_bfloat16>(K2Args);
template __global__ void k2_budgets<kKeyArgmax, float>(K2Args);
template __global__ void k2_budgets<kGivenCmax, float>(K2Args);

}  // namespace mca_dev

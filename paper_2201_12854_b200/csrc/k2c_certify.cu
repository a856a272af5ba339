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
// the pass's error bound (relative) of an integer boundary that changes (r, exact) and
// defers it here (eq9_ambiguous / cert_push, with the pass's own cmax). This
// kernel re-derives those column maxima in binary64 the way the oracle does
// (oracle/tensor.cpp softmax_rows, col_max). One CTA per (b, h) item with
// flagged keys, all of the item's flagged keys at once:
//   1. the item's flagged keys (read from the flag list) and their k rows;
//   2. one pass over the queries: v_if = t_if - lse_i (fp32 dot, fp32 lse)
//      against every flagged key f; the candidates are the (f, i) with v_if
//      within the fp32 error of ln(cmax_f) (the pass's maximum), and for them
//      t_if in binary64 (bf16 products and their sums are exact in binary64,
//      so t_if is the oracle's value bit for bit);
//   3. each candidate row's exact statistics, one pass over the keys with one
//      exp per entry against the score pass's row max m~_i:
//      L_i = sum_j' exp(t_ij' - m~_i) in binary64 (cached per row for the
//      forward: the budget pass clears row_done[], the first CTA fills it);
//   4. cmax_f = max over its candidates of exp(t_if - m~_i) / L_i (the
//      oracle's exp(t - m) / l with both terms scaled by exp(m - m~)), Eq. 9,
//      the FLOP counters and the budget histogram the work lists read.
// What remains between device and oracle is summation order and exp's last
// ulp: ~1e-15 relative, so budgets equal the fp64 oracle's end to end
// (tests/test_gpu_configs.py, tests/test_gpu_parity.py).
#pragma once

#include <type_traits>

#include "mca_common.cuh"

namespace mca_dev {

// Error model of the fp32-accumulated score passes. cmax = exp(v), v = t - lse:
// the absolute error of v grows with the magnitudes fp32 carries, |t| and
// |lse| (tensor-core fp32 accumulation rounds every K step). Measured
// (scripts/tf32_accuracy.py, tests/test_gpu_configs.py): relative cmax error
// <= ~1e-7 x M for the bf16 passes and <= ~3.4e-7 x M for the 3xTF32 passes,
// M = 1 + |ln cmax| + 2 max|lse|. raw ~ cmax^2 doubles it; the flag threshold
// on raw is tau_rel x M with a >= 4x margin.
constexpr float kCertTauBf16 = 1e-6f;
constexpr float kCertTauTf32 = 3e-6f;

// Flag sink of the budget passes (K12 group B, k2_budgets): null list = off.
// A flagged key goes to its (b, h) item's slots (item_cnt counts them; zeroed
// per forward), so the certification kernel visits only items with flags and
// finds their keys without scanning; past kCertSlots per item, keys spill to
// the global list (scanned by that item's CTA only).
constexpr int kCertSlots = 32;
struct CertSink {
    long long* list;                 // [B*H*n] spilled token-head indices t = (b*H + h)*n + j
    double* cm;                      // [B*H*n] the score pass's cmax of each spilled entry
    unsigned long long* count;       // number of spilled entries (zeroed per forward)
    uint8_t* row_done;               // [B*H*n] exact row statistics cached (cleared by the budget pass)
    float tau_rel;                   // flag threshold per unit of M (kCertTauBf16 / kCertTauTf32)
    unsigned* item_cnt;              // [B*H] flagged keys per item (zeroed per forward)
    int* slot_j;                     // [B*H][kCertSlots] key index j
    double* slot_cm;                 // [B*H][kCertSlots] the score pass's cmax
};

// (r, exact) of Eq. 9 could change under the score pass's cmax error: raw lies
// within tau of an integer m whose two sides give different outcomes
// (m >= min_samples: below it both clamp to min_samples; m <= d - 1: at or
// above d both are exact). tau = tau_rel x mag, mag = 1 + |ln cm| + 2 max|lse|.
__device__ __forceinline__ bool eq9_ambiguous(double cm, int n, double alpha, int min_samples, int d, double tau) {
    const double t = __ddiv_rn(__dmul_rn((double)n, cm), alpha);
    const double raw = __dmul_rn(t, t);
    const double m = rint(raw);
    return m >= (double)min_samples && m <= (double)(d - 1) && fabs(raw - m) <= tau * fmax(raw, 1.0);
}

__device__ __forceinline__ void cert_push(const CertSink& c, long long t, double cm, int n) {
    const long long bh = t / n;
    const unsigned pos = atomicAdd(c.item_cnt + bh, 1u);
    if (pos < (unsigned)kCertSlots) {
        c.slot_j[bh * kCertSlots + pos] = (int)(t - bh * n);
        c.slot_cm[bh * kCertSlots + pos] = cm;
    } else {
        const unsigned long long g = atomicAdd(c.count, 1ull);
        c.list[g] = t;
        c.cm[g] = cm;
    }
}

struct K2cArgs {
    const void* q;                   // [B, n, H*64]
    const void* k;
    const float* lse;                // [B, H, n] natural-log lse of the scaled score rows (score pass)
    double scale;
    int n, heads, items, d, dh, min_samples;
    double alpha;
    CertSink cert;
    const double* row_m;             // [B, H, n] the score pass's row max m~ (the reference point)
    double* row_l;                   // [B, H, n] exact L_i (filled on demand)
    int32_t* budgets;
    uint8_t* exact;
    double* cmax_out;                // nullable
    unsigned long long* counters;    // [0] approx cost, [1] sampled draws, [2] exact token-heads
    unsigned int* hist;              // [H, d + 1] (nullable)
    unsigned long long* cert_total;  // number of re-derived token-heads (FlopsReport.certified)
};

constexpr int kCertThreads = 128;    // 4 warps; a thread pair per staged query / key row
constexpr int kCertKeys = 32;        // flagged keys of one item processed together
constexpr int kCertCands = 256;      // (key, query) candidates per batch
constexpr int kCertRows = 8;         // candidate rows whose statistics one pass over the keys computes
constexpr int kCertMaxN = 65536;     // bitmap of an item's rows (n <= 65535, mca_forward's limit)
constexpr int kCertStage = 64;       // rows staged in shared memory per chunk (one L2 round trip each)

// max of positive doubles through their bit patterns (monotone for x >= 0)
__device__ __forceinline__ void atomic_max_pos(double* p, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(p), (unsigned long long)__double_as_longlong(v));
}

// Rows [c0, c0 + cnt) of a [n][HD]-strided 64-wide operand -> s_stage (fp32):
// every thread issues its 16-byte loads at once, so a chunk costs one round trip.
// Pull the next chunk's rows into L2 while this one is computed (the staging
// loads are otherwise full DRAM round trips: q / k were written long before).
template <class T>
__device__ __forceinline__ void prefetch_rows(const T* __restrict__ base, size_t stride, int c0, int n) {
    constexpr int kLines = kDh * (int)sizeof(T) / 128;   // 128-byte lines per row
    const int e = threadIdx.x, r = e / kLines;
    if (r < kCertStage && c0 + r < n)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (size_t)(c0 + r) * stride + (e % kLines) * (128 / sizeof(T))));
}

template <class T>
__device__ __forceinline__ void stage_rows(float (*st)[kDh + 1], const T* __restrict__ base, size_t stride, int c0,
                                           int cnt) {
    constexpr int kPerRow = kDh / 8;                                  // pieces of 8 elements
    constexpr int kPer = kCertStage * kPerRow / kCertThreads;        // pieces per thread (all loads in flight)
    float v[kPer][8];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int e = threadIdx.x + u * kCertThreads, r = e / kPerRow, c = (e - r * kPerRow) * 8;
        if (r < cnt) load8(base + (size_t)(c0 + r) * stride + c, v[u]);
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int e = threadIdx.x + u * kCertThreads, r = e / kPerRow, c = (e - r * kPerRow) * 8;
        if (r < cnt)
#pragma unroll
            for (int q = 0; q < 8; ++q) st[r][c + q] = v[u][q];
    }
}

// One CTA per (b, h) item; items without flags exit after reading their count.
template <class T>
__global__ void __launch_bounds__(kCertThreads) k2c_certify(K2cArgs a) {
    __shared__ float s_k[kCertKeys][kDh];            // the batch's flagged keys (fp32 = exact bf16 / fp32 values)
    __shared__ int s_j[kCertKeys];
    __shared__ double s_lcm[kCertKeys], s_best[kCertKeys];
    __shared__ int s_cf[kCertCands], s_ci[kCertCands];
    __shared__ double s_ct[kCertCands];
    __shared__ int s_rows[kCertCands];
    __shared__ unsigned s_bm[kCertMaxN / 32];        // rows already queued in this batch
    __shared__ double s_qr[kCertRows][kDh];          // candidate rows of one statistics pass (binary64)
    __shared__ double s_mref[kCertRows];
    __shared__ double s_part[kCertThreads / 32][kCertRows];
    __shared__ int s_nkeys, s_ncand, s_nrows, s_slot_next;
    __shared__ float s_stage[kCertStage][kDh + 1];   // a chunk of the item's q or k rows (padded: a row per thread)
    griddep_trigger();
    griddep_wait();                                  // flags, provisional budgets, lse of the budget pass
    const int bh = blockIdx.x;
    const unsigned cnt = *(volatile const unsigned*)(a.cert.item_cnt + bh);
    if (cnt == 0) return;
    if (threadIdx.x == 0 && a.cert_total) atomicAdd(a.cert_total, (unsigned long long)cnt);
    const int tid = threadIdx.x, lane = tid & 31;
    const long long nflag = (long long)*(volatile const unsigned long long*)a.cert.count;
    const size_t HD = (size_t)a.heads * kDh;
    const int b = bh / a.heads, h = bh - b * a.heads;
    const T* Qb = reinterpret_cast<const T*>(a.q) + (size_t)b * a.n * HD + (size_t)h * kDh;
    const T* Kb = reinterpret_cast<const T*>(a.k) + (size_t)b * a.n * HD + (size_t)h * kDh;
    const float* lse = a.lse + (size_t)bh * a.n;
    const double* rowm = a.row_m + (size_t)bh * a.n;
    double* rowl = a.row_l + (size_t)bh * a.n;
    uint8_t* done = a.cert.row_done + (size_t)bh * a.n;
    const long long lo = (long long)bh * a.n, hi = lo + a.n;
    const int nslots = min(cnt, (unsigned)kCertSlots);
    if (tid == 0) s_slot_next = 0;
    for (;;) {
        // 1. up to kCertKeys flagged keys: the item's slots first, then its spilled
        // entries in the global list (consumed: -1, so the next batch takes the rest)
        __syncthreads();
        const int s0 = s_slot_next;
        __syncthreads();                             // every thread has read s0 before it advances
        if (tid == 0) {
            s_nkeys = 0;
            s_ncand = 0;
            s_nrows = 0;
        }
        __syncthreads();
        if (s0 < nslots) {
            const int take = min(nslots - s0, kCertKeys);
            if (tid < take) {
                s_j[tid] = a.cert.slot_j[(size_t)bh * kCertSlots + s0 + tid];
                s_lcm[tid] = log(a.cert.slot_cm[(size_t)bh * kCertSlots + s0 + tid]);
                s_best[tid] = 0.0;
            }
            if (tid == 0) {
                s_nkeys = take;
                s_slot_next = s0 + take;
            }
        } else if (cnt > (unsigned)kCertSlots) {
            for (long long f0 = 0; f0 < nflag; f0 += kCertThreads) {
                const long long f = f0 + tid;
                if (f < nflag) {
                    const long long t = a.cert.list[f];
                    if (t >= lo && t < hi) {
                        const int slot = atomicAdd(&s_nkeys, 1);
                        if (slot < kCertKeys) {
                            s_j[slot] = (int)(t - lo);
                            s_lcm[slot] = log(a.cert.cm[f]);
                            s_best[slot] = 0.0;
                            a.cert.list[f] = -1;
                        }
                    }
                }
            }
        }
        __syncthreads();
        const int nk = min(s_nkeys, kCertKeys);
        if (nk == 0) break;
        for (int e = tid; e < nk * kDh; e += kCertThreads) {
            const int f = e / kDh, c = e - f * kDh;
            s_k[f][c] = to_f32(Kb[(size_t)s_j[f] * HD + c]);
        }
        for (int e = tid; e < (a.n + 31) / 32; e += kCertThreads) s_bm[e] = 0u;
        __syncthreads();
        // 2. one pass over the queries (an octet per query): fp32 partial dots locate
        // the candidates, binary64 partial dots give their exact t
        for (int c0 = 0; c0 < a.n; c0 += kCertStage) {
            const int cn = min(kCertStage, a.n - c0);
            __syncthreads();
            stage_rows(s_stage, Qb, HD, c0, cn);
            __syncthreads();
            prefetch_rows(Qb, HD, c0 + kCertStage, a.n);
            static_assert(kCertThreads == 2 * kCertStage, "two threads per staged row");
            const int ii = tid % kCertStage, half = tid / kCertStage;
            if (ii < cn) {   // a query row per thread pair, the keys split between the two
                const int i = c0 + ii;
                const double l = (double)lse[i];
                for (int f = half; f < nk; f += 2) {
                    float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
                    for (int e = 0; e < kDh; e += 2) {
                        acc0 = fmaf(s_stage[ii][e], s_k[f][e], acc0);
                        acc1 = fmaf(s_stage[ii][e + 1], s_k[f][e + 1], acc1);
                    }
                    const double v = a.scale * (double)(acc0 + acc1) - l;
                    if (v >= s_lcm[f] - (1e-3 + 1e-5 * (fabs(l) + fabs(s_lcm[f])))) {
                        // the same binary64 chain (e = 0 .. 63 in order) as the row pass, so a
                        // candidate's exp(t - m~) / L is exactly 1 when it is the row's only term
                        double t = 0.0;
#pragma unroll
                        for (int e = 0; e < kDh; ++e) t = fma((double)s_stage[ii][e], (double)s_k[f][e], t);
                        const int slot = atomicAdd(&s_ncand, 1);
                        if (slot < kCertCands) {
                            s_cf[slot] = f;
                            s_ci[slot] = i;
                            s_ct[slot] = a.scale * t;
                        }
                    }
                }
            }
        }
        __syncthreads();
        // more near-ties than candidate slots (degenerate, e.g. uniform rows):
        // every query row is a candidate of every key of the batch
        const bool all_rows = s_ncand > kCertCands;
        const int nc = min(s_ncand, kCertCands);
        // 3. the distinct candidate rows without cached statistics
        if (!all_rows) {
            for (int c = tid; c < nc; c += kCertThreads) {
                const int i = s_ci[c];
                if (!done[i]) {
                    const unsigned bit = 1u << (i & 31);
                    if (!(atomicOr(&s_bm[i >> 5], bit) & bit)) s_rows[atomicAdd(&s_nrows, 1)] = i;
                }
            }
        }
        __syncthreads();
        const int nrows_total = all_rows ? a.n : s_nrows;
        // row statistics, kCertRows rows per pass over the item's keys (an octet per key)
        for (int r0 = 0; r0 < nrows_total; r0 += kCertRows) {
            const int nr = min(kCertRows, nrows_total - r0);
            __syncthreads();
            for (int e = tid; e < nr * kDh; e += kCertThreads) {
                const int r = e / kDh, c = e - r * kDh;
                const int i = all_rows ? r0 + r : s_rows[r0 + r];
                s_qr[r][c] = (double)to_f32(Qb[(size_t)i * HD + c]);
            }
            if (tid < nr) s_mref[tid] = rowm[all_rows ? r0 + tid : s_rows[r0 + tid]];
            __syncthreads();
            double part[kCertRows];
#pragma unroll
            for (int r = 0; r < kCertRows; ++r) part[r] = 0.0;
            for (int c0 = 0; c0 < a.n; c0 += kCertStage) {
                const int cn = min(kCertStage, a.n - c0);
                __syncthreads();
                stage_rows(s_stage, Kb, HD, c0, cn);
                __syncthreads();
                prefetch_rows(Kb, HD, c0 + kCertStage, a.n);
                const int jj = tid % kCertStage, half = tid / kCertStage;
                // a key row per thread pair, the candidate rows split between the two (rows
                // half, half + 2, ...); each key element converted to binary64 once; the
                // per-thread row count kQ is the smallest of 1 / 2 / 4 that covers nr
                auto rows_pass = [&](auto kq) {
                    constexpr int kQ = decltype(kq)::value;
                    double t[kQ];
#pragma unroll
                    for (int q = 0; q < kQ; ++q) t[q] = 0.0;
#pragma unroll 8
                    for (int e = 0; e < kDh; ++e) {
                        const double kd = (double)s_stage[jj][e];
#pragma unroll
                        for (int q = 0; q < kQ; ++q) t[q] = fma(kd, s_qr[2 * q + half][e], t[q]);
                    }
#pragma unroll
                    for (int q = 0; q < kQ; ++q) {   // compile-time indices into part[]
                        if (half == 0 && 2 * q < nr) part[2 * q] += exp(a.scale * t[q] - s_mref[2 * q]);
                        if (half == 1 && 2 * q + 1 < nr) part[2 * q + 1] += exp(a.scale * t[q] - s_mref[2 * q + 1]);
                    }
                };
                if (jj < cn) {
                    if (nr <= 2) rows_pass(std::integral_constant<int, 1>{});
                    else if (nr <= 4) rows_pass(std::integral_constant<int, 2>{});
                    else rows_pass(std::integral_constant<int, kCertRows / 2>{});
                }
            }
#pragma unroll
            for (int r = 0; r < kCertRows; ++r) {
                double v = part[r];
                for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0) s_part[tid >> 5][r] = v;
            }
            __syncthreads();
            if (tid < nr) {
                double L = 0.0;
                for (int w2 = 0; w2 < kCertThreads / 32; ++w2) L += s_part[w2][tid];
                const int i = all_rows ? r0 + tid : s_rows[r0 + tid];
                rowl[i] = L;
                done[i] = 1;
            }
        }
        __syncthreads();
        // 4. cmax_f = max over its candidates of exp(t - m~_i) / L_i
        if (all_rows) {
            for (int f = 0; f < nk; ++f) {
                double best = 0.0;
                for (int i = tid; i < a.n; i += kCertThreads) {   // a query row per thread, the row pass's chain
                    const T* qi = Qb + (size_t)i * HD;
                    double t = 0.0;
                    for (int e0 = 0; e0 < kDh; e0 += 8) {
                        float qv[8];
                        load8(qi + e0, qv);
#pragma unroll
                        for (int e = 0; e < 8; ++e) t = fma((double)qv[e], (double)s_k[f][e0 + e], t);
                    }
                    best = fmax(best, exp(a.scale * t - rowm[i]) / rowl[i]);
                }
                atomic_max_pos(&s_best[f], best);
            }
        } else {
            for (int c = tid; c < nc; c += kCertThreads) {
                const int i = s_ci[c];
                atomic_max_pos(&s_best[s_cf[c]], exp(s_ct[c] - rowm[i]) / rowl[i]);
            }
        }
        __syncthreads();
        // Eq. 9 for the batch's keys
        if (tid < nk) {
            const long long t = lo + s_j[tid];
            const double cm = s_best[tid];
            const double tt = __ddiv_rn(__dmul_rn((double)a.n, cm), a.alpha);
            const double raw = __dmul_rn(tt, tt);
            const double cc = ceil(raw);
            const bool ex = cc >= (double)a.d;
            int r = ex ? a.d : (int)cc;
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
        __syncthreads();
        if (s_slot_next >= nslots && cnt <= (unsigned)kCertSlots) break;   // slots done, nothing spilled
    }
}

}  // namespace mca_dev

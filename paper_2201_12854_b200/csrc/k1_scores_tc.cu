// k1_scores_tc.cu — K1 on the 5th-generation tensor cores: the score pass of
// attention_matrix + col_max (matrix.hpp:46-53), bf16.
//
// Softmax needs a reduction along rows (max and sum per query) and Eq. 9 needs
// one along columns (max per key). Each is made lane-local by putting the
// reduced index on the TMEM lane axis, so neither needs shuffles or atomics:
//
//   K1a (kRowStats), CTA = (b, h, 128 queries):  S   = Q K_blk^T (lane = query)
//       per lane: online m = max t, l = sum exp(t - m) over all keys,
//       t = scale * S (log2 domain, ex2.approx)  -> row_m, row_l (fp64), lse
//   K1b (kColMax),   CTA = (b, h, 128 keys):     S^T = K Q_blk^T (lane = key)
//       per lane: max over all queries of v = t - lse_q and its first argmax
//       q*, written as the argmax key plus the winner's raw score S (fp32),
//       which K2 re-evaluates in fp64 as exp(scale S - m_q*) / l_q* (the
//       oracle's softmax form; k1_scores_simt.cu describes the key; one writer
//       per key, no atomics)
//
// Same kernel body for both: the resident 128-row operand (Q or K) arrives by
// TMA once, the streamed operand (K or Q blocks of 128) through a 3-stage TMA
// ring; one thread issues tcgen05.mma M=128 N=128 K=16 x4 per block into a
// double-buffered TMEM accumulator (2 x 128 columns, so two CTAs fit per SM).
// Eight consumer warps: two per TMEM lane quadrant, each owning 64 of the 128
// columns of a block; the two halves combine through shared memory at the end.
// Warp 0: TMA producer, warp 1: TMEM allocator + MMA issuer.
#include "mca_common.cuh"
#include "tc_common.cuh"

#ifndef MCA_K1_POLY
#define MCA_K1_POLY 6   // (measured at C4: 0 / 6 / 10 / 14 -> 901 / 818 / 830 / 935 us) pairs of each 64-score chunk whose exp2 runs as an FMA-pipe polynomial (K1a)
#endif

namespace mca_dev {

namespace k1tc {
constexpr int kBM = 128, kBN = 128;
constexpr int kConsumers = 8;
constexpr int kThreads = 64 + kConsumers * 32;
constexpr int kMaxN = 4096;
constexpr uint32_t kAtomBytes = 128 * 128;                        // 128 rows x 128 B: one 128B-swizzled K atom
// Operand layout per 128-row tile: bf16, one atom of 64 elements; or, for the
// fp32 path (3xTF32), the hi and lo tf32 parts of the fp32 values, each two
// atoms of 32 fp32 (part p, atom a at p * kPartBytes + a * kAtomBytes).
template <bool kTf32>
struct Lay {
    static constexpr int kParts = kTf32 ? 2 : 1;
    static constexpr int kAtoms = kTf32 ? 2 : 1;
    static constexpr uint32_t kPartBytes = kAtoms * kAtomBytes;
    static constexpr uint32_t kTileBytes = kParts * kPartBytes;   // 16 KB / 64 KB
    static constexpr int kStages = kTf32 ? 2 : 3;
    static constexpr uint32_t kSmemA = 0;                          // resident operand
    static constexpr uint32_t kSmemB = kTileBytes;                 // kStages streamed tiles
    static constexpr uint32_t kSmemLse = kSmemB + kStages * kTileBytes;   // [kMaxN] f32 (K1b)
    static constexpr uint32_t kSmemComb = kSmemLse + kMaxN * 4;    // partner exchange, 3 x [128] x 4 B
    static constexpr uint32_t kSmemBar = kSmemComb + 4 * 128 * 4;
    static constexpr uint32_t kSmemBytes = kSmemBar + 256 + 1024;
    static constexpr uint32_t kIdesc = kTf32 ? mca_tc::idesc_tf32(kBM, kBN) : mca_tc::idesc_f16(1, 0, kBM, kBN);
};
constexpr uint32_t kSmemBytes = Lay<false>::kSmemBytes;
constexpr uint32_t kSmemBytesTf32 = Lay<true>::kSmemBytes;
}  // namespace k1tc

enum K1Mode { kRowStats = 0, kColMax = 1 };

// kTf32: the fp32 path. tm_q / tm_k hold the tf32-exact hi parts of q, k and
// tm_q2 / tm_k2 the lo parts (fp32 - hi); S = hi.hi + hi.lo + lo.hi (3xTF32,
// ~2^-22 relative per product), fp32 accumulation in TMEM.
template <int kMode, bool kTf32 = false>
__global__ void __launch_bounds__(k1tc::kThreads, kTf32 ? 1 : 2)
    k1_scores_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_q2, const __grid_constant__ CUtensorMap tm_k2, int n,
                 int heads, float scale, double* __restrict__ row_m, double* __restrict__ row_l,
                 float* __restrict__ lse, unsigned long long* __restrict__ colkey,
                 float* __restrict__ colscore) {
    using namespace k1tc;
    using namespace mca_tc;
    using Ly = Lay<kTf32>;
    constexpr int kStages = Ly::kStages;
    constexpr uint32_t kTileBytes = Ly::kTileBytes, kSmemA = Ly::kSmemA, kSmemB = Ly::kSmemB;
    constexpr uint32_t kSmemLse = Ly::kSmemLse, kSmemComb = Ly::kSmemComb, kSmemBar = Ly::kSmemBar;
    constexpr uint32_t kIdesc = Ly::kIdesc;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* a_full = bars;
    uint64_t* b_full = bars + 1;              // [kStages]
    uint64_t* b_empty = b_full + kStages;     // [kStages]
    uint64_t* s_full = b_empty + kStages;     // [2]
    uint64_t* s_empty = s_full + 2;           // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_empty + 2);
    float* s_lse = reinterpret_cast<float*>(smem + kSmemLse);
    float* comb = reinterpret_cast<float*>(smem + kSmemComb);

    const CUtensorMap* tm_a = kMode == kRowStats ? &tm_q : &tm_k;   // resident rows
    const CUtensorMap* tm_b = kMode == kRowStats ? &tm_k : &tm_q;   // streamed blocks
    const CUtensorMap* tm_a2 = kMode == kRowStats ? &tm_q2 : &tm_k2;
    const CUtensorMap* tm_b2 = kMode == kRowStats ? &tm_k2 : &tm_q2;
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;   // uniform: see k4_apply_tf32
    const int b = blockIdx.z, h = blockIdx.y, r0 = blockIdx.x * kBM;
    const int nblk = (n + kBN - 1) / kBN;
    const size_t bh = (size_t)b * heads + h;
    // one 128-row operand tile: every part and atom of it, arriving on `bar`
    auto load_tile = [&](uint8_t* dst, const CUtensorMap* m1, const CUtensorMap* m2, uint64_t* bar, int row0) {
#pragma unroll
        for (int p = 0; p < Ly::kParts; ++p)
#pragma unroll
            for (int at = 0; at < Ly::kAtoms; ++at)
                tma_load_3d(dst + p * Ly::kPartBytes + at * kAtomBytes, p ? m2 : m1, bar,
                            h * kDh + at * (kTf32 ? 32 : 64), row0, b);
    };

    if (threadIdx.x == 0) {
        mbar_init(a_full, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(b_full + s, 1);
            mbar_init(b_empty + s, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(s_empty + i, kConsumers * 32);
        }
        fence_barrier_init();
    }
    if (kMode == kColMax) {   // query log-sum-exps of this (b, h), log2 domain
        for (int i = threadIdx.x; i < n; i += k1tc::kThreads) s_lse[i] = lse[bh * n + i] * 1.4426950408889634f;
    }
    if (warp == 1) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            tma_prefetch(tm_a);
            tma_prefetch(tm_b);
            mbar_expect_tx(a_full, kTileBytes);
            load_tile(smem + kSmemA, tm_a, tm_a2, a_full, r0);
            for (int i = 0; i < nblk; ++i) {
                const int s = i % kStages;
                mbar_wait(b_empty + s, ((i / kStages) & 1) ^ 1);
                mbar_expect_tx(b_full + s, kTileBytes);
                load_tile(smem + kSmemB + s * kTileBytes, tm_b, tm_b2, b_full + s, i * kBN);
            }
        }
    } else if (warp == 1) {   // ---------------- MMA issuer (whole warp; one elected lane issues)
        const uint64_t da = sw128_desc(smem_u32(smem + kSmemA), 16, 1024);
        const uint64_t db0 = sw128_desc(smem_u32(smem + kSmemB), 16, 1024);
        mbar_wait(a_full, 0);
        for (int i = 0; i < nblk; ++i) {
            const int s = i % kStages, sb = i & 1;
            mbar_wait(b_full + s, (i / kStages) & 1);
            mbar_wait(s_empty + sb, ((i >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint64_t db = desc_add(db0, s * kTileBytes);
            if constexpr (!kTf32) {
#pragma unroll
                for (int kk = 0; kk < kDh / 16; ++kk)
                    umma_f16_w(tmem + sb * kBN, desc_add(da, kk * 32), desc_add(db, kk * 32), kIdesc, kk > 0 ? 1u : 0u);
            } else {   // hi.lo + lo.hi + hi.hi, K = 8 fp32 (32 B) per instruction. The small
                       // products go first: every instruction rounds the fp32 accumulator,
                       // and only the last eight (hi.hi) do so at the magnitude of S
#pragma unroll
                for (int pr = 0; pr < 3; ++pr) {
                    const uint32_t ap = pr == 1 ? Ly::kPartBytes : 0u, bp = pr == 0 ? Ly::kPartBytes : 0u;
#pragma unroll
                    for (int at = 0; at < 2; ++at)
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            umma_tf32_w(tmem + sb * kBN, desc_add(da, ap + at * kAtomBytes + kk * 32),
                                        desc_add(db, bp + at * kAtomBytes + kk * 32), kIdesc, (pr | at | kk) != 0);
                }
            }
            umma_commit_w(s_full + sb);
            umma_commit_w(b_empty + s);
        }
    } else {  // ------------------------------- consumers (warps 2..9)
        const int cw = warp - 2;
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int half = cw >> 2;                  // which 64 columns of each block
        const int row = quad * 32 + lane;          // TMEM lane = resident row (query or key)
        const int grow = r0 + row;
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16) + half * 64;
        const float c2 = scale * 1.4426950408889634f;
        float m2 = -INFINITY, l = 0.0f;            // kRowStats
        float best = -INFINITY;                    // kColMax
        int best_i = 0x7FFFFFFF;
        for (int i = 0; i < nblk; ++i) {
            const int sb = i & 1;
            mbar_wait(s_full + sb, (i >> 1) & 1);
            tc_fence_after();
            uint32_t sv[2][32];
            tmem_ld32(lane_base + sb * kBN, sv[0]);
            tmem_ld32(lane_base + sb * kBN + 32, sv[1]);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(s_empty + sb);
            const int c0 = i * kBN + half * 64;        // global column index of sv[0][0]
            const int valid = min(64, n - c0);         // <= 0 for the right half of a short last block
            if constexpr (kMode == kRowStats) {
                float bmax = -INFINITY;
                if (valid >= 64) {
#pragma unroll
                    for (int e = 0; e < 64; ++e) bmax = fmaxf(bmax, __uint_as_float(sv[e >> 5][e & 31]));
                } else {
#pragma unroll
                    for (int e = 0; e < 64; ++e)
                        if (e < valid) bmax = fmaxf(bmax, __uint_as_float(sv[e >> 5][e & 31]));
                }
                if (valid > 0) {
                    const float mn = fmaxf(m2, bmax * c2);
                    float acc0 = 0.f, acc1 = 0.f;
                    if (valid >= 64) {
                        // MUFU-bound: MCA_K1_POLY of the 32 pairs take the FMA-pipe exp2 (same accuracy)
#pragma unroll
                        for (int e = 0; e < 64; e += 2) {
                            if (e < 2 * MCA_K1_POLY) {
                                const float2 xv = __ffma2_rn(make_float2(__uint_as_float(sv[e >> 5][e & 31]),
                                                                         __uint_as_float(sv[(e + 1) >> 5][(e + 1) & 31])),
                                                             make_float2(c2, c2), make_float2(-mn, -mn));
                                const float2 pv = ex2_poly5x2(xv);
                                acc0 += pv.x;
                                acc1 += pv.y;
                            } else {
                                acc0 += ex2_approx(__fmaf_rn(__uint_as_float(sv[e >> 5][e & 31]), c2, -mn));
                                acc1 += ex2_approx(__fmaf_rn(__uint_as_float(sv[(e + 1) >> 5][(e + 1) & 31]), c2, -mn));
                            }
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 64; ++e)
                            if (e < valid) acc0 += ex2_approx(__fmaf_rn(__uint_as_float(sv[e >> 5][e & 31]), c2, -mn));
                    }
                    l = (m2 == -INFINITY ? 0.0f : l * ex2_approx(m2 - mn)) + (acc0 + acc1);
                    m2 = mn;
                }
            } else {
                // v = t2 - lse2_q; strict > keeps the first (smallest) query on ties
                if (valid >= 64) {   // full chunk: no per-element bounds checks
#pragma unroll
                    for (int g = 0; g < 64; g += 4) {
                        const float4 ls = *reinterpret_cast<const float4*>(s_lse + c0 + g);
                        const float lv[4] = {ls.x, ls.y, ls.z, ls.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float v = __fmaf_rn(__uint_as_float(sv[(g + e) >> 5][(g + e) & 31]), c2, -lv[e]);
                            if (v > best) {
                                best = v;
                                best_i = c0 + g + e;
                            }
                        }
                    }
                } else {
#pragma unroll
                    for (int g = 0; g < 64; g += 4) {
                        if (g < valid) {
                            const float4 ls = *reinterpret_cast<const float4*>(s_lse + c0 + g);
                            const float lv[4] = {ls.x, ls.y, ls.z, ls.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float v = __fmaf_rn(__uint_as_float(sv[(g + e) >> 5][(g + e) & 31]), c2, -lv[e]);
                                if (g + e < valid && v > best) {
                                    best = v;
                                    best_i = c0 + g + e;
                                }
                            }
                        }
                    }
                }
            }
        }
        // combine the two column halves of each row through shared memory
        if constexpr (kMode == kRowStats) {
            if (half == 1) {
                comb[row] = m2;
                comb[128 + row] = l;
            }
        } else {
            if (half == 1) {
                comb[row] = best;
                reinterpret_cast<int*>(comb)[128 + row] = best_i;
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
        if (half == 0 && grow < n) {
            if constexpr (kMode == kRowStats) {
                const float m2b = comb[row], lb = comb[128 + row];
                const float mn = fmaxf(m2, m2b);
                const float lt = (m2 == -INFINITY ? 0.f : l * ex2_approx(m2 - mn)) +
                                 (m2b == -INFINITY ? 0.f : lb * ex2_approx(m2b - mn));
                const size_t t = bh * n + grow;
                row_m[t] = (double)mn * 0.6931471805599453;
                row_l[t] = (double)lt;
                lse[t] = (mn + __log2f(lt)) * 0.6931471805599453f;
            } else {
                const float vb = comb[row];
                const int ib = reinterpret_cast<int*>(comb)[128 + row];
                // ties go to the smaller query index (deterministic, order-independent)
                if (vb > best || (vb == best && ib < best_i)) {
                    best = vb;
                    best_i = ib;
                }
                // the winner's raw score, rebuilt from v = fma(S, c2, -lse2_q*) (exact when S = 0)
                colscore[bh * n + grow] = (best + s_lse[best_i]) / c2;
                colkey[bh * n + grow] = ((unsigned long long)float_to_ordered(best) << 32) |
                                        (unsigned long long)(0xFFFFFFFFu - (uint32_t)best_i);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<256>(tmem);
}

}  // namespace mca_dev

namespace mca_dev {
// fp32 -> (hi, lo) for the 3xTF32 passes: hi keeps the top 11 significand bits
// (exactly representable in tf32, whatever rounding the tensor core applies),
// lo = v - hi exactly. n4 = element count / 4.
__global__ void k_split_tf32(const float4* __restrict__ src, float4* __restrict__ hi, float4* __restrict__ lo,
                             size_t n4) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = src[i];
        float4 a, c;
        a.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
        a.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
        a.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
        a.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
        c.x = v.x - a.x;
        c.y = v.y - a.y;
        c.z = v.z - a.z;
        c.w = v.w - a.w;
        if (hi) hi[i] = a;   // nullptr: the caller uses src itself as the hi operand
        lo[i] = c;
    }
}
}  // namespace mca_dev

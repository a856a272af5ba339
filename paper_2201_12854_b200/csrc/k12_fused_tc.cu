// k12_fused_tc.cu — K1 + K2 fused for BERT-length sequences (bf16, n <= 768):
// the score pass (attention_matrix + softmax_rows + col_max, SPEC.md:286-294,
// matrix.hpp:46-53) and Eq. 9 (sample_budgets) for every
// (b, h) "item", persistent CTAs (one per SM) walking the items.
//
// Same formulas as k1_scores_tc (K1a then K1b) followed by k2_budgets; the
// fp32 row sums are accumulated in 4 partial sums per row instead of 2, so lse
// may differ from the three-kernel path in the last bits, and the budgets are
// Eq. 9 of this kernel's own cmax (what the parity tests check). Q and K of an
// item stay resident in shared memory for both passes.
//
//   phase 1, block (qt, kt):  S = Q_qt K_kt^T   (TMEM lane = query)
//       online row max / sum of t = scale S (log2 domain, ex2.approx) by
//       group A: 4 partial (max, sum) per row, handed to group B at the end
//       of each query tile
//   phase 2, block (qt, kt):  S^T = K_kt Q_qt^T (TMEM lane = key)
//       group B combines the partials of query tile qt into lse (global
//       lse / row_m / row_l, and -lse2 in smem), then per key the max over
//       queries of v = log2(e) (t - lse_q) (one FFMA2 and one three-input
//       max per two scores, two running maxima per thread), accumulated over
//       qt; at the end of the item group B evaluates
//       cmax = max_q exp(t_qj - lse_q) = 2^max v in fp64 and Eq. 9 (budget,
//       exact flag, FLOP counters, the per-head budget histogram). No argmax:
//       the maximum itself is the softmax entry.
// The two phases run CONCURRENTLY: group A (bound by the MUFU, one exponential
// per score) streams blocks without ever waiting for group B; group B trails it
// by a query tile.
//
// Group A is split into two sub-groups that take alternate blocks (even /
// odd block counter, S buffer 0 / 1), 64 columns per warp. On each SM
// sub-partition two warps exponentiate block u while the other two load and
// reduce block u + 1, so the exponential unit stays busy across block
// boundaries (with all four warps on one block they reached the row max /
// load / wait phases together and the MUFU idled meanwhile).
//
// Warp roles (864 threads, one persistent CTA per SM): warp 0 the phase-2 MMA
// issuer, warp 1 TMEM allocator + phase-1 MMA issuer, warps 2-17 group A (four
// warps per TMEM lane quadrant), warps 18-25 group B (two per quadrant, 64
// columns each), warp 26 the TMA producer.
// TMEM: A buffers [0,256), B buffers [256,512).
#include "k2c_certify.cu"
#include "mca_common.cuh"
#include "tc_common.cuh"

namespace mca_dev {

#ifndef MCA_K12_PROF
#define MCA_K12_PROF 0
#endif
// Diagnostics (build with EXTRA=-DMCA_K12_PROF=1): clock64 stamps of CTA 0:
// [0] start, [1 + u] group A block u done, [40 + u] group B block u done, [80] end
__device__ long long g_k12_prof[MCA_K12_PROF ? 256 : 1];   // + [96 + U] A wait done, [128 + U] / [160 + U] A piece loads done, [192 + U] phase-1 MMA issued, [224 + qt] lse of tile qt
// per CTA: smid, globaltimer at start and at exit (ns), clocks at exit - start
__device__ unsigned long long g_k12_cta[MCA_K12_PROF ? 4096 : 1][4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

namespace k12 {
constexpr int kT = 128;                           // tile rows (= block columns)
constexpr int kMaxTiles = 6;                      // n <= 768
constexpr int kAWarps = 16;                       // group A: 4 per TMEM lane quadrant (2 sub-groups x 2 column halves)
constexpr int kBWarps = 8;                        // group B: 2 per TMEM lane quadrant, 64 columns each
constexpr int kAThreads = kAWarps * 32, kBThreads = kBWarps * 32;
constexpr int kCThreads = kAThreads + kBThreads;
constexpr int kThreads = 64 + kCThreads + 32;     // 864: + the TMA producer warp
constexpr uint32_t kTileBytes = kT * kDh * 2;     // 16 KB: 128 rows x 64 bf16, 128B-swizzled
constexpr uint32_t kIdesc = mca_tc::idesc_f16(1, 0, kT, kT);

struct Layout {
    uint32_t q, k, lse2, comb, hist, lmax, bars, bytes;
};
__host__ __device__ inline Layout layout(int nt, int d) {
    Layout L;
    L.q = 0;
    L.k = nt * kTileBytes;
    L.lse2 = 2 * nt * kTileBytes;                              // [2][128] f32: -lse2 of a query tile (qt parity)
    L.comb = L.lse2 + 2 * kT * 4;                              // A partials [2][4][128] x 8 B; B maxima [kMaxTiles][2][128] x 4 B
    L.hist = L.comb + 2 * 4 * kT * 8 + 2 * kMaxTiles * kT * 4; // [d + 1] u32 budget histogram
    L.lmax = L.hist + (uint32_t)(d + 1) * 4;                   // [4] u32: per-warp max |lse| of an item; [4] last-unit flag
    L.bars = (L.lmax + 32 + 15) & ~15u;
    L.bytes = L.bars + 512 + 1024;                             // barriers; + alignment slack
    return L;
}
}  // namespace k12

struct K12Args {
    int n, heads, items, d, dh, min_samples;   // items = B * H (b, h) pairs
    float scale;
    double scale_d, alpha;
    bool force_exact;
    const int32_t* budgets_override;   // debug hooks (mca_debug)
    const uint8_t* exact_override;
    double* cmax_out;
    double* row_m;                     // [B, H, n]
    double* row_l;
    float* lse;
    int32_t* budgets;
    uint8_t* exact;
    unsigned long long* counters;      // [0] approx cost, [1] sampled draws, [2] exact token-heads
    unsigned int* hist;                // [H, d + 1] (nullable)
    CertSink cert;                     // Eq. 9 values at an integer boundary: deferred to k2c_certify
    // Work units: items [0, items - tail_items) whole, then each of the last
    // tail_items items split into tail_parts query-tile ranges (the grid's last
    // wave). A split item's units merge their per-key maxima and max |lse| into
    // tail[slot] = [n] ordered-u32 maxima | lse max | unit counter; the last unit
    // to finish evaluates Eq. 9 and resets the slot to zero for the next launch.
    int units, tail_items, tail_parts;
    unsigned* tail;                    // [tail_items][n + 2], zero between launches
};

namespace k12 {
struct Unit {
    int it, q0, q1, slot;   // item, query tiles [q0, q1), split slot (-1: whole item)
};
__device__ __forceinline__ Unit unit_of(const K12Args& a, int k, int nt) {
    const int nfull = a.items - a.tail_items;
    if (k < nfull) return {k, 0, nt, -1};
    k -= nfull;
    const int ti = k / a.tail_parts, p = k - ti * a.tail_parts;
    return {nfull + ti, p * nt / a.tail_parts, (p + 1) * nt / a.tail_parts, ti};
}
// float <-> u32 keys whose unsigned order is the float order (0 is below every float)
__device__ __forceinline__ unsigned f32_key(float v) {
    const unsigned b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_f32(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
}  // namespace k12

// Persistent: one CTA per SM walks the items (b, h) = blockIdx.x, + gridDim.x, ...
// Every stream (TMA, the two MMA issuers, both consumer groups) runs ahead into
// the next item as far as its buffers allow, so the next item's tile loads and
// group A's first query tile overlap group B's last query tile and Eq. 9.
// Q tile t / K tile t of item i is overwritten for item i + 1 once the last
// MMA of each phase reading it completed (tile_empty1 / tile_empty2, committed
// by the phase's issuer after its last block using the tile).
__global__ void __maxnreg__(72)
    k12_fused_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k, K12Args a) {
    using namespace k12;
    using namespace mca_tc;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int n = a.n, heads = a.heads;
    const int nt = (n + kT - 1) / kT;
    const Layout L = layout(nt, a.d);
    float* s_lse2b = reinterpret_cast<float*>(smem + L.lse2);          // [2][128]
    float2* combA = reinterpret_cast<float2*>(smem + L.comb);        // [2][4][128] (query-tile parity, part)
    float* combB = reinterpret_cast<float*>(combA + 2 * 4 * kT);      // [kMaxTiles][2][128] running maxima
    unsigned int* s_hist = reinterpret_cast<unsigned int*>(smem + L.hist);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* tile_full = bars;                  // [2 * kMaxTiles]: Q tiles, then K tiles
    uint64_t* tile_empty1 = bars + 2 * kMaxTiles;   // phase 1 is done with the tile
    uint64_t* tile_empty2 = bars + 4 * kMaxTiles;   // phase 2 is done with the tile
    uint64_t* a_full = bars + 6 * kMaxTiles;     // [2] phase-1 S buffers
    uint64_t* a_empty = a_full + 2;              // [2]
    uint64_t* b_full = a_empty + 2;              // [2] phase-2 S^T buffers
    uint64_t* b_empty = b_full + 2;              // [2]
    uint64_t* comb_full = b_empty + 2;           // [2] A's partials of a query tile are in combA
    uint64_t* comb_empty = comb_full + 2;        // [2] B has read them
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(comb_empty + 2);

    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;   // uniform: see k4_apply_tf32
    const bool prof0 = MCA_K12_PROF && blockIdx.x == 0;
    griddep_trigger();   // the work-list kernels may launch (they wait for this grid to complete)
    if (prof0 && threadIdx.x == 0) g_k12_prof[0] = clock64();
    long long c_start = 0;
    if (MCA_K12_PROF && threadIdx.x == 0 && blockIdx.x < 4096) {
        unsigned int sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_k12_cta[blockIdx.x][0] = sm;
        g_k12_cta[blockIdx.x][1] = gtimer();
        c_start = clock64();
    }
    const bool use_hist = a.hist != nullptr && a.d <= 1024;

    if (threadIdx.x == 0) {
        for (int t = 0; t < 2 * nt; ++t) {
            mbar_init(tile_full + t, 1);
            mbar_init(tile_empty1 + t, 1);
            mbar_init(tile_empty2 + t, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(a_full + i, 1);
            mbar_init(a_empty + i, kAThreads / 2);   // one sub-group per buffer
            mbar_init(b_full + i, 1);
            mbar_init(b_empty + i, kBThreads);
            mbar_init(comb_full + i, kAThreads);
            mbar_init(comb_empty + i, 1);
        }
        fence_barrier_init();
    }
    if (use_hist)
        for (int i = threadIdx.x; i <= a.d; i += k12::kThreads) s_hist[i] = 0;
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // block (qt, kt) of a unit; U counts the CTA's blocks across units (S buffer
    // index and barrier parity), li its units (tile slot parity: every unit loads
    // every Q and K tile once). Phase 1: S =
    // Q_qt K_kt^T into the A buffers; phase 2: S^T = K_kt Q_qt^T into the B
    // buffers. Each stream has its own issuing thread (tcgen05.commit tracks the
    // issuing thread's MMAs), so neither waits on the other's buffer recycling.
    const uint64_t dbase = sw128_desc(smem_u32(smem), 16, 1024);
    // Whole-warp MMA streams (one elected lane issues and commits; see tc_common.cuh)
    auto issue = [&](int phase, int li, int U, int qt, int kt, const Unit& un) {
        const int sb = U & 1;
        uint64_t* full = phase ? b_full : a_full;
        uint64_t* empty = phase ? b_empty : a_empty;
        mbar_wait(empty + sb, ((U >> 1) & 1) ^ 1);
        mbar_wait(tile_full + qt, li & 1);
        mbar_wait(tile_full + nt + kt, li & 1);
        tc_fence_after();
        const uint64_t dq = desc_add(dbase, L.q + qt * kTileBytes);
        const uint64_t dk = desc_add(dbase, L.k + kt * kTileBytes);
        const uint64_t da = phase ? dk : dq, db = phase ? dq : dk;
        const uint32_t d = tmem + (uint32_t)(phase * 2 + sb) * kT;
#pragma unroll
        for (int kk = 0; kk < kDh / 16; ++kk)
            umma_f16_w(d, desc_add(da, kk * 32), desc_add(db, kk * 32), kIdesc, kk > 0 ? 1u : 0u);
        umma_commit_w(full + sb);
        if (prof0 && lane == 0 && phase == 0 && U < 32) g_k12_prof[192 + U] = clock64();
        uint64_t* tile_empty = phase ? tile_empty2 : tile_empty1;   // this phase's last read of a tile
        if (kt == nt - 1) umma_commit_w(tile_empty + qt);
        if (qt == un.q1 - 1) umma_commit_w(tile_empty + nt + kt);
        if (qt == un.q0 && kt == 0)   // a split unit's other Q tiles: loaded (one load per slot per unit), unused
            for (int t = 0; t < nt; ++t)
                if (t < un.q0 || t >= un.q1) {
                    mbar_wait(tile_full + t, li & 1);   // landed before the slot is released
                    umma_commit_w(tile_empty + t);
                }
    };
    if (warp == k12::kThreads / 32 - 1) {
        if (lane == 0) {  // ---------------- TMA: every Q and K tile of each item once
            tma_prefetch(&tm_q);
            tma_prefetch(&tm_k);
            griddep_wait();   // q, k may be the projection GEMM's output
            for (int k = blockIdx.x, li = 0; k < a.units; k += gridDim.x, ++li) {
                const int it = unit_of(a, k, nt).it;
                const int b = it / heads, h = it - b * heads;
                for (int t = 0; t < nt; ++t)
                    for (int op = 0; op < 2; ++op) {   // 0: Q tile t, 1: K tile t
                        if (li > 0) {   // both phases of the previous item are done with the slot
                            mbar_wait(tile_empty1 + op * nt + t, (li - 1) & 1);
                            mbar_wait(tile_empty2 + op * nt + t, (li - 1) & 1);
                        }
                        mbar_expect_tx(tile_full + op * nt + t, kTileBytes);
                        tma_load_3d(smem + (op ? L.k : L.q) + t * kTileBytes, op ? &tm_k : &tm_q,
                                    tile_full + op * nt + t, h * kDh, t * kT, b);
                    }
            }
        }
    } else if (warp < 2) {   // ---------------- warp 0: the phase-2 MMA stream; warp 1: phase 1
        for (int k = blockIdx.x, li = 0, ub = 0; k < a.units; k += gridDim.x, ++li) {
            const Unit un = unit_of(a, k, nt);
            for (int qt = un.q0; qt < un.q1; ++qt)
                for (int kt = 0; kt < nt; ++kt, ++ub) issue(warp == 0, li, ub, qt, kt, un);
        }
    } else if (warp < 2 + kAWarps) {
        // ---------------- group A: partial row statistics. Sub-group sub takes the
        // blocks with U & 1 == sub (S buffer sub), 64 columns [64 ch, +64) per warp.
        const int gt = threadIdx.x - 64;
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int part = gt >> 7;                  // 0..3: (sub, ch) = (part >> 1, part & 1)
        const int sub = part >> 1, ch = part & 1;
        const int row = quad * 32 + lane;          // TMEM lane = query row of the tile
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)sub * kT + (uint32_t)ch * 64u;
        const float c2 = a.scale * 1.4426950408889634f;
        for (int k = blockIdx.x, ub = 0, qb = 0; k < a.units; k += gridDim.x) {
            const Unit un = unit_of(a, k, nt);
            for (int qt = un.q0; qt < un.q1; ++qt, ub += nt, ++qb) {
                float m2 = -INFINITY, l = 0.0f;
                for (int kt = 0; kt < nt; ++kt) {
                    const int U = ub + kt;
                    if ((U & 1) != sub) continue;
                    mbar_wait(a_full + sub, (U >> 1) & 1);
                    if (prof0 && (gt & 255) == 0 && U < 32) g_k12_prof[96 + U] = clock64();
                    tc_fence_after();
#pragma unroll 1
                    for (int pc = 0; pc < 2; ++pc) {
                        uint32_t sv[32];
                        tmem_ld32(lane_base + pc * 32, sv);
                        tmem_ld_wait();
                        if (pc == 1) {
                            tc_fence_before();
                            mbar_arrive(a_empty + sub);
                        }
                        if (prof0 && (gt & 255) == 0 && U < 32) g_k12_prof[128 + 32 * pc + U] = clock64();
                        const int valid = n - (kt * kT + ch * 64 + pc * 32);   // <= 0: this piece is past n
                        float bmax = -INFINITY;
                        if (valid >= 32) {   // pairwise tree: 5 dependent levels instead of 32
                            float t16[16];
#pragma unroll
                            for (int e = 0; e < 16; ++e) t16[e] = fmaxf(__uint_as_float(sv[e]), __uint_as_float(sv[e + 16]));
#pragma unroll
                            for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
                                for (int e = 0; e < w; ++e) t16[e] = fmaxf(t16[e], t16[e + w]);
                            bmax = t16[0];
                        } else {
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (e < valid) bmax = fmaxf(bmax, __uint_as_float(sv[e]));
                        }
                        if (valid > 0) {
                            const float mn = fmaxf(m2, bmax * c2);
                            float acc0 = 0.f, acc1 = 0.f;
                            if (valid >= 32) {   // packed: one FFMA2 and one FADD2 per two scores
                                float2 acc = make_float2(0.f, 0.f);
                                const float2 cc = make_float2(c2, c2), nm = make_float2(-mn, -mn);
#pragma unroll
                                for (int e = 0; e < 32; e += 2) {
                                    const float2 x = __ffma2_rn(make_float2(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), cc, nm);
                                    acc = __fadd2_rn(acc, make_float2(ex2_approx(x.x), ex2_approx(x.y)));
                                }
                                acc0 = acc.x;
                                acc1 = acc.y;
                            } else {
#pragma unroll
                                for (int e = 0; e < 32; ++e)
                                    if (e < valid) acc0 += ex2_approx(__fmaf_rn(__uint_as_float(sv[e]), c2, -mn));
                            }
                            l = (m2 == -INFINITY ? 0.0f : l * ex2_approx(m2 - mn)) + (acc0 + acc1);
                            m2 = mn;
                        }
                    }
                    if (prof0 && (gt & 255) == 0 && U < 39) g_k12_prof[1 + U] = clock64();
                }
                // hand this row's partial (max, sum) to group B
                const int gq = qb;
                mbar_wait(comb_empty + (gq & 1), ((gq >> 1) & 1) ^ 1);
                combA[((gq & 1) * 4 + part) * kT + row] = make_float2(m2, l);
                mbar_arrive(comb_full + (gq & 1));
            }
        }
    } else {
        // ---------------- group B: lse of each query tile, per-key column maxima, Eq. 9
        const int gt = threadIdx.x - 64 - kAThreads;
        const int quad = warp & 3;
        const int half = gt >> 7;                  // columns (queries) [64 half, +64) of a block
        const int row = quad * 32 + lane;          // TMEM lane = key row of the tile
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16) + 2u * kT + (uint32_t)half * 64u;
        const float c2 = a.scale * 1.4426950408889634f;
        for (int k = blockIdx.x, ub = 0, qb = 0; k < a.units; k += gridDim.x) {
            const Unit un = unit_of(a, k, nt);
            const int it = un.it, h = it % heads;
            const size_t rbase = (size_t)it * n;
            float lmax = 0.f;                          // max |lse| of the unit's queries (certification scale)
            for (int qt = un.q0; qt < un.q1; ++qt, ub += nt, ++qb) {
                const int gq = qb;
                float* s_lse2 = s_lse2b + (gq & 1) * kT;
                mbar_wait(comb_full + (gq & 1), (gq >> 1) & 1);   // acquire: group A's partials of tile qt
                if (gt < kT) {   // combine the four partials of query row gt
                    const float2* cb = combA + (gq & 1) * 4 * kT + gt;
                    float mn = cb[0].x;
#pragma unroll
                    for (int p = 1; p < 4; ++p) mn = fmaxf(mn, cb[p * kT].x);
                    // canonical order, the even key tiles' partials first: sub-group
                    // U & 1 took them, and U of (qt, 0) is odd when nt is odd and an
                    // odd number of query tiles preceded qt on this CTA -- lse then
                    // does not depend on where the item ran
                    const int par = (ub & 1) << 1;
                    float lt = 0.f;
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        const float2 o = cb[(p ^ par) * kT];
                        lt += o.x == -INFINITY ? 0.f : o.y * ex2_approx(o.x - mn);
                    }
                    const int q = qt * kT + gt;
                    if (q < n) {
                        const float lse_nat = (mn + __log2f(lt)) * 0.6931471805599453f;
                        lmax = fmaxf(lmax, fabsf(lse_nat));
                        s_lse2[gt] = -(lse_nat * 1.4426950408889634f);   // stored negated (FFMA2 addend)
                        a.lse[rbase + q] = lse_nat;
                        a.row_m[rbase + q] = (double)mn * 0.6931471805599453;
                        a.row_l[rbase + q] = (double)lt;
                    } else {
                        s_lse2[gt] = -INFINITY;         // padded queries never win a column maximum
                    }
                }
                named_bar_sync(2, kBThreads);          // -lse2 of tile qt is in smem; the partials are read
                if (gt == 0) mbar_arrive(comb_empty + (gq & 1));
                if (prof0 && gt == 0 && gq < 32) g_k12_prof[224 + gq] = clock64();
                for (int kt = 0; kt < nt; ++kt) {
                    const int U = ub + kt, sb = U & 1;
                    // two running maxima break the dependency chain
                    float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
                    for (int pc = 0; pc < 2; ++pc) {   // 64 columns in two 32-column pieces (registers)
                        uint32_t sv[32];
                        if (pc == 0) {
                            mbar_wait(b_full + sb, (U >> 1) & 1);
                            tc_fence_after();
                        }
                        tmem_ld32(lane_base + sb * kT + pc * 32, sv);
                        tmem_ld_wait();
                        if (pc == 1) {
                            tc_fence_before();
                            mbar_arrive(b_empty + sb);
                        }
                        const int c0 = half * 64 + pc * 32;   // query (in the tile) of sv[0]
#pragma unroll
                        for (int g = 0; g < 32; g += 4) {
                            const float4 nl = *reinterpret_cast<const float4*>(s_lse2 + c0 + g);   // -lse2
                            const float2 cc = make_float2(c2, c2);
                            const float2 va = __ffma2_rn(make_float2(__uint_as_float(sv[g]), __uint_as_float(sv[g + 1])),
                                                         cc, make_float2(nl.x, nl.y));
                            const float2 vb = __ffma2_rn(make_float2(__uint_as_float(sv[g + 2]), __uint_as_float(sv[g + 3])),
                                                         cc, make_float2(nl.z, nl.w));
                            m0 = fmaxf(m0, fmaxf(va.x, va.y));   // FMNMX3
                            m1 = fmaxf(m1, fmaxf(vb.x, vb.y));
                        }
                    }
                    float* slot = combB + (kt * 2 + half) * kT + row;
                    *slot = qt == un.q0 ? fmaxf(m0, m1) : fmaxf(*slot, fmaxf(m0, m1));
                    if (prof0 && gt == 0 && U < 39) g_k12_prof[40 + U] = clock64();
                }
            }
            // ---------------- Eq. 9, one key per group-B thread
            unsigned* s_lmax = reinterpret_cast<unsigned*>(smem + L.lmax);
            if (gt < kT) {                         // the four warps that combined the lse rows
                const unsigned wm = __reduce_max_sync(0xffffffffu, __float_as_uint(lmax));
                if (lane == 0) s_lmax[gt >> 5] = wm;
            }
            named_bar_sync(2, kBThreads);          // the running maxima of this unit are final
            float item_lmax = __uint_as_float(max(max(s_lmax[0], s_lmax[1]), max(s_lmax[2], s_lmax[3])));
            unsigned* tmax = nullptr;              // split item: the merged maxima
            if (un.slot >= 0) {
                tmax = a.tail + (size_t)un.slot * (n + 2);
                for (int j = gt; j < n; j += kBThreads) {
                    const int kt = j / kT, r0 = j - kt * kT;
                    atomicMax(tmax + j, f32_key(fmaxf(combB[(kt * 2) * kT + r0], combB[(kt * 2 + 1) * kT + r0])));
                }
                if (gt == 0) atomicMax(tmax + n, __float_as_uint(item_lmax));   // >= 0: u32 order is float order
                __threadfence();
                named_bar_sync(2, kBThreads);      // this unit's maxima are visible device-wide
                if (gt == 0) s_lmax[4] = atomicAdd(tmax + n + 1, 1u) == (unsigned)(a.tail_parts - 1);
                named_bar_sync(2, kBThreads);
                if (!s_lmax[4]) continue;          // another unit of the item finishes it
                __threadfence();
                item_lmax = __uint_as_float(__ldcg(tmax + n));
            }
            unsigned long long cost = 0, samples = 0, nexact = 0;
            for (int j = gt; j < n; j += kBThreads) {
                const int kt = j / kT, r0 = j - kt * kT;
                // v = t - lse in the log2 domain, maximised over both query halves (and the item's units)
                float vmax;
                if (tmax) {
                    vmax = key_f32(__ldcg(tmax + j));
                    tmax[j] = 0u;
                } else {
                    vmax = fmaxf(combB[(kt * 2) * kT + r0], combB[(kt * 2 + 1) * kT + r0]);
                }
                const size_t t = rbase + j;
                if (a.cert.row_done) a.cert.row_done[t] = 0;   // k2c's row-statistics cache
                int r;
                bool ex;
                if (a.force_exact) {
                    r = a.d;
                    ex = true;
                } else if (a.budgets_override) {
                    r = a.budgets_override[t];
                    ex = a.exact_override[t] != 0;
                } else {
                    // cmax = max_q exp(t_qj - lse_q) = 2^vmax, evaluated in fp64
                    const double cm = exp2((double)vmax);
                    if (a.cmax_out) a.cmax_out[t] = cm;
                    budget_for(cm, n, a.alpha, a.min_samples, a.d, &r, &ex);
                    if (a.cert.list && eq9_ambiguous(cm, n, a.alpha, a.min_samples, a.d,
                                                     (double)a.cert.tau_rel *
                                                         (1.0 + fabs((double)vmax) * 0.6931471805599453 +
                                                          2.0 * (double)item_lmax))) {
                        cert_push(a.cert, (long long)t, cm, n);   // k2c re-derives it in fp64 and accounts it
                        continue;
                    }
                }
                a.budgets[t] = r;
                a.exact[t] = ex ? 1 : 0;
                if (ex) {
                    cost += 2ull * (unsigned long long)a.d * (unsigned long long)a.dh;
                    nexact += 1;
                } else {
                    cost += (unsigned long long)r * (2ull * a.dh + 3ull);
                    samples += (unsigned long long)r;
                }
                if (use_hist) atomicAdd(&s_hist[ex ? a.d : min(r, a.d - 1)], 1u);
            }
            if (a.counters) {
                for (int off = 16; off; off >>= 1) {
                    cost += __shfl_xor_sync(0xffffffffu, cost, off);
                    samples += __shfl_xor_sync(0xffffffffu, samples, off);
                    nexact += __shfl_xor_sync(0xffffffffu, nexact, off);
                }
                if (lane == 0) {
                    if (cost) atomicAdd(a.counters + 0, cost);
                    if (samples) atomicAdd(a.counters + 1, samples);
                    if (nexact) atomicAdd(a.counters + 2, nexact);
                }
            }
            named_bar_sync(2, kBThreads);          // Eq. 9 has read the maxima and the histogram is complete
            if (tmax && gt == 0) {
                tmax[n] = 0u;
                tmax[n + 1] = 0u;
            }
            if (use_hist)
                for (int i = gt; i <= a.d; i += kBThreads) {
                    const unsigned int v = s_hist[i];
                    if (v) {
                        atomicAdd(&a.hist[(size_t)h * (a.d + 1) + i], v);
                        s_hist[i] = 0;
                    }
                }
        }
        if (prof0 && gt == 0) g_k12_prof[79] = clock64();   // group B done (incl. Eq. 9)
    }
    tc_fence_before();
    __syncthreads();
    if (prof0 && threadIdx.x == 0) g_k12_prof[80] = clock64();
    if (MCA_K12_PROF && threadIdx.x == 0 && blockIdx.x < 4096) {
        g_k12_cta[blockIdx.x][2] = gtimer();
        g_k12_cta[blockIdx.x][3] = clock64() - c_start;
    }
    if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace mca_dev

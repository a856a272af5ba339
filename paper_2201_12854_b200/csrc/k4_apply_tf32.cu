// k4_apply_tf32.cu — K4 for the fp32 path on the tensor cores (3xTF32):
// y = attn . H~ (matmul, matrix.hpp:33-34) with the attention
// never materialised, as in k4_apply_tc (bf16):
//   S = q_i . k_j (3xTF32: hi.lo + lo.hi + hi.hi on the split operands K1
//       left in the workspace, fp32 accumulation in TMEM)
//   P = 2^(scale log2e S - lse2_i)   (ex2.approx.f32, the row statistics of K1)
//   O += P . H~ (3xTF32 again: P and H~ split into tf32 hi + lo parts)
// CTA = (b, h, 128-query tile); 32-key blocks, two stages of every per-block
// operand. Operands in 128B-swizzled K-major atoms of 32 fp32 (tc_common.cuh):
//   Q  [128 q x 64 d]  hi | lo, resident                              64 KB
//   K  [32 keys x 64 d] hi | lo, 2 stages                            2 x 16 KB
//   V  [64 d x 32 keys] hi | lo (H~ transposed per head, k_split_transpose_h), 2 stages  2 x 16 KB
//   P  [128 q x 32 keys] hi | lo, written by the softmax warps, 2 stages  2 x 32 KB
// TMEM: S in two 32-column buffers, O (64 columns).
// Warp 0: TMA producer; warp 1: TMEM allocator + MMA issuer; warps 2-5:
// softmax (one query row per thread) and the epilogue.
// Overlap: the TMA loads of blocks kb + 1 and kb + 2 are in flight, S(kb + 1)
// is computed while the softmax warps turn S(kb) into P(kb), and P(kb) . V(kb)
// runs while the softmax warps work on block kb + 1.
#pragma once

#include "mca_common.cuh"
#include "tc_common.cuh"

namespace mca_dev {

#ifndef MCA_K4TF_EXP
#define MCA_K4TF_EXP 0   // diagnostics: 1 = softmax stores no P (MMA + TMA only), 2 = no MMAs (softmax + TMA only)
#endif
namespace k4tf {
constexpr int kBM = 128, kBK = 32, kStages = 2;
constexpr int kOAcc = 4;   // interleaved O accumulators (TMEM columns 64 .. 319)
constexpr int kThreads = 192;
constexpr uint32_t kAtom128 = 128 * 128;     // 128 rows x 128 B
constexpr uint32_t kAtom64 = 64 * 128;       // 64 rows x 128 B
constexpr uint32_t kAtom32 = 32 * 128;       // 32 rows x 128 B
constexpr uint32_t kQBytes = 2 * 2 * kAtom128;    // 2 parts x 2 atoms (d) = 64 KB
constexpr uint32_t kKBytes = 2 * 2 * kAtom32;     // 2 parts x 2 atoms (d) = 16 KB per stage
constexpr uint32_t kVBytes = 2 * kAtom64;         // 2 parts x 1 atom (keys) = 16 KB per stage
constexpr uint32_t kPBytes = 2 * kAtom128;        // 2 parts x 1 atom (keys) = 32 KB per stage
constexpr uint32_t kSmemQ = 0, kSmemK = kQBytes, kSmemV = kSmemK + kStages * kKBytes;
constexpr uint32_t kSmemP = kSmemV + kStages * kVBytes;
constexpr uint32_t kSmemBar = kSmemP + kStages * kPBytes;
constexpr uint32_t kSmemBytes = kSmemBar + 256 + 1024;
constexpr uint32_t kIdescS = mca_tc::idesc_tf32(kBM, kBK);   // S: N = 32 keys
constexpr uint32_t kIdescO = mca_tc::idesc_tf32(kBM, kDh);   // O: N = 64 dims
}  // namespace k4tf

// 3xTF32 of one [128 x 32 kAtoms] x [N x 32 kAtoms]^T product into d: K = 8 per
// instruction, small products first (hi.lo, lo.hi, then hi.hi; see k1_scores_tc).
// Warp-wide: a / b are the descriptors of the hi parts' first atoms.
template <int kAtoms>
__device__ __forceinline__ void umma_3xtf32(uint32_t d, uint32_t idesc, uint64_t a, uint32_t a_part, uint32_t a_atom,
                                            uint64_t b, uint32_t b_part, uint32_t b_atom, bool accumulate) {
    using namespace mca_tc;
    if (MCA_K4TF_EXP == 2) return;
#pragma unroll
    for (int pr = 0; pr < 3; ++pr) {
        const uint32_t ap = pr == 1 ? a_part : 0u, bp = pr == 0 ? b_part : 0u;
#pragma unroll
        for (int at = 0; at < kAtoms; ++at)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                umma_tf32_w(d, desc_add(a, ap + at * a_atom + kk * 32), desc_add(b, bp + at * b_atom + kk * 32), idesc,
                            (accumulate || (pr | at | kk) != 0) ? 1u : 0u);
    }
}

// maps: tm_qh / tm_ql: [B][n][H*64] fp32 views, box {32, 128}; tm_kh / tm_kl:
// box {32, 32}; tm_vh / tm_vl: [B*H][64][n] fp32 (H~ transposed), box {32, 64}.
__global__ void __launch_bounds__(k4tf::kThreads, 1)
    k4_apply_tf32(const __grid_constant__ CUtensorMap tm_qh, const __grid_constant__ CUtensorMap tm_ql,
                  const __grid_constant__ CUtensorMap tm_kh, const __grid_constant__ CUtensorMap tm_kl,
                  const __grid_constant__ CUtensorMap tm_vh, const __grid_constant__ CUtensorMap tm_vl,
                  const float* __restrict__ lse, int n, int heads, float scale, float* __restrict__ y) {
    using namespace k4tf;
    using namespace mca_tc;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // per stage s: k_full, k_empty, v_full, v_empty, s_full, s_free, p_full, p_free (8 x 2), then q_full, o_full
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* k_full = bars + 0;
    uint64_t* k_empty = bars + 2;
    uint64_t* v_full = bars + 4;
    uint64_t* v_empty = bars + 6;
    uint64_t* s_full = bars + 8;
    uint64_t* s_free = bars + 10;
    uint64_t* p_full = bars + 12;
    uint64_t* p_free = bars + 14;
    uint64_t* q_full = bars + 16;
    uint64_t* o_full = bars + 17;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);
    // warp index through a shuffle: provably warp-uniform, so role branches keep
    // the MMA descriptors in uniform registers
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
    const int b = blockIdx.z, h = blockIdx.y, i0 = blockIdx.x * kBM;
    const int nblk = (n + kBK - 1) / kBK;
    const size_t bh = (size_t)b * heads + h;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 18; ++i) mbar_init(bars + i, (i >= 10 && i < 14) ? 4 : 1);   // s_free, p_full: 4 warps
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;          // S buffers: columns [0, 32), [32, 64); O_a: [64 + 64 a, 128 + 64 a)
    griddep_trigger();

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer
            griddep_wait();   // H~ (transposed) and the split q / k of this forward
            mbar_expect_tx(q_full, kQBytes);
            for (int p = 0; p < 2; ++p)
                for (int at = 0; at < 2; ++at)
                    tma_load_3d(smem + kSmemQ + p * 2 * kAtom128 + at * kAtom128, p ? &tm_ql : &tm_qh, q_full,
                                h * kDh + at * 32, i0, b);
            for (int kb = 0; kb < nblk; ++kb) {
                const int st = kb & 1;
                const uint32_t ph = (kb >> 1) & 1;
                mbar_wait(k_empty + st, ph ^ 1);
                if (MCA_K4TF_EXP == 3) {   // diagnostics: no K / V loads (MMAs on stale operands)
                    mbar_arrive(k_full + st);
                    mbar_wait(v_empty + st, ph ^ 1);
                    mbar_arrive(v_full + st);
                    continue;
                }
                mbar_expect_tx(k_full + st, kKBytes);
                for (int p = 0; p < 2; ++p)
                    for (int at = 0; at < 2; ++at)
                        tma_load_3d(smem + kSmemK + st * kKBytes + p * 2 * kAtom32 + at * kAtom32, p ? &tm_kl : &tm_kh,
                                    k_full + st, h * kDh + at * 32, kb * kBK, b);
                mbar_wait(v_empty + st, ph ^ 1);
                mbar_expect_tx(v_full + st, kVBytes);
                for (int p = 0; p < 2; ++p)
                    tma_load_3d(smem + kSmemV + st * kVBytes + p * kAtom64, p ? &tm_vl : &tm_vh, v_full + st, kb * kBK,
                                0, (int)bh);
            }
        }
    } else if (warp == 1) {   // ---------------- MMA issuer (whole warp; one elected lane issues)
        const uint64_t dq = sw128_desc(smem_u32(smem + kSmemQ), 16, 1024);
        const uint64_t dk = sw128_desc(smem_u32(smem + kSmemK), 16, 1024);
        const uint64_t dv = sw128_desc(smem_u32(smem + kSmemV), 16, 1024);
        const uint64_t dp = sw128_desc(smem_u32(smem + kSmemP), 16, 1024);
        auto issue_s = [&](int m) {   // S(m) -> TMEM buffer m & 1
            const int st = m & 1;
            const uint32_t ph = (m >> 1) & 1;
            mbar_wait(k_full + st, ph);
            mbar_wait(s_free + st, ph ^ 1);         // the softmax warps have read S(m - 2)
            tc_fence_after();
            umma_3xtf32<2>(tmem + st * kBK, kIdescS, dq, 2 * kAtom128, kAtom128, desc_add(dk, st * kKBytes),
                           2 * kAtom32, kAtom32, false);
            umma_commit_w(s_full + st);
            umma_commit_w(k_empty + st);
        };
        mbar_wait(q_full, 0);
        issue_s(0);
        for (int kb = 0; kb < nblk; ++kb) {
            if (kb + 1 < nblk) issue_s(kb + 1);   // S(kb + 1) runs while the softmax warps turn S(kb) into P(kb)
            const int st = kb & 1;
            const uint32_t ph = (kb >> 1) & 1;
            mbar_wait(p_full + st, ph);
            mbar_wait(v_full + st, ph);
            tc_fence_after();
            // block kb accumulates into O_(kb % kOAcc): kOAcc shorter fp32 accumulation chains (the
            // epilogue adds them), a ~2x smaller rounding error over long rows (n = 1000: 1.1e-5 -> ~5e-6)
            umma_3xtf32<1>(tmem + 64 + 64 * (kb % kOAcc), kIdescO, desc_add(dp, st * kPBytes), kAtom128, 0,
                           desc_add(dv, st * kVBytes),
                           kAtom64, 0, kb >= kOAcc);   // the first block of each accumulator starts it
            umma_commit_w(p_free + st);
            umma_commit_w(v_empty + st);
        }
        umma_commit_w(o_full);
    } else {   // ------------------------------- softmax + epilogue (warps 2-5)
        const int quad = warp & 3;
        const int r = quad * 32 + lane;                 // TMEM lane = query row of the tile
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
        const float c2 = scale * 1.4426950408889634f;
        const float l2 = (i0 + r < n) ? lse[bh * n + i0 + r] * 1.4426950408889634f : 0.f;
        for (int kb = 0; kb < nblk; ++kb) {
            const int st = kb & 1;
            const uint32_t ph = (kb >> 1) & 1;
            mbar_wait(s_full + st, ph);
            tc_fence_after();
            uint32_t sv[32];
            tmem_ld32(lane_base + st * kBK, sv);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_free + st);
            const int valid = min(kBK, n - kb * kBK);
            mbar_wait(p_free + st, ph ^ 1);             // P(kb - 2) . V has read this P buffer
            uint8_t* pb = smem + kSmemP + st * kPBytes;
#pragma unroll
            for (int g = 0; g < (MCA_K4TF_EXP == 1 ? 0 : 8); ++g) {               // 16-byte chunk g: keys 4 g ..
                float hi[4], lo[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int c = g * 4 + e;
                    const float p = c < valid ? ex2_approx(__fmaf_rn(__uint_as_float(sv[c]), c2, -l2)) : 0.f;
                    hi[e] = __uint_as_float(__float_as_uint(p) & 0xFFFFE000u);
                    lo[e] = p - hi[e];
                }
                const uint32_t off = sw128_offset((uint32_t)r, (uint32_t)g * 16);
                *reinterpret_cast<float4*>(pb + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<float4*>(pb + kAtom128 + off) = make_float4(lo[0], lo[1], lo[2], lo[3]);
            }
            fence_proxy_async_smem();                   // generic-proxy writes -> the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full + st);
        }
        // epilogue: O (fp32, exact 3xTF32 accumulation) -> y
        mbar_wait(o_full, 0);
        tc_fence_after();
        uint32_t ov[2][32];
        tmem_ld32(lane_base + 64, ov[0]);
        tmem_ld32(lane_base + 96, ov[1]);
        tmem_ld_wait();
#pragma unroll 1
        for (int acc = 1; acc < kOAcc && acc < nblk; ++acc) {   // fold O_1 .. O_3 into O_0
            uint32_t ow[2][32];
            tmem_ld32(lane_base + 64 + 64 * acc, ow[0]);
            tmem_ld32(lane_base + 96 + 64 * acc, ow[1]);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    ov[u][e] = __float_as_uint(__uint_as_float(ov[u][e]) + __uint_as_float(ow[u][e]));
        }
        if (i0 + r < n) {
            float4* dst = reinterpret_cast<float4*>(y + ((size_t)b * n + i0 + r) * heads * kDh + (size_t)h * kDh);
#pragma unroll
            for (int g = 0; g < 16; ++g)
                dst[g] = make_float4(__uint_as_float(ov[(4 * g) >> 5][(4 * g) & 31]),
                                     __uint_as_float(ov[(4 * g + 1) >> 5][(4 * g + 1) & 31]),
                                     __uint_as_float(ov[(4 * g + 2) >> 5][(4 * g + 2) & 31]),
                                     __uint_as_float(ov[(4 * g + 3) >> 5][(4 * g + 3) & 31]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

// H~ [B, n, H*64] fp32 -> per head transposed, split: V^T hi / lo [B*H][64][ld]
// (the K-major B operand of P . H~; ld = n rounded up to 4 for TMA's 16-byte
// stride rule). A block moves 64 tokens x 64 dims of one (b, h) with 16-byte
// loads and stores on both sides (through a padded shared tile).
// grid (ceil(n / 64), H, B), block 256.
__global__ void __launch_bounds__(256) k_split_transpose_h(const float* __restrict__ hm, int n, int ld, int heads,
                                                           float* __restrict__ vh, float* __restrict__ vl) {
    __shared__ float tile[64][65];   // tile[d][j]
    const int j0 = blockIdx.x * 64, h = blockIdx.y, b = blockIdx.z, tid = threadIdx.x;
    const size_t HD = (size_t)heads * kDh;
    const size_t bh = (size_t)b * heads + h;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int e = tid + 256 * u, jj = e >> 4, d4 = (e & 15) * 4;
        const int j = j0 + jj;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < n) v = *reinterpret_cast<const float4*>(hm + ((size_t)b * n + j) * HD + (size_t)h * kDh + d4);
        tile[d4][jj] = v.x;
        tile[d4 + 1][jj] = v.y;
        tile[d4 + 2][jj] = v.z;
        tile[d4 + 3][jj] = v.w;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int e = tid + 256 * u, d = e >> 4, j4 = (e & 15) * 4;
        if (j0 + j4 >= ld) continue;
        float v[4], hi[4], lo[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            v[q] = tile[d][j4 + q];
            hi[q] = __uint_as_float(__float_as_uint(v[q]) & 0xFFFFE000u);
            lo[q] = v[q] - hi[q];
        }
        const size_t o = (bh * kDh + d) * (size_t)ld + j0 + j4;
        *reinterpret_cast<float4*>(vh + o) = make_float4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<float4*>(vl + o) = make_float4(lo[0], lo[1], lo[2], lo[3]);
    }
}

}  // namespace mca_dev

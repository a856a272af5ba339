// k4_apply_tc.cu — K4 on the 5th-generation tensor cores: y = A . H~ for one
// (b, h, 128-query tile) per CTA (matrix.hpp:33-34 `matmul`).
//
// A is never materialised. Per 64-key block:
//   S  = Q K_blk^T                  tcgen05.mma M=128 N=64 K=64 -> TMEM (fp32)
//   P  = 2^(log2e (scale*S - lse))  8 softmax warps, 2 per TMEM lane quadrant
//                                   (lane = query row), 32 keys each; lse from
//                                   K1, so no online rescaling; two exponentials
//                                   per MUFU op (ex2.approx.f16x2), P written
//                                   fp16 into a 128B-swizzled K-major smem tile
//   O += P H~_blk                   tcgen05.mma kind::f16, fp16 x fp16, M=128 N=64 K=64 (H~ MN-major)
// Warp roles (320 threads): warp 0 TMA producers (lane 0: Q once, then a K ring
// released as soon as S is computed; lane 16: an H~ ring released after P.H~), warp 1 TMEM allocator + single-thread MMA issuer, warps 2-9
// softmax + epilogue. S is double-buffered in TMEM and P in smem; the issuer
// keeps S two blocks ahead (S(kb+2) is issued right after P(kb).H~(kb)), so the
// softmax warps always find the next S ready. 64-key blocks keep
// shared memory at ~98 KB and TMEM at 256 columns (S0 [0,64), S1 [64,128),
// O [128,192)), so two CTAs run per SM and hide each other's prologue.
#include "mca_common.cuh"
#include "tc_common.cuh"

namespace mca_dev {

namespace k4tc {
constexpr int kBM = 128, kBK = 64, kStages = 3;   // separate K and H~ rings of kStages each (2 CTAs/SM fit)
constexpr int kConsumers = 8;                        // 2 warps per TMEM lane quadrant
constexpr int kThreads = 64 + kConsumers * 32;
constexpr uint32_t kQBytes = kBM * kDh * 2;         // 16 KB: Q tile (128 x 64 bf16)
constexpr uint32_t kTileBytes = kBK * kDh * 2;       // 8 KB: one 64-key K or H~ block
constexpr uint32_t kPBytes = kBM * kBK * 2;          // 16 KB: P tile (one 64-key swizzle atom)
constexpr uint32_t kSmemQ = 0;
constexpr uint32_t kSmemK = kSmemQ + kQBytes;                        // kStages tiles
constexpr uint32_t kSmemH = kSmemK + kStages * kTileBytes;           // kStages tiles
constexpr uint32_t kSmemP = kSmemH + kStages * kTileBytes;           // 2 P tiles
constexpr uint32_t kSmemBar = kSmemP + 2 * kPBytes;
constexpr uint32_t kSmemBytes = kSmemBar + 256 + 1024;               // + alignment slack
constexpr uint32_t kIdescS = mca_tc::idesc_f16(1, 0, kBM, kBK);      // bf16, B K-major
constexpr uint32_t kOCol = 2 * kBK;                                 // TMEM: S0 [0,64), S1 [64,128), O [128,192)
constexpr uint32_t kIdescO = mca_tc::idesc_f16(0, 1, kBM, kDh);      // fp16 P x fp16 H~, B MN-major
}  // namespace k4tc

__global__ void __launch_bounds__(k4tc::kThreads, 2)
    k4_apply_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_h, const float* __restrict__ lse, int n, int heads,
                float scale, __nv_bfloat16* __restrict__ y) {
    using namespace k4tc;
    using namespace mca_tc;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* q_full = bars + 0;
    uint64_t* k_full = bars + 1;               // [kStages]  K ring: freed when S(kb) completes
    uint64_t* k_empty = k_full + kStages;      // [kStages]
    uint64_t* h_full = k_empty + kStages;      // [kStages]  H~ ring: freed when P(kb).H~(kb) completes
    uint64_t* h_empty = h_full + kStages;      // [kStages]
    uint64_t* s_full = h_empty + kStages;      // [2]
    uint64_t* s_empty = s_full + 2;            // [2]
    uint64_t* p_full = s_full + 4;             // [2]
    uint64_t* p_empty = s_full + 6;            // [2]
    uint64_t* o_full = s_full + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 9);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.z, h = blockIdx.y, m0 = blockIdx.x * kBM;
    const int nkb = (n + kBK - 1) / kBK;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(k_full + s, 1);
            mbar_init(k_empty + s, 1);
            mbar_init(h_full + s, 1);
            mbar_init(h_empty + s, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(s_empty + i, kConsumers * 32);
            mbar_init(p_full + i, kConsumers * 32);
            mbar_init(p_empty + i, 1);
        }
        mbar_init(o_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer: Q, then the K ring
            tma_prefetch(&tm_q);
            tma_prefetch(&tm_k);
            mbar_expect_tx(q_full, kQBytes);
            tma_load_3d(smem + kSmemQ, &tm_q, q_full, h * kDh, m0, b);
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kStages;
                mbar_wait(k_empty + s, ((kb / kStages) & 1) ^ 1);
                mbar_expect_tx(k_full + s, kTileBytes);
                tma_load_3d(smem + kSmemK + s * kTileBytes, &tm_k, k_full + s, h * kDh, kb * kBK, b);
            }
        } else if (lane == 16) {  // ---------------- TMA producer: the H~ ring
            tma_prefetch(&tm_h);
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % kStages;
                mbar_wait(h_empty + s, ((kb / kStages) & 1) ^ 1);
                mbar_expect_tx(h_full + s, kTileBytes);
                tma_load_3d(smem + kSmemH + s * kTileBytes, &tm_h, h_full + s, h * kDh, kb * kBK, b);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            const uint32_t q_addr = smem_u32(smem + kSmemQ);
            auto issue_pv = [&](int j) {
                const int pb = j & 1, s = j % kStages;
                mbar_wait(h_full + s, (j / kStages) & 1);
                mbar_wait(p_full + pb, (j >> 1) & 1);
                tc_fence_after();
                const uint32_t p_addr = smem_u32(smem + kSmemP + pb * kPBytes);
                const uint32_t h_addr = smem_u32(smem + kSmemH + s * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                    const uint64_t ad = sw128_desc(p_addr + kk * 32, 16, 1024);
                    const uint64_t bd = sw128_desc(h_addr + kk * 2048, kBK * 128, 1024);
                    umma_f16(tmem + kOCol, ad, bd, kIdescO, (j > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(p_empty + pb);
                umma_commit(h_empty + s);
            };
            // S runs two blocks ahead of P.H~ (as deep as the double-buffered S allows):
            // while the softmax warps exponentiate S(kb+1), S(kb+2) is already computing.
            auto issue_s = [&](int kb) {
                const int s = kb % kStages, sb = kb & 1;
                mbar_wait(k_full + s, (kb / kStages) & 1);
                mbar_wait(s_empty + sb, ((kb >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t k_addr = smem_u32(smem + kSmemK + s * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < kDh / 16; ++kk) {
                    const uint64_t ad = sw128_desc(q_addr + kk * 32, 16, 1024);
                    const uint64_t bd = sw128_desc(k_addr + kk * 32, 16, 1024);
                    umma_f16(tmem + sb * kBK, ad, bd, kIdescS, kk > 0 ? 1u : 0u);
                }
                umma_commit(s_full + sb);
                umma_commit(k_empty + s);
            };
            mbar_wait(q_full, 0);
            issue_s(0);
            if (nkb > 1) issue_s(1);
            for (int kb = 0; kb < nkb; ++kb) {
                issue_pv(kb);
                if (kb + 2 < nkb) issue_s(kb + 2);
            }
            umma_commit(o_full);
        }
    } else {  // ------------------------------- softmax + epilogue (warps 2..9)
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int half = (warp - 2) >> 2;          // keys [32*half, 32*half+32) of each block
        const int row = quad * 32 + lane;          // query row within the tile
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
        const float c = scale * 1.4426950408889634f;
        const int grow = m0 + row;
        const float lse2 = grow < n ? lse[((size_t)b * heads + h) * n + grow] * 1.4426950408889634f : 0.0f;
        for (int kb = 0; kb < nkb; ++kb) {
            const int sb = kb & 1;
            const uint32_t ph = (kb >> 1) & 1;
            mbar_wait(s_full + sb, ph);
            tc_fence_after();
            uint32_t sv[32];
            tmem_ld32(lane_base + sb * kBK + half * 32, sv);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(s_empty + sb);
            mbar_wait(p_empty + sb, ph ^ 1);
            // this warp's 32 keys are chunks [4*half, 4*half+4) of the P tile's 128-byte rows
            uint8_t* pt = smem + kSmemP + sb * kPBytes;
            const int kbase = kb * kBK + half * 32;
            const int valid = n - kbase;          // keys >= n contribute nothing
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {       // 16-byte chunks of 8 keys
                uint32_t pk[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int col = ch * 8 + 2 * e;
                    // exponent in fp32, 2^x of the pair in one fp16x2 MUFU op; keys past n
                    // get -inf (2^-inf = 0)
                    float x0 = __fmaf_rn(__uint_as_float(sv[col]), c, -lse2);
                    float x1 = __fmaf_rn(__uint_as_float(sv[col + 1]), c, -lse2);
                    if (col >= valid) x0 = -INFINITY;
                    if (col + 1 >= valid) x1 = -INFINITY;
                    pk[e] = ex2_f16x2(pack_f16x2(x0, x1));
                }
                *reinterpret_cast<uint4*>(pt + sw128_offset(row, (half * 4 + ch) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
            fence_proxy_async_smem();
            mbar_arrive(p_full + sb);
        }
        // epilogue: O (fp32, TMEM cols 256..319) -> bf16 -> y; each half writes 32 columns
        mbar_wait(o_full, 0);
        tc_fence_after();
        uint32_t ov[32];
        tmem_ld32(lane_base + kOCol + half * 32, ov);
        tmem_ld_wait();
        if (grow < n) {
            __nv_bfloat16* dst = y + ((size_t)b * n + grow) * (size_t)heads * kDh + (size_t)h * kDh + half * 32;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                uint32_t pk[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    pk[e] = pack_bf16x2(__uint_as_float(ov[g * 8 + 2 * e]), __uint_as_float(ov[g * 8 + 2 * e + 1]));
                reinterpret_cast<uint4*>(dst)[g] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<256>(tmem);
}

}  // namespace mca_dev

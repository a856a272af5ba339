// k4_apply_tc.cu — K4 on the 5th-generation tensor cores: y = A . H~ for one
// (b, h, 128-query tile) per CTA (matrix.hpp:33-34 `matmul`).
//
// A is never materialised. Per 64-key block:
//   S  = Q K_blk^T                  tcgen05.mma M=128 N=64 K=64, A = Q from TMEM -> S in TMEM (fp32)
//   P  = 2^(log2e (scale*S - lse))  8 softmax warps, 2 per TMEM lane quadrant
//                                   (lane = query row), 32 keys each; lse from
//                                   K1, so no online rescaling; P is written
//                                   back into TMEM as fp16 over the S columns
//                                   the warp just read
//   O += P H~_blk                   tcgen05.mma kind::f16, A = P from TMEM, B = H~ (MN-major smem)
// Only K and H~ blocks pass through shared memory (TMA rings); Q and P live in
// tensor memory, which is what keeps this kernel off the shared-memory
// bandwidth ceiling (an smem P tile costs a store and a tensor-core read of
// 16 KB per block, Q another 16 KB read per block).
// S/P buffers: S(kb) and P(kb) share TMEM columns [64 (kb&1), +64); the
// issuer puts S(kb+2) into that buffer only after P(kb).H~ was issued (the
// tensor pipe executes one thread's MMAs in order), and the softmax warps
// overwrite it with P(kb+2) only after S(kb+2) completed, so no buffer-empty
// barriers are needed.
// Persistent: two CTAs per SM walk tiles t = blockIdx.x + i * gridDim.x. TMEM
// and barriers are set up once; block numbering continues across tiles, so the
// K / H~ rings prefetch the next tile while this one computes, the next tile's
// Q is loaded during the last block and its first S MMAs run during this
// tile's epilogue (O is handed back through o_empty before the next P.H~).
// Warp roles (320 threads): warp 0 TMA producers (lane 0: K ring, lane 16: H~
// ring), warp 1 TMEM allocator + single-thread MMA issuer, warps 2-9 load Q
// into TMEM, then softmax and the epilogue. TMEM (256 columns, two CTAs per
// SM): S/P0 [0,64), S/P1 [64,128), O [128,192), Q [192,224).
#include "k4o_overflow.cu"
#include "mca_common.cuh"
#include "tc_common.cuh"

#ifndef MCA_K4_STAGES
#define MCA_K4_STAGES 4
#endif
#ifndef MCA_K4_EXP
#define MCA_K4_EXP 0   // diagnostics: 1 = no exponentials in the softmax warps, 2 = no MMAs
#endif

namespace mca_dev {

#ifndef MCA_K4_QAHEAD
#define MCA_K4_QAHEAD 2   // blocks before the last at which the next tile's Q loads are issued
#endif
#ifndef MCA_K4_PROF
#define MCA_K4_PROF 0
#endif
// Diagnostics (build with EXTRA=-DMCA_K4_PROF=1): clock64 stamps of the first
// CTA's softmax thread 0 into this device buffer.
__device__ long long g_k4_prof[MCA_K4_PROF ? 64 : 1];

namespace k4tc {
constexpr int kBM = 128, kBK = 64, kStages = MCA_K4_STAGES;   // separate K and H~ rings of kStages each
constexpr int kConsumers = 8;                        // 2 warps per TMEM lane quadrant
constexpr int kThreads = 64 + kConsumers * 32;
constexpr uint32_t kTileBytes = kBK * kDh * 2;       // 8 KB: one 64-key K or H~ block
constexpr uint32_t kSmemK = 0;                                       // kStages tiles
constexpr uint32_t kSmemH = kSmemK + kStages * kTileBytes;           // kStages tiles
constexpr uint32_t kSmemBar = kSmemH + kStages * kTileBytes;
constexpr uint32_t kSmemBytes = kSmemBar + 256 + 1024;               // + alignment slack
constexpr uint32_t kIdescS = mca_tc::idesc_f16(1, 0, kBM, kBK);      // bf16 Q (TMEM) x bf16 K, B K-major
constexpr uint32_t kIdescO = mca_tc::idesc_f16(0, 1, kBM, kDh);      // fp16 P (TMEM) x fp16 H~, B MN-major
constexpr uint32_t kOCol = 2 * kBK;                                  // O [128,192)
constexpr uint32_t kQCol = kOCol + kDh;                              // Q [192,224): 64 bf16 per lane
#ifndef MCA_K4_POLY
#define MCA_K4_POLY 4
#endif
constexpr int kPolyPairs = MCA_K4_POLY;   // per thread and block: pairs exponentiated on the FMA pipe (of 16)
}  // namespace k4tc

// TMEM column of P's K-step kk (16 keys) in S/P buffer sb: the warp owning keys
// [32 half, 32 half + 32) wrote them to the first 16 of its 32 S columns.
__device__ __forceinline__ uint32_t k4_p_col(int sb, int kk) {
    return (uint32_t)(sb * k4tc::kBK + 32 * (kk >> 1) + 8 * (kk & 1));
}

__global__ void __launch_bounds__(k4tc::kThreads, 2)
    k4_apply_tc(const __nv_bfloat16* __restrict__ q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_h, const float* __restrict__ lse, int n, int heads,
                int batch, float scale, __nv_bfloat16* __restrict__ y, const K4oArgs oa,
                unsigned long long* __restrict__ done_ctas) {
    using namespace k4tc;
    using namespace mca_tc;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* q_full = bars + 0;               // softmax warps -> issuer: the tile's Q is in TMEM
    uint64_t* o_empty = bars + 1;              // softmax warps -> issuer: the previous tile's O was read out
    uint64_t* k_full = bars + 2;               // [kStages]  K ring: freed when S(kb) completes
    uint64_t* k_empty = k_full + kStages;      // [kStages]
    uint64_t* h_full = k_empty + kStages;      // [kStages]  H~ ring: freed when P(kb).H~(kb) completes
    uint64_t* h_empty = h_full + kStages;      // [kStages]
    uint64_t* s_full = h_empty + kStages;      // [2]
    uint64_t* p_full = s_full + 2;             // [2]
    uint64_t* o_full = s_full + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 5);

    if (MCA_K4_PROF && blockIdx.x == 0 && threadIdx.x == 64) g_k4_prof[60] = clock64();
    griddep_trigger();
    // Q and K are inputs: their loads and the first S MMAs may run while the
    // encoders drain; lse (score pass) and H~ (encoders) are read after griddep_wait()
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;   // uniform: see k4_apply_tf32
    const int nmt = (n + kBM - 1) / kBM;                   // query tiles per (b, h)
    const int nkb = (n + kBK - 1) / kBK;
    const int ntiles = batch * heads * nmt;
    const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto tile_coords = [&](int i, int& b, int& h, int& m0) {   // tile i of this CTA
        const int t = (int)blockIdx.x + i * (int)gridDim.x;
        const int mt = t % nmt, bh = t / nmt;
        h = bh % heads;
        b = bh / heads;
        m0 = mt * kBM;
    };

    if (threadIdx.x == 0) {
        mbar_init(q_full, kConsumers * 32);
        mbar_init(o_empty, kConsumers * 32);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(k_full + s, 1);
            mbar_init(k_empty + s, 1);
            mbar_init(h_full + s, 1);
            mbar_init(h_empty + s, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(p_full + i, kConsumers * 32);
        }
        mbar_init(o_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // Blocks are numbered across the CTA's tiles (g = i * nkb + kb), so the rings,
    // S/P buffers and their phases simply continue from one tile to the next.
    if (warp == 0) {
        if (lane == 0 || lane == 16) {  // ---------------- TMA producers: lane 0 the K ring, lane 16 the H~ ring
            const CUtensorMap* tm = lane == 0 ? &tm_k : &tm_h;
            uint64_t* full = lane == 0 ? k_full : h_full;
            uint64_t* empty = lane == 0 ? k_empty : h_empty;
            const uint32_t base = lane == 0 ? kSmemK : kSmemH;
            tma_prefetch(tm);
            if (lane == 16) griddep_wait();   // H~ is the encoders' output
            for (int i = 0, g = 0; i < my_tiles; ++i) {
                int b, h, m0;
                tile_coords(i, b, h, m0);
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int s = g % kStages;
                    mbar_wait(empty + s, ((g / kStages) & 1) ^ 1);
                    mbar_expect_tx(full + s, kTileBytes);
                    tma_load_3d(smem + base + s * kTileBytes, tm, full + s, h * kDh, kb * kBK, b);
                }
            }
        }
    } else if (warp == 1) {   // ---------------- MMA issuer (whole warp; one elected lane issues)
        const uint64_t dk0 = sw128_desc(smem_u32(smem + kSmemK), 16, 1024);
        const uint64_t dh0 = sw128_desc(smem_u32(smem + kSmemH), kBK * 128, 1024);
        auto issue_s = [&](int g) {
            const int s = g % kStages, sb = g & 1;
            mbar_wait(k_full + s, (g / kStages) & 1);
            tc_fence_after();
            const uint64_t dk = desc_add(dk0, s * kTileBytes);
#pragma unroll
            for (int kk = 0; kk < kDh / 16; ++kk)
                if (MCA_K4_EXP != 2)   // diagnostics: 2 = no MMAs
                    umma_f16_ts_w(tmem + sb * kBK, tmem + kQCol + kk * 8, desc_add(dk, kk * 32), kIdescS, kk > 0 ? 1u : 0u);
            umma_commit_w(s_full + sb);
            umma_commit_w(k_empty + s);
        };
        auto issue_pv = [&](int g, bool first) {
            const int s = g % kStages, sb = g & 1;
            mbar_wait(p_full + sb, (g >> 1) & 1);
            mbar_wait(h_full + s, (g / kStages) & 1);
            tc_fence_after();
            const uint64_t dh = desc_add(dh0, s * kTileBytes);
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
                if (MCA_K4_EXP != 2)
                umma_f16_ts_w(tmem + kOCol, tmem + k4_p_col(sb, kk), desc_add(dh, kk * 2048), kIdescO,
                              (!first || kk > 0) ? 1u : 0u);
            umma_commit_w(h_empty + s);
        };
        for (int i = 0; i < my_tiles; ++i) {
            const int g0 = i * nkb;
            mbar_wait(q_full, i & 1);
            tc_fence_after();
            // S runs two blocks ahead of P.H~ (S(kb+2) goes into the buffer P(kb) just left)
            issue_s(g0);
            if (nkb > 1) issue_s(g0 + 1);
            mbar_wait(o_empty, (i & 1) ^ 1);   // the previous tile's O has been read out
            for (int kb = 0; kb < nkb; ++kb) {
                issue_pv(g0 + kb, kb == 0);
                if (kb + 2 < nkb) issue_s(g0 + kb + 2);
            }
            umma_commit_w(o_full);
        }
    } else {  // ------------------------------- Q -> TMEM, softmax, epilogue (warps 2..9)
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int half = (warp - 2) >> 2;          // keys [32*half, 32*half+32) of each block; Q dims likewise
        const int row = quad * 32 + lane;          // query row within the tile
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
        const float c = scale * 1.4426950408889634f;
        const size_t HD = (size_t)heads * kDh;
        const bool prof = MCA_K4_PROF && blockIdx.x == 0 && warp == 2 && lane == 0;
        // this thread's 32 Q values (64 bytes) of tile i and its row's lse (log2 domain)
        uint32_t qv[16];
        float lse_next = 0.f;   // raw: scaled at the next tile's start, so the load overlaps the last block
        bool waited = false;
        auto load_q = [&](int i) {
            int b, h, m0;
            tile_coords(i, b, h, m0);
            const int grow = m0 + row;
            if (i < my_tiles && grow < n) {
                const uint4* src = reinterpret_cast<const uint4*>(q + ((size_t)b * n + grow) * HD + (size_t)h * kDh + 32 * half);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint4 t = __ldg(src + u);
                    qv[4 * u] = t.x;
                    qv[4 * u + 1] = t.y;
                    qv[4 * u + 2] = t.z;
                    qv[4 * u + 3] = t.w;
                }
                if (!waited) {   // lse is the score pass's output
                    griddep_wait();
                    waited = true;
                }
                lse_next = lse[((size_t)b * heads + h) * n + grow];
            } else {
#pragma unroll
                for (int u = 0; u < 16; ++u) qv[u] = 0u;
                lse_next = 0.f;
            }
        };
        auto publish_q = [&]() {   // Q registers -> TMEM columns kQCol + [16 half, 16 half + 16)
            tmem_st16(lane_base + kQCol + 16 * half, qv);
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(q_full);
        };
        load_q(0);
        publish_q();
        for (int i = 0; i < my_tiles; ++i) {
            int b, h, m0;
            tile_coords(i, b, h, m0);
            const int grow = m0 + row;
            const float lse2 = lse_next * 1.4426950408889634f;
            const int g0 = i * nkb;
            if (prof && i == 1) g_k4_prof[0] = clock64();
            for (int kb = 0; kb < nkb; ++kb) {
                const int g = g0 + kb, sb = g & 1;
                if (kb == (nkb > MCA_K4_QAHEAD ? nkb - 1 - MCA_K4_QAHEAD : 0))
                    load_q(i + 1);   // next tile's Q (and lse) in flight during the tile's last blocks
                mbar_wait(s_full + sb, (g >> 1) & 1);
                if (prof && i == 1 && kb < 16) g_k4_prof[1 + 3 * kb] = clock64();
                tc_fence_after();
                const uint32_t col = lane_base + sb * kBK + 32 * half;
                uint32_t sv[32];
                tmem_ld32(col, sv);
                tmem_ld_wait();
                if (prof && i == 1 && kb < 16) g_k4_prof[2 + 3 * kb] = clock64();
                // P = 2^(S c - lse2) as fp16 pairs (two exponentials per ex2.approx.f16x2);
                // keys past n get 2^-inf = 0
                uint32_t pk[16];
                const int valid = n - (kb * kBK + 32 * half);
                if (MCA_K4_EXP == 1) {   // diagnostics: no exponentials (P = S bits)
#pragma unroll
                    for (int e = 0; e < 16; ++e) pk[e] = sv[2 * e] ^ sv[2 * e + 1];
                } else if (valid >= 32) {
                    // the MUFU is this loop's bound: kPolyPairs of the 16 pairs take the FMA-pipe exp2
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const float2 xv = __ffma2_rn(make_float2(__uint_as_float(sv[2 * e]), __uint_as_float(sv[2 * e + 1])),
                                                     make_float2(c, c), make_float2(-lse2, -lse2));
                        if (e < kPolyPairs) {
                            const float2 pv = ex2_poly2(xv);
                            pk[e] = pack_f16x2(pv.x, pv.y);
                        } else {
                            pk[e] = ex2_f16x2(pack_f16x2(xv.x, xv.y));
                        }
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        float x0 = __fmaf_rn(__uint_as_float(sv[2 * e]), c, -lse2);
                        float x1 = __fmaf_rn(__uint_as_float(sv[2 * e + 1]), c, -lse2);
                        if (2 * e >= valid) x0 = -INFINITY;
                        if (2 * e + 1 >= valid) x1 = -INFINITY;
                        pk[e] = ex2_f16x2(pack_f16x2(x0, x1));
                    }
                }
                tmem_st16(col, pk);
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(p_full + sb);
                if (prof && i == 1 && kb < 16) g_k4_prof[3 + 3 * kb] = clock64();
            }
            // all of tile i's S are consumed, so Q may be replaced: the issuer starts
            // tile i+1's S while this tile's epilogue runs
            if (i + 1 < my_tiles) publish_q();
            // epilogue: O (fp32, TMEM cols 128..191) -> bf16 -> y; each half writes 32 columns
            mbar_wait(o_full, i & 1);
            if (prof && i == 1) g_k4_prof[50] = clock64();
            tc_fence_after();
            uint32_t ov[32];
            tmem_ld32(lane_base + kOCol + half * 32, ov);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(o_empty);
            if (grow < n) {
                __nv_bfloat16* dst = y + ((size_t)b * n + grow) * HD + (size_t)h * kDh + half * 32;
#pragma unroll
                for (int gq = 0; gq < 4; ++gq) {
                    uint32_t pk[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        pk[e] = pack_bf16x2(__uint_as_float(ov[gq * 8 + 2 * e]), __uint_as_float(ov[gq * 8 + 2 * e + 1]));
                    reinterpret_cast<uint4*>(dst)[gq] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
            }
            if (prof && i == 1) g_k4_prof[51] = clock64();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<256>(tmem);
    // fp16 range guard (k4o_overflow.cu): the last CTA to finish adds P[:, j] H~_j for
    // the encodings the encoders queued (normally none: one atomic per CTA)
    if (done_ctas) {
        int* s_last = reinterpret_cast<int*>(smem);
        if (threadIdx.x == 0) {
            __threadfence();
            s_last[0] = atomicAdd(done_ctas, 1ull) == (unsigned long long)gridDim.x - 1;
        }
        __syncthreads();
        if (s_last[0]) {
            __threadfence();
            const unsigned long long cnt = *(volatile const unsigned long long*)oa.ovf.count;
            if (cnt > (unsigned long long)oa.ovf.cap) __trap();
            if (cnt) ovf_fixup<false>(oa, cnt, 0, 1, reinterpret_cast<float*>(smem + 1024),
                                      reinterpret_cast<float*>(smem + 2048));
        }
    }
}

}  // namespace mca_dev

// k3b_exact_tc.cu — exact-branch encodings on the tensor cores (bf16):
// H~[j] = X[j] . W_h for the token-heads Eq. 9 clamps to the exact branch
// (SPEC.md:309, 348). Those are ~6% of token-heads at BERT shapes, but each is
// a full d_in x 64 dot product, so as CUDA-core work they rival the whole
// sampled encoding; here they are one small GEMM per head over K2's exact list.
//
// Grid (G, heads), persistent: CTA x of head h walks the head's tiles of 128
// listed tokens x, x + G, ... (the exact count is device-side, so the host
// sizes G for one wave and idle CTAs exit at once).
//   A = X rows of the 128 listed tokens  [128 x d_in], K-major, gathered with
//       16-byte cp.async into 128B-swizzled K chunks of 64
//   B = W_h                              [d_in x 64], MN-major chunks of 64 rows
//   D = tcgen05.mma M=128 N=64 K=16 (x4 per chunk), fp32 in TMEM (64 columns)
// Warps 0-3: producers (cp.async of A and B, 4-stage ring) and then the
// epilogue (TMEM -> fp16 -> H~ rows); warp 4: TMEM allocator + MMA issuer.
#include "mca_common.cuh"
#include "tc_common.cuh"

namespace mca_dev {

namespace k3btc {
constexpr int kBM = 128, kBK = 64, kStages = 4;
constexpr int kThreads = 160;
constexpr uint32_t kABytes = kBM * kBK * 2;          // 16 KB
constexpr uint32_t kBBytes = kBK * kDh * 2;          // 8 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr uint32_t kSmemBar = kStages * kStageBytes;
constexpr uint32_t kSmemBytes = kSmemBar + 128 + 1024;
constexpr uint32_t kIdesc = mca_tc::idesc_f16(1, 1, kBM, kDh);   // bf16, B MN-major
}  // namespace k3btc

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_zero16(uint32_t dst, const void* any_valid) {   // src-size 0: zeros
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;" ::"r"(dst), "l"(any_valid) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

#ifndef MCA_K3B_PROF
#define MCA_K3B_PROF 0
#endif
// Diagnostics (EXTRA=-DMCA_K3B_PROF=1): CTA (0, 0)'s clock64 at entry, after the
// dependency wait, per chunk landed / MMA issued, epilogue start and end.
__device__ long long g_k3b_prof[MCA_K3B_PROF ? 64 : 1];

__global__ void __launch_bounds__(k3btc::kThreads, 2) k3b_exact_tc(K3Args a) {
    using namespace k3btc;
    using namespace mca_tc;
    const int h = blockIdx.y;
    const bool prof = MCA_K3B_PROF && blockIdx.x == 0 && blockIdx.y == 0;
    if (prof && threadIdx.x == 0) g_k3b_prof[0] = clock64();
    griddep_trigger();
    // No dependency wait up front: the exact lists come from the scan, which completed
    // before the sampled encoder K3 (the PDL predecessor) let this grid launch (K3
    // triggers only after its own wait), and the two encoders write disjoint rows of
    // H~, so these CTAs run in K3's tail. Every CTA waits for K3 before it exits, so
    // K4 (which waits for this grid) sees all of H~.
    if (prof && threadIdx.x == 0) g_k3b_prof[1] = clock64();
    const int ne = a.counts[2 * h + 1];
    if ((int)blockIdx.x * kBM >= ne) {   // uniform early exit, before any barrier / TMEM use
        griddep_wait();
        return;
    }
    if (a.dense_min > 0) {   // the dense X W_V GEMM encoded every exact token-head (kp_project_tc's gate)
        long ex = 0;
        for (int hh = 0; hh < a.heads; ++hh) ex += a.counts[2 * hh + 1];
        if (ex >= a.dense_min) {
            griddep_wait();
            return;
        }
    }
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* full = bars;               // [kStages], 128 producer arrivals
    uint64_t* empty = bars + kStages;    // [kStages], MMA commit
    uint64_t* acc_full = bars + 2 * kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 1);
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;   // uniform: see k4_apply_tf32
    const int d_in = a.d_in, n = a.n;
    const int nchunks = (d_in + kBK - 1) / kBK;
    const size_t HD = (size_t)a.heads * kDh;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full + s, 128);
            mbar_init(empty + s, 1);
        }
        mbar_init(acc_full, 1);
        fence_barrier_init();
    }
    if (warp == 4) tmem_alloc<64>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    int it = 0;
    for (int tile = blockIdx.x; tile * kBM < ne; tile += gridDim.x, ++it) {
        const int g0 = it * nchunks;
        if (warp < 4) {
            // ---------------- producers: thread t owns A row t (one token) and 4 16-byte pieces of B
            const int t = threadIdx.x;
            const int idx = tile * kBM + t;
            const int bj = idx < ne ? a.exact_list[(size_t)h * a.tokens + idx] : -1;   // (b << 16) | j
            const size_t tok = bj < 0 ? 0 : (size_t)(bj >> 16) * n + (bj & 0xFFFF);
            const __nv_bfloat16* wh = reinterpret_cast<const __nv_bfloat16*>(a.wv) + (size_t)h * kDh;
            // A's gather is warp-cooperative: per chunk, lanes 8k..8k+7 copy one row's
            // 128 bytes (one coalesced line request) instead of each thread copying its
            // own row in 16-byte pieces (eight requests per line: the gather was bound
            // by L2 request throughput). Lane l covers rows 32 warp + 4 j + (l >> 3).
            const __nv_bfloat16* grow[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int r = 32 * warp + 4 * j + (lane >> 3), gi = tile * kBM + r;
                const int gbj = gi < ne ? a.exact_list[(size_t)h * a.tokens + gi] : -1;
                grow[j] = gbj < 0 ? nullptr
                                  : reinterpret_cast<const __nv_bfloat16*>(a.x) +
                                        ((size_t)(gbj >> 16) * n + (gbj & 0xFFFF)) * d_in;
            }
            auto issue = [&](int c, int s) {
                const uint32_t sa = smem_u32(smem + s * kStageBytes);
                const uint32_t sb = sa + kABytes;
                const int k0 = c * kBK;
                const int q = lane & 7;                // A: this lane's 16-byte piece of 8 rows
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int r = 32 * warp + 4 * j + (lane >> 3);
                    const uint32_t dst = sa + sw128_offset(r, q * 16);
                    if (grow[j] && k0 + q * 8 + 8 <= d_in) cp_async16(dst, grow[j] + k0 + q * 8);
                    else cp_async_zero16(dst, a.wv);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {          // B: 64 rows x 8 pieces; thread t takes 4
                    const int piece = t * 4 + q, r = piece >> 3, p8 = piece & 7;
                    const uint32_t dst = sb + sw128_offset(r, p8 * 16);
                    if (k0 + r < d_in) cp_async16(dst, wh + (size_t)(k0 + r) * HD + p8 * 8);
                    else cp_async_zero16(dst, a.wv);
                }
                cp_async_commit();
            };
            // prologue: kStages - 1 chunks in flight
            // ring slots / parities continue across tiles: chunk c of this tile is global chunk g0 + c
            for (int c = 0; c < kStages - 1; ++c)
                if (c < nchunks) {
                    const int g = g0 + c;
                    mbar_wait(empty + g % kStages, ((g / kStages) & 1) ^ 1);
                    issue(c, g % kStages);
                } else {
                    cp_async_commit();
                }
            for (int c = 0; c < nchunks; ++c) {
                const int cn = c + kStages - 1;
                if (cn < nchunks) {
                    const int g = g0 + cn;
                    mbar_wait(empty + g % kStages, ((g / kStages) & 1) ^ 1);
                    issue(cn, g % kStages);
                } else {
                    cp_async_commit();
                }
                cp_async_wait<kStages - 1>();          // chunk c has landed (this thread's copies)
                fence_proxy_async_smem();               // make them visible to the tensor core (async proxy)
                mbar_arrive(full + (g0 + c) % kStages);
                if (prof && threadIdx.x == 0 && it == 0 && c < 16) g_k3b_prof[2 + c] = clock64();
            }
            // ---------------- epilogue: TMEM row t -> bf16 -> H~
            mbar_wait(acc_full, it & 1);
            if (prof && threadIdx.x == 0 && it == 0) g_k3b_prof[40] = clock64();
            tc_fence_after();
            uint32_t v[2][32];
            const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
            tmem_ld32(lane_base, v[0]);
            tmem_ld32(lane_base + 32, v[1]);
            tmem_ld_wait();
            if (bj >= 0) {
                __half* dst = reinterpret_cast<__half*>(a.h_out) + tok * HD + (size_t)h * kDh;   // H~ is fp16
                const long long tokh = ((long long)(bj >> 16) * a.heads + h) * n + (bj & 0xFFFF);
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    float f[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[(g * 8 + e) >> 5][(g * 8 + e) & 31]);
                    f16_guard8(a.ovf, tokh, g, f);    // fp16 range guard (mca_common.cuh)
                    uint32_t pk[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) pk[e] = pack_f16x2(f[2 * e], f[2 * e + 1]);
                    reinterpret_cast<uint4*>(dst)[g] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                if (a.draws_out) {                     // exact token-heads draw nothing
                    const size_t tokh = ((size_t)(bj >> 16) * a.heads + h) * n + (bj & 0xFFFF);
                    for (int k = 0; k < a.draws_stride; ++k) a.draws_out[tokh * a.draws_stride + k] = -1;
                }
            }
        } else if (lane == 0) {
            // ---------------- MMA issuer
            for (int c = 0; c < nchunks; ++c) {
                const int g = g0 + c, s = g % kStages;
                mbar_wait(full + s, (g / kStages) & 1);
                if (prof && it == 0 && c < 16) g_k3b_prof[20 + c] = clock64();
                tc_fence_after();
                const uint32_t sa = smem_u32(smem + s * kStageBytes);
                const uint32_t sb = sa + kABytes;
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk)
                    umma_f16(tmem, sw128_desc(sa + kk * 32, 16, 1024), sw128_desc(sb + kk * 2048, 8192, 1024), kIdesc,
                             (c > 0 || kk > 0) ? 1u : 0u);
                umma_commit(empty + s);
            }
            umma_commit(acc_full);
        }
        tc_fence_before();
        __syncthreads();   // the accumulator is read out before the next tile's MMAs overwrite it
        tc_fence_after();
    }
    tc_fence_before();
    __syncthreads();
    if (prof && threadIdx.x == 0) g_k3b_prof[41] = clock64();
    if (warp == 4) tmem_dealloc<64>(tmem);
    griddep_wait();   // K3 has finished too: K4 may read every row of H~
}

}  // namespace mca_dev

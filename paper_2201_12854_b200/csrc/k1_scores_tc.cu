// k1_scores_tc.cu — K1 on the 5th-generation tensor cores: the score pass of
// attention_matrix + col_max (matrix.hpp:46-53) for one
// (b, h, 128-query tile) per CTA, bf16 inputs.
//
//   S_kb = Q K_kb^T     tcgen05.mma M=128 N=128 K=64 into TMEM (fp32), issued by
//                       one thread; Q and K tiles arrive by TMA (128B swizzle)
//   sweep 1 (per row):  online m = max t, l = sum exp(t - m), t = scale*S, in
//                       the log2 domain with ex2.approx (one TMEM lane per row)
//   sweep 2 (per col):  v = t - m - log l; warp butterfly max (reduce-scatter),
//                       cross-warp max in smem, then the winning row is found by
//                       exact comparison and packed into the argmax key that K2
//                       re-evaluates in fp64 (k1_scores_simt.cu explains the key)
// For n <= 512 every S block stays resident in TMEM (4 x 128 columns), so
// sweep 2 re-reads TMEM instead of recomputing; for n > 512 the K blocks stream
// twice through a 4-stage TMA ring and S is recomputed in sweep 2.
// Warp roles (192 threads): 0 TMA producer, 1 TMEM allocator + MMA issuer,
// 2-5 softmax / column reduction.
#include "mca_common.cuh"
#include "tc_common.cuh"

namespace mca_dev {

namespace k1tc {
constexpr int kBM = 128, kBK = 128, kBufs = 4;
constexpr int kThreads = 192;
constexpr uint32_t kTileBytes = 128 * kDh * 2;                 // 16 KB
constexpr uint32_t kSmemQ = 0;
constexpr uint32_t kSmemK = kTileBytes;                         // kBufs tiles
constexpr uint32_t kSmemRed = kSmemK + kBufs * kTileBytes;      // [4][128] f32 warp maxima
constexpr uint32_t kSmemColM = kSmemRed + 4 * 128 * 4;          // [128] f32
constexpr uint32_t kSmemWin = kSmemColM + 128 * 4;              // [128] i32
constexpr uint32_t kSmemBar = kSmemWin + 128 * 4;
constexpr uint32_t kSmemBytes = kSmemBar + 256 + 1024;
constexpr uint32_t kIdescS = mca_tc::idesc_f16(1, 0, kBM, kBK);
}  // namespace k1tc

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__global__ void __launch_bounds__(k1tc::kThreads, 1)
    k1_scores_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k, int n,
                 int heads, float scale, double* __restrict__ row_m, double* __restrict__ row_l,
                 float* __restrict__ lse_out, unsigned long long* __restrict__ colkey) {
    using namespace k1tc;
    using namespace mca_tc;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;            // [kBufs]
    uint64_t* kv_empty = kv_full + kBufs;    // [kBufs]
    uint64_t* s_full = kv_empty + kBufs;     // [kBufs]
    uint64_t* s_empty = s_full + kBufs;      // [kBufs]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_empty + kBufs);
    float* red = reinterpret_cast<float*>(smem + kSmemRed);
    float* colM = reinterpret_cast<float*>(smem + kSmemColM);
    int* win = reinterpret_cast<int*>(smem + kSmemWin);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.z, h = blockIdx.y, m0 = blockIdx.x * kBM;
    const int nkb = (n + kBK - 1) / kBK;
    const bool resident = nkb <= kBufs;
    const int items = resident ? nkb : 2 * nkb;   // S blocks the tensor core produces

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < kBufs; ++s) {
            mbar_init(kv_full + s, 1);
            mbar_init(kv_empty + s, 1);
            mbar_init(s_full + s, 1);
            mbar_init(s_empty + s, 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            tma_prefetch(&tm_q);
            tma_prefetch(&tm_k);
            mbar_expect_tx(q_full, kTileBytes);
            tma_load_3d(smem + kSmemQ, &tm_q, q_full, h * kDh, m0, b);
            for (int i = 0; i < items; ++i) {
                const int s = i % kBufs;
                mbar_wait(kv_empty + s, ((i / kBufs) & 1) ^ 1);
                mbar_expect_tx(kv_full + s, kTileBytes);
                tma_load_3d(smem + kSmemK + s * kTileBytes, &tm_k, kv_full + s, h * kDh, (i % nkb) * kBK, b);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            const uint32_t q_addr = smem_u32(smem + kSmemQ);
            mbar_wait(q_full, 0);
            for (int i = 0; i < items; ++i) {
                const int s = i % kBufs;
                const uint32_t ph = (i / kBufs) & 1;
                mbar_wait(kv_full + s, ph);
                mbar_wait(s_empty + s, ph ^ 1);
                tc_fence_after();
                const uint32_t k_addr = smem_u32(smem + kSmemK + s * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < kDh / 16; ++kk)
                    umma_f16(tmem + s * kBK, sw128_desc(q_addr + kk * 32, 16, 1024),
                             sw128_desc(k_addr + kk * 32, 16, 1024), kIdescS, kk > 0 ? 1u : 0u);
                umma_commit(s_full + s);
                umma_commit(kv_empty + s);
            }
        }
    } else {  // ------------------------------- softmax / column reduction (warps 2..5)
        const int quad = warp & 3;
        const int wi = warp - 2;                   // 0..3, index into the smem reduction buffers
        const int row = quad * 32 + lane;
        const int grow = m0 + row;
        const bool row_ok = grow < n;
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
        const float c2 = scale * 1.4426950408889634f;   // t2 = S * c2 (log2 domain)
        // ---- sweep 1: row max / sum
        float m2 = -INFINITY, l = 0.0f;
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kBufs;
            mbar_wait(s_full + s, (kb / kBufs) & 1);
            tc_fence_after();
            uint32_t sv[4][32];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) tmem_ld32(lane_base + s * kBK + q4 * 32, sv[q4]);
            tmem_ld_wait();
            if (!resident) {
                tc_fence_before();
                mbar_arrive(s_empty + s);
            }
            const int valid = min(kBK, n - kb * kBK);
            float bmax = -INFINITY;
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    if (q4 * 32 + e < valid) bmax = fmaxf(bmax, __uint_as_float(sv[q4][e]) * c2);
            const float mn = fmaxf(m2, bmax);
            float acc = 0.0f;
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    if (q4 * 32 + e < valid) acc += ex2_approx(__uint_as_float(sv[q4][e]) * c2 - mn);
            l = (m2 == -INFINITY ? 0.0f : l * ex2_approx(m2 - mn)) + acc;
            m2 = mn;
        }
        const float lse2 = m2 + __log2f(l);        // log2-domain log-sum-exp
        if (row_ok) {
            const size_t t = ((size_t)b * heads + h) * n + grow;
            row_m[t] = (double)m2 * 0.6931471805599453;
            row_l[t] = (double)l;
            lse_out[t] = lse2 * 0.6931471805599453f;
        }
        // ---- sweep 2: per-column maxima of v = t2 - lse2 and their argmax rows
        for (int kb = 0; kb < nkb; ++kb) {
            const int item = resident ? kb : nkb + kb;
            const int s = item % kBufs;
            if (!resident) {
                mbar_wait(s_full + s, (item / kBufs) & 1);
                tc_fence_after();
            }
            const int kbase = kb * kBK;
            for (int q4 = 0; q4 < 4; ++q4) {
                uint32_t sv[32];
                tmem_ld32(lane_base + s * kBK + q4 * 32, sv);
                tmem_ld_wait();
                float v[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = row_ok ? __fmaf_rn(__uint_as_float(sv[e]), c2, -lse2) : -INFINITY;
                // butterfly reduce-scatter: lane L ends with the warp max of column L
#pragma unroll
                for (int wdt = 16; wdt >= 1; wdt >>= 1) {
                    const bool upper = (lane & wdt) != 0;
#pragma unroll
                    for (int i = 0; i < wdt; ++i) {
                        const float send = upper ? v[i] : v[i + wdt];
                        const float keep = upper ? v[i + wdt] : v[i];
                        v[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, wdt));
                    }
                }
                red[wi * 128 + q4 * 32 + lane] = v[0];
            }
            named_bar_sync(1, 128);
            {   // thread `row` now owns column kbase + row of this block
                const float M = fmaxf(fmaxf(red[row], red[128 + row]), fmaxf(red[256 + row], red[384 + row]));
                colM[row] = M;
                win[row] = 0x7FFFFFFF;
            }
            named_bar_sync(1, 128);
            // exact re-comparison finds the winning row(s); smallest row wins. The
            // TMEM load is warp-collective (.sync.aligned): every lane executes it.
            for (int q4 = 0; q4 < 4; ++q4) {
                uint32_t sv[32];
                tmem_ld32(lane_base + s * kBK + q4 * 32, sv);
                tmem_ld_wait();
                if (row_ok) {
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float vv = __fmaf_rn(__uint_as_float(sv[e]), c2, -lse2);
                        if (vv == colM[q4 * 32 + e]) atomicMin(&win[q4 * 32 + e], grow);
                    }
                }
            }
            if (!resident) {
                tc_fence_before();
                mbar_arrive(s_empty + s);
            }
            named_bar_sync(1, 128);
            if (kbase + row < n) {
                const unsigned long long key = ((unsigned long long)float_to_ordered(colM[row]) << 32) |
                                               (unsigned long long)(0xFFFFFFFFu - (uint32_t)win[row]);
                atomicMax(colkey + ((size_t)b * heads + h) * n + kbase + row, key);
            }
            named_bar_sync(1, 128);   // red / colM / win are reused by the next block
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace mca_dev

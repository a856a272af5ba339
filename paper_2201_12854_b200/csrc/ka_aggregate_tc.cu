// ka_aggregate_tc.cu — the given-attention aggregation on the tensor cores:
// y[b, i, h*64 + c] = sum_j A[b, h, i, j] H~[b, j, h*64 + c]   (matmul(A, H~),
// matrix.hpp:33-34, the layer cmd_bench drives with an
// imported or synthetic attention dump). The dump A is fp64; each entry is
// rounded to fp32 (relative 2^-24) and split into tf32 hi + lo, H~ comes from
// k_split_transpose_h (per head transposed, [B*H][64][ld]): hi + lo on the fp32
// path (3xTF32: A_hi.H_lo + A_lo.H_hi + A_hi.H_hi, small products first), hi
// alone on the bf16 path (fp16 H~ is exact in tf32: A_lo.H + A_hi.H).
// Bound: HBM, the dump itself (8 B per entry; 1.6 GB at C2's shape).
//
// CTA = (128-row tile i0, h, b); 320 threads, ~97 KB of shared memory (two CTAs
// per SM):
//   warp 0      TMA producer: H~^T hi (| lo) of 32-key blocks, 2 stages
//   warp 1      TMEM allocator (64 columns: O) + MMA issuer (whole warp, elect.sync)
//   warps 2-9   loaders: warp w reads 16 rows of the block, one row (32 keys,
//               256 coalesced bytes) per instruction, the next block's rows in
//               flight while it writes this block's fp32 hi / lo parts into the
//               128B-swizzled K-major P tile; warps 2-5 then run the epilogue
//               (TMEM lane = row).
#pragma once

#include "mca_common.cuh"
#include "tc_common.cuh"

namespace mca_dev {

namespace katc {
constexpr int kBM = 128, kBK = 32, kStages = 2;
constexpr int kLoaders = 8;                    // loader warps: 16 rows each
constexpr int kThreads = 64 + 32 * kLoaders;   // + TMA warp + MMA warp
constexpr uint32_t kAtom128 = 128 * 128;   // P: 128 rows x 128 B (32 fp32 keys)
constexpr uint32_t kAtom64 = 64 * 128;     // H~^T: 64 dims x 128 B (32 fp32 keys)
constexpr uint32_t kPBytes = 2 * kAtom128;   // hi | lo: 32 KB per stage
constexpr uint32_t kVBytes = 2 * kAtom64;    // hi | lo: 16 KB per stage (fp16 H~: hi only, 8 KB used)
constexpr uint32_t kSmemP = 0, kSmemV = kStages * kPBytes, kSmemBar = kSmemV + kStages * kVBytes;
constexpr uint32_t kSmemBytes = kSmemBar + 256 + 1024;
constexpr uint32_t kIdesc = mca_tc::idesc_tf32(kBM, kDh);
}  // namespace katc

// kHLo: H~^T carries a lo part (fp32 path). Y: float (fp32 path) or __nv_bfloat16.
template <bool kHLo, class Y>
__global__ void __launch_bounds__(katc::kThreads, 2)
    ka_aggregate_tc(const __grid_constant__ CUtensorMap tm_vh, const __grid_constant__ CUtensorMap tm_vl,
                    const double* __restrict__ attn, int n, int heads, Y* __restrict__ y) {
    using namespace katc;
    using namespace mca_tc;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* v_full = bars + 0;     // [2] TMA
    uint64_t* v_empty = bars + 2;    // [2] MMA commit
    uint64_t* p_full = bars + 4;     // [2] kLoaders loader warps
    uint64_t* p_free = bars + 6;     // [2] MMA commit
    uint64_t* o_full = bars + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
    const int b = blockIdx.z, h = blockIdx.y, i0 = blockIdx.x * kBM;
    const int nblk = (n + kBK - 1) / kBK;
    const size_t bh = (size_t)b * heads + h;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 9; ++i) mbar_init(bars + i, (i >= 4 && i < 6) ? kLoaders : 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<64>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;   // O: columns [0, 64)
    griddep_trigger();

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer: H~^T blocks
            griddep_wait();   // H~ (transposed) of this forward
            constexpr uint32_t bytes = kHLo ? kVBytes : kAtom64;
            for (int kb = 0; kb < nblk; ++kb) {
                const int st = kb & 1;
                const uint32_t ph = (kb >> 1) & 1;
                mbar_wait(v_empty + st, ph ^ 1);
                mbar_expect_tx(v_full + st, bytes);
                tma_load_3d(smem + kSmemV + st * kVBytes, &tm_vh, v_full + st, kb * kBK, 0, (int)bh);
                if constexpr (kHLo)
                    tma_load_3d(smem + kSmemV + st * kVBytes + kAtom64, &tm_vl, v_full + st, kb * kBK, 0, (int)bh);
            }
        }
    } else if (warp == 1) {   // ---------------- MMA issuer (whole warp)
        const uint64_t dp = sw128_desc(smem_u32(smem + kSmemP), 16, 1024);
        const uint64_t dv = sw128_desc(smem_u32(smem + kSmemV), 16, 1024);
        for (int kb = 0; kb < nblk; ++kb) {
            const int st = kb & 1;
            const uint32_t ph = (kb >> 1) & 1;
            mbar_wait(p_full + st, ph);
            mbar_wait(v_full + st, ph);
            tc_fence_after();
            const uint64_t pa = desc_add(dp, st * kPBytes), va = desc_add(dv, st * kVBytes);
            // products, small first: A_hi . H_lo (fp32 path), A_lo . H_hi, A_hi . H_hi
#pragma unroll
            for (int pr = kHLo ? 0 : 1; pr < 3; ++pr) {
                const uint32_t ap = pr == 1 ? kAtom128 : 0u, bp = pr == 0 ? kAtom64 : 0u;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    umma_tf32_w(tmem, desc_add(pa, ap + kk * 32), desc_add(va, bp + kk * 32), kIdesc,
                                (kb > 0 || pr != (kHLo ? 0 : 1) || kk > 0) ? 1u : 0u);
            }
            umma_commit_w(p_free + st);
            umma_commit_w(v_empty + st);
        }
        umma_commit_w(o_full);
    } else {   // ------------------------------- loaders (warps 2-9) + epilogue (warps 2-5)
        const int lw = warp - 2;                    // rows [16 lw, 16 lw + 16) of the tile
        const double* abase = attn + bh * (size_t)n * n;
        double v[16];
        auto fetch = [&](int kb) {
            const int key = kb * kBK + lane;
#pragma unroll
            for (int rr = 0; rr < 16; ++rr) {
                const int i = i0 + lw * 16 + rr;
                v[rr] = (i < n && key < n) ? __ldg(abase + (size_t)i * n + key) : 0.0;
            }
        };
        fetch(0);
        for (int kb = 0; kb < nblk; ++kb) {
            const int st = kb & 1;
            const uint32_t ph = (kb >> 1) & 1;
            float hi[16], lo[16];
#pragma unroll
            for (int rr = 0; rr < 16; ++rr) {
                const float f = __double2float_rn(v[rr]);
                hi[rr] = __uint_as_float(__float_as_uint(f) & 0xFFFFE000u);
                lo[rr] = f - hi[rr];
            }
            if (kb + 1 < nblk) fetch(kb + 1);        // the next block's rows in flight
            mbar_wait(p_free + st, ph ^ 1);          // P(kb - 2) . H~ has read this buffer
            uint8_t* pb = smem + kSmemP + st * kPBytes;
#pragma unroll
            for (int rr = 0; rr < 16; ++rr) {
                const uint32_t off = sw128_offset((uint32_t)(lw * 16 + rr), (uint32_t)lane * 4);
                *reinterpret_cast<float*>(pb + off) = hi[rr];
                *reinterpret_cast<float*>(pb + kAtom128 + off) = lo[rr];
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full + st);
        }
        if (warp >= 6) goto done;   // warps 2-5 hold TMEM lane quadrants 0-3 (warp % 4)
        {
        const int quad = warp & 3;
        // epilogue: O -> y, TMEM lane = row
        mbar_wait(o_full, 0);
        tc_fence_after();
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
        uint32_t ov[2][32];
        tmem_ld32(lane_base, ov[0]);
        tmem_ld32(lane_base + 32, ov[1]);
        tmem_ld_wait();
        const int i = i0 + quad * 32 + lane;
        if (i < n) {
            Y* dst = y + ((size_t)b * n + i) * heads * kDh + (size_t)h * kDh;
            if constexpr (sizeof(Y) == 4) {
#pragma unroll
                for (int g = 0; g < 16; ++g)
                    reinterpret_cast<float4*>(dst)[g] =
                        make_float4(__uint_as_float(ov[(4 * g) >> 5][(4 * g) & 31]), __uint_as_float(ov[(4 * g + 1) >> 5][(4 * g + 1) & 31]),
                                    __uint_as_float(ov[(4 * g + 2) >> 5][(4 * g + 2) & 31]), __uint_as_float(ov[(4 * g + 3) >> 5][(4 * g + 3) & 31]));
            } else {
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    uint32_t pk[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int c = 8 * g + 2 * e;
                        pk[e] = pack_bf16x2(__uint_as_float(ov[c >> 5][c & 31]), __uint_as_float(ov[(c + 1) >> 5][(c + 1) & 31]));
                    }
                    reinterpret_cast<uint4*>(dst)[g] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
            }
        }
        }
    }
done:
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<64>(tmem);
}

// fp16 H~ (bf16 path) -> per head transposed fp32 [B*H][64][ld] (exact: fp16 values are
// tf32-representable, so there is no lo part). grid (ceil(n / 64), H, B), block 256.
__global__ void __launch_bounds__(256) k_transpose_h16(const __half* __restrict__ hm, int n, int ld, int heads,
                                                       float* __restrict__ vh) {
    __shared__ float tile[64][65];
    const int j0 = blockIdx.x * 64, h = blockIdx.y, b = blockIdx.z, tid = threadIdx.x;
    const size_t HD = (size_t)heads * kDh;
    const size_t bh = (size_t)b * heads + h;
#pragma unroll
    for (int u = 0; u < 2; ++u) {   // 64 tokens x 64 dims = 512 pieces of 8 halves
        const int e = tid + 256 * u, jj = e >> 3, d8 = (e & 7) * 8;
        const int j = j0 + jj;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (j < n) v = *reinterpret_cast<const uint4*>(hm + ((size_t)b * n + j) * HD + (size_t)h * kDh + d8);
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[q]));
            tile[d8 + 2 * q][jj] = f.x;
            tile[d8 + 2 * q + 1][jj] = f.y;
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int e = tid + 256 * u, d = e >> 4, j4 = (e & 15) * 4;
        if (j0 + j4 >= ld) continue;
        *reinterpret_cast<float4*>(vh + (bh * kDh + d) * (size_t)ld + j0 + j4) =
            make_float4(tile[d][j4], tile[d][j4 + 1], tile[d][j4 + 2], tile[d][j4 + 3]);
    }
}

}  // namespace mca_dev

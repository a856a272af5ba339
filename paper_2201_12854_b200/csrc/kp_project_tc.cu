// kp_project_tc.cu — KP: the layer's dense projections on tcgen05.
//
// attention_matrix forms Q = X W_q and
// K = X W_k before the softmax. With W_q / W_k attached to the weights
// (mca_set_projections) the forward takes x alone and this kernel computes
//   [q | k] = x . [W_q | W_k]        x [M = B n, d_in],  W [d_in, 2 H 64]
// in one persistent GEMM whose epilogue writes q and k straight into the
// [B, n, H*64] layout the score kernels' TMA maps read. regular_forward
// adds a third segment, the exact encoding H = X W_V (fp16,
// K4's operand), so the exact layer is one dense GEMM + the row statistics +
// K4. Output segment s (columns [s HD, (s + 1) HD) of the product) goes to
// tensor map s, in fp16 when bit s of f16_mask is set, else bf16.
//
// Operands (tc_common.cuh layout): A = x rows [128 x 64] per K step (K-major,
// TMA 128B swizzle); B = W^T rows [BN x 64] (K-major: the handle keeps W_q /
// W_k transposed, prepared once in mca_set_projections). D = fp32 in TMEM.
//
// Persistent, one CTA per SM, warp-specialised (192 threads):
//   warp 0      TMA producer: kStages-deep ring of (A, B) K-steps
//   warp 1      TMEM allocator + MMA issuer: tcgen05.mma M=128 N=BN K=16, four
//               per K step; two accumulators (2 x BN columns) so the epilogue of
//               tile i overlaps the main loop of tile i + 1
//   warps 2-5   epilogue: tcgen05.ld (warp w reads TMEM lanes 32 (w % 4) ..),
//               fp32 -> bf16 into a 128B-swizzled [128 x 64] staging tile
//               (double-buffered), written out by one TMA bulk tensor store
//               per 64 columns. Direct 16-byte stores of each thread's row
//               (one L2 request per lane) held the kernel at 80 us at C2; the
//               main loop alone runs in 53 us.
// Tiles are visited m-major (t -> m = t / nN, n = t % nN), so the CTAs working
// at one time share x tiles in L2 across the N tiles; W (2.4 MB at BERT-base)
// stays L2-resident.
#include "mca_common.cuh"
#include "tc_common.cuh"

namespace mca_dev {

#ifndef KP_STAGES_256
#define KP_STAGES_256 4
#endif
#ifndef KP_STORE_HINT
#define KP_STORE_HINT 0
#endif
#ifndef KP_OUTBUFS_256
#define KP_OUTBUFS_256 2
#endif
namespace kp {
constexpr int kBM = 128;
constexpr int kThreads = 192;
// kTf32 (the fp32 path, 3xTF32): x and W^T arrive as tf32-exact hi and lo
// parts; a K step is one 128-byte atom of 32 fp32 per part, and the product
// is hi.lo + lo.hi + hi.hi (small products first, k1_scores_tc.cu). bf16: a
// K step is one atom of 64 bf16. Outputs are staged [128 x 128 B] per chunk
// (64 bf16 / fp16 or 32 fp32 columns).
template <int BN, bool kTf32 = false>
struct Cfg {
    static constexpr int kBK = kTf32 ? 32 : 64;                  // elements per K step (one 128-byte atom)
    static constexpr int kParts = kTf32 ? 2 : 1;
    static constexpr int kStages = kTf32 ? (BN >= 192 ? 2 : 3) : (BN >= 192 ? KP_STAGES_256 : 6);
    static constexpr int kOutBufs = (kTf32 || BN < 192) ? 2 : KP_OUTBUFS_256;   // staging tiles in flight
    static constexpr uint32_t kAPart = kBM * 128;                // 16 KB
    static constexpr uint32_t kBPart = BN * 128;                 // 8 / 16 / 32 KB
    static constexpr uint32_t kABytes = kParts * kAPart;
    static constexpr uint32_t kBBytes = kParts * kBPart;
    static constexpr uint32_t kStageBytes = kABytes + kBBytes;
    static constexpr uint32_t kSmemOut = kStages * kStageBytes;  // 2 x [128 x 128 B] staging tiles
    static constexpr uint32_t kOutBytes = kBM * 128;             // 16 KB
    static constexpr int kOutCols = kTf32 ? 32 : 64;             // output columns per staging tile
    static constexpr uint32_t kSmemBar = kSmemOut + kOutBufs * kOutBytes;
    static constexpr uint32_t kSmemBytes = kSmemBar + 256 + 1024;   // barriers + 1 KB alignment slack
    static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
    static constexpr uint32_t kIdesc = kTf32 ? mca_tc::idesc_tf32(kBM, BN) : mca_tc::idesc_f16(1, 0, kBM, BN);
};
}  // namespace kp

struct KpArgs {
    int M;          // rows of x (B * n)
    int d_in;       // K
    int HD;         // H * 64: segment s = product columns [s HD, (s + 1) HD)
    int nseg;       // 1..3 output segments
    int f16_mask;   // bit s: segment s stored as fp16 (else bf16)
    // fp16 segments (H~): chunks of 8 values outside fp16's range are zeroed and,
    // for exact token-heads (exact == nullptr: all of them), queued for the
    // aggregation's fp32 fix-up (mca_common.cuh f16_guard8); n = tokens per sequence.
    OvfSink ovf;
    const uint8_t* exact;   // [B, H, n] or nullptr
    int n;
    // Device-side dispatch of the MCA layer's exact encodings (gate != nullptr):
    // the GEMM runs only when sum_h gate[2 h + 1] >= gate_min (K2's exact counts),
    // otherwise every CTA exits at once and k3b_exact_tc encodes the listed tokens.
    const int* gate;
    long gate_min;
    // 3xTF32, lo_tma != 0: the lo parts v - hi(v) of segments 0 / 1 also go out,
    // through tm_o2 = a [2][M][HD] map (q_lo | k_lo: the score passes' lo
    // operands, so q / k need no split pass); each chunk stages hi and lo in the
    // two staging tiles.
    int lo_tma;
};

// kTf32: tm_x / tm_w carry the hi parts and tm_x2 / tm_w2 the lo parts.
template <int BN, bool kTf32 = false>
__global__ void __launch_bounds__(kp::kThreads, 1) kp_project_tc(const __grid_constant__ CUtensorMap tm_x,
                                                                 const __grid_constant__ CUtensorMap tm_w,
                                                                 const __grid_constant__ CUtensorMap tm_x2,
                                                                 const __grid_constant__ CUtensorMap tm_w2,
                                                                 const __grid_constant__ CUtensorMap tm_o0,
                                                                 const __grid_constant__ CUtensorMap tm_o1,
                                                                 const __grid_constant__ CUtensorMap tm_o2, KpArgs a) {
    using namespace mca_tc;
    using C = kp::Cfg<BN, kTf32>;
    constexpr int S = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kSmemBar);
    uint64_t* full = bars;               // [S] TMA tx
    uint64_t* empty = bars + S;          // [S] MMA commit
    uint64_t* acc_full = bars + 2 * S;   // [2] MMA commit after a tile's last K step
    uint64_t* acc_empty = bars + 2 * S + 2;   // [2] 4 epilogue warps
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;   // uniform: see k4_apply_tf32
    if (a.gate) {   // the exact fraction decides between this dense GEMM and the gathered one
        griddep_wait();
        long ex = 0;
        for (int hh = 0; hh < a.HD / kDh; ++hh) ex += a.gate[2 * hh + 1];
        if (ex < a.gate_min) return;
    }
    const int nK = (a.d_in + C::kBK - 1) / C::kBK;
    const int nM = (a.M + kp::kBM - 1) / kp::kBM;
    const int nN = a.nseg * a.HD / BN;
    const int tiles = nM * nN;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(acc_full + b, 1);
            mbar_init(acc_empty + b, 4);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_x);
        tma_prefetch(&tm_w);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_trigger();

    if (warp == 0) {
        if (lane == 0) {
            griddep_wait();   // x may be the previous kernel's output (a chained layer)
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int m0 = (t / nN) * kp::kBM, n0 = (t % nN) * BN;
                for (int kb = 0; kb < nK; ++kb) {
                    mbar_wait(empty + s, ph ^ 1);
                    uint8_t* st = smem + s * C::kStageBytes;
                    mbar_expect_tx(full + s, C::kStageBytes);
                    tma_load_3d(st, &tm_x, full + s, kb * C::kBK, m0, 0);
                    tma_load_3d(st + C::kABytes, &tm_w, full + s, kb * C::kBK, n0, 0);
                    if constexpr (kTf32) {
                        tma_load_3d(st + C::kAPart, &tm_x2, full + s, kb * C::kBK, m0, 0);
                        tma_load_3d(st + C::kABytes + C::kBPart, &tm_w2, full + s, kb * C::kBK, n0, 0);
                    }
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {   // ---------------- MMA issuer (whole warp; one elected lane issues)
        const uint64_t d0 = sw128_desc(smem_u32(smem), 16, 1024);
        int s = 0;
        uint32_t ph = 0;
        int acc = 0;
        uint32_t aph = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            mbar_wait(acc_empty + acc, aph ^ 1);    // the epilogue drained this accumulator
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)(acc * BN);
            for (int kb = 0; kb < nK; ++kb) {
                mbar_wait(full + s, ph);
                tc_fence_after();
                const uint64_t da = desc_add(d0, s * C::kStageBytes);
                const uint64_t db = desc_add(da, C::kABytes);
                if constexpr (kTf32) {   // hi.lo + lo.hi + hi.hi, K = 8 fp32 per instruction
#pragma unroll
                    for (int pr = 0; pr < 3; ++pr) {
                        const uint32_t ap = pr == 1 ? C::kAPart : 0u, bp = pr == 0 ? C::kBPart : 0u;
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            umma_tf32_w(d, desc_add(da, ap + kk * 32), desc_add(db, bp + kk * 32), C::kIdesc,
                                        (kb | pr | kk) != 0);
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_f16_w(d, desc_add(da, kk * 32), desc_add(db, kk * 32), C::kIdesc, (kb | kk) != 0);
                }
                umma_commit_w(empty + s);             // the stage is free once these MMAs read it
                if (++s == S) {
                    s = 0;
                    ph ^= 1;
                }
            }
            umma_commit_w(acc_full + acc);            // the tile's accumulator is complete
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
    } else {
        // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 = rows of the tile
        const int quarter = warp & 3;
        const int et = threadIdx.x - 64;                 // 0..127 (warps 2-5)
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t r = (uint32_t)(quarter * 32 + lane);   // row within the tile
        uint8_t* stage_out = smem + C::kSmemOut;
        int acc = 0, ob = 0;
        uint32_t aph = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            const int m0 = (t / nN) * kp::kBM, n0 = (t % nN) * BN;
            const int seg = n0 / a.HD;
            const CUtensorMap* om = seg == 0 ? &tm_o0 : seg == 1 ? &tm_o1 : &tm_o2;
            const int oc = n0 - seg * a.HD;
            const bool f16 = (a.f16_mask >> seg) & 1;
            mbar_wait(acc_full + acc, aph);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < BN; c += C::kOutCols) {
                if (et == 0) {   // the store that used this buffer has read it (both buffers when lo goes out too)
                    if (kTf32 && a.lo_tma) bulk_wait_read<0>();
                    else bulk_wait_read<C::kOutBufs - 1>();
                }
                named_bar_sync(1, 128);
                uint8_t* st = stage_out + ob * C::kOutBytes;
                if constexpr (kTf32) {                    // 32 fp32 columns: one 128-byte row per thread
                    uint32_t v[32];
                    tmem_ld32(lane_base + (uint32_t)(acc * BN + c), v);
                    tmem_ld_wait();
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        *reinterpret_cast<uint4*>(st + sw128_offset(r, (uint32_t)g * 16)) =
                            make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                    if (a.lo_tma) {   // the lo parts into the other staging tile (both are free: see above)
                        uint8_t* sl = stage_out + (ob ^ 1) * C::kOutBytes;
#pragma unroll
                        for (int g = 0; g < 8; ++g) {
                            uint32_t e[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const uint32_t b = v[4 * g + u];
                                e[u] = __float_as_uint(__uint_as_float(b) - __uint_as_float(b & 0xFFFFE000u));
                            }
                            *reinterpret_cast<uint4*>(sl + sw128_offset(r, (uint32_t)g * 16)) = make_uint4(e[0], e[1], e[2], e[3]);
                        }
                    }
                } else {
                    uint32_t v[2][32];
                    tmem_ld32(lane_base + (uint32_t)(acc * BN + c), v[0]);
                    tmem_ld32(lane_base + (uint32_t)(acc * BN + c + 32), v[1]);
                    tmem_ld_wait();
#pragma unroll
                    for (int g = 0; g < 8; ++g) {        // 16-byte chunk g = columns 8g .. 8g + 7
                        const uint32_t* src = &v[g >> 2][(g & 3) * 8];
                        uint4 u;
                        if (f16 && a.ovf.count) {   // fp16 range guard (H~ segments)
                            float f[8];
                            bool big = false;
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                f[e] = __uint_as_float(src[e]);
                                big |= f16_overflows(f[e]);
                            }
                            const int t = m0 + (int)r;
                            if (big && t < a.M) {
                                const int col = oc + c + 8 * g, hh = col / kDh, bb = t / a.n, j = t - bb * a.n;
                                const long long tokh = ((long long)bb * (a.HD / kDh) + hh) * a.n + j;
                                if (!a.exact || a.exact[tokh]) {   // sampled token-heads: K3 rewrites the row
                                    const unsigned long long pos = atomicAdd(a.ovf.count, 1ull);
                                    if (pos < (unsigned long long)a.ovf.cap) {
                                        a.ovf.list[pos] = tokh * 8 + ((col % kDh) >> 3);
#pragma unroll
                                        for (int e = 0; e < 8; ++e) a.ovf.rows[pos * 8 + e] = f[e];
                                    }
                                }
                            }
                            if (big) {
                                u = make_uint4(0u, 0u, 0u, 0u);
                            } else {
                                u.x = pack_f16x2(f[0], f[1]);
                                u.y = pack_f16x2(f[2], f[3]);
                                u.z = pack_f16x2(f[4], f[5]);
                                u.w = pack_f16x2(f[6], f[7]);
                            }
                        } else if (f16) {
                            u.x = pack_f16x2(__uint_as_float(src[0]), __uint_as_float(src[1]));
                            u.y = pack_f16x2(__uint_as_float(src[2]), __uint_as_float(src[3]));
                            u.z = pack_f16x2(__uint_as_float(src[4]), __uint_as_float(src[5]));
                            u.w = pack_f16x2(__uint_as_float(src[6]), __uint_as_float(src[7]));
                        } else {
                            u.x = pack_bf16x2(__uint_as_float(src[0]), __uint_as_float(src[1]));
                            u.y = pack_bf16x2(__uint_as_float(src[2]), __uint_as_float(src[3]));
                            u.z = pack_bf16x2(__uint_as_float(src[4]), __uint_as_float(src[5]));
                            u.w = pack_bf16x2(__uint_as_float(src[6]), __uint_as_float(src[7]));
                        }
                        *reinterpret_cast<uint4*>(st + sw128_offset(r, (uint32_t)g * 16)) = u;
                    }
                }
                fence_proxy_async_smem();                // generic-proxy writes -> visible to the TMA store
                named_bar_sync(1, 128);
                if (et == 0) {
#if KP_STORE_HINT == 1
                    tma_store_3d_hint(om, st, oc + c, m0, 0, l2_policy_evict_first());
#elif KP_STORE_HINT == 2
                    tma_store_3d_hint(om, st, oc + c, m0, 0, l2_policy_evict_last());
#else
                    tma_store_3d(om, st, oc + c, m0, 0);  // rows past M are clipped by the tensor map
#endif
                    if (kTf32 && a.lo_tma) tma_store_3d(&tm_o2, stage_out + (ob ^ 1) * C::kOutBytes, oc + c, m0, seg);
                    bulk_commit();
                }
                if (kTf32 && a.lo_tma) continue;   // both tiles used: the next chunk waits for both
                if (++ob == C::kOutBufs) ob = 0;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty + acc);
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
        if (et == 0) bulk_wait<0>();                     // the last stores have left shared memory
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
}

}  // namespace mca_dev

namespace mca_dev {
// W [d_in, HD] (x W convention) -> W^T [HD, d_in] (the K-major B operand above),
// once per mca_set_projections. grid (ceil(HD / 32), ceil(d_in / 32)), block (32, 8).
__global__ void kp_transpose(const __nv_bfloat16* __restrict__ w, int d_in, int HD, __nv_bfloat16* __restrict__ wt) {
    __shared__ __nv_bfloat16 tile[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += 8)
        if (r0 + r < d_in && c0 + (int)threadIdx.x < HD) tile[r][threadIdx.x] = w[(size_t)(r0 + r) * HD + c0 + threadIdx.x];
    __syncthreads();
    for (int c = threadIdx.y; c < 32; c += 8)
        if (c0 + c < HD && r0 + (int)threadIdx.x < d_in)
            wt[(size_t)(c0 + c) * d_in + r0 + threadIdx.x] = tile[threadIdx.x][c];
}
}  // namespace mca_dev

namespace mca_dev {
// fp32 W [d_in, HD] -> W^T hi / lo [HD, d_in] (tf32-exact hi, lo = w - hi): the
// 3xTF32 projection's K-major B parts. grid (ceil(HD / 32), ceil(d_in / 32)), block (32, 8).
__global__ void kp_transpose_split_f32(const float* __restrict__ w, int d_in, int HD, float* __restrict__ wt_hi,
                                       float* __restrict__ wt_lo) {
    __shared__ float tile[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += 8)
        if (r0 + r < d_in && c0 + (int)threadIdx.x < HD) tile[r][threadIdx.x] = w[(size_t)(r0 + r) * HD + c0 + threadIdx.x];
    __syncthreads();
    for (int c = threadIdx.y; c < 32; c += 8)
        if (c0 + c < HD && r0 + (int)threadIdx.x < d_in) {
            const float v = tile[threadIdx.x][c];
            const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
            const size_t o = (size_t)(c0 + c) * d_in + r0 + threadIdx.x;
            wt_hi[o] = hi;
            wt_lo[o] = v - hi;
        }
}
}  // namespace mca_dev

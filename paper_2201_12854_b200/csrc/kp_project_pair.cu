// kp_project_pair.cu — KP on CTA pairs (tcgen05 cta_group::2), bf16 only.
//
// The same product as kp_project_tc ([q | k (| H)] = x . [W_q | W_k (| W_V)],
// SPEC.md:286-294) with 256 x 256 tiles shared by the two CTAs of a cluster:
// CTA r loads rows [128 r, 128 r + 128) of the x tile and rows
// [128 r, 128 r + 128) of the W^T tile (its half of N) into its own shared
// memory, and the leader (r = 0) issues M = 256, N = 256 MMAs that read both
// CTAs' operands and write 128 rows x 256 columns of fp32 into each CTA's TMEM.
// Per SM and K step that is 32 KB of operands for 512 MMA cycles, against 48 KB
// in the single-CTA 128 x 256 tile (tensor pipe ~60% active there). Measured at
// C2: 60 vs 64 us; 3 / 4 / 6 stages 69.5 / 59.8 / 62.0 us
// (scripts/kp2_stage_exp.sh).
//
//   warp 0      TMA producer of its CTA; every load completes on the LEADER's
//               full barrier (the leader expects both CTAs' bytes)
//   warp 1      TMEM allocator (cta_group::2, both CTAs) + MMA issuer (leader)
//   warps 2-5   epilogue of the CTA's 128 rows (tcgen05.ld -> bf16 / fp16 ->
//               swizzled staging tile -> TMA store); they release an
//               accumulator on the leader's barrier (8 arrivals: both CTAs)
#pragma once

#include "mca_common.cuh"
#include "tc_common.cuh"

#ifndef MCA_KP2_STAGES
#define MCA_KP2_STAGES 4
#endif

namespace mca_dev {

namespace kp2 {
// kTf32: 3xTF32 (hi.lo + lo.hi + hi.hi; x and W^T raw as their hi parts, their
// lo parts from their own maps), 32 fp32 per K step, fp32 outputs staged 32
// columns at a time, and (KpArgs::lo_tma) the q / k lo parts out through tm_o2.
template <bool kTf32>
struct Cfg {
    static constexpr int kBK = kTf32 ? 32 : 64, kBN = 256;
    static constexpr int kParts = kTf32 ? 2 : 1;
    static constexpr int kStages = kTf32 ? 3 : MCA_KP2_STAGES, kOutBufs = 2;
    static constexpr int kThreads = 192;
    static constexpr uint32_t kPart = 128 * 128;                  // 16 KB: 128 rows x 128 B
    static constexpr uint32_t kABytes = kParts * kPart;           // the CTA's 128 x rows
    static constexpr uint32_t kBBytes = kParts * kPart;           // the CTA's 128 W^T rows
    static constexpr uint32_t kStageBytes = kABytes + kBBytes;
    static constexpr uint32_t kSmemOut = kStages * kStageBytes;
    static constexpr uint32_t kOutBytes = 128 * 128;              // [128 x 128 B] staging tile
    static constexpr int kOutCols = kTf32 ? 32 : 64;
    static constexpr uint32_t kSmemBar = kSmemOut + kOutBufs * kOutBytes;
    static constexpr uint32_t kSmemBytes = kSmemBar + 256 + 1024;
    static constexpr uint32_t kIdesc = kTf32 ? mca_tc::idesc_tf32(256, kBN) : mca_tc::idesc_f16(1, 0, 256, kBN);
};
}  // namespace kp2

template <bool kTf32>
__global__ void __launch_bounds__(192, 1)
    kp_project_pair(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                    const __grid_constant__ CUtensorMap tm_x2, const __grid_constant__ CUtensorMap tm_w2,
                    const __grid_constant__ CUtensorMap tm_o0, const __grid_constant__ CUtensorMap tm_o1,
                    const __grid_constant__ CUtensorMap tm_o2, KpArgs a) {
    using namespace mca_tc;
    using C = kp2::Cfg<kTf32>;
    constexpr int S = C::kStages, kBK = C::kBK, kBN = C::kBN, kOutBufs = C::kOutBufs;
    constexpr uint32_t kStageBytes = C::kStageBytes, kABytes = C::kABytes, kSmemOut = C::kSmemOut,
                       kOutBytes = C::kOutBytes, kSmemBar = C::kSmemBar, kIdesc = C::kIdesc;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* full = bars;                    // [S] leader's: TMA bytes of both CTAs
    uint64_t* empty = bars + S;               // [S] each CTA's: pair MMA commit
    uint64_t* acc_full = bars + 2 * S;        // [2] each CTA's: pair MMA commit
    uint64_t* acc_empty = bars + 2 * S + 2;   // [2] leader's: 8 epilogue warps
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    if (a.gate) {   // dense exact encoding gate (kp_project_tc): uniform over the cluster
        griddep_wait();
        long ex = 0;
        for (int hh = 0; hh < a.HD / kDh; ++hh) ex += a.gate[2 * hh + 1];
        if (ex < a.gate_min) return;
    }
    const int nK = (a.d_in + kBK - 1) / kBK;
    const int nM = (a.M + 255) / 256;
    const int nN = a.nseg * a.HD / kBN;
    const int tiles = nM * nN;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(acc_full + b, 1);
            mbar_init(acc_empty + b, 8);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc2<512>(tmem_slot);
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_x);
        tma_prefetch(&tm_w);
    }
    tc_fence_before();
    cluster_sync();   // both CTAs' barriers initialised before any cross-CTA arrival
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_trigger();

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer (both CTAs)
            griddep_wait();
            int s = 0;
            uint32_t ph = 0;
            for (int t = pair; t < tiles; t += npairs) {
                const int m0 = (t / nN) * 256, n0 = (t % nN) * kBN;
                for (int kb = 0; kb < nK; ++kb) {
                    mbar_wait(empty + s, ph ^ 1);
                    uint8_t* st = smem + s * kStageBytes;
                    if (rank == 0) mbar_expect_tx(full + s, 2 * kStageBytes);
                    tma_load_3d_pair(st, &tm_x, full + s, kb * kBK, m0 + 128 * (int)rank, 0);
                    tma_load_3d_pair(st + kABytes, &tm_w, full + s, kb * kBK, n0 + 128 * (int)rank, 0);
                    if constexpr (kTf32) {
                        tma_load_3d_pair(st + C::kPart, &tm_x2, full + s, kb * kBK, m0 + 128 * (int)rank, 0);
                        tma_load_3d_pair(st + kABytes + C::kPart, &tm_w2, full + s, kb * kBK, n0 + 128 * (int)rank, 0);
                    }
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {   // ---------------- MMA issuer (leader, whole warp)
            const uint64_t d0 = sw128_desc(smem_u32(smem), 16, 1024);
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t aph = 0;
            for (int t = pair; t < tiles; t += npairs) {
                mbar_wait(acc_empty + acc, aph ^ 1);   // both CTAs drained this accumulator
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * kBN);
                for (int kb = 0; kb < nK; ++kb) {
                    mbar_wait(full + s, ph);
                    tc_fence_after();
                    const uint64_t da = desc_add(d0, s * kStageBytes);
                    const uint64_t db = desc_add(da, kABytes);
                    if constexpr (kTf32) {   // hi.lo + lo.hi + hi.hi, K = 8 fp32 per instruction
#pragma unroll
                        for (int pr = 0; pr < 3; ++pr) {
                            const uint32_t ap = pr == 1 ? C::kPart : 0u, bp = pr == 0 ? C::kPart : 0u;
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                umma_tf32_pair_w(d, desc_add(da, ap + kk * 32), desc_add(db, bp + kk * 32), kIdesc,
                                                 (kb | pr | kk) != 0);
                        }
                    } else {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            umma_f16_pair_w(d, desc_add(da, kk * 32), desc_add(db, kk * 32), kIdesc, (kb | kk) != 0);
                    }
                    umma_commit_pair_w(empty + s);   // the stage is free in both CTAs
                    if (++s == S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                umma_commit_pair_w(acc_full + acc);
                if (++acc == 2) {
                    acc = 0;
                    aph ^= 1;
                }
            }
        }
    } else {   // ---------------- epilogue (warps 2-5): this CTA's 128 rows x 256 columns
        const int quarter = warp & 3;
        const int et = threadIdx.x - 64;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t r = (uint32_t)(quarter * 32 + lane);
        const uint32_t release0 = cluster_addr(acc_empty, 0), release1 = cluster_addr(acc_empty + 1, 0);
        uint8_t* stage_out = smem + kSmemOut;
        int acc = 0, ob = 0;
        uint32_t aph = 0;
        for (int t = pair; t < tiles; t += npairs) {
            const int m0 = (t / nN) * 256 + 128 * (int)rank, n0 = (t % nN) * kBN;
            const int seg = n0 / a.HD;
            const CUtensorMap* om = seg == 0 ? &tm_o0 : seg == 1 ? &tm_o1 : &tm_o2;
            const int oc = n0 - seg * a.HD;
            const bool f16 = (a.f16_mask >> seg) & 1;
            mbar_wait(acc_full + acc, aph);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < kBN; c += C::kOutCols) {
                if (et == 0) {   // the store that used this buffer has read it (both when lo goes out too)
                    if (kTf32 && a.lo_tma) bulk_wait_read<0>();
                    else bulk_wait_read<kOutBufs - 1>();
                }
                named_bar_sync(1, 128);
                uint8_t* st = stage_out + ob * kOutBytes;
                if constexpr (kTf32) {   // 32 fp32 columns: one 128-byte row per thread (+ its lo parts)
                    uint32_t v[32];
                    tmem_ld32(lane_base + (uint32_t)(acc * kBN + c), v);
                    tmem_ld_wait();
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        *reinterpret_cast<uint4*>(st + sw128_offset(r, (uint32_t)g * 16)) =
                            make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                    if (a.lo_tma) {
                        uint8_t* sl = stage_out + (ob ^ 1) * kOutBytes;
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
                    fence_proxy_async_smem();
                    named_bar_sync(1, 128);
                    if (et == 0) {
                        tma_store_3d(om, st, oc + c, m0, 0);
                        if (a.lo_tma) tma_store_3d(&tm_o2, stage_out + (ob ^ 1) * kOutBytes, oc + c, m0, seg);
                        bulk_commit();
                    }
                    if (!a.lo_tma && ++ob == kOutBufs) ob = 0;
                    continue;
                }
                uint32_t v[2][32];
                tmem_ld32(lane_base + (uint32_t)(acc * kBN + c), v[0]);
                tmem_ld32(lane_base + (uint32_t)(acc * kBN + c + 32), v[1]);
                tmem_ld_wait();
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const uint32_t* src = &v[g >> 2][(g & 3) * 8];
                    uint4 u;
                    if (f16 && a.ovf.count) {   // fp16 range guard (H~ segments), as kp_project_tc
                        float fv[8];
                        bool big = false;
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            fv[e] = __uint_as_float(src[e]);
                            big |= f16_overflows(fv[e]);
                        }
                        const int tt = m0 + (int)r;
                        if (big && tt < a.M) {
                            const int col = oc + c + 8 * g, hh = col / kDh, bb = tt / a.n, j = tt - bb * a.n;
                            const long long tokh = ((long long)bb * (a.HD / kDh) + hh) * a.n + j;
                            if (!a.exact || a.exact[tokh]) {
                                const unsigned long long pos = atomicAdd(a.ovf.count, 1ull);
                                if (pos < (unsigned long long)a.ovf.cap) {
                                    a.ovf.list[pos] = tokh * 8 + ((col % kDh) >> 3);
#pragma unroll
                                    for (int e = 0; e < 8; ++e) a.ovf.rows[pos * 8 + e] = fv[e];
                                }
                            }
                        }
                        if (big) {
                            u = make_uint4(0u, 0u, 0u, 0u);
                        } else {
                            u.x = pack_f16x2(fv[0], fv[1]);
                            u.y = pack_f16x2(fv[2], fv[3]);
                            u.z = pack_f16x2(fv[4], fv[5]);
                            u.w = pack_f16x2(fv[6], fv[7]);
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
                fence_proxy_async_smem();
                named_bar_sync(1, 128);
                if (et == 0) {
                    tma_store_3d(om, st, oc + c, m0, 0);   // rows past M are clipped by the tensor map
                    bulk_commit();
                }
                if (++ob == kOutBufs) ob = 0;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc == 0 ? release0 : release1);   // the leader's acc_empty
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
        if (et == 0) bulk_wait<0>();
    }
    tc_fence_before();
    cluster_sync();   // no CTA leaves while its pair may still use its barriers / TMEM
    if (warp == 1) tmem_dealloc2<512>(tmem);
}

}  // namespace mca_dev

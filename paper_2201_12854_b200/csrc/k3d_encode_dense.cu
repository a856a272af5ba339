// k3d_encode_dense.cu — sampled encodings on the tensor cores ("densified").
//
// Same estimator as k3_encode_sampled, regrouped:
//   H~[j] = sum_k X[j, s_k] / (r_j p(s_k)) W_h[s_k] = C[j, :] . W_h,
//   C[j, i] = sum_{k : s_k = i} X[j, i] / (r_j p(i))        (sparse, ~r_j nonzeros)
// A persistent CTA owns one head: W_h (d_in x 64 bf16, MN-major 128B-swizzled
// chunks of 64 rows) arrives once by TMA and stays in shared memory. Per tile
// of 64 tokens of the head's budget-sorted list:
//   1. zero the tile (64 x d_in, 128B-swizzled K-major: the UMMA A operand)
//   2. every lane draws its own samples (Philox4x32-10 + guide-table inverse
//      CDF: the same draws as the gather kernel) and counts them: one 32-bit
//      shared atomic on the 16-bit count of (token, row). No X is read here,
//      so the draw loop has no global-memory latency in it.
//   3. scale in place: C[m, i] = bf16(count * x[m, i] * (1/p_i) * (1/r_m)),
//      reading X only for 16-byte chunks that hold a nonzero count (coalesced
//      row pieces instead of one scattered gather per draw)
//   4. one thread issues tcgen05.mma M=64 N=64 K=16 over C and W_h, fp32 in TMEM
//   5. warps 0-3 read the 64 rows back (M=64 layout: row m in TMEM lane
//      (m % 16) + 32 (m / 16)) and write H~ in bf16
// Per draw this costs one Philox half-call, the search and one shared atomic,
// instead of a 128-byte W_h row read and 64 FMAs; the contraction with W_h
// runs on the tensor core (2 * 64 * 64 * d_in flops per tile). Counts are
// exact integers, so the result is independent of the atomics' order; each
// coefficient is rounded to bf16 once (relative 2^-9), within the bf16 path's
// tolerance. The fp32 parity path keeps the gather kernel.
#include "mca_common.cuh"
#include "tc_common.cuh"

namespace mca_dev {

namespace k3d {
constexpr int kBM = 64;                   // tokens per tile (UMMA M)
constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kBK = 64;                   // K rows per swizzle atom / W_h chunk
constexpr uint32_t kAtomBytes = kBM * 128;       // one 64-column atom of C: 8 KB
constexpr uint32_t kWChunkBytes = kBK * kDh * 2; // 8 KB
constexpr int kGuideD = 11;                      // guide table (2048 buckets) rebuilt at this size
constexpr uint32_t kIdesc = mca_tc::idesc_f16(1, 1, kBM, kDh);   // bf16, B (W_h) MN-major
__host__ __device__ constexpr uint32_t smem_bytes(int d_in) {
    return (uint32_t)(2 * ((d_in + 63) / 64) * 8192 + d_in * 12 + (1 << kGuideD) * 2 + 256 + 1024);
}
}  // namespace k3d

__device__ __forceinline__ void atomic_add_bf16_smem(uint32_t addr, float v) {
    const __nv_bfloat16 b = __float2bfloat16_rn(v);
    asm volatile("red.shared.add.noftz.bf16 [%0], %1;" ::"r"(addr), "h"(*reinterpret_cast<const unsigned short*>(&b))
                 : "memory");
}

__global__ void __launch_bounds__(k3d::kThreads, 1)
    k3d_encode_dense(K3Args a, const __grid_constant__ CUtensorMap tm_w) {
    using namespace k3d;
    using namespace mca_tc;
    const int h = blockIdx.y;
    const int nsamp = a.counts[2 * h];
    const int ntiles = (nsamp + kBM - 1) / kBM;
    if ((int)blockIdx.x >= ntiles) return;       // uniform early exit
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int d_in = a.d_in, n = a.n, heads = a.heads;
    const int natoms = (d_in + 63) / 64;
    uint8_t* wbuf = smem;                                              // natoms x 8 KB (W_h, resident)
    uint8_t* cbuf = smem + natoms * kWChunkBytes;                      // natoms x 8 KB (C tile)
    uint64_t* s_thr = reinterpret_cast<uint64_t*>(cbuf + natoms * kAtomBytes);
    float* s_invp = reinterpret_cast<float*>(s_thr + d_in);
    uint16_t* s_guide = reinterpret_cast<uint16_t*>(s_invp + d_in);
    uint64_t* bars = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(s_guide + (1 << kGuideD)) + 7) & ~uintptr_t(7));
    uint64_t* w_full = bars;
    uint64_t* acc_full = bars + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tid = threadIdx.x;

    if (tid == 0) {
        mbar_init(w_full, 1);
        mbar_init(acc_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<64>(tmem_slot);
    for (int i = tid; i < d_in; i += k3d::kThreads) {
        s_thr[i] = a.thr[(size_t)h * d_in + i];
        s_invp[i] = a.invp[(size_t)h * d_in + i];
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (tid == 0) {   // W_h -> smem once (overlaps the guide-table build and the first tile's draws)
        tma_prefetch(&tm_w);
        mbar_expect_tx(w_full, natoms * kWChunkBytes);
        for (int c = 0; c < natoms; ++c) tma_load_3d(wbuf + c * kWChunkBytes, &tm_w, w_full, h * kDh, c * kBK, 0);
    }
    for (int g = tid; g < (1 << kGuideD); g += k3d::kThreads) {   // first i with thr[i] > g * 2^(53 - kGuideD)
        const uint64_t key = (uint64_t)g << (53 - kGuideD);
        int lo = 0, hi = d_in - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s_thr[mid] > key) hi = mid; else lo = mid + 1;
        }
        s_guide[g] = (uint16_t)lo;
    }

    const int32_t* list = a.samp_list + (size_t)h * a.tokens;
    const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(a.x);
    const uint32_t cbase = smem_u32(cbuf);
    unsigned long long my_samples = 0;
    uint32_t acc_phase = 0;

    __shared__ int s_bj[kBM];
    __shared__ int s_r[kBM];
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // 1. zero the tile; fetch the tile's list entries and budgets once
        for (uint32_t off = tid * 16; off < natoms * kAtomBytes; off += k3d::kThreads * 16)
            *reinterpret_cast<uint4*>(cbuf + off) = make_uint4(0, 0, 0, 0);
        if (tid < kBM) {
            const int e = tile * kBM + tid;
            const int bj = e < nsamp ? list[e] : -1;
            s_bj[tid] = bj;
            s_r[tid] = bj >= 0 ? a.budgets[((size_t)(bj >> 16) * heads + h) * n + (bj & 0xFFFF)] : 0;
        }
        __syncthreads();
        // 2. draws -> counts (16-bit, at the element's position in the swizzled tile)
        for (int m = warp; m < kBM; m += kWarps) {
            const int bj = s_bj[m];
            if (bj < 0) break;                       // warp-uniform (entries are contiguous)
            const int b = bj >> 16, j = bj & 0xFFFF;
            const int r = s_r[m];
            const size_t tokh = ((size_t)b * heads + h) * n + j;
            const uint64_t stream = ((uint64_t)(a.b_offset + b) * heads + h) * (uint64_t)n + (uint64_t)j;
            const uint32_t row_off = cbase + (uint32_t)(m >> 3) * 1024u + (uint32_t)(m & 7) * 128u;
            const uint32_t sw = (uint32_t)(m & 7);
            for (int base = 0; base < r; base += 64) {
                uint64_t m0, m1;
                philox_pair53(a.seed, stream, a.layer, (uint32_t)(base / 2 + lane), &m0, &m1);
                const int k0 = base + 2 * lane;
                int i0 = s_guide[(uint32_t)(m0 >> (53 - kGuideD))], i1 = s_guide[(uint32_t)(m1 >> (53 - kGuideD))];
                bool a0 = s_thr[i0] <= m0, a1 = s_thr[i1] <= m1;
                while (a0 || a1) {
                    if (a0) a0 = s_thr[++i0] <= m0;
                    if (a1) a1 = s_thr[++i1] <= m1;
                }
                if (k0 < r) {
                    const uint32_t ad = row_off + (uint32_t)(i0 >> 6) * kAtomBytes +
                                        ((((uint32_t)(i0 & 63) >> 3) ^ sw) << 4) + (uint32_t)(i0 & 7) * 2;
                    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(ad & ~3u), "r"(1u << ((ad & 2u) * 8)) : "memory");
                    if (a.draws_out && k0 < a.draws_stride) a.draws_out[tokh * a.draws_stride + k0] = i0;
                }
                if (k0 + 1 < r) {
                    const uint32_t ad = row_off + (uint32_t)(i1 >> 6) * kAtomBytes +
                                        ((((uint32_t)(i1 & 63) >> 3) ^ sw) << 4) + (uint32_t)(i1 & 7) * 2;
                    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(ad & ~3u), "r"(1u << ((ad & 2u) * 8)) : "memory");
                    if (a.draws_out && k0 + 1 < a.draws_stride) a.draws_out[tokh * a.draws_stride + k0 + 1] = i1;
                }
            }
            if (lane == 0) my_samples += (unsigned long long)r;
            if (a.draws_out)
                for (int k = r + lane; k < a.draws_stride; k += 32) a.draws_out[tokh * a.draws_stride + k] = -1;
        }
        __syncthreads();
        // 3. counts -> coefficients in place; X read only where a chunk has a count
        {
            constexpr int kChunksPerRow = 8;                    // 16-byte chunks per 128-byte row of an atom
            const int nwork = kBM * natoms * kChunksPerRow;     // (row, atom, chunk)
            for (int base = 0; base < nwork; base += k3d::kThreads * 4) {
                uint4 cnt[4], xv[4];
                uint32_t adr[4];
                int col[4], row[4];
                bool live[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {                   // pass A: read counts, issue X loads
                    const int wi = base + u * k3d::kThreads + tid;
                    live[u] = false;
                    if (wi >= nwork) continue;
                    const int atom = wi / (kBM * kChunksPerRow);
                    const int rem = wi - atom * (kBM * kChunksPerRow);
                    const int m = rem / kChunksPerRow, q = rem - m * kChunksPerRow;
                    row[u] = m;
                    col[u] = atom * 64 + q * 8;
                    adr[u] = (uint32_t)atom * kAtomBytes + (uint32_t)(m >> 3) * 1024u + (uint32_t)(m & 7) * 128u +
                             (((uint32_t)q ^ (uint32_t)(m & 7)) << 4);
                    cnt[u] = *reinterpret_cast<const uint4*>(cbuf + adr[u]);
                    live[u] = (cnt[u].x | cnt[u].y | cnt[u].z | cnt[u].w) != 0u;
                    if (live[u]) {
                        const int bj = s_bj[m];
                        const __nv_bfloat16* xr = x + ((size_t)(bj >> 16) * n + (bj & 0xFFFF)) * d_in;
                        xv[u] = *reinterpret_cast<const uint4*>(xr + col[u]);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {                   // pass B: scale and store bf16
                    if (!live[u]) continue;
                    const float inv_r = 1.0f / (float)s_r[row[u]];
                    const uint32_t cw[4] = {cnt[u].x, cnt[u].y, cnt[u].z, cnt[u].w};
                    const uint32_t xw[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
                    uint32_t outw[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int i = col[u] + 2 * e;
                        const float c0 = (float)(cw[e] & 0xFFFFu), c1 = (float)(cw[e] >> 16);
                        const float x0 = __uint_as_float(xw[e] << 16), x1 = __uint_as_float(xw[e] & 0xFFFF0000u);
                        outw[e] = pack_bf16x2(c0 * x0 * s_invp[i] * inv_r, c1 * x1 * s_invp[i + 1] * inv_r);
                    }
                    *reinterpret_cast<uint4*>(cbuf + adr[u]) = make_uint4(outw[0], outw[1], outw[2], outw[3]);
                }
            }
        }
        fence_proxy_async_smem();                     // C (generic-proxy writes) -> tensor core (async proxy)
        __syncthreads();
        // 3. H~ tile = C . W_h
        if (tid == 0) {
            mbar_wait(w_full, 0);
            tc_fence_after();
            for (int c = 0; c < natoms; ++c) {
                const uint32_t a_addr = cbase + c * kAtomBytes;
                const uint32_t b_addr = smem_u32(wbuf + c * kWChunkBytes);
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk)
                    umma_f16(tmem, sw128_desc(a_addr + kk * 32, 16, 1024), sw128_desc(b_addr + kk * 2048, 8192, 1024),
                             kIdesc, (c > 0 || kk > 0) ? 1u : 0u);
            }
            umma_commit(acc_full);
        }
        // 4. epilogue: warps 0-3, lanes 0-15 (M = 64 accumulator layout)
        if (warp < 4) {
            mbar_wait(acc_full, acc_phase);
            tc_fence_after();
            uint32_t v[2][32];
            const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
            tmem_ld32(lane_base, v[0]);
            tmem_ld32(lane_base + 32, v[1]);
            tmem_ld_wait();
            const int m = warp * 16 + lane;
            const int bj = lane < 16 ? s_bj[m] : -1;
            if (bj >= 0) {
                const size_t tok = (size_t)(bj >> 16) * n + (bj & 0xFFFF);
                __half* dst = reinterpret_cast<__half*>(a.h_out) + tok * (size_t)heads * kDh + (size_t)h * kDh;
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    uint32_t pk[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c = g * 8 + 2 * q;
                        pk[q] = pack_f16x2(__uint_as_float(v[c >> 5][c & 31]),
                                           __uint_as_float(v[(c + 1) >> 5][(c + 1) & 31]));
                    }
                    reinterpret_cast<uint4*>(dst)[g] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
            }
            tc_fence_before();
        }
        acc_phase ^= 1;
        __syncthreads();   // C and the accumulator are free for the next tile
    }
    if (a.sample_counter) {
        for (int off = 16; off; off >>= 1) my_samples += __shfl_xor_sync(0xffffffffu, my_samples, off);
        if (lane == 0 && my_samples) atomicAdd(a.sample_counter, my_samples);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<64>(tmem);
}

}  // namespace mca_dev

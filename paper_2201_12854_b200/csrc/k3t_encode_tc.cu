// k3t_encode_tc.cu — K3 for the bf16 path on the tensor cores: every
// token-head's encoding (sampled and exact) as one tile GEMM.
//
// The estimator of SPEC.md:221-229, 238 (Eq. 5), regrouped by row:
//   H~[j] = (1/r_j) sum_k X[j, s_k] / p(s_k) W_h[s_k]
//         = (1/r_j) sum_i  c_ji X[j, i] . W'[i],    W'[i] = W_h[i] / p(i)
// with c_ji the number of draws of row i for token j (an exact integer, so
// the result does not depend on the order the draws are counted in). An exact
// token-head (r_j >= d, Eq. 9) is H~[j] = X[j] W_h = sum_i (X[j, i] p(i)) W'[i].
// W' (bf16, per head) and bf16 p are built once with the weights (K0).
//
// A CTA owns one head (W'_h resident in shared memory, 96 KB at d_in = 768)
// and walks tiles of 64 consecutive tokens j of one sequence b. Per tile:
//   setup    warp 0 reads the 64 budgets / exact flags, compacts the sampled
//            rows and prefix-sums their draw pairs (one Philox call = 2 draws)
//   draw     512 threads take the tile's draw pairs in flat order (no lane
//            idles on a token boundary): Philox4x32-10, guide-table inverse
//            CDF (the same draws as the oracle, bit for bit), and one shared
//            atomic on the 16-bit count c_ji
//   convert  per 64-column chunk of the tile: A = bf16(c * x) (one HFMA2.BF16,
//            exact product rounded once), or bf16(x * p) for exact rows; the
//            count tile is zeroed as it is read; chunks stream through a
//            2-slot ring to the tensor core
//   MMA      one thread: tcgen05.mma M=64 N=64 K=16 (bf16 in, fp32 in TMEM),
//            4 per chunk, double-buffered accumulators
//   epilogue the previous tile's accumulator x (1/r or 1) -> fp16 H~
// The 12 CTAs of a head advance over the same sequences together, so the X
// rows a tile reads (64 x d_in bf16) are shared through L2 by all heads.
// Per draw: half a Philox call, the guide-table search and one shared atomic;
// per (token, input row): ~2 instructions of the convert pass; the
// contraction (2 * 64 * 64 * d_in flops per tile) is on the tensor core.
#include "mca_common.cuh"
#include "tc_common.cuh"

namespace mca_dev {

namespace k3t {
constexpr int kBM = 64;                          // tokens per tile (UMMA M)
constexpr int kWorkers = 16;                     // setup / draw / convert / epilogue warps
constexpr int kWorkerThreads = kWorkers * 32;
constexpr int kThreads = kWorkerThreads + 32;    // + the TMA / MMA warp
constexpr uint32_t kChunkBytes = kBM * 128;      // one 64-column chunk of the tile: 8 KB
constexpr uint32_t kIdesc = mca_tc::idesc_f16(1, 1, kBM, kDh);   // bf16 x bf16, B (W') MN-major
constexpr int kPre = kBM + 33;                   // pair prefix + padding read by the lane search
constexpr int kMaxAtoms = 12;                    // d_in <= 768: X row chunks a convert thread holds
constexpr int kGuideBitsT = 12;                  // coarser guide table in smem: every 4th entry of K0's
constexpr int kGuideT = 1 << kGuideBitsT;

struct Plan {                     // one tile's draw plan (double-buffered)
    int rb[kBM];                  // budgets of sampled rows (0 otherwise)
    int pre[kPre];                // exclusive prefix of draw pairs over compacted sampled rows, padded
    uint8_t cm[kBM];              // compacted index -> tile row
    int total;                    // draw pairs in the tile
};
struct Meta {
    uint64_t bars[5];             // w_full, a_full, a_free, acc_full[2]
    uint64_t acc_empty[2];
    float scale[3][kBM];          // epilogue row scale: 1/r (sampled), 1 (exact), 0 (no row)
    uint8_t kind[3][kBM];         // 0 none, 1 sampled, 2 exact
    Plan plan[2];
    uint32_t tmem_slot;
};

struct Layout {
    uint32_t natoms, dpad, w, tile, thr, guide, pbf, meta, bytes;
};
__host__ __device__ inline Layout layout(int d_in) {
    Layout L;
    L.natoms = (uint32_t)(d_in + 63) / 64;
    L.dpad = L.natoms * 64;
    L.w = 0;                                               // W'_h: natoms x [64 rows x 64 cols] (MN-major B)
    L.tile = L.natoms * 8192u;                             // counts, then A in place: natoms x [64 x 64] (K-major A)
    L.thr = L.tile + L.natoms * kChunkBytes;
    L.guide = L.thr + (((uint32_t)d_in * 8u + 15u) & ~15u);
    L.pbf = L.guide + kGuideT * 2u;
    L.meta = L.pbf + L.dpad * 2u;
    L.bytes = L.meta + (uint32_t)((sizeof(Meta) + 15) & ~(size_t)15) + 1024u;   // + alignment slack
    if (L.natoms > (uint32_t)kMaxAtoms) L.bytes = 0xFFFFFFFFu;                   // not supported: gather path
    return L;
}
}  // namespace k3t

// +1 on the 16-bit count at shared address `addr` (no carry: counts <= r < 2^16).
__device__ __forceinline__ void red_count16(uint32_t addr) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr & ~3u), "r"(1u << ((addr & 2u) * 8u)) : "memory");
}

__device__ __forceinline__ uint32_t bf2_as_u32(__nv_bfloat162 v) { return *reinterpret_cast<uint32_t*>(&v); }
__device__ __forceinline__ __nv_bfloat162 u32_as_bf2(uint32_t u) { return *reinterpret_cast<__nv_bfloat162*>(&u); }

// bf16(c * x) for two packed 16-bit counts c < 128 and two bf16 x: (128 + c) is
// exact in bf16 (0x4300 | c), and fma((128 + c), x, -128 x) rounds c * x once.
__device__ __forceinline__ uint32_t count_times_x(uint32_t c2, uint32_t x2) {
    const __nv_bfloat162 x = u32_as_bf2(x2);
    const __nv_bfloat162 nx = __hmul2(x, __floats2bfloat162_rn(-128.f, -128.f));
    return bf2_as_u32(__hfma2(u32_as_bf2(c2 | 0x43004300u), x, nx));
}
// Same products for any counts (exact in fp32: c < 2^16, x has 8 significant
// bits). Rare (a count >= 128), so kept out of line: the compiler must not
// if-convert it into the common path.
__device__ __noinline__ uint4 count_times_x_wide(uint4 c, uint4 x) {
    const uint32_t cw[4] = {c.x, c.y, c.z, c.w}, xw[4] = {x.x, x.y, x.z, x.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
        o[e] = mca_tc::pack_bf16x2((float)(cw[e] & 0xFFFFu) * __uint_as_float(xw[e] << 16),
                                   (float)(cw[e] >> 16) * __uint_as_float(xw[e] & 0xFFFF0000u));
    return make_uint4(o[0], o[1], o[2], o[3]);
}

// Byte offset of tile element (row m, column i) in the chunked 128B-swizzled layout.
__device__ __forceinline__ uint32_t tile_offset(uint32_t m, uint32_t i) {
    return (i >> 6) * k3t::kChunkBytes + (m >> 3) * 1024u + (m & 7u) * 128u + ((((i & 63u) >> 3) ^ (m & 7u)) << 4) +
           (i & 7u) * 2u;
}

#ifndef MCA_K3T_PROF
#define MCA_K3T_PROF 0
#endif
constexpr bool kK3tProf = MCA_K3T_PROF;   // build with -DMCA_K3T_PROF=1 for per-phase clocks (MCA_K3_PROF=1)
constexpr int kPreDraw = 4;   // draw pairs per thread computed ahead, while the previous tile's MMAs run

__global__ void __launch_bounds__(k3t::kThreads, 1)
    k3t_encode_tc(K3Args a, const __grid_constant__ CUtensorMap tm_w, const __nv_bfloat16* __restrict__ pbf_g) {
    using namespace k3t;
    using namespace mca_tc;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment by pointer arithmetic on the shared array itself, so
    // every access below compiles to LDS/STS (not generic loads)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int d_in = a.d_in, n = a.n, heads = a.heads;
    const Layout L = layout(d_in);
    Meta& M = *reinterpret_cast<Meta*>(smem + L.meta);
    uint64_t* w_full = M.bars;
    uint64_t* a_full = M.bars + 1;     // workers -> MMA: the tile's A is complete
    uint64_t* a_free = M.bars + 2;     // MMA -> workers: the tile's MMAs finished reading A
    uint64_t* acc_full = M.bars + 3;   // [2]
    uint64_t* acc_empty = M.acc_empty; // [2]
    uint64_t* s_thr = reinterpret_cast<uint64_t*>(smem + L.thr);
    uint16_t* s_guide = reinterpret_cast<uint16_t*>(smem + L.guide);
    __nv_bfloat16* s_pbf = reinterpret_cast<__nv_bfloat16*>(smem + L.pbf);
    uint8_t* s_tile = smem + L.tile;
    const uint32_t tile_base = smem_u32(s_tile);

    const int h = blockIdx.y;
    const int ntj = (n + kBM - 1) / kBM;
    const int ntiles = (int)(a.tokens / n) * ntj;          // B * ntj < 2^31 (B, n <= 65535)
    const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tid = threadIdx.x;

    auto tile_coords = [&](int i, int& b, int& j0) {
        const int tt = (int)blockIdx.x + i * (int)gridDim.x;
        b = tt / ntj;
        j0 = (tt - b * ntj) * kBM;
    };
    // warp 0: a tile's budgets / exact flags (rows lane and lane + 32)
    auto load_plan = [&](int i, int (&r)[2], int (&ex)[2]) {
        int b, j0;
        tile_coords(i, b, j0);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = j0 + lane + 32 * u;
            r[u] = -1;
            ex[u] = 0;
            if (i < my_tiles && j < n) {
                const size_t idx = ((size_t)b * heads + h) * n + j;
                r[u] = __ldg(a.budgets + idx);
                ex[u] = __ldg(a.exact + idx);
            }
        }
    };
    unsigned long long my_samples = 0;
    // warp 0: publish tile i's plan (compaction of sampled rows + prefix of their draw pairs)
    auto setup = [&](int i, const int (&r)[2], const int (&ex)[2]) {
        int b, j0;
        tile_coords(i, b, j0);
        const int buf = i % 3;
        Plan& P = M.plan[i & 1];
        int pr[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int m = lane + 32 * u;
            const int kd = r[u] < 0 ? 0 : (ex[u] ? 2 : 1);
            M.kind[buf][m] = (uint8_t)kd;
            M.scale[buf][m] = kd == 1 ? 1.0f / (float)r[u] : (kd == 2 ? 1.0f : 0.0f);
            P.rb[m] = kd == 1 ? r[u] : 0;
            pr[u] = kd == 1 ? (r[u] + 1) >> 1 : 0;
            if (kd == 1) my_samples += (unsigned long long)r[u];
            if (a.draws_out && kd) {      // entries this tile never writes read -1
                int32_t* dr = a.draws_out + (((size_t)b * heads + h) * n + j0 + m) * a.draws_stride;
                for (int k = kd == 1 ? r[u] : 0; k < a.draws_stride; ++k) dr[k] = -1;
            }
        }
        const unsigned lt = (1u << lane) - 1u;
        const unsigned bal0 = __ballot_sync(0xffffffffu, pr[0] > 0), bal1 = __ballot_sync(0xffffffffu, pr[1] > 0);
        int s0 = pr[0], s1 = pr[1];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t0 = __shfl_up_sync(0xffffffffu, s0, off), t1 = __shfl_up_sync(0xffffffffu, s1, off);
            if (lane >= off) {
                s0 += t0;
                s1 += t1;
            }
        }
        const int tot0 = __shfl_sync(0xffffffffu, s0, 31), tot1 = __shfl_sync(0xffffffffu, s1, 31);
        const int n0 = __popc(bal0), ms = n0 + __popc(bal1);
        if (pr[0]) {
            const int c = __popc(bal0 & lt);
            P.cm[c] = (uint8_t)lane;
            P.pre[c] = s0 - pr[0];
        }
        if (pr[1]) {
            const int c = n0 + __popc(bal1 & lt);
            P.cm[c] = (uint8_t)(lane + 32);
            P.pre[c] = tot0 + s1 - pr[1];
        }
        for (int k = ms + lane; k < kPre; k += 32) P.pre[k] = k == ms ? tot0 + tot1 : 0x7FFFFFFF;
        if (lane == 0) P.total = tot0 + tot1;
    };

    int nr[2], nex[2];
    if (tid == 0) {
        mbar_init(w_full, 1);
        mbar_init(a_full, kWorkerThreads);
        mbar_init(a_free, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(acc_full + s, 1);
            mbar_init(acc_empty + s, kWorkerThreads);
        }
        fence_barrier_init();
    }
    if (warp == kWorkers) {
        tmem_alloc<128>(&M.tmem_slot);
    } else {
        for (int i = tid; i < d_in; i += kWorkerThreads) s_thr[i] = a.thr[(size_t)h * d_in + i];
        for (int g = tid; g < kGuideT; g += kWorkerThreads)   // coarse entries, clean bits masked off
            s_guide[g] = a.guide[(size_t)h * kGuide + ((size_t)g << (kGuideBits - kGuideBitsT))] & kGuideRow;
        for (int i = tid; i < (int)L.dpad; i += kWorkerThreads)
            s_pbf[i] = i < d_in ? pbf_g[(size_t)h * d_in + i] : __float2bfloat16(0.f);
        if (warp == 0 && my_tiles > 0) {
            load_plan(0, nr, nex);
            setup(0, nr, nex);
            load_plan(1, nr, nex);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = M.tmem_slot;

    if (warp == kWorkers) {
        if (lane == 0 && my_tiles > 0) {   // ---------------- W'_h once, then one MMA batch per tile
            tma_prefetch(&tm_w);
            mbar_expect_tx(w_full, L.natoms * 8192u);
            for (uint32_t c = 0; c < L.natoms; ++c) tma_load_3d(smem + L.w + c * 8192u, &tm_w, w_full, h * kDh, c * 64, 0);
            mbar_wait(w_full, 0);
            for (int i = 0; i < my_tiles; ++i) {
                const int ab = i & 1;
                mbar_wait(acc_empty + ab, ((i >> 1) & 1) ^ 1);
                mbar_wait(a_full, i & 1);
                tc_fence_after();
                for (uint32_t c = 0; c < L.natoms; ++c) {
                    const uint32_t a_addr = tile_base + c * kChunkBytes;
                    const uint32_t b_addr = smem_u32(smem + L.w + c * 8192u);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_f16(tmem + ab * kDh, sw128_desc(a_addr + kk * 32, 16, 1024),
                                 sw128_desc(b_addr + kk * 2048, 8192, 1024), kIdesc, (c | kk) ? 1u : 0u);
                }
                umma_commit(a_free);
                umma_commit(acc_full + ab);
            }
        }
    } else {
        const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(a.x);
        __half* hout = reinterpret_cast<__half*>(a.h_out);
        const size_t HD = (size_t)heads * kDh;
        const bool prof = kK3tProf && a.prof && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0;
        auto stamp = [&](int i, int k) {
            if constexpr (kK3tProf)
                if (prof && i < 64) a.prof[i * 8 + k] = clock64();
        };

        auto epilogue = [&](int i) {
            int b, j0;
            tile_coords(i, b, j0);
            const int ab = i & 1, buf = i % 3;
            mbar_wait(acc_full + ab, (i >> 1) & 1);
            tc_fence_after();
            const int qd = warp & 3, part = warp >> 2;   // TMEM lane quadrant, 16-column part
            uint32_t v[16];
            tmem_ld16(tmem + ((uint32_t)(qd * 32) << 16) + ab * kDh + part * 16, v);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(acc_empty + ab);
            const int m = qd * 16 + lane;                 // M = 64 layout: row m in lane (m % 16) + 32 (m / 16)
            if (lane < 16 && M.kind[buf][m]) {
                const float sc = M.scale[buf][m];
                uint32_t pk[8];
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    pk[e] = pack_f16x2(__uint_as_float(v[2 * e]) * sc, __uint_as_float(v[2 * e + 1]) * sc);
                uint4* dst = reinterpret_cast<uint4*>(hout + ((size_t)b * n + j0 + m) * HD + (size_t)h * kDh + part * 16);
                dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            }
        };
        // One draw pair f of the tile: Philox + inverse CDF. Returns the pair packed
        // as m | i0 << 6 | i1 << 16 | second << 26 (i < 1024: d_in <= 768 here).
        auto draw_pair = [&](const Plan& P, int b, int j0, int f0) -> uint32_t {
            // compacted row k of pair f = f0 + lane: rows whose prefix is <= f
            const int kf = __popc(__ballot_sync(0xffffffffu, P.pre[1 + lane] <= f0)) +
                           __popc(__ballot_sync(0xffffffffu, P.pre[33 + lane] <= f0));
            const int nb = P.pre[kf + 1 + lane] - f0;   // > 0: start offsets of later rows
            const unsigned starts = __reduce_or_sync(0xffffffffu, nb < 32 ? (1u << nb) : 0u);
            const int k = kf + __popc(starts & ((2u << lane) - 1u));
            const int f = f0 + lane;
            if (f >= P.total) return 0xFFFFFFFFu;
            const int m = P.cm[k], p = f - P.pre[k], r = P.rb[m];
            const uint64_t stream = ((uint64_t)(a.b_offset + b) * heads + h) * (uint64_t)n + (uint64_t)(j0 + m);
            uint64_t m0, m1;
            philox_pair53(a.seed, stream, a.layer, (uint32_t)p, &m0, &m1);
            int i0, i1;
            sample_index2<kGuideBitsT>(s_thr, s_guide, m0, m1, i0, i1);
            const bool second = 2 * p + 1 < r;
            if (a.draws_out) {
                int32_t* dr = a.draws_out + (((size_t)b * heads + h) * n + j0 + m) * a.draws_stride;
                if (2 * p < a.draws_stride) dr[2 * p] = i0;
                if (second && 2 * p + 1 < a.draws_stride) dr[2 * p + 1] = i1;
            }
            return (uint32_t)m | ((uint32_t)i0 << 6) | ((uint32_t)i1 << 16) | ((uint32_t)second << 26);
        };
        auto count_pair = [&](uint32_t pk) {
            if (pk == 0xFFFFFFFFu) return;
            const uint32_t m = pk & 63u;
            red_count16(tile_base + tile_offset(m, (pk >> 6) & 1023u));
            if (pk & (1u << 26)) red_count16(tile_base + tile_offset(m, (pk >> 16) & 1023u));
        };

        for (int i = 0; i < my_tiles; ++i) {
            int b, j0;
            tile_coords(i, b, j0);
            const int buf = i % 3;
            const Plan& P = M.plan[i & 1];
            stamp(i, 0);
            // ---------------- draw ahead (registers): overlaps tile i-1's MMAs
            uint32_t pk[kPreDraw];
#pragma unroll
            for (int u = 0; u < kPreDraw; ++u) pk[u] = draw_pair(P, b, j0, warp * 32 + u * kWorkerThreads);
            stamp(i, 1);
            // ---------------- the tile's X pieces (thread: row m, 16-byte column piece g of every chunk)
            const int m = tid >> 3, g = tid & 7;
            const int kd = M.kind[buf][m];
            const __nv_bfloat16* xrow = x + ((size_t)b * n + j0 + m) * d_in;
            uint4 xs[kMaxAtoms];
#pragma unroll
            for (int c = 0; c < kMaxAtoms; ++c)
                xs[c] = (kd && c < (int)L.natoms && c * 64 + 8 * g < d_in)
                            ? __ldg(reinterpret_cast<const uint4*>(xrow + c * 64 + 8 * g))
                            : make_uint4(0, 0, 0, 0);
            // ---------------- warp 0 publishes the next tile's plan meanwhile
            if (warp == 0 && i + 1 < my_tiles) {
                setup(i + 1, nr, nex);
                load_plan(i + 2, nr, nex);
            }
            // ---------------- tile buffer free once tile i-1's MMAs are done: zero it
            if (i >= 1) {
                if (tid == 0) mbar_wait(a_free, (i - 1) & 1);
            }
            named_bar_sync(2, kWorkerThreads);
            stamp(i, 2);
            for (uint32_t off = tid * 16u; off < L.natoms * kChunkBytes; off += kWorkerThreads * 16u)
                *reinterpret_cast<uint4*>(s_tile + off) = make_uint4(0, 0, 0, 0);
            named_bar_sync(1, kWorkerThreads);
            stamp(i, 3);
            // ---------------- counts: the pairs drawn ahead, then the rest of the tile
#pragma unroll
            for (int u = 0; u < kPreDraw; ++u) count_pair(pk[u]);
            for (int f0 = warp * 32 + kPreDraw * kWorkerThreads; f0 < P.total; f0 += kWorkerThreads)
                count_pair(draw_pair(P, b, j0, f0));
            named_bar_sync(1, kWorkerThreads);
            stamp(i, 4);
            // ---------------- convert in place: counts (+ X) -> bf16 A
            if (kd) {
                uint8_t* tp = s_tile + sw128_offset((uint32_t)m, (uint32_t)g * 16u);
#pragma unroll
                for (int c = 0; c < kMaxAtoms; ++c) {
                    if (c >= (int)L.natoms) break;
                    uint8_t* tc = tp + c * kChunkBytes;
                    const uint4 xv = xs[c];
                    uint4 o;
                    if (kd == 1) {
                        const uint4 cn = *reinterpret_cast<const uint4*>(tc);
                        const uint32_t any = cn.x | cn.y | cn.z | cn.w;
                        if (!any) continue;                          // all-zero counts are already bf16 zeros
                        if (!(any & 0xFF80FF80u)) {
                            o.x = count_times_x(cn.x, xv.x);
                            o.y = count_times_x(cn.y, xv.y);
                            o.z = count_times_x(cn.z, xv.z);
                            o.w = count_times_x(cn.w, xv.w);
                        } else {
                            o = count_times_x_wide(cn, xv);
                        }
                    } else {
                        const uint4 pv = *reinterpret_cast<const uint4*>(s_pbf + c * 64 + 8 * g);
                        o.x = bf2_as_u32(__hmul2(u32_as_bf2(xv.x), u32_as_bf2(pv.x)));
                        o.y = bf2_as_u32(__hmul2(u32_as_bf2(xv.y), u32_as_bf2(pv.y)));
                        o.z = bf2_as_u32(__hmul2(u32_as_bf2(xv.z), u32_as_bf2(pv.z)));
                        o.w = bf2_as_u32(__hmul2(u32_as_bf2(xv.w), u32_as_bf2(pv.w)));
                    }
                    *reinterpret_cast<uint4*>(tc) = o;
                }
            }
            fence_proxy_async_smem();
            mbar_arrive(a_full);
            stamp(i, 5);
            // ---------------- epilogue of tile i-1 (complete: its MMAs freed the buffer)
            if (i >= 1) epilogue(i - 1);
            stamp(i, 6);
        }
        if (my_tiles > 0) epilogue(my_tiles - 1);
        if (a.sample_counter && warp == 0) {
            for (int off = 16; off; off >>= 1) my_samples += __shfl_xor_sync(0xffffffffu, my_samples, off);
            if (lane == 0 && my_samples) atomicAdd(a.sample_counter, my_samples);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kWorkers) tmem_dealloc<128>(tmem);
}

// K0 extension for the bf16 path: W' = W_h / p (0 where p = 0) and bf16 p.
__global__ void k0_wprime(const __nv_bfloat16* __restrict__ w, const double* __restrict__ probs, int d_in, int heads,
                          __nv_bfloat16* __restrict__ wp, __nv_bfloat16* __restrict__ pbf) {
    const int HD = heads * kDh;
    const size_t total = (size_t)d_in * HD;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / HD), col = (int)(e % HD), h = col / kDh;
        const double p = probs[(size_t)h * d_in + i];
        wp[e] = p > 0.0 ? __double2bfloat16((double)__bfloat162float(w[e]) / p) : __float2bfloat16(0.f);
        if (col % kDh == 0) pbf[(size_t)h * d_in + i] = __double2bfloat16(p);
    }
}

}  // namespace mca_dev

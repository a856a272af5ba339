// k3_encode.cu — K3: the MCA value encoding (gather-scale-accumulate).
//
// For every token-head (b, j, h) with budget r_j:
//   exact_mask: H~[j] = X[j] . W_h
//   otherwise:  H~[j] = sum_k X[j, s_k] / (r_j p(s_k)) * W_h[s_k]
// with s_k = first i such that thr_h[i] > m_k, m_k = draw k of Philox stream
// ((b_offset + b) * heads + h) * n + j, layer `layer`.
//
// Layout / scheduling:
//   - grid = (G, heads); a CTA owns one head: W_h (d_in x 64) is staged in
//     shared memory once with 16-byte coalesced loads, together with the
//     sampler tables (53-bit thresholds, 1024-entry guide table, 1/p).
//   - CTAs pull 64-token chunks of their head from a per-head atomic counter.
//     Each chunk is rank-sorted by budget (exact tokens first) so the four
//     tokens a warp processes together have similar sample counts, and warps
//     pull groups of 4 tokens in that order (LPT): tokens bucketed by sample
//     count keep warps balanced.
//   - An octet of 8 lanes encodes one token; lane l owns output columns
//     [8l, 8l+8). Per round the octet draws 16 samples (8 Philox calls, 2
//     53-bit draws each), resolves them with the guide table, then all 8 lanes
//     walk the 16 samples in draw order: one 16/32-byte shared-memory load of
//     the sampled W_h row and 8 FMAs per lane per sample.
// The fp32 path (Acc = double) forms each coefficient exactly as the oracle
// does, x / (r * p) in binary64, and accumulates in fp64; the bf16 path uses
// fp32 coefficients x * (1/p) * (1/r) and fp32 accumulation.
#include "mca_common.cuh"

namespace mca_dev {

constexpr int kChunk = 64;   // tokens per chunk
constexpr int kK3Threads = 256;

template <class T>
struct CoefT;  // per-index factor kept in shared memory
template <>
struct CoefT<float> { using type = double; };          // p(i) in fp64 (exact oracle coefficient)
template <>
struct CoefT<__nv_bfloat16> { using type = float; };   // 1/p(i) in fp32

__device__ __forceinline__ void load8w(const __nv_bfloat16* p, float v[8]) { load8(p, v); }
__device__ __forceinline__ void load8w(const float* p, float v[8]) { load8(p, v); }

template <class T, class Acc, bool kWSmem>
__global__ void __launch_bounds__(kK3Threads) k3_encode(
    const T* __restrict__ x, const T* __restrict__ wv, int d_in, int heads, int n, int B, long b_offset,
    uint32_t layer, uint64_t seed, const int32_t* __restrict__ budgets, const uint8_t* __restrict__ exact,
    const uint64_t* __restrict__ thr_all, const uint16_t* __restrict__ guide_all,
    const double* __restrict__ probs_all, const float* __restrict__ invp_all, T* __restrict__ h_out,
    int32_t* __restrict__ draws_out, int draws_stride, unsigned long long* __restrict__ sample_counter,
    int* __restrict__ chunk_counter) {
    using Coef = typename CoefT<T>::type;
    extern __shared__ __align__(16) unsigned char smem[];
    const int h = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31;
    const int oct = lane >> 3, l8 = lane & 7;
    const unsigned omask = 0xFFu << (oct * 8);

    // ---- shared memory carve-up
    uint64_t* s_thr = reinterpret_cast<uint64_t*>(smem);
    Coef* s_coef = reinterpret_cast<Coef*>(s_thr + d_in);
    uint16_t* s_guide = reinterpret_cast<uint16_t*>(s_coef + d_in);
    int* s_order = reinterpret_cast<int*>(s_guide + kGuide);
    int* s_key = s_order + kChunk;
    int* s_misc = s_key + kChunk;  // [0] chunk id, [1] group counter
    T* s_w = reinterpret_cast<T*>(smem + ((((size_t)d_in * (8 + sizeof(Coef)) + kGuide * 2 + (2 * kChunk + 4) * 4) + 127) & ~(size_t)127));

    const size_t HD = (size_t)heads * kDh;
    for (int i = tid; i < d_in; i += kK3Threads) {
        s_thr[i] = thr_all[(size_t)h * d_in + i];
        if constexpr (sizeof(Coef) == 8) s_coef[i] = (Coef)probs_all[(size_t)h * d_in + i];
        else s_coef[i] = (Coef)invp_all[(size_t)h * d_in + i];
    }
    for (int g = tid; g < kGuide; g += kK3Threads) s_guide[g] = guide_all[(size_t)h * kGuide + g];
    if constexpr (kWSmem) {
        constexpr int kVec = 16 / sizeof(T);            // elements per 16-byte vector
        const int vecs_per_row = kDh / kVec;
        for (int e = tid; e < d_in * vecs_per_row; e += kK3Threads) {
            const int i = e / vecs_per_row, v = e % vecs_per_row;
            reinterpret_cast<uint4*>(s_w + (size_t)i * kDh)[v] =
                reinterpret_cast<const uint4*>(wv + (size_t)i * HD + (size_t)h * kDh)[v];
        }
    }
    const T* wsrc = kWSmem ? s_w : (wv + (size_t)h * kDh);
    const size_t wstride = kWSmem ? (size_t)kDh : HD;

    const int chunks_per_seq = (n + kChunk - 1) / kChunk;
    const int nchunks = B * chunks_per_seq;
    unsigned long long my_samples = 0;

    for (;;) {
        __syncthreads();  // previous chunk fully consumed (and tables staged on the first pass)
        if (tid == 0) {
            s_misc[0] = atomicAdd(chunk_counter + h, 1);
            s_misc[1] = 0;
        }
        __syncthreads();
        const int c = s_misc[0];
        if (c >= nchunks) break;
        const int b = c / chunks_per_seq, j0 = (c % chunks_per_seq) * kChunk;
        const size_t tok_base = ((size_t)b * heads + h) * n;  // [B, H, n] index of token 0

        // rank-sort the chunk by cost: exact tokens first, then budget descending
        if (tid < kChunk) {
            const int j = j0 + tid;
            int key = -1;
            if (j < n) key = exact[tok_base + j] ? (1 << 30) : budgets[tok_base + j];
            s_key[tid] = key;
        }
        __syncthreads();
        if (tid < kChunk) {
            const int key = s_key[tid];
            int rank = 0;
            for (int u = 0; u < kChunk; ++u) {
                const int ku = s_key[u];
                rank += (ku > key) || (ku == key && u < tid);
            }
            s_order[rank] = tid;
        }
        __syncthreads();

        for (;;) {
            int grp = 0;
            if (lane == 0) grp = atomicAdd(&s_misc[1], 1);
            grp = __shfl_sync(0xffffffffu, grp, 0);
            if (grp * 4 >= kChunk) break;
            const int t = s_order[grp * 4 + oct];
            const int j = j0 + t;
            if (s_key[t] < 0) continue;  // padding past n (octet-uniform)
            const size_t tok = tok_base + j;
            const int r = budgets[tok];
            const bool ex = exact[tok] != 0;
            const T* xrow = x + ((size_t)b * n + j) * d_in;
            Acc acc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] = (Acc)0;

            if (ex) {
                for (int i0 = 0; i0 < d_in; i0 += 8) {
                    const float xv = (i0 + l8 < d_in) ? to_f32(xrow[i0 + l8]) : 0.0f;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float xi = __shfl_sync(omask, xv, u, 8);
                        if (i0 + u < d_in) {
                            float wr[8];
                            load8w(wsrc + (size_t)(i0 + u) * wstride + 8 * l8, wr);
#pragma unroll
                            for (int q = 0; q < 8; ++q) acc[q] += (Acc)xi * (Acc)wr[q];
                        }
                    }
                }
                if (draws_out && l8 == 0)
                    for (int k = 0; k < draws_stride; ++k) draws_out[tok * draws_stride + k] = -1;
            } else {
                const uint64_t stream = ((uint64_t)(b_offset + b) * heads + h) * (uint64_t)n + (uint64_t)j;
                const float inv_r = 1.0f / (float)r;
                const double rd = (double)r;
                for (int base = 0; base < r; base += 16) {
                    uint64_t m0, m1;
                    philox_pair53(seed, stream, layer, (uint32_t)(base / 2 + l8), &m0, &m1);
                    const int k0 = base + 2 * l8, k1 = k0 + 1;
                    int i0 = 0, i1 = 0;
                    Acc c0 = 0, c1 = 0;
                    if (k0 < r) {
                        i0 = sample_index(s_thr, s_guide, m0);
                        const float xv = to_f32(xrow[i0]);
                        if constexpr (sizeof(Coef) == 8) c0 = (Acc)__ddiv_rn((double)xv, __dmul_rn(rd, (double)s_coef[i0]));
                        else c0 = (Acc)(xv * (float)s_coef[i0] * inv_r);
                    }
                    if (k1 < r) {
                        i1 = sample_index(s_thr, s_guide, m1);
                        const float xv = to_f32(xrow[i1]);
                        if constexpr (sizeof(Coef) == 8) c1 = (Acc)__ddiv_rn((double)xv, __dmul_rn(rd, (double)s_coef[i1]));
                        else c1 = (Acc)(xv * (float)s_coef[i1] * inv_r);
                    }
                    if (draws_out) {
                        if (k0 < r && k0 < draws_stride) draws_out[tok * draws_stride + k0] = i0;
                        if (k1 < r && k1 < draws_stride) draws_out[tok * draws_stride + k1] = i1;
                    }
                    const int cnt = min(16, r - base);
                    for (int s = 0; s < cnt; ++s) {
                        const int src = s >> 1;
                        const int idx = __shfl_sync(omask, (s & 1) ? i1 : i0, src, 8);
                        const Acc cf = __shfl_sync(omask, (s & 1) ? c1 : c0, src, 8);
                        float wr[8];
                        load8w(wsrc + (size_t)idx * wstride + 8 * l8, wr);
#pragma unroll
                        for (int q = 0; q < 8; ++q) acc[q] += cf * (Acc)wr[q];
                    }
                    if (l8 == 0) my_samples += (unsigned long long)cnt;
                }
                if (draws_out && l8 == 0)
                    for (int k = r; k < draws_stride; ++k) draws_out[tok * draws_stride + k] = -1;
            }
            float o[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) o[u] = (float)acc[u];
            T* dst = h_out + ((size_t)b * n + j) * HD + (size_t)h * kDh + 8 * l8;
            store8(dst, o);
        }
    }
    if (sample_counter) {
        for (int off = 16; off; off >>= 1) my_samples += __shfl_xor_sync(0xffffffffu, my_samples, off);
        if (lane == 0 && my_samples) atomicAdd(sample_counter, my_samples);
    }
}

size_t k3_smem_bytes(int d_in, size_t elem, size_t coef, bool wsmem) {
    size_t head = (((size_t)d_in * (8 + coef) + kGuide * 2 + (2 * kChunk + 4) * 4) + 127) & ~(size_t)127;
    return head + (wsmem ? (size_t)d_in * kDh * elem : 0);
}

#define MCA_K3_INST(T, A, S)                                                                                       \
    template __global__ void k3_encode<T, A, S>(const T*, const T*, int, int, int, int, long, uint32_t, uint64_t,    \
                                                const int32_t*, const uint8_t*, const uint64_t*, const uint16_t*,    \
                                                const double*, const float*, T*, int32_t*, int, unsigned long long*, \
                                                int*);
MCA_K3_INST(float, double, true)
MCA_K3_INST(float, double, false)
MCA_K3_INST(__nv_bfloat16, float, true)
MCA_K3_INST(__nv_bfloat16, float, false)

}  // namespace mca_dev

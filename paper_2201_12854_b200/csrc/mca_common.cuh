// mca_common.cuh — device primitives shared by the MCA kernels (sm_100a).
//
// Philox4x32-10 here is the device generator; the fp64 oracle has its own,
// independently written copy (oracle/sampling.cpp) and both are pinned to the
// Random123 known-answer vectors, so index parity GPU-vs-oracle is a real check.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mca_dev {

constexpr int kDh = 64;            // head dimension the kernels implement (BERT base/large)
constexpr int kGuideBits = 14;     // guide table: 16384 buckets over the 53-bit uniform (~21 per row at d = 768)
constexpr int kGuide = 1 << kGuideBits;
// Guide entry: bits 0-14 the first row whose threshold exceeds the bucket's
// lower end; bit 15 set when the whole bucket maps to that row ("clean":
// thr[row] >= the bucket's upper end), so the draw needs no threshold compare.
constexpr uint16_t kGuideClean = 0x8000u;   // the bucket lies inside one row: the entry is the answer
constexpr uint16_t kGuideOne = 0x4000u;     // the bucket holds exactly one row boundary: entry or entry + 1
constexpr uint16_t kGuideRow = 0x3FFFu;     // row bits (d_in <= 16384)

// ----------------------------------------------- programmatic dependent launch
// Kernels of the forward are launched with programmatic stream serialization
// (mca_capi.cu launch_pdl): a kernel may start while its predecessor drains.
// griddep_trigger() lets the next kernel launch; griddep_wait() blocks the
// calling thread until the predecessor grid has completed and its writes are
// visible, so it goes before the first read of a predecessor's output. Both
// are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// (b, h) row index of the [B*H]-row grids: gridDim.y caps at 65535, so the
// host splits B*H over (y, z) (bh_grid in mca_capi.cu); rows past B*H exit.
__device__ __forceinline__ long grid_bh() { return (long)blockIdx.z * gridDim.y + blockIdx.y; }

// ----------------------------------------------------------------- Philox
__device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                              uint32_t k1, uint32_t out[4]) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

// Draws 2*blk and 2*blk+1 of stream (seed, stream_id, layer) as 53-bit integers
// m (the uniform is m * 2^-53), DESIGN.md §3.
__device__ __forceinline__ void philox_pair53(uint64_t seed, uint64_t stream_id, uint32_t layer, uint32_t blk,
                                              uint64_t* m0, uint64_t* m1) {
    uint32_t x[4];
    philox4x32_10(blk, layer, (uint32_t)stream_id, (uint32_t)(stream_id >> 32), (uint32_t)seed,
                  (uint32_t)(seed >> 32), x);
    *m0 = ((((uint64_t)x[1]) << 32) | x[0]) >> 11;
    *m1 = ((((uint64_t)x[3]) << 32) | x[2]) >> 11;
}

// Inverse CDF: first i with thr[i] > m, thr[i] = ceil(cdf[i] * 2^53). The guide
// entry for m's top kGuideBits bits is a lower bound on the answer, so the
// forward scan returns exactly std::upper_bound(cdf, m * 2^-53).
// kBits < kGuideBits: a coarser table (entry g = entry g << (kGuideBits - kBits)
// of the full one, with the clean bits masked off: a fine bucket's flag says
// nothing about the coarse bucket containing it).
template <int kBits = kGuideBits>
__device__ __forceinline__ int sample_index(const uint64_t* __restrict__ thr, const uint16_t* __restrict__ guide,
                                            uint64_t m) {
    const uint32_t e = guide[(uint32_t)(m >> (53 - kBits))];
    int i = (int)(e & kGuideRow);
    if (e & kGuideClean) return i;
    while (thr[i] <= m) ++i;
    return i;
}
// Two draws resolved together. Clean buckets need no compare; a bucket with
// exactly one boundary needs one (branch-free); only buckets with several
// boundaries (rows of tiny p) fall into the scan loop.
template <int kBits = kGuideBits>
__device__ __forceinline__ void sample_index2(const uint64_t* __restrict__ thr, const uint16_t* __restrict__ guide,
                                              uint64_t m0, uint64_t m1, int& i0, int& i1) {
    const uint32_t e0 = guide[(uint32_t)(m0 >> (53 - kBits))], e1 = guide[(uint32_t)(m1 >> (53 - kBits))];
    i0 = (int)(e0 & kGuideRow);
    i1 = (int)(e1 & kGuideRow);
    if (e0 & e1 & kGuideClean) return;   // both buckets clean: no threshold compare
    if (!(e0 & kGuideClean)) i0 += thr[i0] <= m0;
    if (!(e1 & kGuideClean)) i1 += thr[i1] <= m1;
    if ((e0 & (kGuideClean | kGuideOne)) && (e1 & (kGuideClean | kGuideOne))) return;   // resolved
    bool a0 = !(e0 & (kGuideClean | kGuideOne)) && thr[i0] <= m0;   // several boundaries: keep scanning
    bool a1 = !(e1 & (kGuideClean | kGuideOne)) && thr[i1] <= m1;
    while (a0 || a1) {
        if (a0) a0 = thr[++i0] <= m0;
        if (a1) a1 = thr[++i1] <= m1;
    }
}

// ------------------------------------------------ order-preserving float keys
__device__ __forceinline__ uint32_t float_to_ordered(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ordered_to_float(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

// ------------------------------------------------------------ dtype helpers
template <class T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <class T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ uint32_t mca_pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

// Load 8 consecutive elements as floats (16 B for bf16, 32 B for f32).
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float v[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        v[2 * i] = __uint_as_float(w[i] << 16);
        v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}
__device__ __forceinline__ void load8(const float* p, float v[8]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0];
    const float4 b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float v[8]) {
    uint4 u;
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    u.x = w[0]; u.y = w[1]; u.z = w[2]; u.w = w[3];
    *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void store8(__half* p, const float v[8]) {
    uint4 u;
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    u.x = w[0]; u.y = w[1]; u.z = w[2]; u.w = w[3];
    *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void load8(const __half* p, float v[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}
template <>
__device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }

// H~ (the encodings) is fp32 on the fp32 path and fp16 on the bf16 path: fp16
// has 3 more mantissa bits than bf16 and feeds K4's fp16 x fp16 tensor-core
// P.H~ product, whose P comes straight out of ex2.approx.f16x2.
template <class T>
struct HType { using type = float; };
template <>
struct HType<__nv_bfloat16> { using type = __half; };

// ------------------------------------------------- fp16 H~ range guard
// H~ is stored as fp16 on the bf16 path (K4's fp16 x fp16 P.H~ product). A
// sampled contribution x[j,s] w[s] / (r p(s)) is unbounded (tiny p(s), outlier
// x), so an 8-column chunk of an encoding that leaves fp16's range is stored as
// zeros in H~ and its fp32 values are queued here; the fix-up adds P[:, j] times
// the chunk into y after the aggregation. Chunk-granular, so
// every lane decides alone (no warp collectives in the encoders' store path).
#ifndef MCA_F16_GUARD
#define MCA_F16_GUARD 1   // 0: diagnostics builds only (measures the guard's cost)
#endif
constexpr float kH16Max = 65504.f;
struct OvfSink {
    unsigned long long* count;       // queued chunks (zeroed per forward)
    long long* list;                 // [cap] (token-head t = (b H + h) n + j) * 8 + chunk (8 columns each)
    float* rows;                     // [cap][8] the fp32 values of each chunk
    int cap;
};
__device__ __forceinline__ bool f16_overflows(float v) { return !(fabsf(v) <= kH16Max); }   // also inf / NaN
// Queue chunk `chunk` (columns [8 chunk, 8 chunk + 8)) of token-head t if any
// of its 8 values leaves fp16's range; zero them in v (the fp16 store). Past
// the capacity the entry is dropped and the count still grows: the fix-up traps.
__device__ __forceinline__ void f16_guard8(const OvfSink& o, long long t, int chunk, float v[8]) {
#if MCA_F16_GUARD
    bool big = false;
#pragma unroll
    for (int u = 0; u < 8; ++u) big |= f16_overflows(v[u]);
    if (big) {
        const unsigned long long pos = atomicAdd(o.count, 1ull);
        if (pos < (unsigned long long)o.cap) {
            o.list[pos] = t * 8 + chunk;
#pragma unroll
            for (int u = 0; u < 8; ++u) o.rows[pos * 8 + u] = v[u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = 0.f;
    }
#endif
}

__device__ __forceinline__ void store8(float* p, const float v[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

}  // namespace mca_dev

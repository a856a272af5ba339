// ka_given_attn.cu — the layer on a GIVEN attention matrix (mca_forward_attn):
// what the reference's cli drives with imported or synthetic attention
// (cmd_bench / cmd_attn_import): the budgets come from the
// dump's column maxima and the aggregation multiplies by the dump itself,
// while the encoding is the same K3 / K3b path as the forward.
//
//   ka_colmax     cmax[b,h,j] = max_i A[b,h,i,j]  (col_max, matrix.hpp:52-53;
//                 exact: the fp64 entries themselves), then K2 (kGivenCmax)
//   ka_aggregate  y[b,i,h*64+c] = sum_j A[b,h,i,j] H~[b,j,h*64+c]
//                 (matmul(A, H~), matrix.hpp:33-34), fp64 accumulation
// Both are plain CUDA-core kernels: this path serves analysis of dumps at
// desk scale, not the BERT-shape hot path.
#include "mca_common.cuh"

namespace mca_dev {

// grid ((n + 31) / 32, B * H), block (32, 8): thread (x, y) = column j = 32 blockIdx.x + x
// over the rows i = y (mod 8) (a warp reads 256 contiguous bytes per row), then the
// eight partial maxima of each column meet in shared memory.
__global__ void __launch_bounds__(256) ka_colmax(const double* __restrict__ attn, int n, long bh_count,
                                                 double* __restrict__ cmax) {
    __shared__ double part[8][33];
    const long bh = grid_bh();
    const int j = blockIdx.x * 32 + threadIdx.x;
    if (bh >= bh_count) return;
    double m = -INFINITY;
    if (j < n) {
        const double* a = attn + (size_t)bh * n * n + j;
        double m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
        int i = threadIdx.y;
        for (; i + 24 < n; i += 32) {   // four independent loads in flight
            m = fmax(m, __ldg(a + (size_t)i * n));
            m1 = fmax(m1, __ldg(a + (size_t)(i + 8) * n));
            m2 = fmax(m2, __ldg(a + (size_t)(i + 16) * n));
            m3 = fmax(m3, __ldg(a + (size_t)(i + 24) * n));
        }
        for (; i < n; i += 8) m = fmax(m, __ldg(a + (size_t)i * n));
        m = fmax(fmax(m, m1), fmax(m2, m3));
    }
    part[threadIdx.y][threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.y == 0 && j < n) {
#pragma unroll
        for (int y = 1; y < 8; ++y) m = fmax(m, part[y][threadIdx.x]);
        cmax[(size_t)bh * n + j] = m;
    }
}

// grid (n, H, B), 64 threads: thread = output column c of row i, head h
template <class T, class HT>
__global__ void ka_aggregate(const double* __restrict__ attn, const HT* __restrict__ hbuf, int n, int heads,
                             T* __restrict__ y) {
    const int i = blockIdx.x, h = blockIdx.y, b = blockIdx.z, c = threadIdx.x;
    const size_t HD = (size_t)heads * kDh;
    const double* arow = attn + (((size_t)b * heads + h) * n + i) * n;
    const HT* hc = hbuf + (size_t)b * n * HD + (size_t)h * kDh + c;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc = fma(arow[j], (double)to_f32(hc[(size_t)j * HD]), acc);
    y[((size_t)b * n + i) * HD + (size_t)h * kDh + c] = from_f32<T>((float)acc);
}

}  // namespace mca_dev

// mca_diag.cuh — host-side dumps of the kernels' diagnostic timelines.
//
// Diagnostics builds only (make EXTRA=-DMCA_K12_PROF=1 etc.): each kernel
// then keeps clock64 / globaltimer stamps in a __device__ array, and the
// functions here synchronise the stream and print them to stderr. In the
// product build every MCA_*_PROF switch is 0, the device arrays shrink to one
// element, and these functions compile to nothing.
#pragma once

#include <cstdio>

namespace mca_diag {

#if MCA_K12_PROF
// CTA 0's group A / B block timeline, then every CTA's SM and start / end.
inline void dump_k12(cudaStream_t stream, int n, int grid) {
    long long t[256];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(t, mca_dev::g_k12_prof, sizeof(t));
    const int nb = ((n + 127) / 128) * ((n + 127) / 128), ntq = (n + 127) / 128;
    auto rel = [&](long long v) { return v ? v - t[0] : -1; };
    fprintf(stderr, "k12 CTA0: A end");
    for (int u = 0; u < 2 * nb && u < 39; ++u) fprintf(stderr, " %lld", rel(t[1 + u]));
    fprintf(stderr, " | B end");
    for (int u = 0; u < 2 * nb && u < 39; ++u) fprintf(stderr, " %lld", rel(t[40 + u]));
    fprintf(stderr, " | Bdone %lld end %lld\n", rel(t[79]), rel(t[80]));
    fprintf(stderr, "k12 CTA0 A issue/wait/ld0/ld1/end:");
    for (int u = 0; u < 2 * nb && u < 32; ++u)
        fprintf(stderr, " %lld/%lld/%lld/%lld/%lld", rel(t[192 + u]), rel(t[96 + u]), rel(t[128 + u]),
                rel(t[160 + u]), rel(t[1 + u]));
    fprintf(stderr, " | lse");
    for (int q = 0; q < 2 * ntq && q < 32; ++q) fprintf(stderr, " %lld", rel(t[224 + q]));
    fprintf(stderr, "\n");
    static unsigned long long c[4096][4];
    const int nc = grid < 4096 ? grid : 4096;
    cudaMemcpyFromSymbol(c, mca_dev::g_k12_cta, sizeof(unsigned long long) * 4 * nc);
    unsigned long long t0 = ~0ull;
    for (int i = 0; i < nc; ++i) t0 = c[i][1] < t0 ? c[i][1] : t0;
    fprintf(stderr, "k12 CTAS");
    for (int i = 0; i < nc; ++i) fprintf(stderr, " %llu:%llu:%llu:%llu", c[i][0], c[i][1] - t0, c[i][2] - t0, c[i][3]);
    fprintf(stderr, "\n");
}
#else
inline void dump_k12(cudaStream_t, int, int) {}
#endif

#if MCA_K3S_PROF
// Per head: the last prologue end, the first and the last CTA exit (us).
inline void dump_k3s(cudaStream_t stream, int ctas, int heads) {
    static unsigned long long c[1024][4];
    const int nc = ctas < 1024 ? ctas : 1024;
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(c, mca_dev::g_k3s_cta, sizeof(unsigned long long) * 4 * nc);
    unsigned long long t0 = ~0ull;
    for (int i = 0; i < nc; ++i) t0 = c[i][0] < t0 ? c[i][0] : t0;
    fprintf(stderr, "k3s heads (prologue end, first exit, last exit in us):");
    for (int hh = 0; hh < heads; ++hh) {
        unsigned long long pe = 0, e0 = ~0ull, e1 = 0;
        for (int i = 0; i < nc; ++i)
            if ((int)c[i][3] == hh) {
                pe = c[i][1] - t0 > pe ? c[i][1] - t0 : pe;
                e0 = c[i][2] - t0 < e0 ? c[i][2] - t0 : e0;
                e1 = c[i][2] - t0 > e1 ? c[i][2] - t0 : e1;
            }
        fprintf(stderr, " | h%d %.1f %.1f %.1f", hh, pe / 1e3, e0 / 1e3, e1 / 1e3);
    }
    fprintf(stderr, "\n");
}
#else
inline void dump_k3s(cudaStream_t, int, int) {}
#endif

#if MCA_K3B_PROF
inline void dump_k3b(cudaStream_t stream) {
    long long t[64];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(t, mca_dev::g_k3b_prof, sizeof(t));
    fprintf(stderr, "k3b CTA0: waited %lld | landed", t[1] - t[0]);
    for (int c = 0; c < 12; ++c) fprintf(stderr, " %lld", t[2 + c] - t[0]);
    fprintf(stderr, " | mma");
    for (int c = 0; c < 12; ++c) fprintf(stderr, " %lld", t[20 + c] - t[0]);
    fprintf(stderr, " | acc %lld end %lld\n", t[40] - t[0], t[41] - t[0]);
}
#else
inline void dump_k3b(cudaStream_t) {}
#endif

#if MCA_K4_PROF
inline void dump_k4(cudaStream_t stream, int n, int block_keys) {
    long long t[64];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(t, mca_dev::g_k4_prof, sizeof(t));
    fprintf(stderr, "k4 CTA0 (2nd tile): start->softmax %lld |", t[0] - t[60]);
    for (int kb = 0; kb < (n + block_keys - 1) / block_keys && kb < 16; ++kb)
        fprintf(stderr, " kb%d S@%lld P@%lld done@%lld", kb, t[1 + 3 * kb] - t[60], t[2 + 3 * kb] - t[60],
                t[3 + 3 * kb] - t[60]);
    fprintf(stderr, " | O@%lld end@%lld\n", t[50] - t[60], t[51] - t[60]);
}
#else
inline void dump_k4(cudaStream_t, int, int) {}
#endif

#if MCA_K3T_PROF
// k3t phase clocks (MCA_K3_PROF=1 at run time): allocate before the launch,
// print the mean cycles per tile of CTA 0 after it.
inline long long* k3t_prof_begin(cudaStream_t stream) {
    if (!getenv("MCA_K3_PROF")) return nullptr;
    long long* p = nullptr;
    if (cudaMalloc(&p, 64 * 8 * sizeof(long long)) != cudaSuccess) return nullptr;
    cudaMemsetAsync(p, 0, 64 * 8 * sizeof(long long), stream);
    return p;
}
inline void k3t_prof_end(cudaStream_t stream, long long* pbuf) {
    if (!pbuf) return;
    long long h[64 * 8];
    cudaMemcpyAsync(h, pbuf, sizeof(h), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    cudaFree(pbuf);
    double acc[7] = {};
    int nt = 0;
    for (int i = 1; i < 64 && h[i * 8]; ++i, ++nt) {
        for (int k = 0; k < 6; ++k) acc[k] += (double)(h[i * 8 + k + 1] - h[i * 8 + k]);
        if (i + 1 < 64 && h[(i + 1) * 8]) acc[6] += (double)(h[(i + 1) * 8] - h[i * 8]);
    }
    if (nt)
        fprintf(stderr, "k3t CTA0 mean cycles/tile over %d tiles: predraw %.0f xload+setup+afree %.0f zero %.0f count %.0f "
                        "convert %.0f epi %.0f | tile %.0f\n", nt, acc[0] / nt, acc[1] / nt, acc[2] / nt,
                acc[3] / nt, acc[4] / nt, acc[5] / nt, acc[6] / (nt > 1 ? nt - 1 : 1));
}
#else
inline long long* k3t_prof_begin(cudaStream_t) { return nullptr; }
inline void k3t_prof_end(cudaStream_t, long long*) {}
#endif

}  // namespace mca_diag

// mca_capi.cu — host side of the C ABI (include/mca/mca_cuda.h).
//
// Owns the prepared weights and the forward's workspace, validates arguments
// into SPEC error classes, and enqueues K0..K4 on the caller's stream. There
// is no CPU compute path: every stage of the forward runs on the GPU, and a
// missing device is reported as MCA_ERR_CUDA.
//
// Unity build: the kernel translation units are included here so one nvcc
// invocation produces libmca_b200.so (no relocatable device code needed).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "mca/mca_cuda.h"

#include "k0_weights.cu"
#include "k1_scores_simt.cu"
#include "k1_scores_tc.cu"
#include "k2_budgets.cu"
#include "k12_fused_tc.cu"
#include "k3_encode.cu"
#include "k3b_exact_tc.cu"
#include "k3t_encode_tc.cu"
#include "k4_apply_simt.cu"
#include "k4_apply_tc.cu"
#include "k4_apply_tf32.cu"
#include "kp_project_tc.cu"
#include "kp_project_pair.cu"
#include "ka_given_attn.cu"
#include "ka_aggregate_tc.cu"
#include "mca_diag.cuh"

#ifndef MCA_K2_FUSED_SCAN
#define MCA_K2_FUSED_SCAN 1   // work lists by one scan + scatter kernel
#endif
#ifndef MCA_K3_SPECIALIZE
#define MCA_K3_SPECIALIZE 1   // d_in = 768 / 1024 encoders with compile-time table offsets
#endif

using namespace mca_dev;

namespace {

thread_local std::string g_err;

mca_status fail(mca_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define MCA_CUDA_TRY(expr)                                                                                   \
    do {                                                                                                     \
        cudaError_t e_ = (expr);                                                                             \
        if (e_ != cudaSuccess)                                                                               \
            return fail(MCA_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

#define MCA_LAUNCH_CHECK(name)                                                                               \
    do {                                                                                                     \
        cudaError_t e_ = cudaGetLastError();                                                                 \
        if (e_ != cudaSuccess) return fail(MCA_ERR_CUDA, "launch of %s failed: %s", name, cudaGetErrorString(e_)); \
        ++launches;                                                                                          \
    } while (0)

size_t dtype_size(mca_dtype t) { return t == MCA_BF16 ? 2 : 4; }

constexpr int kCertCounter = 6;                // counters[6]: k2c-flagged token-heads spilled past their item's slots
constexpr int kCertTotal = 4;                  // counters[4]: token-heads k2c re-derived (FlopsReport.certified)
constexpr int kOvfCounter = 7;                 // counters[7]: fp16-overflowing encodings queued for k4o_overflow
constexpr int kK4DoneCounter = 5;              // counters[5]: K4 CTAs finished (its last CTA runs the range-guard fix-up)
constexpr long kOvfCap = 1 << 18;              // queue capacity (8-column chunks per forward)
constexpr size_t kMaxGraphs = 256;              // captured forwards kept per handle (LRU)

// Per-device facts and settings. Everything here is keyed by the current
// device: one process may drive several GPUs (one handle per device), and
// kernel attributes such as the >48 KB shared-memory opt-in are per device.
int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

int sm_count() {
    static std::mutex mu;
    static std::map<int, int> by_dev;
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu);
    auto it = by_dev.find(dev);
    if (it != by_dev.end()) return it->second;
    int c = 0;
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    if (c <= 0) c = 148;
    by_dev[dev] = c;
    return c;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel),
// raised when a launch needs more than the last setting.
cudaError_t ensure_smem(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> set;
    const auto key = std::make_pair(current_device(), fn);
    std::lock_guard<std::mutex> lock(mu);
    auto it = set.find(key);
    if (it != set.end() && it->second >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) set[key] = bytes;
    return e;
}
template <class F>
cudaError_t ensure_smem(F* fn, size_t bytes) {
    return ensure_smem(reinterpret_cast<const void*>(fn), bytes);
}

// [B*H]-row grid: x covers a row's tokens, (y, z) the B*H rows (grid_bh()).
dim3 bh_grid(unsigned x, long bh) {
    const unsigned y = (unsigned)std::min<long>(bh, 65535);
    return dim3(x, y, (unsigned)((bh + y - 1) / y));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D bf16 view [batch][rows][inner] with a {64, box_rows, 1} box and 128-byte
// swizzle: the UMMA operand layout of tc_common.cuh. Rows past `rows` read as 0.
bool make_tmap_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t batch,
                    uint32_t box_rows, CUtensorMapDataType type = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {inner, rows, batch};
    cuuint64_t strides[2] = {inner * 2, rows * inner * 2};
    cuuint32_t box[3] = {64, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, type, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D fp32 view [batch][rows][inner] with a {32, box_rows, 1} box (128 bytes) and
// 128-byte swizzle: the tf32 operand atoms of k1_scores_tc<*, true>.
// H~ transposed per head, [BH][64][n_pad] fp32 (k_split_transpose_h / k_transpose_h16): box {32 keys, 64 dims}
bool make_vt_map(CUtensorMap* m, const float* base, int n, int n_pad, long BH) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)kDh, (cuuint64_t)BH};
    cuuint64_t strides[2] = {(cuuint64_t)n_pad * 4, (cuuint64_t)kDh * n_pad * 4};
    cuuint32_t box[3] = {32, 64, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_f32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t batch, uint32_t box_rows) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {inner, rows, batch};
    cuuint64_t strides[2] = {inner * 4, rows * inner * 4};
    cuuint32_t box[3] = {32, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// MCA_K3_TILE=1 selects the tile-GEMM encoder (k3t) on the bf16 path; the
// default there is the gather-scale-accumulate encoder + exact tensor-core
// kernel (measured faster at BERT shapes).
bool tile_k3_requested() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MCA_K3_TILE");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

bool force_simt() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MCA_FORCE_SIMT");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

}  // namespace

struct mca_weights {
    int d_in = 0, heads = 0, dh = 0;
    mca_dtype wdt = MCA_F32;
    int device = 0;
    void* w = nullptr;            // [d_in, heads*dh] copy of W_V
    double* probs = nullptr;      // [heads, d_in]
    double* cdf = nullptr;        // [heads, d_in]
    uint64_t* thr = nullptr;      // [heads, d_in]
    float* invp = nullptr;        // [heads, d_in]
    uint16_t* guide = nullptr;    // [heads, kGuide]
    void* wprime = nullptr;       // bf16 path: [d_in, heads*dh] W_h / p (k3t's B operand)
    void* wqkv_t = nullptr;       // [3*heads*dh][d_in] W_q^T | W_k^T | W_V^T (kp_project_tc's K-major B): bf16, or
                                  // for fp32 the tf32-exact hi parts, with the lo parts in wqkv_t_lo
    void* wqkv_t_lo = nullptr;
    void* x_split = nullptr;      // fp32 path: x - hi(x) [B*n, d_in] (3xTF32 projection lo part; x is the hi part)
    long cap_x = 0;
    bool has_qk_t = false;        // the W_q^T | W_k^T rows are set (mca_set_projections)
    void* qk = nullptr;           // [2][B*n][heads*dh] projected q, k (workspace, grown on demand)
    long cap_qk = 0;
    void* pbf = nullptr;          // bf16 path: [heads, d_in] bf16 p
    // workspace (grown on demand)
    long cap_tokens = 0;          // capacity in B*n tokens
    float* lse = nullptr;                     // [B, H, n]
    double* row_m = nullptr;                  // [B, H, n] row max of the scaled scores
    double* row_l = nullptr;                  // [B, H, n] row sum of exp(t - m)
    unsigned long long* colkey = nullptr;     // [B, H, n]
    float* colscore = nullptr;                // [B, H, n] winning raw score (tensor-core score pass)
    int32_t* budgets = nullptr;               // [B, H, n]
    uint8_t* exact = nullptr;                 // [B, H, n]
    void* hbuf = nullptr;                     // [B, n, H*dh]
    int32_t* samp_list = nullptr;             // [H, B*n] sampled tokens per head, budget-descending
    int32_t* exact_list = nullptr;            // [H, B*n] exact tokens per head
    long long* cert_list = nullptr;           // [B, H, n] Eq. 9 values at an integer boundary (k2c_certify)
    double* cert_cm = nullptr;                // [B, H, n] the score pass's cmax of each flagged entry
    unsigned* cert_item_cnt = nullptr;        // [B*H] flagged keys per item (k2c)
    int* cert_slot_j = nullptr;               // [B*H][kCertSlots]
    double* cert_slot_cm = nullptr;           // [B*H][kCertSlots]
    long cap_items = 0;
    long long* ovf_list = nullptr;            // [kOvfCap] fp16-overflowing 8-column chunks (bf16 path)
    float* ovf_rows = nullptr;                // [kOvfCap][8] their fp32 values
    void* qk_split = nullptr;                 // fp32 path: q_lo | k_lo [B, n, H*64] (3xTF32; q, k are the hi parts)
    float* vt_split = nullptr;                // fp32 path: H~ transposed hi | lo [B*H][64][n_pad] (K4 3xTF32)
    size_t cap_vt = 0;                        // floats
    long ovf_cap = 0;
    uint8_t* row_done = nullptr;              // [B, H, n] k2c's exact row-statistics cache flags
    void* zeroed = nullptr;                   // counters | task_cursor | hist | fill (zeroed once per forward)
    unsigned int* fill = nullptr;             // [H, d + 1] per-bin list fill counters (k2_scan_scatter)
    unsigned long long* counters = nullptr;   // [8]
    unsigned int* hist = nullptr;             // [H, d_in + 1] budget histogram
    unsigned int* cursor = nullptr;           // [H, d_in + 1] scatter cursors
    int* counts = nullptr;                    // [H, 2] sampled / exact token counts
    int* task_cursor = nullptr;               // [2][H] K3 work cursors
    unsigned* k12_tail = nullptr;             // K12 split items: [SMs][kMaxTiles*128 + 2], zero between launches
    // timing
    bool timing = false;
    cudaEvent_t ev[6] = {};   // stage boundaries: projection | score | budgets | encoding | aggregation
    // MCA_GRAPHS=1: CUDA graphs of repeated identical forwards (key = every argument).
    // The first call of a key runs eagerly (it may size buffers), the second is
    // captured, later ones replay the graph: one launch instead of ~10.
    struct GraphEntry {
        uint64_t key[16];
        uint64_t last_use = 0;        // LRU clock
        bool graphable = true;        // false after a failed capture: always eager
        cudaGraphExec_t exec = nullptr;
    };
    std::vector<GraphEntry> graphs;
    uint64_t graph_clock = 0;
    bool ev_valid = false;
    int last_launches = 0;
};

namespace {

void free_workspace(mca_weights* w) {
    cudaFree(w->lse);
    cudaFree(w->row_m);
    cudaFree(w->row_l);
    cudaFree(w->colkey);
    cudaFree(w->colscore);
    cudaFree(w->budgets);
    cudaFree(w->exact);
    cudaFree(w->hbuf);
    cudaFree(w->samp_list);
    cudaFree(w->exact_list);
    cudaFree(w->cert_list);
    cudaFree(w->cert_cm);
    w->cert_cm = nullptr;
    cudaFree(w->cert_item_cnt);
    cudaFree(w->cert_slot_j);
    cudaFree(w->cert_slot_cm);
    w->cert_item_cnt = nullptr;
    w->cert_slot_j = nullptr;
    w->cert_slot_cm = nullptr;
    w->cap_items = 0;
    cudaFree(w->ovf_list);
    cudaFree(w->ovf_rows);
    cudaFree(w->qk_split);
    w->qk_split = nullptr;
    cudaFree(w->vt_split);
    w->vt_split = nullptr;
    w->cap_vt = 0;
    w->ovf_list = nullptr;
    w->ovf_rows = nullptr;
    w->ovf_cap = 0;
    cudaFree(w->row_done);
    w->cert_list = nullptr;
    w->row_done = nullptr;
    w->samp_list = nullptr;
    w->exact_list = nullptr;
    w->lse = nullptr;
    w->row_m = nullptr;
    w->row_l = nullptr;
    w->colkey = nullptr;
    w->colscore = nullptr;
    w->budgets = nullptr;
    w->exact = nullptr;
    w->hbuf = nullptr;
    w->cap_tokens = 0;
}

// Captured forwards point into the workspace: drop them when it moves.
void drop_graphs(mca_weights* w) {
    for (auto& g : w->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    w->graphs.clear();
}

mca_status ensure_workspace(mca_weights* w, long tokens, mca_stream_t stream) {
    if (tokens <= w->cap_tokens) return MCA_OK;
    if (w->cap_tokens) MCA_CUDA_TRY(cudaStreamSynchronize(stream));  // old buffers may still be in use
    drop_graphs(w);
    free_workspace(w);
    const size_t th = (size_t)tokens * w->heads;
    if (cudaMalloc(&w->lse, th * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&w->row_m, th * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&w->row_l, th * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&w->colkey, th * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&w->colscore, th * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&w->budgets, th * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&w->exact, th * sizeof(uint8_t)) != cudaSuccess ||
        cudaMalloc(&w->hbuf, th * w->dh * dtype_size(w->wdt)) != cudaSuccess ||
        cudaMalloc(&w->samp_list, th * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&w->exact_list, th * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&w->cert_list, th * sizeof(long long)) != cudaSuccess ||
        cudaMalloc(&w->cert_cm, th * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&w->ovf_list, std::min<long>(8L * (long)th, kOvfCap) * sizeof(long long)) != cudaSuccess ||
        cudaMalloc(&w->ovf_rows, std::min<long>(8L * (long)th, kOvfCap) * 8 * sizeof(float)) != cudaSuccess ||
        (w->wdt == MCA_F32 && cudaMalloc(&w->qk_split, 2 * th * w->dh * sizeof(float)) != cudaSuccess) ||
        cudaMalloc(&w->row_done, th * sizeof(uint8_t)) != cudaSuccess) {
        cudaGetLastError();
        free_workspace(w);
        return fail(MCA_ERR_ALLOC, "workspace allocation for %ld tokens failed", tokens);
    }
    w->cap_tokens = tokens;
    w->ovf_cap = std::min<long>(8L * (long)th, kOvfCap);
    return MCA_OK;
}

mca_status check_config(const mca_config* cfg, bool need_alpha) {
    if (!cfg) return fail(MCA_ERR_NULL, "cfg is NULL");
    if (cfg->mode != MCA_MODE_APPROX && cfg->mode != MCA_MODE_REGULAR)
        return fail(MCA_ERR_CONFIG, "unknown mode %d", cfg->mode);
    if (need_alpha && cfg->mode == MCA_MODE_APPROX && !(cfg->alpha > 0.0 && cfg->alpha <= 1.0))
        return fail(MCA_ERR_DOMAIN, "alpha = %g is not in (0, 1] (SPEC.md:270, 353)", cfg->alpha);
    if (cfg->min_samples < 1) return fail(MCA_ERR_DOMAIN, "min_samples = %d must be >= 1", cfg->min_samples);
    return MCA_OK;
}

// bf16 path: K3 as a tile GEMM (k3t) when its shared-memory plan fits.
// Launch with programmatic stream serialization (PDL): the kernel may start
// while its stream predecessor drains; it calls griddep_wait() before reading
// the predecessor's output (mca_common.cuh).
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// counters (64 B) | task cursors | budget histograms [H, d + 1] | list fill counters [H, d + 1]
// counters (64 B) | task cursors [2][H] (K3; the fp32 column halves walk the lists separately)
// | budget histograms [H, d + 1] | list fill counters [H, d + 1]
size_t zeroed_bytes(int heads, int d_in) { return 64 + (((size_t)heads * 8 + 63) & ~(size_t)63) + 2 * (size_t)heads * (d_in + 1) * 4; }

// Exact-fraction threshold of the dense exact encoding (bf16 MCA layer): at C2 the
// gathered k3b_exact_tc costs ~2.7 us per 1% of token-heads and the dense X W_V GEMM
// ~30 us, so the dense GEMM wins above ~12%. MCA_DENSE_EXACT=0 disables it.
constexpr double kDenseExactFrac = 0.12;
bool dense_exact_enabled() {
    static const bool on = [] {
        const char* e = getenv("MCA_DENSE_EXACT");
        return !(e && e[0] == '0');
    }();
    return on;
}
long dense_exact_min(long token_heads) { return std::max(1L, (long)(kDenseExactFrac * (double)token_heads)); }

// MCA_KP_PAIR=0: the single-CTA projection GEMM instead of the CTA-pair one
bool kp_pair_enabled() {
    static const bool on = [] {
        const char* e = getenv("MCA_KP_PAIR");
        return !(e && e[0] == '0');
    }();
    return on;
}

// MCA_K12_SPLIT=0: K12 runs every item whole (no split last wave)
bool k12_split_enabled() {
    static const bool on = [] {
        const char* e = getenv("MCA_K12_SPLIT");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool use_k3t(const mca_weights* w) {
    return w->wdt == MCA_BF16 && w->wprime && !force_simt() && tile_k3_requested() && w->d_in % 8 == 0 &&
           k3t::layout(w->d_in).bytes <= 227u * 1024u;
}

// skip_exact: the exact token-heads' encodings are already in hout (the dense GEMM).
template <class T, class Acc>
mca_status launch_k3(mca_weights* w, const void* x, int B, int n, long b_offset, uint32_t layer, uint64_t seed,
                     void* hout, int32_t* draws, int draws_stride, mca_stream_t stream, int& launches,
                     bool skip_exact = false, long dense_min = 0) {
    using Coef = float;   // K3's per-row factor: 1/p(i) in fp32 (both dtypes accumulate in fp32)
    K3Args a{};
    a.x = x;
    a.wv = w->w;
    a.d_in = w->d_in;
    a.heads = w->heads;
    a.n = n;
    a.tokens = (long)B * n;
    a.b_offset = b_offset;
    a.layer = layer;
    a.seed = seed;
    a.budgets = w->budgets;
    a.exact = w->exact;
    a.thr = w->thr;
    a.guide = w->guide;
    a.probs = w->probs;
    a.invp = w->invp;
    a.h_out = hout;
    a.draws_out = draws;
    a.draws_stride = draws_stride;
    a.sample_counter = w->counters + 3;
    a.samp_list = w->samp_list;
    a.exact_list = w->exact_list;
    a.counts = w->counts;
    a.dense_min = dense_min;
    a.task_cursor = w->task_cursor;
    a.ovf.count = w->counters + kOvfCounter;
    a.ovf.list = w->ovf_list;
    a.ovf.rows = w->ovf_rows;
    a.ovf.cap = (int)w->ovf_cap;
    // W_h staged in smem as fp32 when it fits (no unpacking in the hot loop),
    // else as bf16, else read from global memory (L1/L2).
    if (sizeof(T) == 2 && use_k3t(w)) {
        // bf16: every token-head (sampled and exact) as one tile GEMM per head
        CUtensorMap tw;
        if (!make_tmap_bf16(&tw, w->wprime, (uint64_t)w->heads * kDh, w->d_in, 1, 64))
            return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for W'");
        const uint32_t smem = k3t::layout(w->d_in).bytes;
        MCA_CUDA_TRY(ensure_smem(k3t_encode_tc, smem));
        int G = sm_count() / w->heads;
        const long cap = (long)B * ((n + k3t::kBM - 1) / k3t::kBM);
        if (G > cap) G = (int)cap;
        if (G < 1) G = 1;
        a.prof = mca_diag::k3t_prof_begin(stream);   // diagnostics builds only
        k3t_encode_tc<<<dim3(G, w->heads), k3t::kThreads, smem, stream>>>(a, tw,
                                                                           (const __nv_bfloat16*)w->pbf);
        MCA_LAUNCH_CHECK("k3t_encode_tc");
        mca_diag::k3t_prof_end(stream, a.prof);
        return MCA_OK;
    } else {
    // Gather-scale-accumulate: W_h staged as bf16 (one 128-byte smem wavefront
    // per sample; smem bandwidth, not issue, bounds this loop) / fp32 for the
    // fp32 parity path.
    void (*kern)(K3Args) = nullptr;
    bool launched = false;
    size_t smem = k3_smem_bytes(w->d_in, sizeof(Coef), sizeof(T), true);
    constexpr size_t kMaxSmem = 220 * 1024;
    constexpr size_t kMaxSmemOptIn = 227 * 1024;   // sm_100 per-block opt-in maximum
    int threads = kK3BlockThreads;
    if (sizeof(T) == 2 && k3_bf16_smem_bytes(w->d_in) <= kMaxSmem) {
        smem = k3_bf16_smem_bytes(w->d_in);
        kern = !MCA_K3_SPECIALIZE ? k3_encode_sampled_bf16<0>
               : w->d_in == 768 ? k3_encode_sampled_bf16<768>
               : w->d_in == 1024 ? k3_encode_sampled_bf16<1024>
                                 : k3_encode_sampled_bf16<0>;
    } else if (sizeof(T) == 4 && a.tokens * w->heads <= (1L << 16) &&
               k3_smem_bytes(w->d_in, sizeof(Coef), 4, true, kDh / 2) <= kMaxSmem) {
        // fp32, small batches (latency-bound: C1 0.19 -> 0.10 ms): two CTAs per
        // head-task, each with its fp32 half of W_h resident. At C2 the doubled
        // draws cost more than the L2 row reads save (0.91 vs 0.79 ms).
        if constexpr (sizeof(T) == 4) {
            smem = k3_smem_bytes(w->d_in, sizeof(Coef), 4, true, kDh / 2);
            auto kh = k3_encode_sampled<float, float, float, true, 4>;
            MCA_CUDA_TRY(ensure_smem(kh, smem));
            int occ = 0;
            MCA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kh, kK3BlockThreads, smem));
            if (occ < 1) occ = 1;
            int G = sm_count() * occ / (2 * w->heads);
            const long cap = (a.tokens + 63) / 64;
            if (G > cap) G = (int)cap;
            if (G < 1) G = 1;
            kh<<<dim3(G, w->heads, 2), kK3BlockThreads, smem, stream>>>(a);
            MCA_LAUNCH_CHECK("k3_encode_sampled_f32h");
            launched = true;
        }
    } else if (smem <= kMaxSmem) {
        if constexpr (sizeof(T) == 2) kern = k3_encode_sampled<__nv_bfloat16, __nv_bfloat16, float, true>;
        else kern = k3_encode_sampled<float, float, float, true>;
    } else if (sizeof(T) == 4 && k3_smem_bytes(w->d_in, sizeof(Coef), 4, true, kDh, kK3F32Warps, kK3F32GuideBits) <=
                                     kMaxSmemOptIn) {
        // fp32 at C2 (d_in = 768): the whole fp32 W_h resident beside a coarse
        // guide table, 512 threads per CTA (conflict-free smem row reads instead of
        // L1/L2 gathers of 256-byte rows)
        smem = k3_smem_bytes(w->d_in, sizeof(Coef), 4, true, kDh, kK3F32Warps, kK3F32GuideBits);
        if constexpr (sizeof(T) == 4) kern = k3_encode_sampled<float, float, float, true, 8, kK3F32Warps, kK3F32GuideBits>;
        threads = kK3F32Warps * 32;
    } else {
        smem = k3_smem_bytes(w->d_in, sizeof(Coef), sizeof(T), false);
        if constexpr (sizeof(T) == 2) kern = k3_encode_sampled<__nv_bfloat16, __nv_bfloat16, float, false>;
        else kern = k3_encode_sampled<float, float, float, false>;
    }
    if (!launched) {
    MCA_CUDA_TRY(ensure_smem(kern, smem));
    int occ = 0;
    MCA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
    if (occ < 1) occ = 1;
    int G = sm_count() * occ / w->heads;     // all CTAs resident: no second wave
    const long cap = (a.tokens + 63) / 64;   // at most one CTA per 64 tokens of a head
    if (G > cap) G = (int)cap;
    if (G < 1) G = 1;
    // bf16: a 1-D grid filling every SM (CTA c starts on head c % heads and
    // then joins whichever head has the most work left)
    const int G1 = (int)std::min<long>((long)sm_count() * occ, (long)std::max(G, 1) * w->heads + (long)w->heads);
    const bool bf16_kern = kern == k3_encode_sampled_bf16<768> || kern == k3_encode_sampled_bf16<1024> ||
                           kern == k3_encode_sampled_bf16<0>;
    if (bf16_kern) MCA_CUDA_TRY(launch_pdl(kern, dim3(G1), dim3(kK3BlockThreads), smem, stream, a));
    else kern<<<dim3(G, w->heads), threads, smem, stream>>>(a);
    MCA_LAUNCH_CHECK("k3_encode_sampled");
    if (bf16_kern) mca_diag::dump_k3s(stream, G1, w->heads);   // diagnostics builds only
    }
    }
    if (skip_exact) {
    } else if (sizeof(T) == 2 && !force_simt()) {   // bf16: exact token-heads on the tensor cores
        MCA_CUDA_TRY(ensure_smem(k3b_exact_tc, k3btc::kSmemBytes));
        // persistent: one wave (2 CTAs per SM), CTAs loop over their head's exact tiles
        int Ge = (2 * sm_count() + w->heads - 1) / w->heads;
        const long ecap = (a.tokens + k3btc::kBM - 1) / k3btc::kBM;
        if (Ge > ecap) Ge = (int)ecap;
        if (Ge < 1) Ge = 1;
        MCA_CUDA_TRY(launch_pdl(k3b_exact_tc, dim3((unsigned)Ge, w->heads), dim3(k3btc::kThreads), k3btc::kSmemBytes,
                                stream, a));
        MCA_LAUNCH_CHECK("k3b_exact_tc");
        mca_diag::dump_k3b(stream);   // diagnostics builds only
    } else {                                  // fp32 parity path: fp64 CUDA-core GEMM
        int Ge = (4 * sm_count() + w->heads - 1) / w->heads;   // 128-thread CTAs, several per SM
        const long ecap = (a.tokens + 63) / 64;
        if (Ge > ecap) Ge = (int)ecap;
        if (Ge < 1) Ge = 1;
        // few tiles (C1: 2 per head): split each tile's outputs over two CTAs
        if ((long)Ge * w->heads * 2 <= 2L * sm_count())
            MCA_CUDA_TRY(launch_pdl(k3b_encode_exact<T, Acc, 32>, dim3((unsigned)Ge, w->heads, 2), dim3(128), 0, stream, a));
        else
            MCA_CUDA_TRY(launch_pdl(k3b_encode_exact<T, Acc, 64>, dim3((unsigned)Ge, w->heads), dim3(128), 0, stream, a));
        MCA_LAUNCH_CHECK("k3b_encode_exact");
    }
    return MCA_OK;
}

// Budget-sorted work lists from the histograms: one scan + scatter kernel
// (k2_scan_scatter), or the two-kernel form (MCA_K2_FUSED_SCAN=0).
mca_status launch_lists(mca_weights* w, dim3 grid, int n, long tokens, mca_stream_t stream, int& launches) {
    const int H = w->heads;
    if (MCA_K2_FUSED_SCAN) {
        const size_t smem = 2 * (size_t)(w->d_in + 1) * 4;   // bin bases + this CTA's bin counts
        if (smem > 48 * 1024) MCA_CUDA_TRY(ensure_smem(k2_scan_scatter, smem));
        const dim3 gs((unsigned)((tokens + kScatterThreads * kScatterPerThread - 1) / (kScatterThreads * kScatterPerThread)),
                      (unsigned)H);
        MCA_CUDA_TRY(launch_pdl(k2_scan_scatter, gs, dim3(kScatterThreads), smem, stream,
                                (const int32_t*)w->budgets, (const uint8_t*)w->exact, (const unsigned int*)w->hist, n,
                                H, w->d_in, tokens, w->fill, w->counts, w->samp_list, w->exact_list));
        MCA_LAUNCH_CHECK("k2_scan_scatter");
    } else {
        MCA_CUDA_TRY(launch_pdl(k2_scan, dim3(H), dim3(1024), 0, stream, (const unsigned int*)w->hist, w->d_in,
                                w->cursor, w->counts));
        MCA_LAUNCH_CHECK("k2_scan");
        MCA_CUDA_TRY(launch_pdl(k2_scatter, grid, dim3(256), 0, stream, (const int32_t*)w->budgets,
                                (const uint8_t*)w->exact, n, H, w->d_in, tokens, w->cursor, w->samp_list,
                                w->exact_list));
        MCA_LAUNCH_CHECK("k2_scatter");
    }
    return MCA_OK;
}

// The dense projection GEMM (kp_project_tc) over segments [seg0, seg0 + nseg) of
// W^T = [W_q^T | W_k^T | W_V^T]: segment s of x W goes to outs[s]. bf16 handles:
// bf16 outputs, or fp16 when bit s of f16_mask is set. fp32 handles: 3xTF32 on
// the hi / lo parts of x (split here) and W^T (split at preparation), fp32 outputs.
// guard: the fp16 range guard / device gate fields of KpArgs (ovf, exact, n, gate,
// gate_min); the shape fields are filled here.
mca_status launch_projection(mca_weights* w, const void* x, long tokens, int seg0, int nseg, void* const outs[3],
                             int f16_mask, mca_stream_t stream, int& launches, const KpArgs* guard = nullptr) {
    const int HD = w->heads * w->dh;
    const bool tf32 = w->wdt == MCA_F32;
    if ((size_t)w->d_in * dtype_size(w->wdt) % 16 != 0)   // TMA: a 16-byte multiple row stride
        return fail(MCA_ERR_UNSUPPORTED, "the on-device projections need d_in * %zu bytes to be a multiple of 16 "
                    "(d_in = %d); pass q and k instead", dtype_size(w->wdt), w->d_in);
    // N tile: the widest of 256 / 128 / 64 that divides H*64 (192 for BERT-base's
    // finer wave quantisation measured 72 us vs 66 for 256: per-tile overheads)
    // 3xTF32: 128 (three 64 KB stages instead of two 96 KB ones; measured 291 vs 303 us at C2)
    // Small M (C1: one 128-row tile): 128 x 64 tiles on single CTAs when they fit
    // one wave -- 4x the CTAs of the 256 x 256 pairs on a K loop that is serial
    // per tile (C1 fp32: 33 -> 9 us)
    const bool small = HD % 64 == 0 && ((tokens + kp::kBM - 1) / kp::kBM) * ((long)nseg * HD / 64) <= sm_count();
    const int BN = small ? 64 : (HD % 256 == 0 && !tf32) ? 256 : HD % 128 == 0 ? 128 : 64;
    CUtensorMap tx, tw, tx2, tw2, to[3];
    const size_t wofs = (size_t)seg0 * HD * w->d_in;
    if (tf32) {
        if (tokens > w->cap_x) {   // x hi | lo workspace
            if (w->cap_x) MCA_CUDA_TRY(cudaStreamSynchronize(stream));
            drop_graphs(w);
            cudaFree(w->x_split);
            w->x_split = nullptr;
            w->cap_x = 0;
            if (cudaMalloc(&w->x_split, (size_t)tokens * w->d_in * sizeof(float)) != cudaSuccess) {
                cudaGetLastError();
                return fail(MCA_ERR_ALLOC, "x split workspace allocation failed");
            }
            w->cap_x = tokens;
        }
        const size_t cnt = (size_t)tokens * w->d_in;
        // kind::tf32 reads the top 19 bits of each fp32 operand (the low 13 are
        // ignored: measured bitwise equal to the masked hi part), so x itself is
        // the hi operand and only x - hi(x) is materialised
        float* xl = static_cast<float*>(w->x_split);
        const unsigned gs = (unsigned)std::min<size_t>((cnt / 4 + 255) / 256, 8 * (size_t)sm_count());
        k_split_tf32<<<gs, 256, 0, stream>>>((const float4*)x, nullptr, (float4*)xl, cnt / 4);   // d_in % 4 == 0
        MCA_LAUNCH_CHECK("k_split_tf32");
        if (!make_tmap_f32(&tx, x, (uint64_t)w->d_in, (uint64_t)tokens, 1, kp::kBM) ||
            !make_tmap_f32(&tx2, xl, (uint64_t)w->d_in, (uint64_t)tokens, 1, kp::kBM) ||
            !make_tmap_f32(&tw, static_cast<const float*>(w->wqkv_t) + wofs, (uint64_t)w->d_in, (uint64_t)nseg * HD,
                           1, (uint32_t)BN) ||
            !make_tmap_f32(&tw2, static_cast<const float*>(w->wqkv_t_lo) + wofs, (uint64_t)w->d_in,
                           (uint64_t)nseg * HD, 1, (uint32_t)BN))
            return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for x / W^T (tf32 parts)");
    } else {
        const __nv_bfloat16* wt = static_cast<const __nv_bfloat16*>(w->wqkv_t) + wofs;
        if (!make_tmap_bf16(&tx, x, (uint64_t)w->d_in, (uint64_t)tokens, 1, kp::kBM) ||
            !make_tmap_bf16(&tw, wt, (uint64_t)w->d_in, (uint64_t)nseg * HD, 1, (uint32_t)BN))
            return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for x / W^T");
        tx2 = tx;
        tw2 = tw;
    }
    int mask = 0;
    const bool lo_tma = tf32 && guard && guard->lo_tma;
    for (int i = 0; i < 3; ++i) {
        if (lo_tma && i == 2) {   // q_lo | k_lo: [2][tokens][HD], the third map
            if (!make_tmap_f32(&to[2], outs[2], (uint64_t)HD, (uint64_t)tokens, 2, kp::kBM))
                return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for the lo outputs");
            continue;
        }
        const int sg = std::min(seg0 + i, seg0 + nseg - 1);   // unused maps repeat the last segment
        const bool f16 = !tf32 && ((f16_mask >> sg) & 1);
        if (i < nseg && f16) mask |= 1 << i;
        const bool ok = tf32 ? make_tmap_f32(&to[i], outs[sg], (uint64_t)HD, (uint64_t)tokens, 1, kp::kBM)
                             : make_tmap_bf16(&to[i], outs[sg], (uint64_t)HD, (uint64_t)tokens, 1, kp::kBM,
                                              f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
        if (!ok) return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for the projection outputs");
    }
    KpArgs pa = guard ? *guard : KpArgs{};
    pa.M = (int)tokens;
    pa.d_in = w->d_in;
    pa.HD = HD;
    pa.nseg = nseg;
    pa.f16_mask = mask;
    const long tiles = ((tokens + kp::kBM - 1) / kp::kBM) * ((long)nseg * HD / BN);
    const dim3 grid((unsigned)std::min<long>(tiles, sm_count()));
    if (!small && HD % 256 == 0 && kp_pair_enabled()) {   // a 256-column pair tile never straddles two segments
        // CTA pairs: 256 x 256 tiles (kp_project_pair.cu); W^T with 128-row boxes
        // (each CTA of the pair loads half of the tile's N)
        const long ptiles = ((tokens + 255) / 256) * ((long)nseg * HD / 256);
        const unsigned pairs = (unsigned)std::max<long>(1, std::min<long>(ptiles, sm_count() / 2));
        CUtensorMap twp = tw;
        if (!tf32 && !make_tmap_bf16(&twp, static_cast<const __nv_bfloat16*>(w->wqkv_t) + wofs, (uint64_t)w->d_in,
                                     (uint64_t)nseg * HD, 1, 128))
            return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for W^T (pair)");
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(192);
        cfg.stream = stream;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        if (tf32) {
            cfg.dynamicSmemBytes = kp2::Cfg<true>::kSmemBytes;
            MCA_CUDA_TRY(ensure_smem(kp_project_pair<true>, kp2::Cfg<true>::kSmemBytes));
            MCA_CUDA_TRY(cudaLaunchKernelEx(&cfg, kp_project_pair<true>, tx, twp, tx2, tw2, to[0], to[1], to[2], pa));
        } else {
            cfg.dynamicSmemBytes = kp2::Cfg<false>::kSmemBytes;
            MCA_CUDA_TRY(ensure_smem(kp_project_pair<false>, kp2::Cfg<false>::kSmemBytes));
            MCA_CUDA_TRY(cudaLaunchKernelEx(&cfg, kp_project_pair<false>, tx, twp, tx2, tw2, to[0], to[1], to[2], pa));
        }
        MCA_LAUNCH_CHECK("kp_project_pair");
        return MCA_OK;
    }
    auto go = [&](auto kern, uint32_t smem) -> mca_status {
        MCA_CUDA_TRY(ensure_smem(kern, smem));
        MCA_CUDA_TRY(launch_pdl(kern, grid, dim3(kp::kThreads), smem, stream, tx, tw, tx2, tw2, to[0], to[1], to[2], pa));
        return MCA_OK;
    };
    mca_status ps;
    if (tf32)
        ps = BN == 256   ? go(kp_project_tc<256, true>, kp::Cfg<256, true>::kSmemBytes)
             : BN == 128 ? go(kp_project_tc<128, true>, kp::Cfg<128, true>::kSmemBytes)
                         : go(kp_project_tc<64, true>, kp::Cfg<64, true>::kSmemBytes);
    else
        ps = BN == 256   ? go(kp_project_tc<256>, kp::Cfg<256>::kSmemBytes)
             : BN == 128 ? go(kp_project_tc<128>, kp::Cfg<128>::kSmemBytes)
                         : go(kp_project_tc<64>, kp::Cfg<64>::kSmemBytes);
    if (ps) return ps;
    MCA_LAUNCH_CHECK("kp_project_tc");
    return MCA_OK;
}

// The fp16 range guard of a dense H~ segment (all token-heads exact when exact ==
// nullptr), optionally gated on K2's exact counts (sum >= gate_min).
KpArgs h_guard(mca_weights* w, int n, const uint8_t* exact, const int* gate, long gate_min) {
    KpArgs g{};
    g.ovf.count = w->counters + kOvfCounter;
    g.ovf.list = w->ovf_list;
    g.ovf.rows = w->ovf_rows;
    g.ovf.cap = (int)w->ovf_cap;
    g.exact = exact;
    g.n = n;
    g.gate = gate;
    g.gate_min = gate_min;
    return g;
}

// fp16 range guard's fix-up (k4o_overflow): after the aggregation, add P[:, j] H~_j
// for the token-heads the encoders queued (normally none: one counter read).
mca_status launch_overflow_fixup(mca_weights* w, bool given, const void* q, const void* k, const double* attn,
                                 double scale, int B, int n, void* y, mca_stream_t stream, int& launches) {
    K4oArgs o{};
    o.ovf.count = w->counters + kOvfCounter;
    o.ovf.list = w->ovf_list;
    o.ovf.rows = w->ovf_rows;
    o.ovf.cap = (int)w->ovf_cap;
    o.q = q;
    o.k = k;
    o.lse = w->lse;
    o.attn = attn;
    o.scale = scale;
    o.n = n;
    o.heads = w->heads;
    o.y = static_cast<__nv_bfloat16*>(y);
    const dim3 grid((unsigned)std::min<long>((long)B * w->heads, sm_count()));
    if (given) MCA_CUDA_TRY(launch_pdl(k4o_overflow<true>, grid, dim3(256), 0, stream, o));
    else MCA_CUDA_TRY(launch_pdl(k4o_overflow<false>, grid, dim3(256), 0, stream, o));
    MCA_LAUNCH_CHECK("k4o_overflow");
    return MCA_OK;
}

// FlopsReport of the last plan from the device counters; synchronises.
mca_status read_flops(mca_weights* w, int B, int n, bool approx, mca_flops* out, mca_stream_t stream) {
    unsigned long long c[8];
    MCA_CUDA_TRY(cudaMemcpyAsync(c, w->counters, sizeof(c), cudaMemcpyDeviceToHost, stream));
    MCA_CUDA_TRY(cudaStreamSynchronize(stream));
    const long th = (long)B * n * w->heads;
    out->exact_encoding = (uint64_t)th * 2ull * w->d_in * w->dh;
    out->approx_encoding = approx ? c[0] : out->exact_encoding;
    out->aggregation = (uint64_t)B * w->heads * 2ull * n * n * w->dh;
    out->samples = approx ? c[3] : 0;
    out->exact_tokens = approx ? c[2] : (uint64_t)th;
    out->certified = c[kCertTotal];
    out->reduction_factor = (double)out->exact_encoding / (double)out->approx_encoding;
    out->total_reduction = (double)(out->exact_encoding + out->aggregation) /
                           (double)(out->approx_encoding + out->aggregation);
    return MCA_OK;
}

}  // namespace

extern "C" {

const char* mca_last_error(void) { return g_err.c_str(); }

mca_status mca_device_alloc(size_t bytes, void** out) {
    if (!out) return fail(MCA_ERR_NULL, "out is NULL");
    *out = nullptr;
    if (cudaMalloc(out, bytes) != cudaSuccess) {
        const cudaError_t e = cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? MCA_ERR_ALLOC : MCA_ERR_CUDA, "cudaMalloc(%zu) failed: %s", bytes,
                    cudaGetErrorString(e));
    }
    return MCA_OK;
}

void mca_device_free(void* p) { cudaFree(p); }

mca_status mca_copy(void* dst, const void* src, size_t bytes, mca_copy_kind kind) {
    if ((!dst || !src) && bytes) return fail(MCA_ERR_NULL, "dst / src is NULL");
    const cudaMemcpyKind k = kind == MCA_COPY_H2D   ? cudaMemcpyHostToDevice
                             : kind == MCA_COPY_D2H ? cudaMemcpyDeviceToHost
                                                    : cudaMemcpyDeviceToDevice;
    MCA_CUDA_TRY(cudaMemcpy(dst, src, bytes, k));
    return MCA_OK;
}

mca_status mca_stream_sync(mca_stream_t stream) {
    MCA_CUDA_TRY(cudaStreamSynchronize(stream));
    return MCA_OK;
}
const char* mca_version(void) { return "mca_b200 0.1 (sm_100a)"; }

mca_status mca_prepare_weights(const void* w_v, mca_dtype wdt, int d_in, int heads, int d_h, mca_stream_t stream,
                               mca_weights** out) {
    if (!out || !w_v) return fail(MCA_ERR_NULL, "w_v / out is NULL");
    *out = nullptr;
    if (wdt != MCA_F32 && wdt != MCA_BF16) return fail(MCA_ERR_CONFIG, "unknown dtype %d", (int)wdt);
    if (d_in <= 0 || heads <= 0 || d_h <= 0) return fail(MCA_ERR_SHAPE, "d_in, heads, d_h must be positive");
    if (d_h != kDh) return fail(MCA_ERR_UNSUPPORTED, "d_h = %d: the sm_100a kernels implement d_h = 64", d_h);
    if (d_in > 16384) return fail(MCA_ERR_UNSUPPORTED, "d_in = %d exceeds the guide table's 14-bit rows", d_in);
    if ((size_t)d_in * dtype_size(wdt) % 16 != 0)   // x rows are read with 16-byte vector / TMA / cp.async loads
        return fail(MCA_ERR_UNSUPPORTED, "d_in = %d: x rows must be a multiple of 16 bytes (d_in %% %d == 0)", d_in,
                    (int)(16 / dtype_size(wdt)));
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
        cudaGetLastError();
        return fail(MCA_ERR_CUDA, "no CUDA device: the MCA forward has no CPU path");
    }
    mca_weights* w = new mca_weights();
    w->d_in = d_in;
    w->heads = heads;
    w->dh = d_h;
    w->wdt = wdt;
    cudaGetDevice(&w->device);
    const size_t wbytes = (size_t)d_in * heads * d_h * dtype_size(wdt);
    const size_t hd = (size_t)heads * d_in;
    double* sq = nullptr;
    int* status = nullptr;
    auto cleanup = [&](mca_status s) {
        cudaFree(sq);
        cudaFree(status);
        if (s != MCA_OK) mca_weights_free(w);
        return s;
    };
    if (cudaMalloc(&w->w, wbytes) != cudaSuccess || cudaMalloc(&w->probs, hd * 8) != cudaSuccess ||
        cudaMalloc(&w->cdf, hd * 8) != cudaSuccess || cudaMalloc(&w->thr, hd * 8) != cudaSuccess ||
        cudaMalloc(&w->invp, hd * 4) != cudaSuccess || cudaMalloc(&w->guide, (size_t)heads * kGuide * 2) != cudaSuccess ||
        cudaMalloc(&w->zeroed, zeroed_bytes(heads, d_in)) != cudaSuccess ||
        cudaMalloc(&w->cursor, (size_t)heads * (d_in + 1) * 4) != cudaSuccess ||
        cudaMalloc(&w->counts, heads * 2 * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&sq, hd * 8) != cudaSuccess ||
        cudaMalloc(&status, heads * sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        return cleanup(fail(MCA_ERR_ALLOC, "weight table allocation failed"));
    }
    // counters | task cursors | budget histograms: one region, one memset per forward
    w->counters = static_cast<unsigned long long*>(w->zeroed);
    w->task_cursor = reinterpret_cast<int*>(static_cast<char*>(w->zeroed) + 64);
    w->hist = reinterpret_cast<unsigned int*>(static_cast<char*>(w->zeroed) + 64 + ((heads * 8 + 63) & ~63));
    w->fill = w->hist + (size_t)heads * (d_in + 1);
    if (cudaMemcpyAsync(w->w, w_v, wbytes, cudaMemcpyDeviceToDevice, stream) != cudaSuccess)
        return cleanup(fail(MCA_ERR_CUDA, "copying w_v failed: %s", cudaGetErrorString(cudaGetLastError())));
    const dim3 g0((d_in + 255) / 256, heads);
    if (wdt == MCA_F32) k0_row_sq<float><<<g0, 256, 0, stream>>>((const float*)w->w, d_in, heads, sq);
    else k0_row_sq<__nv_bfloat16><<<g0, 256, 0, stream>>>((const __nv_bfloat16*)w->w, d_in, heads, sq);
    k0_dist<<<heads, 256, 0, stream>>>(sq, d_in, w->probs, w->cdf, w->thr, w->invp, w->guide, status);
    if (wdt == MCA_F32) {    // W_V^T hi / lo: the third segment of the 3xTF32 projection GEMM (dense H = X W_V)
        if (cudaMalloc(&w->wqkv_t, 3 * wbytes) != cudaSuccess || cudaMalloc(&w->wqkv_t_lo, 3 * wbytes) != cudaSuccess) {
            cudaGetLastError();
            return cleanup(fail(MCA_ERR_ALLOC, "W^T allocation failed"));
        }
        const int HD = heads * d_h;
        kp_transpose_split_f32<<<dim3((HD + 31) / 32, (d_in + 31) / 32), dim3(32, 8), 0, stream>>>(
            (const float*)w->w, d_in, HD, static_cast<float*>(w->wqkv_t) + 2 * (size_t)HD * d_in,
            static_cast<float*>(w->wqkv_t_lo) + 2 * (size_t)HD * d_in);
    }
    if (wdt == MCA_BF16) {   // k3t's operands: W' = W_h / p and bf16 p
        if (cudaMalloc(&w->wprime, wbytes) != cudaSuccess || cudaMalloc(&w->pbf, hd * 2) != cudaSuccess) {
            cudaGetLastError();
            return cleanup(fail(MCA_ERR_ALLOC, "W' allocation failed"));
        }
        k0_wprime<<<2 * sm_count(), 256, 0, stream>>>((const __nv_bfloat16*)w->w, w->probs, d_in, heads,
                                                       (__nv_bfloat16*)w->wprime, (__nv_bfloat16*)w->pbf);
        // W_V^T as the third segment of the projection GEMM's B (the exact layer's H = X W_V)
        if (cudaMalloc(&w->wqkv_t, 3 * wbytes) != cudaSuccess) {
            cudaGetLastError();
            return cleanup(fail(MCA_ERR_ALLOC, "W^T allocation failed"));
        }
        const int HD = heads * d_h;
        kp_transpose<<<dim3((HD + 31) / 32, (d_in + 31) / 32), dim3(32, 8), 0, stream>>>(
            (const __nv_bfloat16*)w->w, d_in, HD, static_cast<__nv_bfloat16*>(w->wqkv_t) + 2 * (size_t)HD * d_in);
    }
    std::vector<int> hs(heads);
    if (cudaMemcpyAsync(hs.data(), status, heads * sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
        return cleanup(fail(MCA_ERR_CUDA, "K0 failed: %s", cudaGetErrorString(cudaGetLastError())));
    for (int h = 0; h < heads; ++h)
        if (hs[h]) return cleanup(fail(MCA_ERR_DEGENERATE, "head %d: W_h is zero or non-finite (SPEC.md:205)", h));
    *out = w;
    return cleanup(MCA_OK);
}

void mca_weights_free(mca_weights* w) {
    if (!w) return;
    free_workspace(w);
    cudaFree(w->w);
    cudaFree(w->probs);
    cudaFree(w->cdf);
    cudaFree(w->thr);
    cudaFree(w->invp);
    cudaFree(w->guide);
    cudaFree(w->wprime);
    cudaFree(w->pbf);
    cudaFree(w->wqkv_t);
    cudaFree(w->wqkv_t_lo);
    cudaFree(w->x_split);
    cudaFree(w->qk);
    for (auto& g : w->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    cudaFree(w->zeroed);
    cudaFree(w->k12_tail);
    cudaFree(w->cursor);
    cudaFree(w->counts);
    for (auto& e : w->ev)
        if (e) cudaEventDestroy(e);
    delete w;
}

mca_status mca_set_projections(mca_weights* w, const void* w_q, const void* w_k, mca_stream_t stream) {
    if (!w || !w_q || !w_k) return fail(MCA_ERR_NULL, "weights / w_q / w_k is NULL");
    if (w->wdt == MCA_BF16) {   // kp_project_tc: W_q^T | W_k^T rows of the handle's K-major W^T
        const int HD = w->heads * w->dh;
        const dim3 g((HD + 31) / 32, (w->d_in + 31) / 32);
        for (int i = 0; i < 2; ++i) {
            kp_transpose<<<g, dim3(32, 8), 0, stream>>>(static_cast<const __nv_bfloat16*>(i ? w_k : w_q), w->d_in, HD,
                                                        static_cast<__nv_bfloat16*>(w->wqkv_t) + (size_t)i * HD * w->d_in);
            MCA_CUDA_TRY(cudaGetLastError());
        }
        w->has_qk_t = true;
        drop_graphs(w);
        return MCA_OK;
    }
    {   // fp32: W_q^T, W_k^T hi / lo parts (3xTF32)
        const int HD = w->heads * w->dh;
        const dim3 g((HD + 31) / 32, (w->d_in + 31) / 32);
        for (int i = 0; i < 2; ++i) {
            kp_transpose_split_f32<<<g, dim3(32, 8), 0, stream>>>(
                static_cast<const float*>(i ? w_k : w_q), w->d_in, HD,
                static_cast<float*>(w->wqkv_t) + (size_t)i * HD * w->d_in,
                static_cast<float*>(w->wqkv_t_lo) + (size_t)i * HD * w->d_in);
            MCA_CUDA_TRY(cudaGetLastError());
        }
        w->has_qk_t = true;
        drop_graphs(w);
        return MCA_OK;
    }
}

mca_status mca_weights_export(const mca_weights* w, double* probs_host, double* cdf_host) {
    if (!w) return fail(MCA_ERR_NULL, "weights is NULL");
    const size_t hd = (size_t)w->heads * w->d_in * 8;
    if (probs_host) MCA_CUDA_TRY(cudaMemcpy(probs_host, w->probs, hd, cudaMemcpyDeviceToHost));
    if (cdf_host) MCA_CUDA_TRY(cudaMemcpy(cdf_host, w->cdf, hd, cudaMemcpyDeviceToHost));
    return MCA_OK;
}

mca_status mca_reserve(mca_weights* w, long max_tokens, mca_stream_t stream) {
    if (!w) return fail(MCA_ERR_NULL, "weights is NULL");
    if (max_tokens < 0) return fail(MCA_ERR_SHAPE, "max_tokens < 0");
    return ensure_workspace(w, max_tokens, stream);
}

mca_status mca_set_timing(mca_weights* w, int enable) {
    if (!w) return fail(MCA_ERR_NULL, "weights is NULL");
    w->timing = enable != 0;
    if (w->timing && !w->ev[0])
        for (auto& e : w->ev) MCA_CUDA_TRY(cudaEventCreate(&e));
    w->ev_valid = false;
    return MCA_OK;
}

int mca_last_stage_ms(const mca_weights* w, float* ms, int max_stages) {
    if (!w || !w->timing || !w->ev_valid) return 0;
    if (cudaEventSynchronize(w->ev[5]) != cudaSuccess) return 0;
    int k = 0;
    for (; k < 5 && k < max_stages; ++k)
        if (cudaEventElapsedTime(&ms[k], w->ev[k], w->ev[k + 1]) != cudaSuccess) return k;
    return k;
}

int mca_last_launch_count(const mca_weights* w) { return w ? w->last_launches : 0; }

mca_status mca_stage_budgets(const double* cmax, long count, int n, int d, const mca_config* cfg, int32_t* budgets,
                             uint8_t* exact, mca_stream_t stream) {
    if (!cmax || !budgets || !exact) return fail(MCA_ERR_NULL, "cmax / budgets / exact is NULL");
    if (mca_status s = check_config(cfg, true)) return s;
    if (count < 0 || n <= 0 || d <= 0) return fail(MCA_ERR_SHAPE, "bad count / n / d");
    if (count == 0) return MCA_OK;
    int launches = 0;
    if (count > 0x7FFFFFFF) return fail(MCA_ERR_SHAPE, "count too large");
    const dim3 grid((unsigned)((count + 255) / 256), 1);   // one row of `count` values
    K2Args a{};
    a.cmax_in = cmax;
    a.count = count;
    a.row_len = (int)count;
    a.n = n;
    a.heads = 1;
    a.d = d;
    a.dh = kDh;
    a.min_samples = cfg->min_samples;
    a.alpha = cfg->alpha;
    a.budgets = budgets;
    a.exact = exact;
    k2_budgets<kGivenCmax, float><<<grid, 256, 0, stream>>>(a);
    MCA_LAUNCH_CHECK("k2_budgets");
    return MCA_OK;
}

mca_status mca_forward_ex(mca_weights* w, const void* q, const void* k, const void* x, mca_dtype dt, int B, int n,
                          long b_offset, uint32_t layer, const mca_config* cfg, uint64_t seed, void* y,
                          int32_t* budgets_out, uint8_t* exact_out, mca_flops* flops_out, const mca_debug* dbg,
                          mca_stream_t stream) {
    if (!w) return fail(MCA_ERR_NULL, "weights is NULL");
    if (mca_status s = check_config(cfg, true)) return s;
    if (B < 0 || n <= 0) return fail(MCA_ERR_SHAPE, "B = %d, n = %d: need B >= 0, n >= 1", B, n);
    if (dt != w->wdt) return fail(MCA_ERR_CONFIG, "activation dtype %d != weight dtype %d", (int)dt, (int)w->wdt);
    if (b_offset < 0) return fail(MCA_ERR_SHAPE, "b_offset < 0");
    if (n > 65535 || B > 65535)
        return fail(MCA_ERR_UNSUPPORTED, "B = %d, n = %d: work lists pack (b, j) into 16 bits each", B, n);
    const bool approx = cfg->mode == MCA_MODE_APPROX;
    if (dbg && dbg->budgets_override && !dbg->exact_override)
        return fail(MCA_ERR_NULL, "budgets_override needs exact_override");
    if (flops_out) std::memset(flops_out, 0, sizeof(*flops_out));
    if (B == 0) {
        w->last_launches = 0;
        return MCA_OK;
    }
    if (!x || !y || (!q) != (!k)) return fail(MCA_ERR_NULL, "x / y is NULL, or only one of q / k is");
    if (!q && !w->has_qk_t) return fail(MCA_ERR_NULL, "q / k are NULL and the weights carry no W_q / W_k");
    const long tokens = (long)B * n;
    if (mca_status s = ensure_workspace(w, tokens, stream)) return s;
    const int H = w->heads;
    int launches = 0;
    if (w->timing) MCA_CUDA_TRY(cudaEventRecord(w->ev[0], stream));
    // The exact encodings as one dense GEMM (H = x W_V, the projection kernel's third
    // segment, straight into K4's fp16 operand): the bf16 exact layer. The fp32
    // path keeps binary64 accumulation for exact encodings (K3b): a 3xTF32 GEMM
    // accumulates its 768 products in fp32 and measured up to 1.3e-5 relative per
    // row at C2 (tests/test_gpu_configs.py::test_fp32_c2_shape_tensor_core_path),
    // above the fp32 contract's 1e-5.
    const bool want_dense_h = !force_simt() && dt == MCA_BF16 && !approx && !budgets_out && !exact_out;
    bool h_dense = false;
    bool qk_lo_done = false;   // fp32: the projection GEMM wrote q_lo | k_lo
    // counters (incl. the fp16 guard's queue, which the dense H~ GEMM below may fill), cursors, histograms
    MCA_CUDA_TRY(cudaMemsetAsync(w->zeroed, 0, zeroed_bytes(H, w->d_in), stream));
    if (!q) {   // q = x W_q, k = x W_k (+ H): one tcgen05 GEMM, outputs in the score kernels' layout
        const size_t HD = (size_t)H * w->dh, esz = dtype_size(dt);
        if (tokens > w->cap_qk) {
            if (w->cap_qk) MCA_CUDA_TRY(cudaStreamSynchronize(stream));
            drop_graphs(w);
            cudaFree(w->qk);
            w->qk = nullptr;
            w->cap_qk = 0;
            if (cudaMalloc(&w->qk, 2 * (size_t)tokens * HD * esz) != cudaSuccess) {
                cudaGetLastError();
                return fail(MCA_ERR_ALLOC, "q / k workspace allocation failed");
            }
            w->cap_qk = tokens;
        }
        void* outs[3] = {w->qk, static_cast<char*>(w->qk) + (size_t)tokens * HD * esz, w->hbuf};
        KpArgs hg = h_guard(w, n, nullptr, nullptr, 0);
        if (dt == MCA_F32 && w->qk_split) {   // the 3xTF32 score passes' q_lo | k_lo, from the GEMM's epilogue
            hg.lo_tma = 1;
            outs[2] = w->qk_split;
            qk_lo_done = true;
        }
        if (mca_status ps = launch_projection(w, x, tokens, 0, want_dense_h ? 3 : 2, outs, 0b100, stream, launches,
                                              (want_dense_h || qk_lo_done) ? &hg : nullptr))
            return ps;
        h_dense = want_dense_h;
        q = w->qk;
        k = static_cast<const char*>(w->qk) + (size_t)tokens * HD * esz;
        if (dbg && dbg->q_out)
            MCA_CUDA_TRY(cudaMemcpyAsync(dbg->q_out, q, (size_t)tokens * HD * esz, cudaMemcpyDeviceToDevice, stream));
        if (dbg && dbg->k_out)
            MCA_CUDA_TRY(cudaMemcpyAsync(dbg->k_out, k, (size_t)tokens * HD * esz, cudaMemcpyDeviceToDevice, stream));
    }
    if (want_dense_h && !h_dense) {   // given q, k: the H segment alone
        void* outs[3] = {nullptr, nullptr, w->hbuf};
        const KpArgs hg = h_guard(w, n, nullptr, nullptr, 0);
        if (mca_status ps = launch_projection(w, x, tokens, 2, 1, outs, 0b100, stream, launches, &hg)) return ps;
        h_dense = true;
    }
    const bool h_done = h_dense && !approx;   // regular mode: no budgets, no encoders
    if (w->timing) MCA_CUDA_TRY(cudaEventRecord(w->ev[1], stream));   // end of the (optional) projection
    const long th = tokens * H;
    const double scale = cfg->scale > 0.0 ? cfg->scale : 1.0 / std::sqrt((double)w->dh);

    if (dt == MCA_F32 || force_simt() || n > k1tc::kMaxN)   // atomicMax column keys (the TC pass writes each once)
        MCA_CUDA_TRY(cudaMemsetAsync(w->colkey, 0, th * sizeof(unsigned long long), stream));
    const bool tile_k3 = dt == MCA_BF16 && use_k3t(w);   // k3t reads budgets directly: no work lists
    // bf16 score passes: Eq. 9 values within kCertTau of an integer boundary are
    // re-derived in binary64 by k2c_certify (the fp32 path's scores are fp64 already)
    // fp32: the score passes run 3xTF32 on the tensor cores (column maxima within
    // ~1e-6 of binary64, like the bf16 passes); their Eq. 9 boundary values are
    // always certified, so the fp32 path keeps budgets equal to the fp64 oracle's
    const bool tf32_scores = dt == MCA_F32 && !force_simt() && n <= k1tc::kMaxN;
    const bool certify = (cfg->certify || tf32_scores) && (dt == MCA_BF16 || tf32_scores) && approx &&
                         !(dbg && (dbg->budgets_override || dbg->cmax_override));
    CertSink cert{};
    if (certify) {
        cert.list = w->cert_list;
        cert.cm = w->cert_cm;
        cert.count = w->counters + kCertCounter;
        cert.row_done = w->row_done;
        cert.tau_rel = tf32_scores ? kCertTauTf32 : kCertTauBf16;
        const long items = (long)B * H;
        if (items > w->cap_items) {   // per-item flag slots
            if (w->cap_items) MCA_CUDA_TRY(cudaStreamSynchronize(stream));
            drop_graphs(w);
            cudaFree(w->cert_item_cnt);
            cudaFree(w->cert_slot_j);
            cudaFree(w->cert_slot_cm);
            w->cert_item_cnt = nullptr;
            w->cert_slot_j = nullptr;
            w->cert_slot_cm = nullptr;
            w->cap_items = 0;
            if (cudaMalloc(&w->cert_item_cnt, items * sizeof(unsigned)) != cudaSuccess ||
                cudaMalloc(&w->cert_slot_j, items * kCertSlots * sizeof(int)) != cudaSuccess ||
                cudaMalloc(&w->cert_slot_cm, items * kCertSlots * sizeof(double)) != cudaSuccess) {
                cudaGetLastError();
                return fail(MCA_ERR_ALLOC, "certification slot allocation failed");
            }
            w->cap_items = items;
        }
        MCA_CUDA_TRY(cudaMemsetAsync(w->cert_item_cnt, 0, items * sizeof(unsigned), stream));
        cert.item_cnt = w->cert_item_cnt;
        cert.slot_j = w->cert_slot_j;
        cert.slot_cm = w->cert_slot_cm;
    }


    // K1 + K2 fused (bf16, n <= 768): both score passes and Eq. 9 in one kernel per (b, h)
    const bool fused12 = dt == MCA_BF16 && !force_simt() && !h_done && n <= k12::kMaxTiles * k12::kT &&
                         !(dbg && dbg->cmax_override) && w->d_in <= 1024 &&
                         k12::layout((n + k12::kT - 1) / k12::kT, w->d_in).bytes <= 227u * 1024u;
    if (fused12) {
        CUtensorMap tq, tk;
        if (!make_tmap_bf16(&tq, q, (uint64_t)H * kDh, n, B, 128) || !make_tmap_bf16(&tk, k, (uint64_t)H * kDh, n, B, 128))
            return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for q/k");
        const uint32_t smem = k12::layout((n + k12::kT - 1) / k12::kT, w->d_in).bytes;
        MCA_CUDA_TRY(ensure_smem(k12_fused_tc, smem));
        K12Args a{};
        a.n = n;
        a.heads = H;
        a.d = w->d_in;
        a.dh = w->dh;
        a.min_samples = cfg->min_samples;
        a.scale = (float)scale;
        a.scale_d = scale;
        a.alpha = cfg->alpha;
        a.force_exact = !approx;
        a.budgets_override = dbg ? dbg->budgets_override : nullptr;
        a.exact_override = dbg ? dbg->exact_override : nullptr;
        a.cmax_out = dbg ? dbg->cmax_out : nullptr;
        a.row_m = w->row_m;
        a.row_l = w->row_l;
        a.lse = w->lse;
        a.budgets = w->budgets;
        a.exact = w->exact;
        a.counters = w->counters;
        a.hist = tile_k3 ? nullptr : w->hist;
        a.cert = cert;
        a.items = B * H;
        // The grid's last wave: split its items into per-query-tile units so the
        // wave's leftover CTAs share them (C2: 768 items = 5 x 148 + 28 -> the 28
        // items as 112 one-tile units instead of 28 CTAs running a sixth item).
        const int sms = sm_count(), nt = (n + k12::kT - 1) / k12::kT;
        const int rem = a.items % sms;
        const int parts = rem ? std::min(nt, sms / rem) : 1;
        a.tail_items = parts > 1 && k12_split_enabled() ? rem : 0;
        a.tail_parts = a.tail_items ? parts : 1;
        a.units = a.items - a.tail_items + a.tail_items * a.tail_parts;
        if (a.tail_items && !w->k12_tail) {
            const size_t bytes = (size_t)sms * (k12::kMaxTiles * k12::kT + 2) * sizeof(unsigned);
            if (cudaMalloc(&w->k12_tail, bytes) != cudaSuccess) {
                cudaGetLastError();
                return fail(MCA_ERR_ALLOC, "K12 tail scratch allocation failed");
            }
            MCA_CUDA_TRY(cudaMemsetAsync(w->k12_tail, 0, bytes, stream));
        }
        a.tail = w->k12_tail;
        const int grid = std::min(a.units, sms);   // persistent: one CTA per SM
        MCA_CUDA_TRY(launch_pdl(k12_fused_tc, dim3((unsigned)grid), dim3(k12::kThreads), smem, stream, tq, tk, a));
        MCA_LAUNCH_CHECK("k12_fused_tc");
        mca_diag::dump_k12(stream, n, grid);   // diagnostics builds only
    }
    // K1: row statistics + column maxima
    if (!fused12) {
        const dim3 grid((n + kQT - 1) / kQT, H, B);
        if (dt == MCA_F32 && tf32_scores) {   // 3xTF32 tensor-core score passes on split q, k
            const size_t cnt = (size_t)tokens * H * kDh;
            // q, k are their own hi operands (kind::tf32 ignores the low 13 bits);
            // the lo parts: q_lo | k_lo
            float* parts = static_cast<float*>(w->qk_split);
            const unsigned gs = (unsigned)std::min<size_t>((cnt / 4 + 255) / 256, 8 * (size_t)sm_count());
            if (!qk_lo_done) {
                k_split_tf32<<<gs, 256, 0, stream>>>((const float4*)q, nullptr, (float4*)parts, cnt / 4);
                k_split_tf32<<<gs, 256, 0, stream>>>((const float4*)k, nullptr, (float4*)(parts + cnt), cnt / 4);
                MCA_LAUNCH_CHECK("k_split_tf32");
                ++launches;
            }
            CUtensorMap tqh, tql, tkh, tkl;
            if (!make_tmap_f32(&tqh, q, (uint64_t)H * kDh, n, B, 128) ||
                !make_tmap_f32(&tql, parts, (uint64_t)H * kDh, n, B, 128) ||
                !make_tmap_f32(&tkh, k, (uint64_t)H * kDh, n, B, 128) ||
                !make_tmap_f32(&tkl, parts + cnt, (uint64_t)H * kDh, n, B, 128))
                return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for the q/k tf32 parts");
            MCA_CUDA_TRY(ensure_smem(k1_scores_tc<kRowStats, true>, k1tc::kSmemBytesTf32));
            MCA_CUDA_TRY(ensure_smem(k1_scores_tc<kColMax, true>, k1tc::kSmemBytesTf32));
            const dim3 g1((n + 127) / 128, H, B);
            k1_scores_tc<kRowStats, true><<<g1, k1tc::kThreads, k1tc::kSmemBytesTf32, stream>>>(
                tqh, tkh, tql, tkl, n, H, (float)scale, w->row_m, w->row_l, w->lse, w->colkey, w->colscore);
            if (!h_done) {   // the exact layer needs the row statistics (lse) only
                MCA_LAUNCH_CHECK("k1a_row_stats_tf32");
                k1_scores_tc<kColMax, true><<<g1, k1tc::kThreads, k1tc::kSmemBytesTf32, stream>>>(
                    tqh, tkh, tql, tkl, n, H, (float)scale, w->row_m, w->row_l, w->lse, w->colkey, w->colscore);
            }
        } else if (dt == MCA_F32)
            k1_scores_simt<float, double><<<grid, kThreads, 0, stream>>>((const float*)q, (const float*)k, n, H, scale,
                                                                         w->row_m, w->row_l, w->lse, w->colkey);
        else if (force_simt() || n > k1tc::kMaxN)
            k1_scores_simt<__nv_bfloat16, float><<<grid, kThreads, 0, stream>>>(
                (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, n, H, scale, w->row_m, w->row_l, w->lse,
                w->colkey);
        else {
            CUtensorMap tq, tk;
            if (!make_tmap_bf16(&tq, q, (uint64_t)H * kDh, n, B, 128) ||
                !make_tmap_bf16(&tk, k, (uint64_t)H * kDh, n, B, 128))
                return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for q/k");
            MCA_CUDA_TRY(ensure_smem(k1_scores_tc<kRowStats>, k1tc::kSmemBytes));
            MCA_CUDA_TRY(ensure_smem(k1_scores_tc<kColMax>, k1tc::kSmemBytes));
            const dim3 g1((n + 127) / 128, H, B);
            k1_scores_tc<kRowStats><<<g1, k1tc::kThreads, k1tc::kSmemBytes, stream>>>(
                tq, tk, tq, tk, n, H, (float)scale, w->row_m, w->row_l, w->lse, w->colkey, w->colscore);
            if (!h_done) {   // the exact layer needs the row statistics (lse) only
                MCA_LAUNCH_CHECK("k1a_row_stats");
                k1_scores_tc<kColMax><<<g1, k1tc::kThreads, k1tc::kSmemBytes, stream>>>(
                    tq, tk, tq, tk, n, H, (float)scale, w->row_m, w->row_l, w->lse, w->colkey, w->colscore);
            }
        }
        MCA_LAUNCH_CHECK("k1_scores");
    }
    if (w->timing) MCA_CUDA_TRY(cudaEventRecord(w->ev[2], stream));
    // K2: Eq. 9 budgets (none for the dense exact layer)
    if (!h_done) {
        const dim3 grid = bh_grid((n + 255) / 256, (long)B * H);
        K2Args a{};
        a.colkey = w->colkey;
        a.cmax_in = dbg ? dbg->cmax_override : nullptr;
        a.row_m = w->row_m;
        a.row_l = w->row_l;
        a.q = q;
        a.k = k;
        // K1b's winning score: exact bf16 products (bf16), 3xTF32 (fp32: measured
        // |dcm/cm| <= 1.6e-7 M against the binary64 oracle, tau_tf32 = 3e-6 M)
        a.colscore = ((dt == MCA_BF16 && !force_simt() && n <= k1tc::kMaxN) || tf32_scores) ? w->colscore : nullptr;
        a.scale = scale;
        a.count = th;
        a.row_len = n;
        a.n = n;
        a.heads = H;
        a.d = w->d_in;
        a.dh = w->dh;
        a.min_samples = cfg->min_samples;
        a.alpha = cfg->alpha;
        a.force_exact = !approx;
        a.budgets_override = dbg ? dbg->budgets_override : nullptr;
        a.exact_override = dbg ? dbg->exact_override : nullptr;
        a.budgets = w->budgets;
        a.exact = w->exact;
        a.cmax_out = dbg ? dbg->cmax_out : nullptr;
        a.counters = w->counters;
        a.hist = tile_k3 ? nullptr : w->hist;
        a.cert = cert;
        if (!fused12) {
            if (a.cmax_in) k2_budgets<kGivenCmax, float><<<grid, 256, 0, stream>>>(a);
            else if (tf32_scores) k2_budgets<kKeyArgmax, float><<<grid, 256, 0, stream>>>(a);   // winner score from K1b
            else if (dt == MCA_F32) k2_budgets<kKeyValue, float><<<grid, 256, 0, stream>>>(a);
            else k2_budgets<kKeyArgmax, __nv_bfloat16><<<grid, 256, 0, stream>>>(a);
            MCA_LAUNCH_CHECK("k2_budgets");
        }
        if (certify) {   // the flagged token-heads' budgets, FLOP counts and histogram entries
            K2cArgs c{};
            c.q = q;
            c.k = k;
            c.lse = w->lse;
            c.scale = scale;
            c.n = n;
            c.heads = H;
            c.items = B * H;
            c.d = w->d_in;
            c.dh = w->dh;
            c.min_samples = cfg->min_samples;
            c.alpha = cfg->alpha;
            c.cert = cert;
            c.row_m = w->row_m;
            c.row_l = w->row_l;
            c.budgets = w->budgets;
            c.exact = w->exact;
            c.cmax_out = dbg ? dbg->cmax_out : nullptr;
            c.counters = w->counters;
            c.hist = tile_k3 ? nullptr : w->hist;
            c.cert_total = w->counters + kCertTotal;
            const int gc = B * H;   // one CTA per (b, h) item; items without flags exit at once
            if (dt == MCA_F32) MCA_CUDA_TRY(launch_pdl(k2c_certify<float>, dim3((unsigned)gc), dim3(kCertThreads), 0, stream, c));
            else MCA_CUDA_TRY(launch_pdl(k2c_certify<__nv_bfloat16>, dim3((unsigned)gc), dim3(kCertThreads), 0, stream, c));
            MCA_LAUNCH_CHECK("k2c_certify");
        }
        if (!tile_k3) {
            if (mca_status s = launch_lists(w, grid, n, tokens, stream, launches)) return s;
        }
    }
    // bf16 MCA layer: when K2 marks at least kDenseExactFrac of the token-heads exact
    // (small alpha), their encodings come from one dense X W_V GEMM (every row; K3
    // then rewrites the sampled token-heads' rows) instead of k3b_exact_tc's gathered
    // tiles. Decided on the device: both kernels read K2's counts, one of them exits.
    const bool dense_gate = dt == MCA_BF16 && approx && !force_simt() && !tile_k3 && dense_exact_enabled();
    if (dense_gate) {
        void* outs[3] = {nullptr, nullptr, w->hbuf};
        const KpArgs hg = h_guard(w, n, w->exact, w->counts, dense_exact_min(th));
        if (mca_status ps = launch_projection(w, x, tokens, 2, 1, outs, 0b100, stream, launches, &hg)) return ps;
    }
    if (w->timing) MCA_CUDA_TRY(cudaEventRecord(w->ev[3], stream));
    // K3: encoding (the dense exact layer's H came out of the projection GEMM)
    if (!h_done) {
        int32_t* draws = dbg ? dbg->draws_out : nullptr;
        const int stride = dbg ? dbg->draws_stride : 0;
        mca_status s = dt == MCA_F32
                           ? launch_k3<float, double>(w, x, B, n, b_offset, layer, seed, w->hbuf, draws, stride,
                                                      stream, launches, h_dense)
                           : launch_k3<__nv_bfloat16, float>(w, x, B, n, b_offset, layer, seed, w->hbuf, draws, stride,
                                                             stream, launches, false, dense_gate ? dense_exact_min(th) : 0);
        if (s) return s;
    }
    if (w->timing) MCA_CUDA_TRY(cudaEventRecord(w->ev[4], stream));
    // K4: y = A . H~
    {
        const dim3 grid((n + kQT4 - 1) / kQT4, H, B);
        if (dt == MCA_F32 && tf32_scores) {   // 3xTF32 on the tensor cores: split q / k from K1, H~^T split here
            const int n_pad = (n + 3) & ~3;     // TMA: the transposed rows' stride is a multiple of 16 B
            const size_t need = 2 * (size_t)B * H * kDh * n_pad;
            if (need > w->cap_vt) {
                if (w->cap_vt) MCA_CUDA_TRY(cudaStreamSynchronize(stream));
                drop_graphs(w);
                cudaFree(w->vt_split);
                w->vt_split = nullptr;
                w->cap_vt = 0;
                if (cudaMalloc(&w->vt_split, need * sizeof(float)) != cudaSuccess) {
                    cudaGetLastError();
                    return fail(MCA_ERR_ALLOC, "H~ split workspace allocation failed");
                }
                w->cap_vt = need;
            }
            float* vh = w->vt_split;
            float* vl = w->vt_split + need / 2;
            k_split_transpose_h<<<dim3((n + 63) / 64, H, B), 256, 0, stream>>>((const float*)w->hbuf, n, n_pad, H, vh,
                                                                                vl);
            MCA_LAUNCH_CHECK("k_split_transpose_h");
            const size_t cnt = (size_t)tokens * H * kDh;
            float* parts = static_cast<float*>(w->qk_split);
            CUtensorMap tqh, tql, tkh, tkl, tvh, tvl;
            auto vmap = [&](CUtensorMap* m, const float* base) { return make_vt_map(m, base, n, n_pad, (long)B * H); };
            if (!make_tmap_f32(&tqh, q, (uint64_t)H * kDh, n, B, 128) ||
                !make_tmap_f32(&tql, parts, (uint64_t)H * kDh, n, B, 128) ||
                !make_tmap_f32(&tkh, k, (uint64_t)H * kDh, n, B, k4tf::kBK) ||
                !make_tmap_f32(&tkl, parts + cnt, (uint64_t)H * kDh, n, B, k4tf::kBK) || !vmap(&tvh, vh) ||
                !vmap(&tvl, vl))
                return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for the K4 tf32 operands");
            MCA_CUDA_TRY(ensure_smem(k4_apply_tf32, k4tf::kSmemBytes));
            const dim3 g4((n + k4tf::kBM - 1) / k4tf::kBM, H, B);
            MCA_CUDA_TRY(launch_pdl(k4_apply_tf32, g4, dim3(k4tf::kThreads), k4tf::kSmemBytes, stream, tqh, tql, tkh,
                                    tkl, tvh, tvl, (const float*)w->lse, n, H, (float)scale, (float*)y));
        } else if (dt == MCA_F32)
            k4_apply_simt<float><<<grid, kT4, 0, stream>>>((const float*)q, (const float*)k, (const float*)w->hbuf,
                                                            w->lse, n, H, (float)scale, (float*)y);
        else if (force_simt())
            k4_apply_simt<__nv_bfloat16><<<grid, kT4, 0, stream>>>(
                (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __half*)w->hbuf, w->lse, n, H,
                (float)scale, (__nv_bfloat16*)y);
        else {
            CUtensorMap tk, th;
            if (!make_tmap_bf16(&tk, k, (uint64_t)H * kDh, n, B, k4tc::kBK) ||
                !make_tmap_bf16(&th, w->hbuf, (uint64_t)H * kDh, n, B, k4tc::kBK, CU_TENSOR_MAP_DATA_TYPE_FLOAT16))
                return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for k/h");
            MCA_CUDA_TRY(ensure_smem(k4_apply_tc, k4tc::kSmemBytes));
            const long tiles = (long)B * H * ((n + k4tc::kBM - 1) / k4tc::kBM);
            const int grid = (int)std::min<long>(tiles, 2L * sm_count());   // persistent: two CTAs per SM
            K4oArgs o{};
            o.ovf.count = w->counters + kOvfCounter;
            o.ovf.list = w->ovf_list;
            o.ovf.rows = w->ovf_rows;
            o.ovf.cap = (int)w->ovf_cap;
            o.q = q;
            o.k = k;
            o.lse = w->lse;
            o.scale = scale;
            o.n = n;
            o.heads = H;
            o.y = (__nv_bfloat16*)y;
            MCA_CUDA_TRY(launch_pdl(k4_apply_tc, dim3(grid), dim3(k4tc::kThreads), k4tc::kSmemBytes, stream,
                                    (const __nv_bfloat16*)q, tk, th, (const float*)w->lse, n, H, B, (float)scale,
                                    (__nv_bfloat16*)y, o, w->counters + kK4DoneCounter));
            mca_diag::dump_k4(stream, n, k4tc::kBK);   // diagnostics builds only
        }
        MCA_LAUNCH_CHECK("k4_apply");
        if (dt == MCA_BF16 && !h_done && force_simt())   // the CUDA-core K4 has no built-in range-guard fix-up
            if (mca_status s = launch_overflow_fixup(w, false, q, k, nullptr, scale, B, n, y, stream, launches)) return s;
    }
    if (w->timing) {
        MCA_CUDA_TRY(cudaEventRecord(w->ev[5], stream));
        w->ev_valid = true;
    }
    // optional outputs
    if (budgets_out)
        MCA_CUDA_TRY(cudaMemcpyAsync(budgets_out, w->budgets, th * sizeof(int32_t), cudaMemcpyDeviceToDevice, stream));
    if (exact_out)
        MCA_CUDA_TRY(cudaMemcpyAsync(exact_out, w->exact, th * sizeof(uint8_t), cudaMemcpyDeviceToDevice, stream));
    if (dbg && dbg->lse_out)
        MCA_CUDA_TRY(cudaMemcpyAsync(dbg->lse_out, w->lse, th * sizeof(float), cudaMemcpyDeviceToDevice, stream));
    if (dbg && dbg->h_out)
        MCA_CUDA_TRY(cudaMemcpyAsync(dbg->h_out, w->hbuf, th * w->dh * dtype_size(dt), cudaMemcpyDeviceToDevice,
                                     stream));
    w->last_launches = launches;
    if (flops_out) return read_flops(w, B, n, approx, flops_out, stream);
    return MCA_OK;
}

mca_status mca_forward_attn(mca_weights* w, const double* attn, const void* x, mca_dtype dt, int B, int n,
                            long b_offset, uint32_t layer, const mca_config* cfg, uint64_t seed, void* y,
                            int32_t* budgets_out, uint8_t* exact_out, mca_flops* flops_out, mca_stream_t stream) {
    if (!w) return fail(MCA_ERR_NULL, "weights is NULL");
    if (mca_status s = check_config(cfg, true)) return s;
    if (B < 0 || n <= 0) return fail(MCA_ERR_SHAPE, "B = %d, n = %d: need B >= 0, n >= 1", B, n);
    if (dt != w->wdt) return fail(MCA_ERR_CONFIG, "activation dtype %d != weight dtype %d", (int)dt, (int)w->wdt);
    if (b_offset < 0) return fail(MCA_ERR_SHAPE, "b_offset < 0");
    if (n > 65535 || B > 65535)
        return fail(MCA_ERR_UNSUPPORTED, "B = %d, n = %d: work lists pack (b, j) into 16 bits each", B, n);
    if (flops_out) std::memset(flops_out, 0, sizeof(*flops_out));
    if (B == 0) {
        w->last_launches = 0;
        return MCA_OK;
    }
    if (!attn || !x || !y) return fail(MCA_ERR_NULL, "attn / x / y is NULL");
    const bool approx = cfg->mode == MCA_MODE_APPROX;
    const long tokens = (long)B * n;
    if (mca_status s = ensure_workspace(w, tokens, stream)) return s;
    const int H = w->heads;
    const long th = tokens * H;
    int launches = 0;
    MCA_CUDA_TRY(cudaMemsetAsync(w->zeroed, 0, zeroed_bytes(H, w->d_in), stream));   // counters, cursors, histograms
    double* cmax = reinterpret_cast<double*>(w->colkey);                             // [B, H, n] scratch
    const dim3 grid = bh_grid((n + 255) / 256, (long)B * H);
    ka_colmax<<<bh_grid((n + 31) / 32, (long)B * H), dim3(32, 8), 0, stream>>>(attn, n, (long)B * H, cmax);
    MCA_LAUNCH_CHECK("ka_colmax");
    K2Args a{};
    a.cmax_in = cmax;
    a.count = th;
    a.row_len = n;
    a.n = n;
    a.heads = H;
    a.d = w->d_in;
    a.dh = w->dh;
    a.min_samples = cfg->min_samples;
    a.alpha = cfg->alpha;
    a.force_exact = !approx;
    a.budgets = w->budgets;
    a.exact = w->exact;
    a.counters = w->counters;
    a.hist = w->hist;
    k2_budgets<kGivenCmax, float><<<grid, 256, 0, stream>>>(a);
    MCA_LAUNCH_CHECK("k2_budgets");
    if (mca_status s = launch_lists(w, grid, n, tokens, stream, launches)) return s;
    mca_status s = dt == MCA_F32 ? launch_k3<float, double>(w, x, B, n, b_offset, layer, seed, w->hbuf, nullptr, 0,
                                                            stream, launches)
                                 : launch_k3<__nv_bfloat16, float>(w, x, B, n, b_offset, layer, seed, w->hbuf, nullptr,
                                                                   0, stream, launches);
    if (s) return s;
    if (force_simt()) {   // CUDA cores, fp64 accumulation
        const dim3 ga(n, H, B);
        if (dt == MCA_F32)
            ka_aggregate<float, float><<<ga, kDh, 0, stream>>>(attn, (const float*)w->hbuf, n, H, (float*)y);
        else
            ka_aggregate<__nv_bfloat16, __half><<<ga, kDh, 0, stream>>>(attn, (const __half*)w->hbuf, n, H,
                                                                       (__nv_bfloat16*)y);
        MCA_LAUNCH_CHECK("ka_aggregate");
    } else {   // tensor cores: the fp64 dump rounded to fp32, split hi / lo; H~ transposed per head
        const int n_pad = (n + 3) & ~3;
        const size_t part = (size_t)B * H * kDh * n_pad;
        const size_t need = (dt == MCA_F32 ? 2 : 1) * part;
        if (need > w->cap_vt) {
            if (w->cap_vt) MCA_CUDA_TRY(cudaStreamSynchronize(stream));
            drop_graphs(w);
            cudaFree(w->vt_split);
            w->vt_split = nullptr;
            w->cap_vt = 0;
            if (cudaMalloc(&w->vt_split, need * sizeof(float)) != cudaSuccess) {
                cudaGetLastError();
                return fail(MCA_ERR_ALLOC, "H~ transpose workspace allocation failed");
            }
            w->cap_vt = need;
        }
        float* vh = w->vt_split;
        float* vl = dt == MCA_F32 ? w->vt_split + part : vh;
        const dim3 gt((n + 63) / 64, H, B);
        if (dt == MCA_F32)
            k_split_transpose_h<<<gt, 256, 0, stream>>>((const float*)w->hbuf, n, n_pad, H, vh, vl);
        else
            k_transpose_h16<<<gt, 256, 0, stream>>>((const __half*)w->hbuf, n, n_pad, H, vh);
        MCA_LAUNCH_CHECK("k_transpose_h");
        CUtensorMap tvh, tvl;
        if (!make_vt_map(&tvh, vh, n, n_pad, (long)B * H) || !make_vt_map(&tvl, vl, n, n_pad, (long)B * H))
            return fail(MCA_ERR_CUDA, "cuTensorMapEncodeTiled failed for H~^T");
        const dim3 g4((n + katc::kBM - 1) / katc::kBM, H, B);
        if (dt == MCA_F32) {
            MCA_CUDA_TRY(ensure_smem(ka_aggregate_tc<true, float>, katc::kSmemBytes));
            MCA_CUDA_TRY(launch_pdl(ka_aggregate_tc<true, float>, g4, dim3(katc::kThreads), katc::kSmemBytes, stream,
                                    tvh, tvl, attn, n, H, (float*)y));
        } else {
            MCA_CUDA_TRY(ensure_smem(ka_aggregate_tc<false, __nv_bfloat16>, katc::kSmemBytes));
            MCA_CUDA_TRY(launch_pdl(ka_aggregate_tc<false, __nv_bfloat16>, g4, dim3(katc::kThreads), katc::kSmemBytes,
                                    stream, tvh, tvl, attn, n, H, (__nv_bfloat16*)y));
        }
        MCA_LAUNCH_CHECK("ka_aggregate_tc");
    }
    if (dt == MCA_BF16)   // encodings outside fp16's range (normally none)
        if (mca_status s2 = launch_overflow_fixup(w, true, nullptr, nullptr, attn, 0.0, B, n, y, stream, launches))
            return s2;
    if (budgets_out)
        MCA_CUDA_TRY(cudaMemcpyAsync(budgets_out, w->budgets, th * sizeof(int32_t), cudaMemcpyDeviceToDevice, stream));
    if (exact_out)
        MCA_CUDA_TRY(cudaMemcpyAsync(exact_out, w->exact, th * sizeof(uint8_t), cudaMemcpyDeviceToDevice, stream));
    w->last_launches = launches;
    if (flops_out) return read_flops(w, B, n, approx, flops_out, stream);
    return MCA_OK;
}

mca_status mca_forward(mca_weights* w, const void* q, const void* k, const void* x, mca_dtype dt, int B, int n,
                       long b_offset, uint32_t layer, const mca_config* cfg, uint64_t seed, void* y,
                       int32_t* budgets_out, uint8_t* exact_out, mca_flops* flops_out, mca_stream_t stream) {
    static const bool use_graphs = !getenv("MCA_GRAPHS") || atoi(getenv("MCA_GRAPHS")) != 0;   // default on
    // graphs need a capturable stream, no host read-back and no stage events
    if (!use_graphs || !w || !cfg || !stream || flops_out || w->timing)
        return mca_forward_ex(w, q, k, x, dt, B, n, b_offset, layer, cfg, seed, y, budgets_out, exact_out, flops_out,
                              nullptr, stream);
    uint64_t key[16] = {(uint64_t)q, (uint64_t)k, (uint64_t)x, (uint64_t)y, (uint64_t)dt, (uint64_t)B, (uint64_t)n,
                        (uint64_t)b_offset, (uint64_t)layer, seed, (uint64_t)budgets_out, (uint64_t)exact_out,
                        (uint64_t)stream, 0, 0,
                        (uint64_t)(uint32_t)cfg->min_samples | ((uint64_t)(cfg->mode & 0xFF) << 32) |
                            ((uint64_t)(cfg->certify != 0) << 40)};
    std::memcpy(&key[13], &cfg->alpha, 8);
    std::memcpy(&key[14], &cfg->scale, 8);
    auto eager = [&]() {
        return mca_forward_ex(w, q, k, x, dt, B, n, b_offset, layer, cfg, seed, y, budgets_out, exact_out, nullptr,
                              nullptr, stream);
    };
    // the caller may itself be capturing this stream (e.g. torch CUDA graphs):
    // then our kernels simply join its capture
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return eager();
    }
    mca_weights::GraphEntry* e = nullptr;
    for (auto& g : w->graphs)
        if (std::memcmp(g.key, key, sizeof(key)) == 0) e = &g;
    if (e) e->last_use = ++w->graph_clock;
    if (e && e->exec) {
        MCA_CUDA_TRY(cudaGraphLaunch(e->exec, stream));
        return MCA_OK;
    }
    if (!e) {   // first sighting: eager (sizes the workspace), remembered
        if (w->graphs.size() >= kMaxGraphs) {   // evict the least recently used key
            auto lru = std::min_element(w->graphs.begin(), w->graphs.end(),
                                        [](const auto& a, const auto& b) { return a.last_use < b.last_use; });
            if (lru->exec) cudaGraphExecDestroy(lru->exec);
            *lru = w->graphs.back();
            w->graphs.pop_back();
        }
        w->graphs.push_back({});
        std::memcpy(w->graphs.back().key, key, sizeof(key));
        w->graphs.back().last_use = ++w->graph_clock;
        return eager();
    }
    if (!e->graphable) return eager();
    // second sighting: capture this forward and replay it from now on. A
    // capture or instantiation failure marks the key eager-only and still
    // runs the forward.
    if (cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        e->graphable = false;
        return eager();
    }
    const mca_status s = mca_forward_ex(w, q, k, x, dt, B, n, b_offset, layer, cfg, seed, y, budgets_out, exact_out,
                                        nullptr, nullptr, stream);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(stream, &graph);
    cudaGraphExec_t exec = nullptr;
    const bool ok = s == MCA_OK && ce == cudaSuccess && graph && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    // the forward may have grown the workspace (drop_graphs cleared the cache): re-find the entry
    e = nullptr;
    for (auto& g : w->graphs)
        if (std::memcmp(g.key, key, sizeof(key)) == 0) e = &g;
    if (!e) {
        w->graphs.push_back({});
        e = &w->graphs.back();
        std::memcpy(e->key, key, sizeof(key));
    }
    if (!ok) {
        if (exec) cudaGraphExecDestroy(exec);
        if (s != MCA_OK && ce == cudaSuccess) return s;    // an argument / launch error: report it
        e->graphable = false;
        return eager();
    }
    e->exec = exec;
    e->last_use = ++w->graph_clock;
    MCA_CUDA_TRY(cudaGraphLaunch(exec, stream));
    return MCA_OK;
}

mca_status mca_regular_forward(mca_weights* w, const void* q, const void* k, const void* x, mca_dtype dt, int B,
                               int n, double scale, void* y, mca_stream_t stream) {
    mca_config cfg{1.0, scale, 1, MCA_MODE_REGULAR, 0, 0};
    return mca_forward_ex(w, q, k, x, dt, B, n, 0, 0, &cfg, 0, y, nullptr, nullptr, nullptr, nullptr, stream);
}

}  // extern "C"

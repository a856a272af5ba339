/* mca/mca_cuda.h — C ABI of the B200 Monte-Carlo Attention forward.
 *
 * This is the drop-in boundary for the reference's MCA path. The reference
 * declares its tensor layer in proj/include/mca/matrix.hpp:7-55 and specifies
 * the attention-layer operations in SPEC.md (no definitions ship). Each entry
 * point below names the reference operation it replaces:
 *
 *   mca_prepare_weights   weight_probs + make_distribution, cached once per W
 *                         (AttentionWeights.cached_dist
 *                         SPEC.md:260-265; "embedded in the model or cached")
 *   mca_forward           multihead_forward / mca_forward in approximation mode
 *                         (SPEC.md:306-314, 326-334): attention_matrix's softmax
 *                         (matrix.hpp:46-50) + col_max (matrix.hpp:52-53) +
 *                         sample_budgets + approx_encode_row /
 *                         draw_indices + matmul(A, H~)
 *                         (matrix.hpp:33-34) + flops_for_plan
 *   mca_set_projections   AttentionWeights.w_q / w_k: with them
 *                         attached, mca_forward takes x alone and computes
 *                         attention_matrix's projections q = x w_q, k = x w_k
 *                          on the device
 *   mca_regular_forward   regular_forward
 *   mca_stage_budgets     sample_budgets on given column maxima
 *   mca_forward_attn      the layer on a given attention matrix: what cmd_bench /
 *                         cmd_attn_import drive
 *
 * Conventions:
 *   - Plain C: pointers and sizes only, no exceptions cross this boundary.
 *     Status codes mirror the SPEC error classes; mca_last_error() returns the
 *     thread-local message of the last failure.
 *   - All tensor pointers are DEVICE pointers (cudaMalloc'd or torch CUDA
 *     storage) unless a parameter says "host". Work is enqueued on `stream`
 *     (a cudaStream_t; NULL = legacy default stream) and is asynchronous,
 *     except where a host output (flops_out) is requested.
 *   - Layouts (row-major, contiguous):
 *       q, k, y, h~   [B, n, heads*d_h]   (the projection-output layout)
 *       x             [B, n, d_in]
 *       w_v           [d_in, heads*d_h]   (x @ w_v convention)
 *       per-token     [B, heads, n]       (budgets, exact mask, cmax, lse)
 *   - Head h of sequence b uses Philox stream ((b_offset + b) * heads + h) * n + j
 *     and counter word 1 = layer; b_offset lets a batch shard
 *     reproduce the unsharded result bit for bit.
 */
#ifndef MCA_CUDA_H_
#define MCA_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* mca_stream_t; /* == cudaStream_t */

typedef enum mca_status {
    MCA_OK = 0,
    MCA_ERR_SHAPE = 1,       /* shape mismatch                       */
    MCA_ERR_DOMAIN = 2,      /* alpha not in (0,1], r == 0               */
    MCA_ERR_DEGENERATE = 3,  /* zero W_h / all-zero weights          */
    MCA_ERR_CONFIG = 4,      /* d not divisible by heads, bad mode        */
    MCA_ERR_CUDA = 5,        /* CUDA runtime error (message has the CUDA error string)       */
    MCA_ERR_ALLOC = 6,       /* device allocation failed                                     */
    MCA_ERR_UNSUPPORTED = 7, /* shape outside what the sm_100a kernels implement */
    MCA_ERR_NULL = 8         /* required pointer is NULL                                     */
} mca_status;

typedef enum mca_dtype { MCA_F32 = 0, MCA_BF16 = 1 } mca_dtype;

typedef enum mca_mode { MCA_MODE_REGULAR = 0, MCA_MODE_APPROX = 1 } mca_mode;

/* McaConfig. scale <= 0 selects 1/sqrt(d_h). */
typedef struct mca_config {
    double alpha;        /* attention error coefficient, (0, 1]            */
    double scale;        /* softmax scale a                                */
    int32_t min_samples; /* budget floor (default 1)                       */
    int32_t mode;        /* mca_mode                                       */
    int32_t certify;     /* bf16: re-derive in binary64 every Eq. 9 value within 1e-5 of
                            an integer boundary (k2c_certify), so the budgets equal the
                            fp64 reference's end to end; 0 = off     */
    int32_t reserved;
} mca_config;

/* FlopsReport, summed over heads and batch. `samples` is
 * the instrumented count of draws the encoding kernel actually processed
 * (must equal sum of sampled budgets). */
typedef struct mca_flops {
    uint64_t exact_encoding;
    uint64_t approx_encoding;
    uint64_t aggregation;
    uint64_t samples;
    uint64_t exact_tokens;
    double reduction_factor;
    double total_reduction;
    uint64_t certified;      /* token-heads whose Eq. 9 value sat within 1e-5 of an integer
                                boundary and was re-derived in binary64 (k2c_certify) */
} mca_flops;

/* Optional stage outputs / overrides for parity testing (all device, [B,heads,n]
 * unless noted; every field nullable). */
typedef struct mca_debug {
    double* cmax_out;                /* column maxima of A (fp64: exactly what Eq. 9 consumed) */
    float* lse_out;                  /* per-row log-sum-exp of the scaled scores             */
    void* h_out;                     /* H~ [B, n, heads*d_h]: fp32 (fp32 path) / fp16 (bf16)  */
    int32_t* draws_out;              /* [B, heads, n, draws_stride]: first draws, -1 padded  */
    int32_t draws_stride;
    int32_t reserved;
    const double* cmax_override;     /* replace the score pass's cmax before Eq. 9           */
    const int32_t* budgets_override; /* replace Eq. 9's budgets (with exact_override)        */
    const uint8_t* exact_override;
    void* q_out;                     /* the projected q [B, n, heads*d_h] (q == NULL forwards) */
    void* k_out;                     /* the projected k                                      */
} mca_debug;

typedef struct mca_weights mca_weights;

/* One-time preparation (K0, on the device): copies w_v, builds per-head
 * p(i) = ||W_h[i]||^2 / ||W_h||_F^2 (fp64, fixed accumulation order), the cdf,
 * the 53-bit integer inverse-CDF thresholds and the guide table. Synchronises
 * `stream` once to report degenerate heads. */
mca_status mca_prepare_weights(const void* w_v, mca_dtype wdt, int d_in, int heads, int d_h,
                               mca_stream_t stream, mca_weights** out);
void mca_weights_free(mca_weights* w);

/* Attach W_q and W_k ([d_in, heads*d_h], the weights' dtype, device
 * pointers; copied, transposed). A forward called with q == k == NULL then
 * computes q = x W_q and k = x W_k on `stream` first (the tcgen05 projection
 * GEMM: bf16 with fp32 accumulation, 3xTF32 on the fp32 path). */
mca_status mca_set_projections(mca_weights* w, const void* w_q, const void* w_k, mca_stream_t stream);

/* Copy the per-head fp64 probabilities / cdf ([heads, d_in], host buffers). */
mca_status mca_weights_export(const mca_weights* w, double* probs_host, double* cdf_host);

/* Pre-size the workspace for up to `max_tokens` = B*n tokens (optional; the
 * forward grows it on demand, which synchronises). */
mca_status mca_reserve(mca_weights* w, long max_tokens, mca_stream_t stream);

/* MCA forward (approximation mode, or cfg->mode == MCA_MODE_REGULAR for the
 * exact layer). q and k may both be NULL when the weights carry W_q / W_k
 * (mca_set_projections): the reference's mca_forward(x, weights, ...).
 * budgets_out / exact_out are optional device outputs; flops_out is an
 * optional HOST output (synchronises the stream). */
mca_status mca_forward(mca_weights* w, const void* q, const void* k, const void* x, mca_dtype dt, int B, int n,
                       long b_offset, uint32_t layer, const mca_config* cfg, uint64_t seed, void* y,
                       int32_t* budgets_out, uint8_t* exact_out, mca_flops* flops_out, mca_stream_t stream);

/* mca_forward plus the parity-testing hooks of mca_debug. */
mca_status mca_forward_ex(mca_weights* w, const void* q, const void* k, const void* x, mca_dtype dt, int B, int n,
                          long b_offset, uint32_t layer, const mca_config* cfg, uint64_t seed, void* y,
                          int32_t* budgets_out, uint8_t* exact_out, mca_flops* flops_out, const mca_debug* dbg,
                          mca_stream_t stream);

/* The layer on a GIVEN attention matrix (the cli's imported or synthetic
 * attention, cmd_bench / cmd_attn_import): budgets from attn's
 * column maxima (Eq. 9 on the exact fp64 entries), H~ by the forward's encoding
 * kernels, y = attn . H~ (fp64 accumulation). attn: DEVICE fp64
 * [B, heads, n, n], row i = query i. cfg->mode == MCA_MODE_REGULAR gives
 * attn . (x W_V). Desk-scale analysis path (CUDA-core aggregation). */
mca_status mca_forward_attn(mca_weights* w, const double* attn, const void* x, mca_dtype dt, int B, int n,
                            long b_offset, uint32_t layer, const mca_config* cfg, uint64_t seed, void* y,
                            int32_t* budgets_out, uint8_t* exact_out, mca_flops* flops_out, mca_stream_t stream);

/* Exact layer Y = softmax(a Q K^T) (X W_V). */
mca_status mca_regular_forward(mca_weights* w, const void* q, const void* k, const void* x, mca_dtype dt, int B,
                               int n, double scale, void* y, mca_stream_t stream);

/* Eq. 9 on given column maxima (device, `count` values): the budget kernel in
 * isolation. */
mca_status mca_stage_budgets(const double* cmax, long count, int n, int d, const mca_config* cfg, int32_t* budgets,
                             uint8_t* exact, mca_stream_t stream);

/* Stage timing with CUDA events recorded on the forward's stream (off by
 * default). mca_last_stage_ms synchronises on the last forward's events and
 * writes per-stage device ms in order: score pass, budgets, encoding,
 * aggregation; it returns the number of stages written (0 if disabled). */
mca_status mca_set_timing(mca_weights* w, int enable);
int mca_last_stage_ms(const mca_weights* w, float* ms, int max_stages);

/* Number of kernels the last forward enqueued. */
int mca_last_launch_count(const mca_weights* w);

/* Device buffers and synchronous copies for host callers that do not link the
 * CUDA runtime themselves (include/mca/mca.hpp uses these, so a C++ caller
 * links -lmca_b200 alone). Allocation is on the current device. */
typedef enum mca_copy_kind { MCA_COPY_H2D = 0, MCA_COPY_D2H = 1, MCA_COPY_D2D = 2 } mca_copy_kind;
mca_status mca_device_alloc(size_t bytes, void** out);
void mca_device_free(void* p);
mca_status mca_copy(void* dst, const void* src, size_t bytes, mca_copy_kind kind);
mca_status mca_stream_sync(mca_stream_t stream);

const char* mca_last_error(void);
const char* mca_version(void);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* MCA_CUDA_H_ */

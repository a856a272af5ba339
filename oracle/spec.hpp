// oracle/spec.hpp — fp64 CPU restatement of the MCA SPEC modules above the
// tensor layer: sampling, amm, attention, metrics.
//
// TEST INFRASTRUCTURE ONLY. This is the checker the GPU path is compared
// against (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline leg and
// `--impl reference`). Nothing in the product (paper_2201_12854_b200/) links,
// imports or calls it.
//
// The reference ships declarations only (proj/include/mca/matrix.hpp) and a
// behavioural spec; every op below cites the SPEC lines it restates.
// Choices the SPEC leaves open are pinned here once, and documented in
// DESIGN.md §3 (generator, uniform, inverse-CDF rule, stream ids, budget
// arithmetic). They are pinned externally by the Philox4x32-10 known-answer
// vectors of Random123 (tests/test_oracle_sampling.py).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "mca/matrix.hpp"

namespace mca {

// SPEC error classes.
struct shape_error : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct domain_error : std::domain_error { using std::domain_error::domain_error; };
struct degenerate_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct config_error : std::runtime_error { using std::runtime_error::runtime_error; };

// ---------------------------------------------------------------- sampling
// Philox4x32-10 block function (Salmon et al., SC'11; Random123 v1.14
// philox.h round/bump constants). ctr/key/out are little-endian 32-bit words.
void philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

// RngStream. Counter-based: draw k of stream (seed, stream_id,
// layer) is a pure function of (seed, stream_id, layer, k):
//   key = {seed_lo, seed_hi}; ctr = {k >> 1, layer, stream_lo, stream_hi}
//   even k -> words (x0 low, x1 high); odd k -> (x2 low, x3 high)
//   m = u64 >> 11 (53 bits);  u = m * 2^-53 in [0, 1)
struct RngStream {
    uint64_t seed = 0;
    uint64_t stream_id = 0;
    uint32_t layer = 0;
    uint64_t counter = 0;  // index k of the next draw
    RngStream(uint64_t s, uint64_t id, uint32_t l = 0) : seed(s), stream_id(id), layer(l) {}
    uint64_t next_bits53();  // m
    double next_uniform();   // m * 2^-53
};
uint64_t philox_bits53(uint64_t seed, uint64_t stream_id, uint32_t layer, uint64_t k);

// SamplingDistribution.
struct SamplingDistribution {
    std::vector<double> probs;
    std::vector<double> cdf;
};

// SPEC.md:136-144 and the <1e-15 clamp of SPEC.md:163. Accumulation orders are
// fixed: total = sequential left-to-right sum; renormalisation happens only
// when an entry was clamped; cdf is the sequential prefix sum, forced to
// exactly 1.0 from the last positive entry onwards (so zero-probability
// trailing entries can never be drawn and the search always terminates).
SamplingDistribution make_distribution(const std::vector<double>& weights);

// inverse transform, first i with cdf[i] > u (binary
// search, std::upper_bound).
std::vector<std::size_t> draw_indices(const SamplingDistribution& dist, std::size_t r, RngStream& rng);

// --------------------------------------------------------------------- amm
// SPEC.md:191-199 (Eq. 4).
SamplingDistribution optimal_probs(const Matrix& a, const Matrix& b);
// SPEC.md:201-209 (Eq. 6). Squared row norms are accumulated left to right
// over the row, never via sqrt-then-square.
SamplingDistribution weight_probs(const Matrix& w);

struct AmmEstimate {
    Matrix value;
    std::size_t samples_used = 0;
};
// SPEC.md:211-219 (Eq. 2); per-sample 1/(r p) scaling.
AmmEstimate approx_matmul(const Matrix& a, const Matrix& b, const SamplingDistribution& dist,
                          std::size_t r, RngStream& rng);
// SPEC.md:221-229 (Lemma 1's H[i]); w may be d x d_out (d_out != d for heads).
std::vector<double> approx_encode_row(const double* x_row, const Matrix& w,
                                      const SamplingDistribution& dist, std::size_t r,
                                      RngStream& rng);

// ---------------------------------------------------------------- attention
enum class Mode { regular = 0, approximation = 1 };

struct McaConfig {
    double alpha = 0.4;
    Mode mode = Mode::approximation;
    std::size_t min_samples = 1;
    std::size_t heads = 1;
};

struct AttentionWeights {
    Matrix w_q, w_k, w;
    SamplingDistribution cached_dist;
};
AttentionWeights make_attention_weights(Matrix w_q, Matrix w_k, Matrix w);

struct SamplePlan {
    std::vector<std::size_t> budgets;
    std::vector<uint8_t> exact_mask;
    std::vector<std::vector<std::size_t>> draws;
};

struct FlopsReport {
    uint64_t exact_encoding = 0;
    uint64_t approx_encoding = 0;
    uint64_t aggregation = 0;
    double reduction_factor = 1.0;
    double total_reduction = 1.0;
};

struct AttentionOutput {
    Matrix y;
    SamplePlan plan;
    FlopsReport flops;
    Matrix attn;
};

// One Eq. 9 budget: t = (n * cmax) / alpha; raw = t * t;
// c = ceil(raw); exact = c >= d; r = clamp(c, min_samples, d). Each operation
// is a single correctly rounded IEEE binary64 op (no contraction).
void budget_for(double cmax, std::size_t n, double alpha, std::size_t min_samples, std::size_t d,
                std::size_t* r, bool* exact);

// A = softmax(a (x w_q)(x w_k)^T) with a = 1/sqrt(w_q.cols) (for a
// head slice d x d_h this is the usual 1/sqrt(d_h)).
Matrix attention_matrix(const Matrix& x, const AttentionWeights& weights);
SamplePlan sample_budgets(const Matrix& attn, const McaConfig& cfg, std::size_t d);
AttentionOutput mca_forward(const Matrix& x, const AttentionWeights& weights, const McaConfig& cfg,
                            uint64_t seed);
AttentionOutput regular_forward(const Matrix& x, const AttentionWeights& weights);
AttentionOutput multihead_forward(const Matrix& x, const std::vector<AttentionWeights>& per_head,
                                  const McaConfig& cfg, uint64_t seed);

// ------------------------------------------------------------------ metrics
// cost(j) = 2 d d_out if exact else r_j (2 d_out + 3) (with
// d_out = d for the square single-head case the SPEC writes).
FlopsReport flops_for_plan(const SamplePlan& plan, std::size_t n, std::size_t d, std::size_t d_out);
double predicted_reduction(const Matrix& attn, const McaConfig& cfg, std::size_t d);

}  // namespace mca

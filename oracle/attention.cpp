// oracle/attention.cpp — SPEC attention + metrics modules
// in fp64, plus the batched multi-head forward in the device layout that the
// GPU parity tests and the CPU baseline use (oracle/batched.hpp).
//
// TEST INFRASTRUCTURE ONLY (see oracle/spec.hpp).
#include <algorithm>
#include <cmath>
#include <string>

#include "batched.hpp"
#include "spec.hpp"

namespace mca {

AttentionWeights make_attention_weights(Matrix w_q, Matrix w_k, Matrix w) {
    AttentionWeights aw;
    aw.w_q = std::move(w_q);
    aw.w_k = std::move(w_k);
    aw.w = std::move(w);
    aw.cached_dist = weight_probs(aw.w);  // SPEC.md:264, cached once per W
    return aw;
}

// SPEC.md:299 (Eq. 9) with the SPEC.md:347-348 rounding and
// clamping rules. `volatile` pins each step to one binary64 rounding.
void budget_for(double cmax, std::size_t n, double alpha, std::size_t min_samples, std::size_t d,
                std::size_t* r, bool* exact) {
    volatile double t = static_cast<double>(n) * cmax;
    t = t / alpha;
    volatile double raw = t * t;
    const double c = std::ceil(raw);
    const bool ex = c >= static_cast<double>(d);
    std::size_t rr;
    if (ex) rr = d;
    else rr = static_cast<std::size_t>(c);
    if (rr < min_samples) rr = min_samples;
    if (rr > d) rr = d;
    *r = rr;
    *exact = ex;
}

// SPEC.md:286-294
Matrix attention_matrix(const Matrix& x, const AttentionWeights& weights) {
    if (x.cols != weights.w_q.rows || x.cols != weights.w_k.rows)
        throw shape_error("attention_matrix: x.cols != d");
    const Matrix q = matmul(x, weights.w_q);
    const Matrix k = matmul(x, weights.w_k);
    const double a = 1.0 / std::sqrt(static_cast<double>(weights.w_q.cols));
    return softmax_rows(matmul_nt(q, k), a);
}

// SPEC.md:296-304
SamplePlan sample_budgets(const Matrix& attn, const McaConfig& cfg, std::size_t d) {
    if (attn.rows != attn.cols) throw shape_error("sample_budgets: attention matrix must be n x n");
    if (!(cfg.alpha > 0.0 && cfg.alpha <= 1.0)) throw domain_error("sample_budgets: alpha must be in (0, 1]");
    const std::size_t n = attn.rows;
    SamplePlan plan;
    plan.budgets.resize(n);
    plan.exact_mask.resize(n);
    plan.draws.resize(n);
    for (std::size_t j = 0; j < n; ++j) {
        bool ex = false;
        budget_for(col_max(attn, j), n, cfg.alpha, cfg.min_samples, d, &plan.budgets[j], &ex);
        plan.exact_mask[j] = ex ? 1 : 0;
    }
    return plan;
}

namespace {

// Encoding + aggregation of one head given A and a plan (budgets filled). H̃ is
// returned through `h_out` when non-null. stream id of token j = stream_base + j.
Matrix encode_and_aggregate(const Matrix& x, const Matrix& attn, const Matrix& w, const SamplingDistribution& dist,
                            SamplePlan& plan, uint64_t seed, uint64_t stream_base, uint32_t layer,
                            bool keep_draws, Matrix* h_out) {
    const std::size_t n = x.rows;
    Matrix h(n, w.cols, 0.0);
    for (std::size_t j = 0; j < n; ++j) {
        if (plan.exact_mask[j]) {
            const double* xr = x.row(j);
            double* hr = h.row(j);
            for (std::size_t i = 0; i < w.rows; ++i) {
                const double* wr = w.row(i);
                for (std::size_t c = 0; c < w.cols; ++c) hr[c] += xr[i] * wr[c];
            }
            continue;
        }
        RngStream rng(seed, stream_base + j, layer);
        if (keep_draws) {
            RngStream replay = rng;
            plan.draws[j] = draw_indices(dist, plan.budgets[j], replay);
        }
        const std::vector<double> hj = approx_encode_row(x.row(j), w, dist, plan.budgets[j], rng);
        for (std::size_t c = 0; c < w.cols; ++c) h.at(j, c) = hj[c];
    }
    if (h_out) *h_out = h;
    return matmul(attn, h);
}

void check_forward_preconditions(const Matrix& x, const AttentionWeights& weights) {
    if (x.cols != weights.w.rows) throw shape_error("forward: x.cols != w.rows");
    if (weights.cached_dist.probs.size() != weights.w.rows)
        throw config_error("forward: cached distribution is missing or stale (SPEC.md:264)");
}

}  // namespace

// SPEC.md:306-314
AttentionOutput mca_forward(const Matrix& x, const AttentionWeights& weights, const McaConfig& cfg, uint64_t seed) {
    if (cfg.mode != Mode::approximation) throw config_error("mca_forward: cfg.mode must be approximation");
    check_forward_preconditions(x, weights);
    AttentionOutput out;
    out.attn = attention_matrix(x, weights);
    out.plan = sample_budgets(out.attn, cfg, weights.w.rows);
    out.y = encode_and_aggregate(x, out.attn, weights.w, weights.cached_dist, out.plan, seed, 0, 0, true, nullptr);
    out.flops = flops_for_plan(out.plan, x.rows, weights.w.rows, weights.w.cols);
    return out;
}

// SPEC.md:316-324
AttentionOutput regular_forward(const Matrix& x, const AttentionWeights& weights) {
    if (x.cols != weights.w.rows) throw shape_error("regular_forward: x.cols != w.rows");
    AttentionOutput out;
    out.attn = attention_matrix(x, weights);
    out.y = matmul(out.attn, matmul(x, weights.w));
    const std::size_t n = x.rows;
    out.plan.budgets.assign(n, weights.w.rows);
    out.plan.exact_mask.assign(n, 1);
    out.plan.draws.assign(n, {});
    out.flops = flops_for_plan(out.plan, n, weights.w.rows, weights.w.cols);
    return out;
}

// SPEC.md:326-334; head h uses stream namespace h*n + j.
AttentionOutput multihead_forward(const Matrix& x, const std::vector<AttentionWeights>& per_head,
                                  const McaConfig& cfg, uint64_t seed) {
    const std::size_t H = cfg.heads;
    if (H == 0 || per_head.size() != H) throw config_error("multihead_forward: per_head.size() != cfg.heads");
    if (x.cols % H != 0) throw config_error("multihead_forward: d not divisible by heads");
    const std::size_t n = x.rows;
    std::size_t d_out = 0;
    for (const auto& hw : per_head) d_out += hw.w.cols;
    AttentionOutput out;
    out.y = Matrix(n, d_out, 0.0);
    out.plan.budgets.reserve(n * H);
    std::size_t col0 = 0;
    for (std::size_t h = 0; h < H; ++h) {
        const AttentionWeights& hw = per_head[h];
        check_forward_preconditions(x, hw);
        const Matrix attn = attention_matrix(x, hw);
        SamplePlan plan;
        Matrix yh;
        if (cfg.mode == Mode::regular) {
            plan.budgets.assign(n, hw.w.rows);
            plan.exact_mask.assign(n, 1);
            plan.draws.assign(n, {});
            yh = matmul(attn, matmul(x, hw.w));
        } else {
            plan = sample_budgets(attn, cfg, hw.w.rows);
            yh = encode_and_aggregate(x, attn, hw.w, hw.cached_dist, plan, seed, h * n, 0, true, nullptr);
        }
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t c = 0; c < hw.w.cols; ++c) out.y.at(i, col0 + c) = yh.at(i, c);
        col0 += hw.w.cols;
        const FlopsReport f = flops_for_plan(plan, n, hw.w.rows, hw.w.cols);
        out.flops.exact_encoding += f.exact_encoding;
        out.flops.approx_encoding += f.approx_encoding;
        out.flops.aggregation += f.aggregation;
        out.plan.budgets.insert(out.plan.budgets.end(), plan.budgets.begin(), plan.budgets.end());
        out.plan.exact_mask.insert(out.plan.exact_mask.end(), plan.exact_mask.begin(), plan.exact_mask.end());
        for (auto& dr : plan.draws) out.plan.draws.push_back(std::move(dr));
        if (h == 0) out.attn = attn;
    }
    out.flops.reduction_factor = static_cast<double>(out.flops.exact_encoding) /
                                 static_cast<double>(out.flops.approx_encoding);
    out.flops.total_reduction = static_cast<double>(out.flops.exact_encoding + out.flops.aggregation) /
                                static_cast<double>(out.flops.approx_encoding + out.flops.aggregation);
    return out;
}

// SPEC.md:384-392
FlopsReport flops_for_plan(const SamplePlan& plan, std::size_t n, std::size_t d, std::size_t d_out) {
    FlopsReport f;
    const uint64_t exact_cost = 2ull * d * d_out;
    f.exact_encoding = exact_cost * n;
    for (std::size_t j = 0; j < plan.budgets.size(); ++j)
        f.approx_encoding += plan.exact_mask[j] ? exact_cost : plan.budgets[j] * (2ull * d_out + 3ull);
    f.aggregation = 2ull * n * n * d_out;
    f.reduction_factor = static_cast<double>(f.exact_encoding) / static_cast<double>(f.approx_encoding);
    f.total_reduction = static_cast<double>(f.exact_encoding + f.aggregation) /
                        static_cast<double>(f.approx_encoding + f.aggregation);
    return f;
}

// SPEC.md:394-402
double predicted_reduction(const Matrix& attn, const McaConfig& cfg, std::size_t d) {
    const SamplePlan plan = sample_budgets(attn, cfg, d);
    return flops_for_plan(plan, attn.rows, d, d).reduction_factor;
}

// ----------------------------------------------------------- batched forward
// Device-layout multi-head forward: q, k, y, h: [B, n, H*dh];
// x: [B, n, d_in]; w: [d_in, H*dh]; per-token outputs [B, H, n]. Head h of
// sequence b uses stream ((b_offset + b) * H + h) * n + j and layer `layer`.
// Parallel over (b, h) with OpenMP; every (b, h) is computed independently in
// a fixed order, so results do not depend on the thread count.
void batched_forward(const BatchedArgs& a, BatchedOut& o) {
    const int B = a.B, n = a.n, H = a.H, dh = a.dh, din = a.d_in, HD = H * dh;
    if (B < 0 || n <= 0 || H <= 0 || dh <= 0 || din <= 0) throw shape_error("batched_forward: bad extents");
    if (a.mode == 1 && !(a.alpha > 0.0 && a.alpha <= 1.0)) throw domain_error("batched_forward: alpha not in (0,1]");
    // One-time per-head distributions.
    std::vector<Matrix> wh(H);
    std::vector<SamplingDistribution> dist(H);
    for (int h = 0; h < H; ++h) {
        wh[h] = Matrix(din, dh);
        for (int i = 0; i < din; ++i)
            for (int c = 0; c < dh; ++c) wh[h].at(i, c) = a.w[(size_t)i * HD + (size_t)h * dh + c];
        if (a.mode == 1) dist[h] = weight_probs(wh[h]);
        if (o.probs) for (int i = 0; i < din; ++i) o.probs[(size_t)h * din + i] = a.mode == 1 ? dist[h].probs[i] : 0.0;
        if (o.cdf) for (int i = 0; i < din; ++i) o.cdf[(size_t)h * din + i] = a.mode == 1 ? dist[h].cdf[i] : 0.0;
    }
    uint64_t approx_total = 0;
    const double scale = a.scale > 0.0 ? a.scale : 1.0 / std::sqrt((double)dh);
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : approx_total)
    for (long bh = 0; bh < (long)B * H; ++bh) {
        const int b = (int)(bh / H), h = (int)(bh % H);
        Matrix q(n, dh), k(n, dh), x(n, din);
        for (int j = 0; j < n; ++j) {
            const size_t row = (size_t)b * n + j;
            for (int c = 0; c < dh; ++c) {
                q.at(j, c) = a.q[row * HD + (size_t)h * dh + c];
                k.at(j, c) = a.k[row * HD + (size_t)h * dh + c];
            }
            for (int i = 0; i < din; ++i) x.at(j, i) = a.x[row * din + i];
        }
        const Matrix scores = matmul_nt(q, k);
        const Matrix attn = softmax_rows(scores, scale);
        SamplePlan plan;
        plan.budgets.resize(n);
        plan.exact_mask.resize(n);
        plan.draws.resize(n);
        const size_t tok0 = ((size_t)b * H + h) * n;
        for (int j = 0; j < n; ++j) {
            const double cm = col_max(attn, j);
            if (o.cmax) o.cmax[tok0 + j] = cm;
            if (a.mode == 0) {
                plan.budgets[j] = din;
                plan.exact_mask[j] = 1;
            } else if (a.budgets_override) {
                plan.budgets[j] = (size_t)a.budgets_override[tok0 + j];
                plan.exact_mask[j] = a.exact_override[tok0 + j];
            } else {
                bool ex = false;
                budget_for(cm, n, a.alpha, a.min_samples, din, &plan.budgets[j], &ex);
                plan.exact_mask[j] = ex;
            }
            if (o.budgets) o.budgets[tok0 + j] = (int32_t)plan.budgets[j];
            if (o.exact) o.exact[tok0 + j] = plan.exact_mask[j];
        }
        if (o.lse) {  // log-sum-exp of each scaled score row (the GPU's row statistic)
            for (int i = 0; i < n; ++i) {
                double mx = -INFINITY;
                for (int j = 0; j < n; ++j) mx = std::max(mx, scale * scores.at(i, j));
                double sum = 0.0;
                for (int j = 0; j < n; ++j) sum += std::exp(scale * scores.at(i, j) - mx);
                o.lse[tok0 + i] = mx + std::log(sum);
            }
        }
        Matrix hmat;
        Matrix yh = encode_and_aggregate(x, attn, wh[h], dist[h], plan, a.seed,
                                         ((uint64_t)(a.b_offset + b) * H + h) * (uint64_t)n, a.layer, false,
                                         o.h ? &hmat : nullptr);
        for (int j = 0; j < n; ++j) {
            const size_t row = (size_t)b * n + j;
            for (int c = 0; c < dh; ++c) {
                if (o.y) o.y[row * HD + (size_t)h * dh + c] = yh.at(j, c);
                if (o.h) o.h[row * HD + (size_t)h * dh + c] = hmat.at(j, c);
            }
        }
        const uint64_t ec = 2ull * din * dh;
        for (int j = 0; j < n; ++j)
            approx_total += plan.exact_mask[j] ? ec : (uint64_t)plan.budgets[j] * (2ull * dh + 3ull);
    }
    o.flops.exact_encoding = (uint64_t)B * H * n * 2ull * din * dh;
    o.flops.approx_encoding = approx_total;
    o.flops.aggregation = (uint64_t)B * H * 2ull * n * n * dh;
    o.flops.reduction_factor = (double)o.flops.exact_encoding / (double)o.flops.approx_encoding;
    o.flops.total_reduction = (double)(o.flops.exact_encoding + o.flops.aggregation) /
                              (double)(o.flops.approx_encoding + o.flops.aggregation);
}

}  // namespace mca

// oracle/capi.cpp — extern "C" surface of the fp64 oracle for the Python test
// suite and bench.py's CPU legs (ctypes). TEST INFRASTRUCTURE ONLY.
//
// Every entry point returns 0 on success and a nonzero SPEC error class on
// failure (1 shape, 2 domain, 3 degenerate, 4 config, 9 other); the message is
// available from oracle_last_error().
#include <cstring>
#include <string>

#include "batched.hpp"
#include "spec.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace mca;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const shape_error& e) { g_err = e.what(); return 1; }
    catch (const std::out_of_range& e) { g_err = e.what(); return 1; }
    catch (const std::invalid_argument& e) { g_err = e.what(); return 1; }
    catch (const domain_error& e) { g_err = e.what(); return 2; }
    catch (const degenerate_error& e) { g_err = e.what(); return 3; }
    catch (const config_error& e) { g_err = e.what(); return 4; }
    catch (const std::exception& e) { g_err = e.what(); return 9; }
}

Matrix from_ptr(const double* p, int rows, int cols) {
    Matrix m((size_t)rows, (size_t)cols);
    std::memcpy(m.data.data(), p, sizeof(double) * (size_t)rows * cols);
    return m;
}
void to_ptr(const Matrix& m, double* p) { std::memcpy(p, m.data.data(), sizeof(double) * m.data.size()); }
void dist_out(const SamplingDistribution& d, double* probs, double* cdf) {
    if (probs) std::memcpy(probs, d.probs.data(), sizeof(double) * d.probs.size());
    if (cdf) std::memcpy(cdf, d.cdf.data(), sizeof(double) * d.cdf.size());
}
SamplingDistribution dist_in(const double* probs, const double* cdf, int k) {
    SamplingDistribution d;
    d.probs.assign(probs, probs + k);
    d.cdf.assign(cdf, cdf + k);
    return d;
}
void flops_out(const FlopsReport& f, uint64_t* counts, double* ratios) {
    if (counts) { counts[0] = f.exact_encoding; counts[1] = f.approx_encoding; counts[2] = f.aggregation; }
    if (ratios) { ratios[0] = f.reduction_factor; ratios[1] = f.total_reduction; }
}
}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

int oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
    return omp_get_max_threads();
#else
    (void)t;
    return 1;
#endif
}

// ------------------------------------------------------------------ tensor
int oracle_matrix_check(int rows, int cols) { return guarded([&] { Matrix m((size_t)rows, (size_t)cols); }); }
int oracle_matmul(const double* a, int m, int k, const double* b, int k2, int n, double* out) {
    return guarded([&] { to_ptr(matmul(from_ptr(a, m, k), from_ptr(b, k2, n)), out); });
}
int oracle_matmul_nt(const double* a, int m, int k, const double* b, int n, int k2, double* out) {
    return guarded([&] { to_ptr(matmul_nt(from_ptr(a, m, k), from_ptr(b, n, k2)), out); });
}
int oracle_transpose(const double* a, int m, int n, double* out) {
    return guarded([&] { to_ptr(transpose(from_ptr(a, m, n)), out); });
}
int oracle_frobenius_norm(const double* a, int m, int n, double* out) {
    return guarded([&] { *out = frobenius_norm(from_ptr(a, m, n)); });
}
int oracle_row_l2_norms(const double* a, int m, int n, double* out) {
    return guarded([&] { auto v = row_l2_norms(from_ptr(a, m, n)); std::memcpy(out, v.data(), sizeof(double) * v.size()); });
}
int oracle_col_l2_norms(const double* a, int m, int n, double* out) {
    return guarded([&] { auto v = col_l2_norms(from_ptr(a, m, n)); std::memcpy(out, v.data(), sizeof(double) * v.size()); });
}
int oracle_softmax_rows(const double* a, int m, int n, double scale, double* out) {
    return guarded([&] { to_ptr(softmax_rows(from_ptr(a, m, n), scale), out); });
}
int oracle_col_max(const double* a, int m, int n, long j, double* out) {
    return guarded([&] { *out = col_max(from_ptr(a, m, n), (size_t)j); });
}
int oracle_all_finite(const double* a, int m, int n) { return from_ptr(a, m, n).all_finite() ? 1 : 0; }

// ---------------------------------------------------------------- sampling
void oracle_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) { philox4x32_10(ctr, key, out); }
uint64_t oracle_bits53(uint64_t seed, uint64_t stream, uint32_t layer, uint64_t k) {
    return philox_bits53(seed, stream, layer, k);
}
int oracle_make_distribution(const double* w, int k, double* probs, double* cdf) {
    return guarded([&] { dist_out(make_distribution(std::vector<double>(w, w + k)), probs, cdf); });
}
int oracle_draw_indices(const double* probs, const double* cdf, int k, uint64_t seed, uint64_t stream, uint32_t layer,
                        long r, int64_t* out) {
    return guarded([&] {
        RngStream rng(seed, stream, layer);
        auto v = draw_indices(dist_in(probs, cdf, k), (size_t)r, rng);
        for (size_t i = 0; i < v.size(); ++i) out[i] = (int64_t)v[i];
    });
}

// --------------------------------------------------------------------- amm
int oracle_optimal_probs(const double* a, int m, int k, const double* b, int k2, int n, double* probs, double* cdf) {
    return guarded([&] { dist_out(optimal_probs(from_ptr(a, m, k), from_ptr(b, k2, n)), probs, cdf); });
}
int oracle_weight_probs(const double* w, int rows, int cols, double* probs, double* cdf) {
    return guarded([&] { dist_out(weight_probs(from_ptr(w, rows, cols)), probs, cdf); });
}
int oracle_approx_matmul(const double* a, int m, int k, const double* b, int k2, int n, const double* probs,
                         const double* cdf, long r, uint64_t seed, uint64_t stream, double* out) {
    return guarded([&] {
        RngStream rng(seed, stream);
        to_ptr(approx_matmul(from_ptr(a, m, k), from_ptr(b, k2, n), dist_in(probs, cdf, k), (size_t)r, rng).value, out);
    });
}
int oracle_approx_encode_row(const double* x, const double* w, int d, int d_out, const double* probs,
                             const double* cdf, long r, uint64_t seed, uint64_t stream, uint32_t layer, double* out) {
    return guarded([&] {
        if (r < 1) throw domain_error("approx_encode_row: r must be >= 1");
        RngStream rng(seed, stream, layer);
        auto v = approx_encode_row(x, from_ptr(w, d, d_out), dist_in(probs, cdf, d), (size_t)r, rng);
        std::memcpy(out, v.data(), sizeof(double) * v.size());
    });
}

// --------------------------------------------------------------- attention
int oracle_budget_for(double cmax, long n, double alpha, long min_samples, long d, long* r, int* exact) {
    size_t rr; bool ex;
    budget_for(cmax, (size_t)n, alpha, (size_t)min_samples, (size_t)d, &rr, &ex);
    *r = (long)rr; *exact = ex;
    return 0;
}
// Stage-isolated Eq. 9 over a vector of column maxima (the GPU-cmax parity check).
int oracle_sample_budgets_from_cmax(const double* cmax, long count, long n, double alpha, long min_samples, long d,
                                    int32_t* budgets, uint8_t* exact) {
    return guarded([&] {
        if (!(alpha > 0.0 && alpha <= 1.0)) throw domain_error("alpha must be in (0, 1]");
        for (long i = 0; i < count; ++i) {
            size_t rr; bool ex;
            budget_for(cmax[i], (size_t)n, alpha, (size_t)min_samples, (size_t)d, &rr, &ex);
            budgets[i] = (int32_t)rr; exact[i] = ex;
        }
    });
}
int oracle_sample_budgets(const double* attn, int n, double alpha, long min_samples, long d, int32_t* budgets,
                          uint8_t* exact) {
    return guarded([&] {
        McaConfig cfg; cfg.alpha = alpha; cfg.min_samples = (size_t)min_samples;
        SamplePlan p = sample_budgets(from_ptr(attn, n, n), cfg, (size_t)d);
        for (int j = 0; j < n; ++j) { budgets[j] = (int32_t)p.budgets[j]; exact[j] = p.exact_mask[j]; }
    });
}
int oracle_attention_matrix(const double* x, int n, int d, const double* wq, const double* wk, int dq, double* out) {
    return guarded([&] {
        AttentionWeights aw; aw.w_q = from_ptr(wq, d, dq); aw.w_k = from_ptr(wk, d, dq);
        to_ptr(attention_matrix(from_ptr(x, n, d), aw), out);
    });
}
// Single-head SPEC forward (mode 1 = mca_forward, 0 = regular_forward).
int oracle_forward(int mode, const double* x, int n, int d, const double* wq, const double* wk, int dq,
                   const double* w, int d_out, double alpha, long min_samples, uint64_t seed, double* y,
                   int32_t* budgets, uint8_t* exact, int64_t* draws /* n*d_out max, -1 padded; may be null */,
                   uint64_t* counts, double* ratios) {
    return guarded([&] {
        AttentionWeights aw = make_attention_weights(from_ptr(wq, d, dq), from_ptr(wk, d, dq), from_ptr(w, d, d_out));
        McaConfig cfg; cfg.alpha = alpha; cfg.min_samples = (size_t)min_samples;
        cfg.mode = mode ? Mode::approximation : Mode::regular;
        AttentionOutput o = mode ? mca_forward(from_ptr(x, n, d), aw, cfg, seed) : regular_forward(from_ptr(x, n, d), aw);
        to_ptr(o.y, y);
        for (int j = 0; j < n; ++j) {
            if (budgets) budgets[j] = (int32_t)o.plan.budgets[j];
            if (exact) exact[j] = o.plan.exact_mask[j];
            if (draws)
                for (int k = 0; k < d; ++k)
                    draws[(size_t)j * d + k] = k < (int)o.plan.draws[j].size() ? (int64_t)o.plan.draws[j][k] : -1;
        }
        flops_out(o.flops, counts, ratios);
    });
}
// SPEC multihead_forward: per-head weights stacked [H, d, dq] / [H, d, dh].
int oracle_multihead_forward(int mode, const double* x, int n, int d, int heads, const double* wq, const double* wk,
                             int dq, const double* w, int dh, double alpha, long min_samples, uint64_t seed, double* y,
                             int32_t* budgets, uint8_t* exact, uint64_t* counts, double* ratios) {
    return guarded([&] {
        std::vector<AttentionWeights> per;
        for (int h = 0; h < heads; ++h)
            per.push_back(make_attention_weights(from_ptr(wq + (size_t)h * d * dq, d, dq),
                                                 from_ptr(wk + (size_t)h * d * dq, d, dq),
                                                 from_ptr(w + (size_t)h * d * dh, d, dh)));
        McaConfig cfg; cfg.alpha = alpha; cfg.min_samples = (size_t)min_samples; cfg.heads = (size_t)(heads > 0 ? heads : 0);
        cfg.mode = mode ? Mode::approximation : Mode::regular;
        AttentionOutput o = multihead_forward(from_ptr(x, n, d), per, cfg, seed);
        to_ptr(o.y, y);
        for (size_t j = 0; j < o.plan.budgets.size(); ++j) {
            if (budgets) budgets[j] = (int32_t)o.plan.budgets[j];
            if (exact) exact[j] = o.plan.exact_mask[j];
        }
        flops_out(o.flops, counts, ratios);
    });
}

// Batched multi-head forward in the device layout (oracle/batched.hpp).
int oracle_batched_forward(const double* q, const double* k, const double* x, const double* w, int B, int n, int H,
                           int dh, int d_in, double alpha, double scale, long min_samples, int mode, uint64_t seed,
                           int b_offset, uint32_t layer, const int32_t* budgets_override, const uint8_t* exact_override,
                           double* y, double* h, int32_t* budgets, uint8_t* exact, double* cmax, double* lse,
                           double* probs, double* cdf, uint64_t* counts, double* ratios) {
    return guarded([&] {
        BatchedArgs a;
        a.q = q; a.k = k; a.x = x; a.w = w; a.B = B; a.n = n; a.H = H; a.dh = dh; a.d_in = d_in;
        a.alpha = alpha; a.scale = scale; a.min_samples = (size_t)min_samples; a.mode = mode; a.seed = seed;
        a.b_offset = b_offset; a.layer = layer; a.budgets_override = budgets_override; a.exact_override = exact_override;
        BatchedOut o;
        o.y = y; o.h = h; o.budgets = budgets; o.exact = exact; o.cmax = cmax; o.lse = lse; o.probs = probs; o.cdf = cdf;
        batched_forward(a, o);
        flops_out(o.flops, counts, ratios);
    });
}

// ---------------------------------------------------------------- metrics
int oracle_flops_for_plan(const int32_t* budgets, const uint8_t* exact, long n, long d, long d_out, uint64_t* counts,
                          double* ratios) {
    return guarded([&] {
        SamplePlan p;
        p.budgets.assign(budgets, budgets + n);
        p.exact_mask.assign(exact, exact + n);
        flops_out(flops_for_plan(p, (size_t)n, (size_t)d, (size_t)d_out), counts, ratios);
    });
}
int oracle_predicted_reduction(const double* attn, int n, double alpha, long min_samples, long d, double* out) {
    return guarded([&] {
        McaConfig cfg; cfg.alpha = alpha; cfg.min_samples = (size_t)min_samples;
        *out = predicted_reduction(from_ptr(attn, n, n), cfg, (size_t)d);
    });
}

}  // extern "C"

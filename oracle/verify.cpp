// oracle/verify.cpp — the SPEC's statistical acceptance suites (SPEC.md:442-450,
// 499-508) run on the fp64 oracle, so the oracle itself is checked against the
// paper's guarantees before it is trusted as the GPU's checker.
// TEST INFRASTRUCTURE ONLY (see oracle/spec.hpp).
//
// Fixtures are filled with uniform values in [-1, 1) drawn from the oracle's
// own Philox streams (fixture generator stream ids start at 2^40 so they never
// collide with attention stream ids).
#include <cmath>
#include <vector>

#include "spec.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace mca;

namespace {

Matrix fixture(std::size_t rows, std::size_t cols, uint64_t seed, uint64_t id, double lo = -1.0, double hi = 1.0) {
    Matrix m(rows, cols);
    RngStream rng(seed, (1ull << 40) + id);
    for (double& v : m.data) v = lo + (hi - lo) * rng.next_uniform();
    return m;
}

double row_err(const Matrix& a, const Matrix& b, std::size_t i) {
    double s = 0.0;
    for (std::size_t c = 0; c < a.cols; ++c) {
        const double d = a.at(i, c) - b.at(i, c);
        s += d * d;
    }
    return std::sqrt(s);
}

double rel_fro(const Matrix& a, const Matrix& b) {
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < a.data.size(); ++i) {
        num += (a.data[i] - b.data[i]) * (a.data[i] - b.data[i]);
        den += b.data[i] * b.data[i];
    }
    return std::sqrt(num) / std::sqrt(den);
}

}  // namespace

extern "C" {

// Criterion 1: regular_forward vs an independent three-step
// reference written with its own loops (column-major accumulation order).
double oracle_verify_exactness(int fixtures, uint64_t seed) {
    double worst = 0.0;
    for (int f = 0; f < fixtures; ++f) {
        const std::size_t n = 4 + (std::size_t)(f * 7) % 29, d = 8 + (std::size_t)(f * 37) % 121;
        const Matrix x = fixture(n, d, seed, 4 * f), wq = fixture(d, d, seed, 4 * f + 1),
                     wk = fixture(d, d, seed, 4 * f + 2), w = fixture(d, d, seed, 4 * f + 3);
        const AttentionWeights aw = make_attention_weights(wq, wk, w);
        const AttentionOutput out = regular_forward(x, aw);
        // independent reference
        std::vector<double> q(n * d, 0.0), k(n * d, 0.0), hh(n * d, 0.0), A(n * n), y(n * d, 0.0);
        for (std::size_t c = 0; c < d; ++c)
            for (std::size_t i = 0; i < n; ++i)
                for (std::size_t t = 0; t < d; ++t) {
                    q[i * d + c] += x.at(i, t) * wq.at(t, c);
                    k[i * d + c] += x.at(i, t) * wk.at(t, c);
                    hh[i * d + c] += x.at(i, t) * w.at(t, c);
                }
        const double a = 1.0 / std::sqrt((double)d);
        for (std::size_t i = 0; i < n; ++i) {
            double mx = -1e300;
            for (std::size_t j = 0; j < n; ++j) {
                double s = 0.0;
                for (std::size_t t = 0; t < d; ++t) s += q[i * d + t] * k[j * d + t];
                A[i * n + j] = a * s;
                mx = std::max(mx, A[i * n + j]);
            }
            double z = 0.0;
            for (std::size_t j = 0; j < n; ++j) z += (A[i * n + j] = std::exp(A[i * n + j] - mx));
            for (std::size_t j = 0; j < n; ++j) A[i * n + j] /= z;
        }
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t j = 0; j < n; ++j)
                for (std::size_t c = 0; c < d; ++c) y[i * d + c] += A[i * n + j] * hh[j * d + c];
        Matrix ym(n, d);
        ym.data = y;
        worst = std::max(worst, rel_fro(out.y, ym));
    }
    return worst;
}

// Criterion 2: fraction of components of the mean of
// approx_matmul over `seeds` seeds within 3 standard errors of the exact product.
double oracle_verify_unbiased(long seeds, uint64_t seed) {
    const Matrix a = fixture(4, 6, seed, 100), b = fixture(6, 5, seed, 101);
    const Matrix exact = matmul(a, b);
    const SamplingDistribution dist = optimal_probs(a, b);
    const std::size_t m = exact.data.size();
    std::vector<double> sum(m, 0.0), sumsq(m, 0.0);
    for (long s = 0; s < seeds; ++s) {
        RngStream rng(seed + 1 + (uint64_t)s, 0);
        const AmmEstimate e = approx_matmul(a, b, dist, 6, rng);
        for (std::size_t c = 0; c < m; ++c) { sum[c] += e.value.data[c]; sumsq[c] += e.value.data[c] * e.value.data[c]; }
    }
    std::size_t ok = 0;
    for (std::size_t c = 0; c < m; ++c) {
        const double mean = sum[c] / seeds;
        const double var = std::max(0.0, sumsq[c] / seeds - mean * mean);
        const double se = std::sqrt(var / seeds);
        if (std::fabs(mean - exact.data[c]) <= 3.0 * se + 1e-12) ++ok;
    }
    return (double)ok / (double)m;
}

// Criterion 3: worst ratio (mean ‖H − xW‖) / (‖x‖‖W‖_F / √r)
// over `fixtures` fixtures (d = 128) and r ∈ {1, 4, 16, 64}.
double oracle_verify_lemma1(int fixtures, long trials, uint64_t seed) {
    const std::size_t d = 128;
    const std::size_t rs[4] = {1, 4, 16, 64};
    double worst = 0.0;
    for (int f = 0; f < fixtures; ++f) {
        const Matrix x = fixture(1, d, seed, 200 + 2 * f), w = fixture(d, d, seed, 201 + 2 * f);
        const SamplingDistribution dist = weight_probs(w);
        const Matrix exact = matmul(x, w);
        const double bound0 = std::sqrt((double)[&] { double s = 0; for (double v : x.data) s += v * v; return s; }()) *
                              frobenius_norm(w);
        for (std::size_t r : rs) {
            double tot = 0.0;
#pragma omp parallel for reduction(+ : tot) schedule(static)
            for (long t = 0; t < trials; ++t) {
                RngStream rng(seed + 7, (uint64_t)f * 1000000 + (uint64_t)t);
                const std::vector<double> h = approx_encode_row(x.row(0), w, dist, r, rng);
                double s = 0.0;
                for (std::size_t c = 0; c < d; ++c) s += (h[c] - exact.at(0, c)) * (h[c] - exact.at(0, c));
                tot += std::sqrt(s);
            }
            worst = std::max(worst, (tot / trials) / (bound0 / std::sqrt((double)r)));
        }
    }
    return worst;
}

// Criterion 4: log-log slope of mean error vs r, r = 1..256.
double oracle_verify_scaling(long trials, uint64_t seed) {
    const std::size_t d = 128;
    const Matrix x = fixture(1, d, seed, 300), w = fixture(d, d, seed, 301);
    const SamplingDistribution dist = weight_probs(w);
    const Matrix exact = matmul(x, w);
    std::vector<double> lx, ly;
    for (std::size_t r = 1; r <= 256; r *= 2) {
        double tot = 0.0;
#pragma omp parallel for reduction(+ : tot) schedule(static)
        for (long t = 0; t < trials; ++t) {
            RngStream rng(seed + 11, r * 1000000 + (uint64_t)t);
            const std::vector<double> h = approx_encode_row(x.row(0), w, dist, r, rng);
            double s = 0.0;
            for (std::size_t c = 0; c < d; ++c) s += (h[c] - exact.at(0, c)) * (h[c] - exact.at(0, c));
            tot += std::sqrt(s);
        }
        lx.push_back(std::log((double)r));
        ly.push_back(std::log(tot / trials));
    }
    double mx = 0, my = 0;
    for (std::size_t i = 0; i < lx.size(); ++i) { mx += lx[i]; my += ly[i]; }
    mx /= lx.size(); my /= ly.size();
    double sxy = 0, sxx = 0;
    for (std::size_t i = 0; i < lx.size(); ++i) { sxy += (lx[i] - mx) * (ly[i] - my); sxx += (lx[i] - mx) * (lx[i] - mx); }
    return sxy / sxx;
}

// Criteria 5, 6, 10: Theorem 1 on an n x d fixture.
// Outputs: worst over rows of mean error / (αβ‖W‖_F); worst over rows of the
// fraction of trials with error > αβ‖W‖_F/δ; mean error over rows and trials.
// The attention matrix and plan are computed once (they do not depend on the
// seed); trial t encodes with seed `seed + 1 + t`, exactly as mca_forward would.
void oracle_verify_theorem1(double alpha, int n, int d, long trials, uint64_t seed, double delta,
                            double* worst_mean_ratio, double* worst_tail_frac, double* mean_err) {
    const Matrix x = fixture((size_t)n, (size_t)d, seed, 400), wq = fixture((size_t)d, (size_t)d, seed, 401),
                 wk = fixture((size_t)d, (size_t)d, seed, 402), w = fixture((size_t)d, (size_t)d, seed, 403);
    const AttentionWeights aw = make_attention_weights(wq, wk, w);
    const Matrix A = attention_matrix(x, aw);
    const Matrix Y = matmul(A, matmul(x, w));
    McaConfig cfg; cfg.alpha = alpha;
    const SamplePlan plan = sample_budgets(A, cfg, (size_t)d);
    double beta = 0.0;
    for (const double v : row_l2_norms(x)) beta += v;
    beta /= n;
    const double bound = alpha * beta * frobenius_norm(w);
    std::vector<double> err((size_t)trials * n);
#pragma omp parallel for schedule(static)
    for (long t = 0; t < trials; ++t) {
        Matrix h((size_t)n, (size_t)d, 0.0);
        for (int j = 0; j < n; ++j) {
            if (plan.exact_mask[j]) {
                for (int i = 0; i < d; ++i)
                    for (int c = 0; c < d; ++c) h.at(j, c) += x.at(j, i) * w.at(i, c);
            } else {
                RngStream rng(seed + 1 + (uint64_t)t, (uint64_t)j);
                const std::vector<double> hj = approx_encode_row(x.row(j), w, aw.cached_dist, plan.budgets[j], rng);
                for (int c = 0; c < d; ++c) h.at(j, c) = hj[c];
            }
        }
        const Matrix yt = matmul(A, h);
        for (int i = 0; i < n; ++i) err[(size_t)t * n + i] = row_err(yt, Y, i);
    }
    double wm = 0.0, wt = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        long exceed = 0;
        for (long t = 0; t < trials; ++t) {
            const double e = err[(size_t)t * n + i];
            s += e;
            if (e > bound / delta) ++exceed;
        }
        tot += s;
        wm = std::max(wm, (s / trials) / bound);
        wt = std::max(wt, (double)exceed / trials);
    }
    *worst_mean_ratio = wm;
    *worst_tail_frac = wt;
    *mean_err = tot / ((double)trials * n);
}

}  // extern "C"

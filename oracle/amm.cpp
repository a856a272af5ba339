// oracle/amm.cpp — SPEC amm module in fp64.
//
// TEST INFRASTRUCTURE ONLY (see oracle/spec.hpp).
#include <cmath>

#include "spec.hpp"

namespace mca {

// SPEC.md:191-199 (Eq. 4): p(i) ∝ ‖a[:,i]‖ ‖b[i]‖.
SamplingDistribution optimal_probs(const Matrix& a, const Matrix& b) {
    if (a.cols != b.rows) throw shape_error("optimal_probs: a.cols != b.rows");
    const std::vector<double> cn = col_l2_norms(a);
    const std::vector<double> rn = row_l2_norms(b);
    std::vector<double> w(cn.size());
    for (std::size_t i = 0; i < w.size(); ++i) w[i] = cn[i] * rn[i];
    return make_distribution(w);
}

// SPEC.md:201-209 (Eq. 6): p(i) = ‖w[i]‖² / ‖w‖_F². The
// squared norms are the weights; make_distribution divides by their
// sequential sum, which is ‖w‖_F² accumulated row by row.
SamplingDistribution weight_probs(const Matrix& w) {
    std::vector<double> sq(w.rows, 0.0);
    for (std::size_t i = 0; i < w.rows; ++i) {
        const double* r = w.row(i);
        double s = 0.0;
        for (std::size_t c = 0; c < w.cols; ++c) s += r[c] * r[c];
        sq[i] = s;
    }
    return make_distribution(sq);  // zero matrix -> degenerate_error
}

// SPEC.md:211-219 (Eq. 2).
AmmEstimate approx_matmul(const Matrix& a, const Matrix& b, const SamplingDistribution& dist,
                          std::size_t r, RngStream& rng) {
    if (a.cols != b.rows || dist.probs.size() != a.cols) throw shape_error("approx_matmul: shape mismatch");
    // Precondition SPEC.md:213,239: every contributing index has p > 0.
    {
        const std::vector<double> cn = col_l2_norms(a), rn = row_l2_norms(b);
        for (std::size_t i = 0; i < a.cols; ++i)
            if (cn[i] * rn[i] > 0.0 && dist.probs[i] == 0.0)
                throw degenerate_error("approx_matmul: contributing index has zero probability");
    }
    const std::vector<std::size_t> s = draw_indices(dist, r, rng);
    AmmEstimate est;
    est.value = Matrix(a.rows, b.cols, 0.0);
    est.samples_used = r;
    const double rd = static_cast<double>(r);
    for (std::size_t k = 0; k < r; ++k) {
        const std::size_t i = s[k];
        const double scale = 1.0 / (rd * dist.probs[i]);
        const double* br = b.row(i);
        for (std::size_t row = 0; row < a.rows; ++row) {
            const double coef = a.at(row, i) * scale;
            double* o = est.value.row(row);
            for (std::size_t c = 0; c < b.cols; ++c) o[c] += coef * br[c];
        }
    }
    return est;
}

// H̃ = Σ_k (x[s_k] / (r p(s_k))) w[s_k], accumulated
// per sample in draw order, fp64, no compensation.
std::vector<double> approx_encode_row(const double* x_row, const Matrix& w, const SamplingDistribution& dist,
                                      std::size_t r, RngStream& rng) {
    if (dist.probs.size() != w.rows) throw shape_error("approx_encode_row: len(probs) != w.rows");
    std::vector<double> h(w.cols, 0.0);
    const double rd = static_cast<double>(r);
    for (std::size_t k = 0; k < r; ++k) {
        const double u = rng.next_uniform();
        std::size_t i = 0;
        {
            std::size_t lo = 0, hi = dist.cdf.size();  // upper_bound: first cdf[i] > u
            while (lo < hi) {
                const std::size_t mid = lo + (hi - lo) / 2;
                if (dist.cdf[mid] > u) hi = mid; else lo = mid + 1;
            }
            i = lo;
        }
        const double coef = x_row[i] / (rd * dist.probs[i]);
        const double* wr = w.row(i);
        for (std::size_t c = 0; c < w.cols; ++c) h[c] += coef * wr[c];
    }
    return h;
}

}  // namespace mca

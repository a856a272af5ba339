// oracle/tensor.cpp — fp64 definitions for the tensor module declared in
// include/mca/matrix.hpp (reference interface: proj/include/mca/matrix.hpp:7-55;
// behaviour: SPEC.md:22-114).
//
// TEST INFRASTRUCTURE ONLY (see oracle/spec.hpp). Compiled with
// -ffp-contract=off so every + and * is one correctly rounded binary64 op and
// results do not depend on the host CPU's FMA support.
#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>

#include "mca/matrix.hpp"

namespace mca {

// matrix.hpp:20 — checked constructor; SPEC.md:28 requires positive extents.
Matrix::Matrix(std::size_t r, std::size_t c, double fill) : rows(r), cols(c) {
    if (r == 0 || c == 0) throw std::invalid_argument("Matrix: rows and cols must be positive");
    data.assign(r * c, fill);
}

// matrix.hpp:23
Matrix Matrix::from_rows(std::initializer_list<std::initializer_list<double>> init) {
    if (init.size() == 0) throw std::invalid_argument("Matrix::from_rows: no rows");
    const std::size_t c = init.begin()->size();
    Matrix m(init.size(), c);
    std::size_t r = 0;
    for (const auto& row : init) {
        if (row.size() != c) throw std::invalid_argument("Matrix::from_rows: ragged rows");
        std::size_t k = 0;
        for (double v : row) m.at(r, k++) = v;
        ++r;
    }
    return m;
}

// matrix.hpp:30 / SPEC.md:31
bool Matrix::all_finite() const {
    for (double v : data)
        if (!std::isfinite(v)) return false;
    return true;
}

// matrix.hpp:33-34 / SPEC.md:35-43. i-k-j loop order; for each output element
// the k-sum runs in increasing k, so results are the plain left-to-right dot
// product (used by the "exact-associative on integers" invariant).
Matrix matmul(const Matrix& a, const Matrix& b) {
    if (a.cols != b.rows)
        throw std::invalid_argument("matmul: a.cols (" + std::to_string(a.cols) + ") != b.rows (" +
                                    std::to_string(b.rows) + ")");
    Matrix out(a.rows, b.cols, 0.0);
    for (std::size_t i = 0; i < a.rows; ++i) {
        double* o = out.row(i);
        const double* ar = a.row(i);
        for (std::size_t k = 0; k < a.cols; ++k) {
            const double aik = ar[k];
            const double* br = b.row(k);
            for (std::size_t j = 0; j < b.cols; ++j) o[j] += aik * br[j];
        }
    }
    return out;
}

// matrix.hpp:36-37 — a * b^T as row-by-row dot products.
Matrix matmul_nt(const Matrix& a, const Matrix& b) {
    if (a.cols != b.cols)
        throw std::invalid_argument("matmul_nt: a.cols != b.cols");
    Matrix out(a.rows, b.rows, 0.0);
    for (std::size_t i = 0; i < a.rows; ++i) {
        const double* ar = a.row(i);
        for (std::size_t j = 0; j < b.rows; ++j) {
            const double* br = b.row(j);
            double s = 0.0;
            for (std::size_t k = 0; k < a.cols; ++k) s += ar[k] * br[k];
            out.at(i, j) = s;
        }
    }
    return out;
}

// matrix.hpp:39
Matrix transpose(const Matrix& m) {
    Matrix t(m.cols, m.rows);
    for (std::size_t i = 0; i < m.rows; ++i)
        for (std::size_t j = 0; j < m.cols; ++j) t.at(j, i) = m.at(i, j);
    return t;
}

// matrix.hpp:41 / SPEC.md:45-53: sqrt of the row-major sequential sum of squares.
double frobenius_norm(const Matrix& m) {
    double s = 0.0;
    for (double v : m.data) s += v * v;
    return std::sqrt(s);
}

// matrix.hpp:43 / SPEC.md:55-63
std::vector<double> row_l2_norms(const Matrix& m) {
    std::vector<double> out(m.rows, 0.0);
    for (std::size_t i = 0; i < m.rows; ++i) {
        double s = 0.0;
        const double* r = m.row(i);
        for (std::size_t j = 0; j < m.cols; ++j) s += r[j] * r[j];
        out[i] = std::sqrt(s);
    }
    return out;
}

// matrix.hpp:44 / SPEC.md:65-71
std::vector<double> col_l2_norms(const Matrix& m) {
    std::vector<double> s(m.cols, 0.0);
    for (std::size_t i = 0; i < m.rows; ++i) {
        const double* r = m.row(i);
        for (std::size_t j = 0; j < m.cols; ++j) s[j] += r[j] * r[j];
    }
    for (double& v : s) v = std::sqrt(v);
    return s;
}

// matrix.hpp:46-50 / SPEC.md:73-81,101: t_j = scale*m_j; e_j = exp(t_j - max t);
// out_j = e_j / sum_j e_j (sum left to right).
Matrix softmax_rows(const Matrix& m, double scale) {
    Matrix out(m.rows, m.cols);
    std::vector<double> t(m.cols);
    for (std::size_t i = 0; i < m.rows; ++i) {
        const double* r = m.row(i);
        double mx = -std::numeric_limits<double>::infinity();
        for (std::size_t j = 0; j < m.cols; ++j) {
            t[j] = scale * r[j];
            if (t[j] > mx) mx = t[j];
        }
        double sum = 0.0;
        for (std::size_t j = 0; j < m.cols; ++j) {
            t[j] = std::exp(t[j] - mx);
            sum += t[j];
        }
        double* o = out.row(i);
        for (std::size_t j = 0; j < m.cols; ++j) o[j] = t[j] / sum;
    }
    return out;
}

// matrix.hpp:52-53 / SPEC.md:83-91
double col_max(const Matrix& m, std::size_t j) {
    if (j >= m.cols)
        throw std::out_of_range("col_max: column " + std::to_string(j) + " >= cols " +
                                std::to_string(m.cols));
    double mx = m.at(0, j);
    for (std::size_t i = 1; i < m.rows; ++i)
        if (m.at(i, j) > mx) mx = m.at(i, j);
    return mx;
}

}  // namespace mca

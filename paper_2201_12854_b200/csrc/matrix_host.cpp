// matrix_host.cpp — libmca_b200's definitions of the reference's tensor module.
//
// The reference declares these functions out of line in
// proj/include/mca/matrix.hpp:20-53 (behaviour: SPEC.md:22-114) and ships no
// definitions. A C++ caller written against that header links them from
// libmca_b200 (`-lmca_b200`, nothing else): the fp64 host Matrix is the value
// type the C++ mirror include/mca/mca.hpp converts to and from the device
// layout, and these are its host-side operations. They are dense fp64 CPU
// routines over caller-owned std::vector storage; the MCA forward itself never
// calls them (it runs on the GPU through include/mca/mca_cuda.h).
//
// Numerics: products are formed as dot products of a row of `a` with a
// contiguous row (matmul_nt) or gathered column (matmul) in increasing k, so
// integer-valued inputs give exact, associativity-independent results
// (SPEC.md:96); softmax is max-subtracted.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>

#include "mca/matrix.hpp"

namespace mca {

namespace {

std::string dims(std::size_t r, std::size_t c) { return std::to_string(r) + "x" + std::to_string(c); }

// sum_k a[k] * b[k * stride], k increasing (no FMA contraction: -ffp-contract=off)
double dot(const double* a, const double* b, std::size_t len, std::size_t stride) {
    double s = 0.0;
    for (std::size_t k = 0; k < len; ++k) s += a[k] * b[k * stride];
    return s;
}

}  // namespace

// matrix.hpp:20. Positive extents; every element = fill.
Matrix::Matrix(std::size_t r, std::size_t c, double fill) : rows(r), cols(c), data() {
    if (r == 0 || c == 0) throw std::invalid_argument("mca::Matrix: extents must be positive, got " + dims(r, c));
    if (c > std::numeric_limits<std::size_t>::max() / r)
        throw std::invalid_argument("mca::Matrix: " + dims(r, c) + " overflows size_t");
    data.resize(r * c, fill);
}

// matrix.hpp:23. Rows of equal, positive length.
Matrix Matrix::from_rows(std::initializer_list<std::initializer_list<double>> init) {
    const std::size_t r = init.size();
    const std::size_t c = r ? init.begin()->size() : 0;
    Matrix m(r, c);   // throws for 0 rows / 0 columns
    double* out = m.data.data();
    for (const auto& row : init) {
        if (row.size() != c)
            throw std::invalid_argument("mca::Matrix::from_rows: row of length " + std::to_string(row.size()) +
                                        ", expected " + std::to_string(c));
        out = std::copy(row.begin(), row.end(), out);
    }
    return m;
}

// matrix.hpp:30
bool Matrix::all_finite() const {
    return std::all_of(data.begin(), data.end(), [](double v) { return std::isfinite(v); });
}

// matrix.hpp:33-34. out(i, j) = sum_k a(i, k) b(k, j).
Matrix matmul(const Matrix& a, const Matrix& b) {
    if (a.cols != b.rows)
        throw std::invalid_argument("mca::matmul: " + dims(a.rows, a.cols) + " * " + dims(b.rows, b.cols));
    Matrix out(a.rows, b.cols);
    for (std::size_t i = 0; i < a.rows; ++i)
        for (std::size_t j = 0; j < b.cols; ++j) out.at(i, j) = dot(a.row(i), b.data.data() + j, a.cols, b.cols);
    return out;
}

// matrix.hpp:36-37. out(i, j) = <a row i, b row j>.
Matrix matmul_nt(const Matrix& a, const Matrix& b) {
    if (a.cols != b.cols)
        throw std::invalid_argument("mca::matmul_nt: " + dims(a.rows, a.cols) + " * (" + dims(b.rows, b.cols) +
                                    ")^T");
    Matrix out(a.rows, b.rows);
    for (std::size_t i = 0; i < a.rows; ++i)
        for (std::size_t j = 0; j < b.rows; ++j) out.at(i, j) = dot(a.row(i), b.row(j), a.cols, 1);
    return out;
}

// matrix.hpp:39
Matrix transpose(const Matrix& m) {
    Matrix t(m.cols, m.rows);
    for (std::size_t j = 0; j < m.cols; ++j)
        for (std::size_t i = 0; i < m.rows; ++i) t.at(j, i) = m.at(i, j);
    return t;
}

// matrix.hpp:41. sqrt of the sum of squares in storage order.
double frobenius_norm(const Matrix& m) {
    return std::sqrt(std::accumulate(m.data.begin(), m.data.end(), 0.0, [](double s, double v) { return s + v * v; }));
}

// matrix.hpp:43
std::vector<double> row_l2_norms(const Matrix& m) {
    std::vector<double> n(m.rows);
    for (std::size_t i = 0; i < m.rows; ++i) n[i] = std::sqrt(dot(m.row(i), m.row(i), m.cols, 1));
    return n;
}

// matrix.hpp:44
std::vector<double> col_l2_norms(const Matrix& m) {
    std::vector<double> n(m.cols, 0.0);
    for (std::size_t i = 0; i < m.rows; ++i)
        for (std::size_t j = 0; j < m.cols; ++j) n[j] += m.at(i, j) * m.at(i, j);
    for (double& v : n) v = std::sqrt(v);
    return n;
}

// matrix.hpp:46-50. Row i: t = scale * m(i, :); out = exp(t - max t) / sum.
Matrix softmax_rows(const Matrix& m, double scale) {
    Matrix out(m.rows, m.cols);
    for (std::size_t i = 0; i < m.rows; ++i) {
        const double* in = m.row(i);
        double* o = out.row(i);
        double top = -std::numeric_limits<double>::infinity();
        for (std::size_t j = 0; j < m.cols; ++j) top = std::max(top, scale * in[j]);
        double sum = 0.0;
        for (std::size_t j = 0; j < m.cols; ++j) sum += (o[j] = std::exp(scale * in[j] - top));
        for (std::size_t j = 0; j < m.cols; ++j) o[j] /= sum;
    }
    return out;
}

// matrix.hpp:52-53
double col_max(const Matrix& m, std::size_t j) {
    if (j >= m.cols)
        throw std::out_of_range("mca::col_max: column " + std::to_string(j) + " of a " + dims(m.rows, m.cols) +
                                " matrix");
    double best = m.at(0, j);
    for (std::size_t i = 1; i < m.rows; ++i) best = std::max(best, m.at(i, j));
    return best;
}

}  // namespace mca

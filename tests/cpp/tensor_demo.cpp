// A reference-style caller of the tensor module (matrix.hpp:7-55), linked
// against libmca_b200 alone (-lmca_b200: no oracle, no libcudart). It runs
// the SPEC's tensor examples plus the error behaviour of matrix.hpp:20,33,52,
// and writes matmul / matmul_nt / softmax_rows / norms / col_max of two
// matrices read from argv[1] to argv[2] for tests/test_cpp_host.py to compare
// with numpy. Compiles against include/mca/matrix.hpp or, unchanged, the
// reference's own proj/include/mca/matrix.hpp.
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <fstream>
#include <stdexcept>
#include <vector>

#include "mca/matrix.hpp"

static int fails = 0;
#define EXPECT(c)                                                      \
    do {                                                               \
        if (!(c)) {                                                    \
            std::fprintf(stderr, "FAILED %s (line %d)\n", #c, __LINE__); \
            ++fails;                                                   \
        }                                                              \
    } while (0)

static mca::Matrix read_matrix(std::ifstream& f) {
    int64_t r = 0, c = 0;
    f.read(reinterpret_cast<char*>(&r), 8);
    f.read(reinterpret_cast<char*>(&c), 8);
    mca::Matrix m(static_cast<std::size_t>(r), static_cast<std::size_t>(c));
    f.read(reinterpret_cast<char*>(m.data.data()), static_cast<std::streamsize>(m.data.size() * 8));
    return m;
}

static void write(std::ofstream& f, const std::vector<double>& v) {
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
}

int main(int argc, char** argv) {
    // softmax of [0, ln 3] is [0.25, 0.75]
    const mca::Matrix s = mca::softmax_rows(mca::Matrix::from_rows({{0.0, std::log(3.0)}}), 1.0);
    EXPECT(std::fabs(s.at(0, 0) - 0.25) < 1e-15 && std::fabs(s.at(0, 1) - 0.75) < 1e-15);
    // matmul of integers is exact; 2x3 * 3x2
    const mca::Matrix a = mca::Matrix::from_rows({{1, 2, 3}, {4, 5, 6}});
    const mca::Matrix b = mca::Matrix::from_rows({{7, 8}, {9, 10}, {11, 12}});
    const mca::Matrix ab = mca::matmul(a, b);
    EXPECT(ab.rows == 2 && ab.cols == 2 && ab.at(0, 0) == 58 && ab.at(0, 1) == 64 && ab.at(1, 0) == 139 &&
           ab.at(1, 1) == 154);
    const mca::Matrix abt = mca::matmul_nt(a, mca::transpose(b));
    EXPECT(abt.data == ab.data);
    EXPECT(mca::frobenius_norm(mca::Matrix::from_rows({{3, 4}})) == 5.0);
    EXPECT(mca::row_l2_norms(mca::Matrix::from_rows({{3, 4}, {0, 2}})) == (std::vector<double>{5.0, 2.0}));
    EXPECT(mca::col_l2_norms(mca::Matrix::from_rows({{3, 0}, {4, 2}})) == (std::vector<double>{5.0, 2.0}));
    EXPECT(mca::col_max(a, 2) == 6.0);
    mca::Matrix f(2, 3, 1.5);
    EXPECT(f.rows == 2 && f.cols == 3 && f.data.size() == 6 && f.at(1, 2) == 1.5 && f.all_finite());
    f.at(0, 1) = NAN;
    EXPECT(!f.all_finite());
    // errors (matrix.hpp:20, 23, 33, 52)
    bool e1 = false, e2 = false, e3 = false, e4 = false;
    try { (void)mca::matmul(a, a); } catch (const std::invalid_argument&) { e1 = true; }
    try { (void)mca::col_max(a, 3); } catch (const std::out_of_range&) { e2 = true; }
    try { mca::Matrix z(0, 3); } catch (const std::invalid_argument&) { e3 = true; }
    try { (void)mca::Matrix::from_rows({{1, 2}, {3}}); } catch (const std::invalid_argument&) { e4 = true; }
    EXPECT(e1 && e2 && e3 && e4);
    if (argc == 3) {
        std::ifstream in(argv[1], std::ios::binary);
        const mca::Matrix p = read_matrix(in), q = read_matrix(in);
        std::ofstream out(argv[2], std::ios::binary);
        write(out, mca::matmul(p, mca::transpose(q)).data);
        write(out, mca::matmul_nt(p, q).data);
        write(out, mca::softmax_rows(p, 0.125).data);
        write(out, mca::row_l2_norms(p));
        write(out, mca::col_l2_norms(p));
        std::vector<double> cm(p.cols);
        for (std::size_t j = 0; j < p.cols; ++j) cm[j] = mca::col_max(p, j);
        write(out, cm);
        write(out, {mca::frobenius_norm(p)});
    }
    if (fails) return 1;
    std::puts("tensor_demo ok");
    return 0;
}

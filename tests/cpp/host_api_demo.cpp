// A C++ caller of the B200 MCA path through include/mca/mca.hpp (the host
// mirror of the reference's SPEC interface over matrix.hpp's Matrix).
// Reads q, k, x (n x ...), W_V, W_q, W_k (d x heads*64) as fp64 from argv[1],
// runs mca_forward and regular_forward for one sequence on (q, k, x), then the
// reference's mca_forward(x, weights) with W_q / W_k on the weights, and
// writes y_mca, y_exact, budgets, exact_mask, flops, y_x, budgets_x to
// argv[2]. tests/test_cpp_host.py drives it.
#include <cstdio>
#include <cstdint>
#include <fstream>
#include <vector>

#include "mca/mca.hpp"

static mca::Matrix read_matrix(std::ifstream& f) {
    int64_t r = 0, c = 0;
    f.read(reinterpret_cast<char*>(&r), 8);
    f.read(reinterpret_cast<char*>(&c), 8);
    mca::Matrix m(static_cast<std::size_t>(r), static_cast<std::size_t>(c));   // matrix.hpp:20, from libmca_b200
    f.read(reinterpret_cast<char*>(m.data.data()), static_cast<std::streamsize>(m.data.size() * 8));
    return m;
}

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: %s in.bin out.bin\n", argv[0]);
        return 2;
    }
    std::ifstream in(argv[1], std::ios::binary);
    int64_t heads = 0, seed = 0;
    double alpha = 0;
    in.read(reinterpret_cast<char*>(&heads), 8);
    in.read(reinterpret_cast<char*>(&seed), 8);
    in.read(reinterpret_cast<char*>(&alpha), 8);
    const mca::Matrix q = read_matrix(in), k = read_matrix(in), x = read_matrix(in), w = read_matrix(in);
    const mca::Matrix wq = read_matrix(in), wk = read_matrix(in);
    try {
        mca::b200::AttentionWeights weights(w, static_cast<int>(heads));
        mca::b200::McaConfig cfg;
        cfg.alpha = alpha;
        const auto approx = mca::b200::mca_forward(q, k, x, weights, cfg, static_cast<uint64_t>(seed));
        const auto exact = mca::b200::regular_forward(q, k, x, weights);
        // error behaviour of the reference: alpha = 0 is a domain error
        bool domain_error = false;
        try {
            mca::b200::McaConfig bad;
            bad.alpha = 0.0;
            (void)mca::b200::mca_forward(q, k, x, weights, bad, 1);
        } catch (const std::domain_error&) {
            domain_error = true;
        }
        bool shape_error = false;
        try {
            mca::Matrix wrong(x.rows, x.cols - 1);
            (void)mca::b200::mca_forward(q, k, wrong, weights, cfg, 1);
        } catch (const std::invalid_argument&) {
            shape_error = true;
        }
        std::ofstream out(argv[2], std::ios::binary);
        out.write(reinterpret_cast<const char*>(approx.y.data.data()), static_cast<std::streamsize>(approx.y.data.size() * 8));
        out.write(reinterpret_cast<const char*>(exact.y.data.data()), static_cast<std::streamsize>(exact.y.data.size() * 8));
        out.write(reinterpret_cast<const char*>(approx.budgets.data()), static_cast<std::streamsize>(approx.budgets.size() * 4));
        out.write(reinterpret_cast<const char*>(approx.exact_mask.data()), static_cast<std::streamsize>(approx.exact_mask.size()));
        const double fl[3] = {approx.flops.reduction_factor, static_cast<double>(approx.flops.samples),
                              (domain_error ? 1.0 : 0.0) + (shape_error ? 2.0 : 0.0)};
        out.write(reinterpret_cast<const char*>(fl), sizeof(fl));
        // SPEC's AttentionWeights{w_q, w_k, w} and mca_forward(x, weights, cfg, seed)
        mca::b200::AttentionWeights full(wq, wk, w, static_cast<int>(heads));
        const auto viax = mca::b200::mca_forward(x, full, cfg, static_cast<uint64_t>(seed));
        out.write(reinterpret_cast<const char*>(viax.y.data.data()), static_cast<std::streamsize>(viax.y.data.size() * 8));
        out.write(reinterpret_cast<const char*>(viax.budgets.data()), static_cast<std::streamsize>(viax.budgets.size() * 4));
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}

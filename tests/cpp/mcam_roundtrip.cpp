// mcam_roundtrip IN OUT: read an MCAM file with include/mca/mcam.hpp and write it
// back (tests/test_mcam_cli.py compares the bytes); prints the error and exits 2
// on a format / domain error (the cli's exit status).
#include <cstdio>

#include "mca/mcam.hpp"

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    try {
        mca::Matrix m = mca::read_mcam(argv[1]);
        mca::validate_attention(m, 1e300);   // sign check only: keep the payload bit-exact
        mca::write_mcam(argv[2], m);
        std::printf("%zu %zu\n", m.rows, m.cols);
        return 0;
    } catch (const mca::format_error& e) {
        std::printf("format_error offset=%zu: %s\n", e.offset, e.what());
    } catch (const std::domain_error& e) {
        std::printf("domain_error: %s\n", e.what());
    }
    return 2;
}

// mca/mcam.hpp — the cli module's matrix file format and
// cmd_attn_import's validation, header-only C++17 over
// matrix.hpp's Matrix (only its inline members: no oracle definitions needed).
//
// MCAM, bit-exact little-endian: "MCAM", u32 version = 1, u64 rows, u64 cols,
// rows*cols float64 row-major. Errors: mca::format_error (with the byte
// offset: bad magic / version, payload length != header, non-finite entry),
// std::domain_error (negative attention entry).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "mca/matrix.hpp"

namespace mca {

struct format_error : std::runtime_error {
    std::size_t offset;
    format_error(const std::string& msg, std::size_t off)
        : std::runtime_error(msg + " (byte offset " + std::to_string(off) + ")"), offset(off) {}
};

namespace mcam_detail {
inline void put_le(std::string& out, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) out.push_back(static_cast<char>((v >> (8 * i)) & 0xFF));
}
inline uint64_t get_le(const std::string& in, std::size_t off, int bytes) {
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(static_cast<unsigned char>(in[off + i])) << (8 * i);
    return v;
}
}  // namespace mcam_detail

inline std::string encode_mcam(const Matrix& m) {
    using namespace mcam_detail;
    std::string out = "MCAM";
    put_le(out, 1, 4);
    put_le(out, m.rows, 8);
    put_le(out, m.cols, 8);
    for (double v : m.data) {
        uint64_t bits;
        std::memcpy(&bits, &v, 8);
        put_le(out, bits, 8);
    }
    return out;
}

inline Matrix decode_mcam(const std::string& buf) {
    using namespace mcam_detail;
    constexpr std::size_t kHeader = 24;
    if (buf.size() < kHeader)
        throw format_error("truncated header: expected 24 bytes, got " + std::to_string(buf.size()), buf.size());
    if (buf.compare(0, 4, "MCAM") != 0) throw format_error("bad magic (expected MCAM)", 0);
    if (get_le(buf, 4, 4) != 1) throw format_error("unsupported version " + std::to_string(get_le(buf, 4, 4)), 4);
    const uint64_t rows = get_le(buf, 8, 8), cols = get_le(buf, 16, 8);
    const uint64_t want = kHeader + rows * cols * 8;
    if (buf.size() != want)
        throw format_error(std::string(buf.size() < want ? "truncated" : "oversized") + " payload: expected " +
                               std::to_string(want) + " bytes for " + std::to_string(rows) + " x " +
                               std::to_string(cols) + ", got " + std::to_string(buf.size()),
                           buf.size() < want ? buf.size() : want);
    Matrix m;
    m.rows = rows;
    m.cols = cols;
    m.data.resize(rows * cols);
    for (std::size_t i = 0; i < m.data.size(); ++i) {
        const uint64_t bits = get_le(buf, kHeader + 8 * i, 8);
        std::memcpy(&m.data[i], &bits, 8);
        if (!std::isfinite(m.data[i])) throw format_error("non-finite entry", kHeader + 8 * i);
    }
    return m;
}

inline void write_mcam(const std::string& path, const Matrix& m) {
    std::ofstream f(path, std::ios::binary);
    const std::string s = encode_mcam(m);
    f.write(s.data(), static_cast<std::streamsize>(s.size()));
    if (!f) throw std::runtime_error("cannot write " + path);
}

inline Matrix read_mcam(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + path);
    const std::string buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    return decode_mcam(buf);
}

// cmd_attn_import's checks on a loaded matrix: negative entries are a domain
// error; rows whose sums miss 1 by more than tol are renormalised (returns
// how many were).
inline std::size_t validate_attention(Matrix& a, double tol = 1e-6) {
    std::size_t fixed = 0;
    for (std::size_t r = 0; r < a.rows; ++r) {
        double s = 0.0;
        for (std::size_t c = 0; c < a.cols; ++c) {
            const double v = a.at(r, c);
            if (v < 0.0)
                throw std::domain_error("negative attention entry at (" + std::to_string(r) + ", " +
                                        std::to_string(c) + ")");
            s += v;
        }
        if (std::fabs(s - 1.0) > tol) {
            if (s <= 0.0) throw std::domain_error("attention row " + std::to_string(r) + " sums to 0");
            for (std::size_t c = 0; c < a.cols; ++c) a.at(r, c) /= s;
            ++fixed;
        }
    }
    return fixed;
}

}  // namespace mca

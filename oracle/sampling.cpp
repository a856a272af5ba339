// oracle/sampling.cpp — SPEC sampling module in fp64.
//
// TEST INFRASTRUCTURE ONLY (see oracle/spec.hpp). This file is written
// independently of the device code in paper_2201_12854_b200/csrc: the GPU
// draws indices with an integer threshold table plus a guide table, the
// oracle with std::upper_bound over the fp64 cdf exactly as SPEC.md:161 says,
// so index parity between the two is a real check, not a shared-code tautology.
#include <algorithm>
#include <cmath>

#include "spec.hpp"

namespace mca {

namespace {
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;  // golden ratio
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;  // sqrt(3) - 1
}  // namespace

// Philox4x32 with 10 rounds: each round multiplies words 0 and 2 by M0/M1,
// permutes, and xors in the key; the key is bumped by (W0, W1) between rounds.
void philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += kPhiloxW0;
            k1 += kPhiloxW1;
        }
        const uint64_t p0 = static_cast<uint64_t>(kPhiloxM0) * c0;
        const uint64_t p1 = static_cast<uint64_t>(kPhiloxM1) * c2;
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n1 = lo1;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        const uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint64_t philox_bits53(uint64_t seed, uint64_t stream_id, uint32_t layer, uint64_t k) {
    const uint32_t ctr[4] = {static_cast<uint32_t>(k >> 1), layer, static_cast<uint32_t>(stream_id),
                             static_cast<uint32_t>(stream_id >> 32)};
    const uint32_t key[2] = {static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)};
    uint32_t x[4];
    philox4x32_10(ctr, key, x);
    const uint64_t w = (k & 1) ? ((static_cast<uint64_t>(x[3]) << 32) | x[2])
                               : ((static_cast<uint64_t>(x[1]) << 32) | x[0]);
    return w >> 11;
}

uint64_t RngStream::next_bits53() { return philox_bits53(seed, stream_id, layer, counter++); }

double RngStream::next_uniform() { return std::ldexp(static_cast<double>(next_bits53()), -53); }

// SPEC.md:136-144,163
SamplingDistribution make_distribution(const std::vector<double>& weights) {
    if (weights.empty()) throw degenerate_error("make_distribution: empty weight vector");
    double total = 0.0;
    for (double w : weights) {
        if (!std::isfinite(w)) throw domain_error("make_distribution: non-finite weight");
        if (w < 0.0) throw domain_error("make_distribution: negative weight");
        total += w;
    }
    if (!(total > 0.0)) throw degenerate_error("make_distribution: all weights are zero");

    SamplingDistribution d;
    d.probs.resize(weights.size());
    bool clamped = false;
    for (std::size_t i = 0; i < weights.size(); ++i) {
        d.probs[i] = weights[i] / total;
        if (d.probs[i] < 1e-15) {
            if (d.probs[i] != 0.0) clamped = true;
            d.probs[i] = 0.0;
        }
    }
    if (clamped) {
        double s = 0.0;
        for (double p : d.probs) s += p;
        if (!(s > 0.0)) throw degenerate_error("make_distribution: every probability below 1e-15");
        for (double& p : d.probs) p = p / s;
    }
    d.cdf.resize(d.probs.size());
    double acc = 0.0;
    std::size_t last_pos = 0;
    for (std::size_t i = 0; i < d.probs.size(); ++i) {
        acc += d.probs[i];
        d.cdf[i] = acc < 1.0 ? acc : 1.0;  // rounding may overshoot 1 by ulps; keep cdf monotone
        if (d.probs[i] > 0.0) last_pos = i;
    }
    for (std::size_t i = last_pos; i < d.cdf.size(); ++i) d.cdf[i] = 1.0;
    return d;
}

// SPEC.md:146-154,161
std::vector<std::size_t> draw_indices(const SamplingDistribution& dist, std::size_t r, RngStream& rng) {
    if (r == 0) throw domain_error("draw_indices: r must be >= 1");
    if (dist.cdf.empty()) throw degenerate_error("draw_indices: empty distribution");
    std::vector<std::size_t> out(r);
    for (std::size_t k = 0; k < r; ++k) {
        const double u = rng.next_uniform();
        const auto it = std::upper_bound(dist.cdf.begin(), dist.cdf.end(), u);
        out[k] = static_cast<std::size_t>(it - dist.cdf.begin());
    }
    return out;
}

}  // namespace mca

// oracle/batched.hpp — batched multi-head forward in the device layout.
// TEST INFRASTRUCTURE ONLY (see oracle/spec.hpp).
#pragma once

#include <cstdint>

#include "spec.hpp"

namespace mca {

struct BatchedArgs {
    const double* q = nullptr;  // [B, n, H*dh]
    const double* k = nullptr;  // [B, n, H*dh]
    const double* x = nullptr;  // [B, n, d_in]
    const double* w = nullptr;  // [d_in, H*dh]
    int B = 0, n = 0, H = 0, dh = 0, d_in = 0;
    double alpha = 0.4;
    double scale = 0.0;  // <= 0 -> 1/sqrt(dh)
    std::size_t min_samples = 1;
    int mode = 1;  // 0 regular, 1 approximation
    uint64_t seed = 0;
    int b_offset = 0;
    uint32_t layer = 0;
    const int32_t* budgets_override = nullptr;  // [B, H, n]; when set, replaces Eq. 9
    const uint8_t* exact_override = nullptr;    // [B, H, n]
};

struct BatchedOut {
    double* y = nullptr;        // [B, n, H*dh]
    double* h = nullptr;        // [B, n, H*dh]  (H̃, the encodings)
    int32_t* budgets = nullptr; // [B, H, n]
    uint8_t* exact = nullptr;   // [B, H, n]
    double* cmax = nullptr;     // [B, H, n]
    double* lse = nullptr;      // [B, H, n]
    double* probs = nullptr;    // [H, d_in]
    double* cdf = nullptr;      // [H, d_in]
    FlopsReport flops;
};

void batched_forward(const BatchedArgs& a, BatchedOut& o);

}  // namespace mca

// mca/mca.hpp — C++ host interface of the B200 MCA forward, header-only,
// layered on the C ABI (mca/mca_cuda.h). It mirrors the reference's
// operator interface for the path (SPEC.md:255-424 over matrix.hpp's Matrix)
// so C++ callers of the reference can switch:
//
//   reference (SPEC op)                          here
//   AttentionWeights{w_q, w_k, w, cached_dist}   mca::b200::AttentionWeights (W_V on device + K0 tables,
//                                     :260-265   optionally W_q / W_k)
//   mca_forward(x, weights, cfg, seed)  :306-314 mca::b200::mca_forward(x, weights, cfg, seed) (x alone)
//   McaConfig{alpha, mode, min_samples, heads}   mca::b200::McaConfig
//   multihead_forward(x, heads, cfg, seed)       mca::b200::multihead_forward(q, k, x, w, cfg, seed)
//   mca_forward / regular_forward                same, cfg.mode approximation / regular
//   sample_budgets(attn, cfg, d)                 mca::b200::sample_budgets(cmax, n, d, cfg) (device)
//   FlopsReport                       :376-381   mca::b200::FlopsReport
//
// Errors follow matrix.hpp:33,52 and the SPEC error classes: shape errors
// throw std::invalid_argument, domain errors std::domain_error, degenerate /
// configuration / CUDA errors std::runtime_error. Every call reaches the GPU;
// there is no host fallback.
//
// Two levels: device-pointer calls (zero copies; any mca_stream_t) and
// Matrix-level calls for one sequence (fp64 host Matrix in, converted to the
// fp32 parity-precision path, result copied back).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "mca/matrix.hpp"
#include "mca/mca_cuda.h"

namespace mca {
namespace b200 {

enum class Mode { regular = MCA_MODE_REGULAR, approximation = MCA_MODE_APPROX };

struct McaConfig {
    double alpha = 0.4;
    Mode mode = Mode::approximation;
    int min_samples = 1;
    double scale = 0.0;  // <= 0: 1/sqrt(d_h)
    bool certify = false;  // bf16: boundary Eq. 9 values re-derived in binary64 (mca_config.certify)
    mca_config c() const {
        return mca_config{alpha, scale, min_samples, static_cast<int32_t>(mode), certify ? 1 : 0, 0};
    }
};

struct FlopsReport {
    uint64_t exact_encoding = 0, approx_encoding = 0, aggregation = 0, samples = 0, exact_tokens = 0;
    double reduction_factor = 1.0, total_reduction = 1.0;
};

inline void check(mca_status s) {
    if (s == MCA_OK) return;
    const std::string msg = std::string("mca: ") + mca_last_error();
    switch (s) {
        case MCA_ERR_SHAPE: throw std::invalid_argument(msg);
        case MCA_ERR_DOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

// Device buffers and copies go through libmca_b200's own helpers (mca_cuda.h),
// so a caller links -lmca_b200 alone (no direct libcudart dependency).
inline void dev_check(mca_status s, const char* what) {
    if (s != MCA_OK) throw std::runtime_error(std::string("mca: ") + what + ": " + mca_last_error());
}

// W_V [d_in, heads*64] on the device plus its cached sampling tables.
class AttentionWeights {
   public:
    // From a device buffer in `dtype` (row-major [d_in, heads*64]).
    AttentionWeights(const void* w_v_device, mca_dtype dtype, int d_in, int heads, mca_stream_t stream = nullptr)
        : dtype_(dtype), d_in_(d_in), heads_(heads) {
        check(mca_prepare_weights(w_v_device, dtype, d_in, heads, 64, stream, &h_));
    }
    // From a host fp64 Matrix (d_in x heads*64): uploaded as fp32 (parity precision).
    AttentionWeights(const Matrix& w_v, int heads, mca_stream_t stream = nullptr)
        : dtype_(MCA_F32), d_in_(static_cast<int>(w_v.rows)), heads_(heads) {
        check_shape(w_v);
        void* d = upload_f32(w_v);
        const mca_status s = mca_prepare_weights(d, MCA_F32, d_in_, heads, 64, stream, &h_);
        mca_device_free(d);  // the handle keeps its own copy
        check(s);
    }
    // SPEC's AttentionWeights{w_q, w_k, w}: host fp64 matrices (all d_in x heads*64),
    // uploaded as fp32; forwards then take x alone.
    AttentionWeights(const Matrix& w_q, const Matrix& w_k, const Matrix& w_v, int heads, mca_stream_t stream = nullptr)
        : AttentionWeights(w_v, heads, stream) {
        check_shape(w_q);
        check_shape(w_k);
        void* dq = upload_f32(w_q);
        void* dk = upload_f32(w_k);
        const mca_status s = mca_set_projections(h_, dq, dk, stream);
        mca_stream_sync(stream);
        mca_device_free(dq);
        mca_device_free(dk);
        check(s);
        projections_ = true;
    }
    // Attach device W_q / W_k (this handle's dtype, d_in x heads*64).
    void set_projections(const void* w_q_device, const void* w_k_device, mca_stream_t stream = nullptr) {
        check(mca_set_projections(h_, w_q_device, w_k_device, stream));
        projections_ = true;
    }
    bool has_projections() const { return projections_; }
    AttentionWeights(const AttentionWeights&) = delete;
    AttentionWeights& operator=(const AttentionWeights&) = delete;
    AttentionWeights(AttentionWeights&& o) noexcept
        : h_(o.h_), dtype_(o.dtype_), d_in_(o.d_in_), heads_(o.heads_), projections_(o.projections_) {
        o.h_ = nullptr;
    }
    ~AttentionWeights() { mca_weights_free(h_); }

    mca_weights* handle() const { return h_; }
    mca_dtype dtype() const { return dtype_; }
    int d_in() const { return d_in_; }
    int heads() const { return heads_; }

    // Per-head p(i) and cdf, [heads * d_in] each (SamplingDistribution).
    void distributions(std::vector<double>& probs, std::vector<double>& cdf) const {
        probs.resize(static_cast<std::size_t>(heads_) * d_in_);
        cdf.resize(probs.size());
        check(mca_weights_export(h_, probs.data(), cdf.data()));
    }

   private:
    void check_shape(const Matrix& m) const {
        if (heads_ <= 0 || m.cols != static_cast<std::size_t>(heads_) * 64 || m.rows != static_cast<std::size_t>(d_in_))
            throw std::invalid_argument("mca: weight matrices must be d_in x heads*64");
    }
    static void* upload_f32(const Matrix& m) {
        std::vector<float> f(m.data.begin(), m.data.end());
        void* d = nullptr;
        dev_check(mca_device_alloc(f.size() * sizeof(float), &d), "device allocation");
        const mca_status e = mca_copy(d, f.data(), f.size() * sizeof(float), MCA_COPY_H2D);
        if (e != MCA_OK) {
            mca_device_free(d);
            dev_check(e, "H2D copy");
        }
        return d;
    }
    mca_weights* h_ = nullptr;
    mca_dtype dtype_;
    int d_in_, heads_;
    bool projections_ = false;
};

// ---------------------------------------------------------------- device level
// q, k, y: [B, n, heads*64]; x: [B, n, d_in] device buffers in w.dtype().
// q = k = nullptr with projection-carrying weights: q, k are computed from x.
inline FlopsReport forward_device(const AttentionWeights& w, const void* q, const void* k, const void* x, int B, int n,
                                  const McaConfig& cfg, uint64_t seed, void* y, int32_t* budgets = nullptr,
                                  uint8_t* exact = nullptr, bool want_flops = false, long b_offset = 0,
                                  uint32_t layer = 0, mca_stream_t stream = nullptr) {
    const mca_config c = cfg.c();
    mca_flops f{};
    check(mca_forward(w.handle(), q, k, x, w.dtype(), B, n, b_offset, layer, &c, seed, y, budgets, exact,
                      want_flops ? &f : nullptr, stream));
    FlopsReport r;
    if (want_flops) {
        r.exact_encoding = f.exact_encoding;
        r.approx_encoding = f.approx_encoding;
        r.aggregation = f.aggregation;
        r.samples = f.samples;
        r.exact_tokens = f.exact_tokens;
        r.reduction_factor = f.reduction_factor;
        r.total_reduction = f.total_reduction;
    }
    return r;
}

// ---------------------------------------------------------------- Matrix level
struct AttentionOutput {   // SPEC.md:280-283 (attn is never materialised on the device)
    Matrix y;                        // n x heads*64
    std::vector<int32_t> budgets;    // [heads, n]
    std::vector<uint8_t> exact_mask; // [heads, n]
    FlopsReport flops;
};

namespace detail {
struct DeviceBuf {
    void* p = nullptr;
    explicit DeviceBuf(std::size_t bytes) { dev_check(mca_device_alloc(bytes ? bytes : 1, &p), "device allocation"); }
    ~DeviceBuf() { mca_device_free(p); }
    DeviceBuf(const DeviceBuf&) = delete;
    DeviceBuf& operator=(const DeviceBuf&) = delete;
};
inline void upload_f32(const Matrix& m, DeviceBuf& d) {
    std::vector<float> f(m.data.begin(), m.data.end());
    dev_check(mca_copy(d.p, f.data(), f.size() * sizeof(float), MCA_COPY_H2D), "H2D copy");
}
}  // namespace detail

// multihead_forward for one sequence with the projections
// given: q, k: n x heads*64, x: n x d_in. Weights must be fp32 (Matrix ctor).
inline AttentionOutput multihead_forward(const Matrix& q, const Matrix& k, const Matrix& x, const AttentionWeights& w,
                                         const McaConfig& cfg, uint64_t seed) {
    const std::size_t H = static_cast<std::size_t>(w.heads()), n = q.rows;
    if (w.dtype() != MCA_F32) throw std::invalid_argument("mca: Matrix-level forward needs fp32 weights");
    if (q.cols != H * 64 || k.rows != n || k.cols != H * 64)
        throw std::invalid_argument("mca: q, k must be n x heads*64");
    if (x.rows != n || x.cols != static_cast<std::size_t>(w.d_in()))
        throw std::invalid_argument("mca: x must be n x d_in");
    detail::DeviceBuf dq(q.data.size() * 4), dk(k.data.size() * 4), dx(x.data.size() * 4), dy(q.data.size() * 4),
        db(H * n * 4), de(H * n);
    detail::upload_f32(q, dq);
    detail::upload_f32(k, dk);
    detail::upload_f32(x, dx);
    AttentionOutput out;
    out.flops = forward_device(w, dq.p, dk.p, dx.p, 1, static_cast<int>(n), cfg, seed, dy.p,
                               static_cast<int32_t*>(db.p), static_cast<uint8_t*>(de.p), true);
    std::vector<float> y(q.data.size());
    dev_check(mca_copy(y.data(), dy.p, y.size() * 4, MCA_COPY_D2H), "D2H copy");
    out.y.rows = n;
    out.y.cols = H * 64;
    out.y.data.assign(y.begin(), y.end());
    out.budgets.resize(H * n);
    out.exact_mask.resize(H * n);
    dev_check(mca_copy(out.budgets.data(), db.p, H * n * 4, MCA_COPY_D2H), "D2H copy");
    dev_check(mca_copy(out.exact_mask.data(), de.p, H * n, MCA_COPY_D2H), "D2H copy");
    return out;
}

// mca_forward(x, weights, cfg, seed) for one sequence with
// projection-carrying weights: x is n x d_in; returns y (n x heads*64).
inline AttentionOutput mca_forward(const Matrix& x, const AttentionWeights& w, const McaConfig& cfg, uint64_t seed) {
    if (!w.has_projections()) throw std::invalid_argument("mca: mca_forward(x, w) needs weights with W_q / W_k");
    if (cfg.mode != Mode::approximation) throw std::runtime_error("mca: mca_forward requires approximation mode");
    if (w.dtype() != MCA_F32) throw std::invalid_argument("mca: Matrix-level forward needs fp32 weights");
    const std::size_t H = static_cast<std::size_t>(w.heads()), n = x.rows;
    if (x.cols != static_cast<std::size_t>(w.d_in())) throw std::invalid_argument("mca: x must be n x d_in");
    detail::DeviceBuf dx(x.data.size() * 4), dy(n * H * 64 * 4), db(H * n * 4), de(H * n);
    detail::upload_f32(x, dx);
    AttentionOutput out;
    out.flops = forward_device(w, nullptr, nullptr, dx.p, 1, static_cast<int>(n), cfg, seed, dy.p,
                               static_cast<int32_t*>(db.p), static_cast<uint8_t*>(de.p), true);
    std::vector<float> y(n * H * 64);
    dev_check(mca_copy(y.data(), dy.p, y.size() * 4, MCA_COPY_D2H), "D2H copy");
    out.y.rows = n;
    out.y.cols = H * 64;
    out.y.data.assign(y.begin(), y.end());
    out.budgets.resize(H * n);
    out.exact_mask.resize(H * n);
    dev_check(mca_copy(out.budgets.data(), db.p, H * n * 4, MCA_COPY_D2H), "D2H copy");
    dev_check(mca_copy(out.exact_mask.data(), de.p, H * n, MCA_COPY_D2H), "D2H copy");
    return out;
}

// mca_forward: the single-sequence forward in approximation mode.
inline AttentionOutput mca_forward(const Matrix& q, const Matrix& k, const Matrix& x, const AttentionWeights& w,
                                   const McaConfig& cfg, uint64_t seed) {
    if (cfg.mode != Mode::approximation) throw std::runtime_error("mca: mca_forward requires approximation mode");
    return multihead_forward(q, k, x, w, cfg, seed);
}

// regular_forward: the exact layer.
inline AttentionOutput regular_forward(const Matrix& q, const Matrix& k, const Matrix& x, const AttentionWeights& w) {
    McaConfig cfg;
    cfg.mode = Mode::regular;
    return multihead_forward(q, k, x, w, cfg, 0);
}

// sample_budgets on column maxima (host vector in, host out).
inline void sample_budgets(const std::vector<double>& cmax, int n, int d, const McaConfig& cfg,
                           std::vector<int32_t>& budgets, std::vector<uint8_t>& exact) {
    const std::size_t m = cmax.size();
    detail::DeviceBuf dc(m * 8), db(m * 4), de(m);
    dev_check(mca_copy(dc.p, cmax.data(), m * 8, MCA_COPY_H2D), "H2D copy");
    const mca_config c = cfg.c();
    check(mca_stage_budgets(static_cast<const double*>(dc.p), static_cast<long>(m), n, d, &c,
                            static_cast<int32_t*>(db.p), static_cast<uint8_t*>(de.p), nullptr));
    budgets.resize(m);
    exact.resize(m);
    dev_check(mca_copy(budgets.data(), db.p, m * 4, MCA_COPY_D2H), "D2H copy");
    dev_check(mca_copy(exact.data(), de.p, m, MCA_COPY_D2H), "D2H copy");
}

}  // namespace b200
}  // namespace mca

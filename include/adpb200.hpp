// adpb200.hpp — C++ façade over the adpb200 C ABI with the reference's host
// interface: ozadp::adp_gemm (proj/include/ozadp/adp.hpp:84-87) and friends,
// on row-major host matrices (ozadp::MatrixF64 layout,
// proj/include/ozadp/matrix.hpp:12-43). Header-only; link libadpb200.so and
// the CUDA runtime. std::invalid_argument where the reference throws it
// (contract violations), std::runtime_error for CUDA failures.
#pragma once

#include <cuda_runtime.h>

#include <charconv>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "adpb200.h"

namespace adpb200 {

class MatrixF64 {
public:
    MatrixF64() = default;
    MatrixF64(std::size_t rows, std::size_t cols, double fill = 0.0) : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return data_.size(); }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    double& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
    double operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

enum class AdpMode : std::uint8_t { Auto = ADPB200_MODE_AUTO, ForceEmulate = ADPB200_MODE_EMULATE, ForceNative = ADPB200_MODE_NATIVE };
enum class AdpPath : std::uint8_t { Emulated = ADPB200_PATH_EMULATED, NativeFallback = ADPB200_PATH_NATIVE };
enum class AdpReason : std::uint8_t { Ok, Forced, ExceptionalValues, EscTooLarge, TooSmall, CostModel };

inline const char* to_string(AdpPath p) { return p == AdpPath::Emulated ? "emulated" : "native_fallback"; }
inline const char* to_string(AdpReason r) {
    switch (r) {
        case AdpReason::Ok: return "ok";
        case AdpReason::Forced: return "forced";
        case AdpReason::ExceptionalValues: return "exceptional_values";
        case AdpReason::EscTooLarge: return "esc_too_large";
        case AdpReason::TooSmall: return "too_small";
        case AdpReason::CostModel: return "cost_model";
    }
    return "?";
}

// ozadp::AdpConfig (adp.hpp:18-33) + the B200 extensions.
struct AdpConfig {
    int target_bits = 53;
    std::size_t esc_block_len = 256;
    int max_slices = 18;
    std::size_t min_dim = 256;
    AdpMode mode = AdpMode::Auto;
    int forced_slices = 7;
    double cost_ratio = 512.0;
    std::size_t chunk_len = 65536;
    int pair_limit = ADPB200_PAIRS_FULL;  // ADPB200_PAIRS_TARGET skips the pairs below the target precision
    bool guardrails_forced = false;
    bool esc_certified = false;  // ADPB200_ESC_CERTIFIED instead of the reference's coarsened ESC

    adpb200_options to_c() const {
        adpb200_options o;
        adpb200_default_options(&o);
        o.target_bits = target_bits;
        o.esc_block_len = static_cast<int64_t>(esc_block_len);
        o.max_slices = max_slices;
        o.min_dim = static_cast<int64_t>(min_dim);
        o.mode = static_cast<int32_t>(mode);
        o.forced_slices = forced_slices;
        o.cost_ratio = cost_ratio;
        o.chunk_len = static_cast<int64_t>(chunk_len);
        o.pair_limit = pair_limit;
        o.guardrails_forced = guardrails_forced ? 1 : 0;
        o.esc_method = esc_certified ? ADPB200_ESC_CERTIFIED : ADPB200_ESC_COARSENED;
        return o;
    }
    void validate() const {
        adpb200_options o = to_c();
        if (adpb200_validate_options(&o) != ADPB200_OK) throw std::invalid_argument(adpb200_last_error());
    }
};

struct ScanReport {
    std::uint64_t nan_count = 0, inf_count = 0, negzero_count = 0;
    bool has_exceptional = false;
};

struct AdpTrace {
    AdpPath path = AdpPath::NativeFallback;
    AdpReason reason = AdpReason::Ok;
    std::optional<int> esc_bits;
    std::optional<int> slices;
    double modeled_cost_ratio = 0.0;
    ScanReport scan_a, scan_b;
    std::size_t m = 0, n = 0, k = 0;
    int pairs = 0;

    static AdpTrace from_c(const adpb200_trace& t) {
        AdpTrace r;
        r.path = static_cast<AdpPath>(t.path);
        r.reason = static_cast<AdpReason>(t.reason);
        if (t.esc_bits >= 0) r.esc_bits = t.esc_bits;
        if (t.slices >= 0) r.slices = t.slices;
        r.modeled_cost_ratio = t.modeled_cost_ratio;
        r.scan_a = {t.nan_a, t.inf_a, t.negzero_a, t.nan_a + t.inf_a > 0};
        r.scan_b = {t.nan_b, t.inf_b, t.negzero_b, t.nan_b + t.inf_b > 0};
        r.m = static_cast<std::size_t>(t.m);
        r.n = static_cast<std::size_t>(t.n);
        r.k = static_cast<std::size_t>(t.k);
        r.pairs = t.pairs;
        return r;
    }
    // AdpTrace::to_json (adp.cpp:98-114): stable keys path, reason, esc_bits, slices, m, n, k
    std::string to_json() const {
        std::string s = "{\"path\":\"";
        s += to_string(path);
        s += "\",\"reason\":\"";
        s += to_string(reason);
        s += "\",\"esc_bits\":" + (esc_bits ? std::to_string(*esc_bits) : std::string("null"));
        s += ",\"slices\":" + (path == AdpPath::Emulated && slices ? std::to_string(*slices) : std::string("null"));
        s += ",\"m\":" + std::to_string(m) + ",\"n\":" + std::to_string(n) + ",\"k\":" + std::to_string(k) + "}";
        return s;
    }
};

// parse_mode (adp.cpp:116-137)
inline bool parse_mode(const std::string& text, AdpConfig& config) {
    if (text == "auto") {
        config.mode = AdpMode::Auto;
        return true;
    }
    if (text == "native") {
        config.mode = AdpMode::ForceNative;
        return true;
    }
    const std::string prefix = "emulate:";
    if (text.size() > prefix.size() && text.compare(0, prefix.size(), prefix) == 0) {
        const char* first = text.data() + prefix.size();
        const char* last = text.data() + text.size();
        int slices = 0;
        auto [ptr, ec] = std::from_chars(first, last, slices);
        if (ec != std::errc{} || ptr != last || slices < 1 || slices > 32) return false;
        config.mode = AdpMode::ForceEmulate;
        config.forced_slices = slices;
        return true;
    }
    return false;
}

namespace detail {
inline void check(int rc) {
    if (rc == ADPB200_OK) return;
    if (rc == ADPB200_ERR_CONTRACT) throw std::invalid_argument(adpb200_last_error());
    throw std::runtime_error(adpb200_last_error());
}
inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t bytes) {
        if (bytes) cuda(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};
}  // namespace detail

// One handle (device workspace) per thread and device.
inline adpb200_handle default_handle(int device = 0) {
    struct Owner {
        adpb200_handle h = nullptr;
        ~Owner() {
            if (h) adpb200_destroy(h);
        }
    };
    thread_local Owner owners[16];
    if (device < 0 || device >= 16) throw std::invalid_argument("device out of range");
    if (!owners[device].h) detail::check(adpb200_create(&owners[device].h, device));
    return owners[device].h;
}

// ozadp::adp_gemm (adp.hpp:84-87 / adp.cpp:139-178): returns alpha*A*B + beta*C
// and the trace. Host in, host out; one synchronisation at the end.
inline std::pair<MatrixF64, AdpTrace> adp_gemm(const MatrixF64& a, const MatrixF64& b, double alpha = 1.0,
                                               double beta = 0.0, const MatrixF64* c = nullptr,
                                               const AdpConfig& config = AdpConfig{}, int device = 0) {
    config.validate();
    if (a.cols() != b.rows()) throw std::invalid_argument("adp_gemm: inner dimensions differ");
    if (beta != 0.0 && c == nullptr) throw std::invalid_argument("adp_gemm: beta != 0 requires C");
    if (c && (c->rows() != a.rows() || c->cols() != b.cols())) throw std::invalid_argument("adp_gemm: C shape mismatch");
    const std::size_t m = a.rows(), n = b.cols(), k = a.cols();
    adpb200_handle h = default_handle(device);
    detail::cuda(cudaSetDevice(device), "cudaSetDevice");
    adpb200_options o = config.to_c();
    MatrixF64 out(m, n);
    adpb200_trace t;
    // host-buffer entry point: copies in, computes, copies C out while the GEMM runs
    detail::check(adpb200_adp_gemm_host(h, int64_t(m), int64_t(n), int64_t(k), alpha, a.data(), b.data(), beta,
                                        c ? c->data() : nullptr, out.data(), &o, &t, nullptr));
    return {std::move(out), AdpTrace::from_c(t)};
}

}  // namespace adpb200

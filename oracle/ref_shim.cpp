// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" wrappers over the UNMODIFIED reference library (ozadp, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). These
// let the Python tests and the C restatement (oracle/adp_oracle.c) be pinned
// against the reference's own code on the same inputs. Only tests/, smoke()
// and bench.py's cpu_baseline / --impl reference leg may load the result.
//
// Every wrapper takes plain pointers + sizes, row-major like ozadp::MatrixF64
// (proj/include/ozadp/matrix.hpp:12-43), and returns 0 on success, 3 for
// std::invalid_argument / std::domain_error (the CLI's contract exit code,
// proj/tools/ozadp_main.cpp:235-244) and 2 for anything else.
#include <chrono>
#include <cstring>
#include <exception>
#include <optional>
#include <vector>
#include <stdexcept>
#include <string>

#include "ozadp/adp.hpp"
#include "ozadp/esc.hpp"
#include "ozadp/fpbits.hpp"
#include "ozadp/grading.hpp"
#include "ozadp/igemm.hpp"
#include "ozadp/oracle.hpp"
#include "ozadp/qr.hpp"
#include "ozadp/matrix_io.hpp"
#include "ozadp/slicing.hpp"
#include "ozadp/threads.hpp"

using namespace ozadp;

namespace {

MatrixF64 wrap(const double* p, std::size_t r, std::size_t c) {
    MatrixF64 m(r, c);
    if (r * c) std::memcpy(m.data(), p, r * c * sizeof(double));
    return m;
}

void unwrap(const MatrixF64& m, double* out) {
    if (m.size()) std::memcpy(out, m.data(), m.size() * sizeof(double));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 3;
    } catch (const std::domain_error&) {
        return 3;
    } catch (...) {
        return 2;
    }
}

GemmParams params(double alpha, double beta, int slices, long long chunk, int limit) {
    GemmParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.slices = slices;
    p.chunk_len = std::size_t(chunk);
    if (limit >= 0) {
        p.policy.kind = PairPolicy::Kind::DiagonalTruncated;
        p.policy.limit = limit;
    }
    return p;
}

}  // namespace

extern "C" {

int ozref_set_threads(int n) {
    set_thread_cap(n);
    return 0;
}

int ozref_gen_uniform_rect(long long rows, long long cols, unsigned long long seed, double lo,
                           double hi, double* out) {
    return guarded([&] { unwrap(gen_uniform_rect(rows, cols, seed, lo, hi), out); });
}

int ozref_gen_test2(long long n, int b, unsigned long long seed, double* lhs, double* rhs) {
    return guarded([&] {
        Test2Instance t = gen_test2(std::size_t(n), b, seed);
        unwrap(t.lhs, lhs);
        unwrap(t.rhs, rhs);
    });
}

// counts[0..2] = nan, inf, -0; returns has_exceptional in *exc.
int ozref_scan(const double* a, long long rows, long long cols, unsigned long long* counts,
               int* exc) {
    return guarded([&] {
        ScanReport r = scan_matrix(wrap(a, rows, cols));
        counts[0] = r.nan_count;
        counts[1] = r.inf_count;
        counts[2] = r.negzero_count;
        *exc = r.has_exceptional ? 1 : 0;
    });
}

// orient 0 = ByRow, 1 = ByCol. Outputs sized lines*blocks, lines*blocks, lines.
int ozref_block_stats(const double* a, long long rows, long long cols, int orient,
                      long long block_len, int* max_exp, int* min_exp, int* line_max) {
    return guarded([&] {
        BlockStats s = block_exponent_stats(wrap(a, rows, cols),
                                            orient ? Orientation::ByCol : Orientation::ByRow,
                                            std::size_t(block_len));
        if (!s.max_exp.empty()) std::memcpy(max_exp, s.max_exp.data(), s.max_exp.size() * 4);
        if (!s.min_exp.empty()) std::memcpy(min_exp, s.min_exp.data(), s.min_exp.size() * 4);
        if (!s.line_max.empty()) std::memcpy(line_max, s.line_max.data(), s.line_max.size() * 4);
    });
}

// out[0..2] = esc_bits, window_bits, slices_required.
int ozref_esc_coarsened(const double* a, const double* b, long long m, long long n, long long k,
                        long long block_len, int target_bits, int* out) {
    return guarded([&] {
        BlockStats sa = block_exponent_stats(wrap(a, m, k), Orientation::ByRow, block_len);
        BlockStats sb = block_exponent_stats(wrap(b, k, n), Orientation::ByCol, block_len);
        EscReport r = esc_coarsened(sa, sb, target_bits);
        out[0] = r.esc_bits;
        out[1] = r.window_bits;
        out[2] = r.slices_required;
    });
}

int ozref_esc_exact(const double* a, const double* b, long long m, long long n, long long k,
                    int target_bits, int* out) {
    return guarded([&] {
        EscReport r = esc_exact(wrap(a, m, k), wrap(b, k, n), target_bits);
        out[0] = r.esc_bits;
        out[1] = r.window_bits;
        out[2] = r.slices_required;
    });
}

int ozref_required_slices(int target_bits, int esc_bits, int* out) {
    return guarded([&] { *out = required_slices(target_bits, esc_bits); });
}

// digits: slices planes of lines*len int8; scale: lines int32.
int ozref_decompose(const double* a, long long rows, long long cols, int orient, int slices,
                    signed char* digits, int* scale) {
    return guarded([&] {
        SlicedMatrix s = decompose(wrap(a, rows, cols),
                                   orient ? Orientation::ByCol : Orientation::ByRow, slices);
        if (!s.digits.empty()) std::memcpy(digits, s.digits.data(), s.digits.size());
        if (!s.scale_exp.empty()) std::memcpy(scale, s.scale_exp.data(), s.scale_exp.size() * 4);
    });
}

// acc: m*n*(2s-1) int64, element-major (igemm.hpp:34-47). limit < 0 = Full.
int ozref_slice_pair_mm(const double* a, const double* b, long long m, long long n, long long k,
                        int slices, long long chunk, int limit, long long* acc) {
    return guarded([&] {
        GemmParams p = params(1.0, 0.0, slices, chunk, limit);
        SlicedMatrix sa = decompose(wrap(a, m, k), Orientation::ByRow, slices);
        SlicedMatrix sb = decompose(wrap(b, k, n), Orientation::ByCol, slices);
        DiagonalAccumulators d = slice_pair_mm(sa, sb, p);
        if (!d.acc.empty()) std::memcpy(acc, d.acc.data(), d.acc.size() * 8);
    });
}

int ozref_emulated_gemm(const double* a, const double* b, long long m, long long n, long long k,
                        double alpha, double beta, const double* c, int slices, long long chunk,
                        int limit, double* out) {
    return guarded([&] {
        GemmParams p = params(alpha, beta, slices, chunk, limit);
        MatrixF64 cm;
        if (c) cm = wrap(c, m, n);
        unwrap(emulated_gemm(wrap(a, m, k), wrap(b, k, n), p, c ? &cm : nullptr), out);
    });
}

int ozref_native_gemm(const double* a, const double* b, long long m, long long n, long long k,
                      double alpha, double beta, const double* c, double* out) {
    return guarded([&] {
        MatrixF64 cm;
        if (c) cm = wrap(c, m, n);
        unwrap(native_gemm(wrap(a, m, k), wrap(b, k, n), alpha, beta, c ? &cm : nullptr), out);
    });
}

int ozref_exact_gemm(const double* a, const double* b, long long m, long long n, long long k,
                     double* out) {
    return guarded([&] { unwrap(exact_gemm(wrap(a, m, k), wrap(b, k, n)), out); });
}

// cfg_i: target_bits, esc_block_len, max_slices, min_dim, mode(0 auto,1 emulate,2 native),
//        forced_slices, chunk_len;  cfg_d: cost_ratio.
// trace_i: path(0 emulated,1 native), reason(0..5 as AdpReason), esc_bits(-1 null),
//          slices(-1 null), m, n, k, scan counts a[3], b[3].
// trace_d: modeled_cost_ratio.  json: optional buffer for AdpTrace::to_json.
int ozref_adp_gemm(const double* a, const double* b, long long m, long long n, long long k,
                   double alpha, double beta, const double* c, const long long* cfg_i,
                   const double* cfg_d, double* out, long long* trace_i, double* trace_d,
                   char* json, int json_cap) {
    return guarded([&] {
        AdpConfig cfg;
        cfg.target_bits = int(cfg_i[0]);
        cfg.esc_block_len = std::size_t(cfg_i[1]);
        cfg.max_slices = int(cfg_i[2]);
        cfg.min_dim = std::size_t(cfg_i[3]);
        cfg.mode = cfg_i[4] == 1 ? AdpMode::ForceEmulate
                                 : (cfg_i[4] == 2 ? AdpMode::ForceNative : AdpMode::Auto);
        cfg.forced_slices = int(cfg_i[5]);
        cfg.chunk_len = std::size_t(cfg_i[6]);
        cfg.cost_ratio = cfg_d[0];
        MatrixF64 cm;
        if (c) cm = wrap(c, m, n);
        auto [res, tr] = adp_gemm(wrap(a, m, k), wrap(b, k, n), alpha, beta, c ? &cm : nullptr, cfg);
        unwrap(res, out);
        trace_i[0] = tr.decision.path == AdpPath::Emulated ? 0 : 1;
        trace_i[1] = int(tr.decision.reason);
        trace_i[2] = tr.decision.esc ? tr.decision.esc->esc_bits : -1;
        trace_i[3] = tr.decision.path == AdpPath::Emulated ? tr.decision.slices : -1;
        trace_i[4] = (long long)tr.m;
        trace_i[5] = (long long)tr.n;
        trace_i[6] = (long long)tr.k;
        trace_i[7] = (long long)tr.scan_a.nan_count;
        trace_i[8] = (long long)tr.scan_a.inf_count;
        trace_i[9] = (long long)tr.scan_a.negzero_count;
        trace_i[10] = (long long)tr.scan_b.nan_count;
        trace_i[11] = (long long)tr.scan_b.inf_count;
        trace_i[12] = (long long)tr.scan_b.negzero_count;
        trace_d[0] = tr.decision.modeled_cost_ratio;
        if (json && json_cap > 0) {
            std::string js = tr.to_json();
            std::strncpy(json, js.c_str(), std::size_t(json_cap) - 1);
            json[json_cap - 1] = 0;
        }
    });
}

// decide() with a fake ESC provider (the reference's own test seam,
// proj/tests/test_adp.cpp:38-54). scan flags: exc_a, exc_b. esc_in = esc_bits
// the fake reports (slices_required = required_slices(target, esc_in)).
// out_i: path, reason, slices, provider_calls, esc_bits(-1 none); out_d: cost ratio.
int ozref_decide(int exc_a, int exc_b, long long m, long long n, long long k, int esc_in,
                 const long long* cfg_i, const double* cfg_d, int* out_i, double* out_d) {
    return guarded([&] {
        AdpConfig cfg;
        cfg.target_bits = int(cfg_i[0]);
        cfg.esc_block_len = std::size_t(cfg_i[1]);
        cfg.max_slices = int(cfg_i[2]);
        cfg.min_dim = std::size_t(cfg_i[3]);
        cfg.mode = cfg_i[4] == 1 ? AdpMode::ForceEmulate
                                 : (cfg_i[4] == 2 ? AdpMode::ForceNative : AdpMode::Auto);
        cfg.forced_slices = int(cfg_i[5]);
        cfg.chunk_len = std::size_t(cfg_i[6]);
        cfg.cost_ratio = cfg_d[0];
        ScanReport sa, sb;
        sa.has_exceptional = exc_a != 0;
        sb.has_exceptional = exc_b != 0;
        int calls = 0;
        auto provider = [&]() {
            ++calls;
            EscReport r;
            r.esc_bits = esc_in;
            r.window_bits = cfg.target_bits + esc_in;
            r.slices_required = required_slices(cfg.target_bits, esc_in);
            r.method = EscMethod::Coarsened;
            return r;
        };
        AdpDecision d = decide(sa, sb, m, n, k, provider, cfg);
        out_i[0] = d.path == AdpPath::Emulated ? 0 : 1;
        out_i[1] = int(d.reason);
        out_i[2] = d.slices;
        out_i[3] = calls;
        out_i[4] = d.esc ? d.esc->esc_bits : -1;
        out_d[0] = d.modeled_cost_ratio;
    });
}

// Wall-clock seconds of one emulated_gemm / adp_gemm / native_gemm call on
// row-major host buffers (bench.py's reference arm). which: 0 emulated(slices,
// Full), 1 adp auto (default AdpConfig), 2 native.
double ozref_time_call(int which, const double* a, const double* b, long long m, long long n,
                       long long k, int slices, double* out) {
    MatrixF64 am = wrap(a, m, k), bm = wrap(b, k, n);
    auto t0 = std::chrono::steady_clock::now();
    MatrixF64 r;
    try {
        if (which == 0)
            r = emulated_gemm(am, bm, params(1.0, 0.0, slices, 65536, -1));
        else if (which == 1)
            r = adp_gemm(am, bm).first;
        else
            r = native_gemm(am, bm);
    } catch (...) {
        return -1.0;
    }
    auto t1 = std::chrono::steady_clock::now();
    if (out) unwrap(r, out);
    return std::chrono::duration<double>(t1 - t0).count();
}

// error_report (grading.cpp:67-90). use_diag: compare the diagonal against
// exact_diag. out: max_err, avg_err, counted, skipped.
int ozref_error_report(const double* c, const double* ref, long long rows, long long cols,
                       int use_diag, double exact_diag, double* out) {
    return guarded([&] {
        std::optional<double> d;
        if (use_diag) d = exact_diag;
        ErrorReport r = error_report(wrap(c, rows, cols), wrap(ref, rows, cols), d);
        out[0] = r.max_err;
        out[1] = r.avg_err;
        out[2] = double(r.counted);
        out[3] = double(r.skipped);
    });
}

// exact_dot(x, y).rounded (oracle.cpp:40-53)
int ozref_exact_dot(const double* x, const double* y, long long n, double* out) {
    return guarded([&] {
        std::vector<double> xv(x, x + n), yv(y, y + n);
        *out = exact_dot(xv, yv).rounded;
    });
}

// grade_uniform_point (grading.cpp:92-134) with the default AdpConfig.
// out: emu_max, emu_avg, nat_max, nat_avg, esc_bits, slices, fallback.
int ozref_grade_uniform_point(long long n, unsigned long long seed, double* out) {
    return guarded([&] {
        GradePoint p = grade_uniform_point(std::size_t(n), seed, AdpConfig{});
        out[0] = p.emu_max_ratio;
        out[1] = p.emu_avg_ratio;
        out[2] = p.nat_max_ratio;
        out[3] = p.nat_avg_ratio;
        out[4] = p.esc_bits;
        out[5] = p.slices;
        out[6] = p.fallback ? 1.0 : 0.0;
    });
}

// run_test2_sweep (grading.cpp:246-275) for one b and one mode string;
// out: max_err, avg_err, esc_bits (-1 none), slices, fallback.
int ozref_test2_row(long long n, int b, const char* mode, unsigned long long seed, double* out) {
    return guarded([&] {
        std::vector<SweepRow> rows = run_test2_sweep(std::size_t(n), {b}, {std::string(mode)}, seed);
        const SweepRow& r = rows.at(0);
        out[0] = r.max_err;
        out[1] = r.avg_err;
        out[2] = r.esc_bits ? *r.esc_bits : -1;
        out[3] = r.slices;
        out[4] = r.fallback ? 1.0 : 0.0;
    });
}

// geqrf_blocked (qr.cpp:98-143) + materialize_q + qr_residual in one call.
// cfg_i / cfg_d as ozref_adp_gemm. t_out: panels slots of panel*panel
// doubles, T of panel p packed pw x pw at slot start. traces_i: 3 per panel x
// {path, reason, esc_bits(-1), slices(-1), m, n, k}. q_out (m x n) and acc[2]
// (residual, orthogonality) optional.
int ozref_qr(const double* a, long long m, long long n, long long panel, const long long* cfg_i,
             const double* cfg_d, double* factors, double* t_out, long long* traces_i, double* q_out,
             double* acc) {
    return guarded([&] {
        AdpConfig cfg;
        cfg.target_bits = int(cfg_i[0]);
        cfg.esc_block_len = std::size_t(cfg_i[1]);
        cfg.max_slices = int(cfg_i[2]);
        cfg.min_dim = std::size_t(cfg_i[3]);
        cfg.mode = cfg_i[4] == 1 ? AdpMode::ForceEmulate
                                 : (cfg_i[4] == 2 ? AdpMode::ForceNative : AdpMode::Auto);
        cfg.forced_slices = int(cfg_i[5]);
        cfg.chunk_len = std::size_t(cfg_i[6]);
        cfg.cost_ratio = cfg_d[0];
        const MatrixF64 am = wrap(a, m, n);
        QrResult qr = geqrf_blocked(am, std::size_t(panel), cfg);
        unwrap(qr.factors, factors);
        for (std::size_t p = 0; p < qr.t_blocks.size(); ++p)
            unwrap(qr.t_blocks[p], t_out + p * std::size_t(panel) * std::size_t(panel));
        for (std::size_t i = 0; i < qr.traces.size(); ++i) {
            const AdpTrace& tr = qr.traces[i];
            long long* o = traces_i + 7 * i;
            o[0] = tr.decision.path == AdpPath::Emulated ? 0 : 1;
            o[1] = int(tr.decision.reason);
            o[2] = tr.decision.esc ? tr.decision.esc->esc_bits : -1;
            o[3] = tr.decision.path == AdpPath::Emulated ? tr.decision.slices : -1;
            o[4] = (long long)tr.m;
            o[5] = (long long)tr.n;
            o[6] = (long long)tr.k;
        }
        if (q_out) unwrap(materialize_q(qr), q_out);
        if (acc) {
            QrAccuracy r = qr_residual(am, qr);
            acc[0] = r.residual;
            acc[1] = r.orthogonality;
        }
    });
}

// Wall-clock seconds of one geqrf_blocked call (bench / CPU baseline).
double ozref_time_qr(const double* a, long long m, long long n, long long panel, long long min_dim) {
    const MatrixF64 am = wrap(a, m, n);
    AdpConfig cfg;
    cfg.min_dim = std::size_t(min_dim);
    auto t0 = std::chrono::steady_clock::now();
    try {
        QrResult qr = geqrf_blocked(am, std::size_t(panel), cfg);
        (void)qr;
    } catch (...) {
        return -1.0;
    }
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// matrix_io (matrix_io.cpp): write_matrix by extension / read_matrix by sniffing.
int ozref_write_matrix(const char* path, const double* a, long long rows, long long cols) {
    return guarded([&] { write_matrix(path, wrap(a, rows, cols)); });
}
// dims[2] out; out may be NULL to query the shape (cap elements max).
int ozref_read_matrix(const char* path, double* out, long long cap, long long* dims) {
    return guarded([&] {
        MatrixF64 m = read_matrix(path);
        dims[0] = (long long)m.rows();
        dims[1] = (long long)m.cols();
        if (out && (long long)m.size() <= cap) unwrap(m, out);
    });
}

}  // extern "C"

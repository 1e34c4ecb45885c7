// Exercises the C++ façade (include/adpb200.hpp) the way a reference user
// would call ozadp::adp_gemm. Built and run by tests/test_cabi.py (CPU part)
// and tests/test_gpu_facade.py (GPU part).
//
//   facade_check cpu            -> config / parse_mode / decide contract checks
//   facade_check gpu in.bin out -> adp_gemm on the matrices in in.bin
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>

#include "adpb200.hpp"

using namespace adpb200;

static int fail(const char* what) {
    std::fprintf(stderr, "FAIL: %s\n", what);
    return 1;
}

static int cpu_checks() {
    AdpConfig cfg;
    cfg.validate();
    // AdpConfig::validate contract (proj/tests/test_adp.cpp:58-80)
    AdpConfig bad = cfg;
    bad.max_slices = 6;
    try {
        bad.validate();
        return fail("max_slices 6 accepted");
    } catch (const std::invalid_argument&) {
    }
    bad = cfg;
    bad.chunk_len = 131072;
    try {
        bad.validate();
        return fail("chunk_len 131072 accepted");
    } catch (const std::invalid_argument&) {
    }
    bad = cfg;
    bad.cost_ratio = 0.0;
    try {
        bad.validate();
        return fail("cost_ratio 0 accepted");
    } catch (const std::invalid_argument&) {
    }
    // the certified-ESC extension maps onto the C options
    AdpConfig cc;
    cc.esc_certified = true;
    cc.validate();
    if (cc.to_c().esc_method != ADPB200_ESC_CERTIFIED || AdpConfig{}.to_c().esc_method != ADPB200_ESC_COARSENED)
        return fail("esc_method mapping");
    // parse_mode (adp.cpp:116-137)
    AdpConfig p;
    if (!parse_mode("emulate:11", p) || p.mode != AdpMode::ForceEmulate || p.forced_slices != 11)
        return fail("emulate:11");
    if (parse_mode("emulate:33", p) || parse_mode("emulate:", p) || parse_mode("emulate:7x", p) || parse_mode("x", p))
        return fail("bad modes accepted");
    if (!parse_mode("native", p) || p.mode != AdpMode::ForceNative) return fail("native");
    if (!parse_mode("auto", p) || p.mode != AdpMode::Auto) return fail("auto");
    // decide (host copy of the device decision function)
    adpb200_options o = AdpConfig{}.to_c();
    int32_t out[5];
    double cost = 0;
    if (adpb200_decide_host(0, 0, 1024, 1024, 1024, 1, &o, out, &cost) != 0) return fail("decide rc");
    if (out[0] != ADPB200_PATH_EMULATED || out[1] != 0 || out[2] != 7 || out[3] != 1) return fail("decide 1024^3");
    if (adpb200_decide_host(0, 1, 1024, 1024, 1024, 1, &o, out, &cost) != 0 || out[1] != 2 || out[3] != 0)
        return fail("decide exceptional");
    AdpTrace t;
    t.path = AdpPath::Emulated;
    t.esc_bits = 1;
    t.slices = 7;
    t.m = t.n = t.k = 4;
    if (t.to_json() != "{\"path\":\"emulated\",\"reason\":\"ok\",\"esc_bits\":1,\"slices\":7,\"m\":4,\"n\":4,\"k\":4}")
        return fail("to_json");
    std::printf("facade cpu checks ok\n");
    return 0;
}

// in.bin: int64 m, n, k, then A (m*k), B (k*n), C (m*n) doubles, alpha, beta
static int gpu_run(const char* in, const char* outp) {
    std::ifstream f(in, std::ios::binary);
    int64_t dims[3];
    f.read(reinterpret_cast<char*>(dims), sizeof(dims));
    MatrixF64 a(dims[0], dims[2]), b(dims[2], dims[1]), c(dims[0], dims[1]);
    f.read(reinterpret_cast<char*>(a.data()), a.size() * 8);
    f.read(reinterpret_cast<char*>(b.data()), b.size() * 8);
    f.read(reinterpret_cast<char*>(c.data()), c.size() * 8);
    double ab[2];
    f.read(reinterpret_cast<char*>(ab), sizeof(ab));
    auto [res, trace] = adp_gemm(a, b, ab[0], ab[1], &c);
    std::ofstream o(outp, std::ios::binary);
    o.write(reinterpret_cast<const char*>(res.data()), res.size() * 8);
    std::printf("%s\n", trace.to_json().c_str());
    return 0;
}

int main(int argc, char** argv) {
    try {
        if (argc >= 2 && std::strcmp(argv[1], "cpu") == 0) return cpu_checks();
        if (argc >= 4 && std::strcmp(argv[1], "gpu") == 0) return gpu_run(argv[2], argv[3]);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 2;
    }
    std::fprintf(stderr, "usage: facade_check cpu | gpu in.bin out.bin\n");
    return 2;
}

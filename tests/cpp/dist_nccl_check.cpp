// Runs the NCCL-driven B-distributed ADP DGEMM (include/adpb200_nccl.hpp) as a
// single-rank communicator on GPU 0 and checks C bitwise against the
// single-GPU adpb200_dgemm, on the emulated path and on the NaN fallback.
// Built and run by tests/test_gpu_golden.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "adpb200_nccl.hpp"

static double lcg(uint64_t& s) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return double(s >> 11) * 0x1p-53 * 2.0 - 1.0;
}

int main() {
    const int64_t m = 700, n = 512, k = 650;
    std::vector<double> A(m * k), B(k * n), C0(m * n);
    uint64_t s = 42;
    for (auto& v : A) v = lcg(s);
    for (auto& v : B) v = lcg(s);
    for (auto& v : C0) v = lcg(s);
    adpb200_handle h;
    if (adpb200_create(&h, 0)) return 2;
    ncclComm_t comm;
    int dev = 0;
    if (ncclCommInitAll(&comm, 1, &dev) != ncclSuccess) {
        std::fprintf(stderr, "ncclCommInitAll failed\n");
        return 2;
    }
    cudaStream_t st;
    cudaStreamCreate(&st);
    adpb200_options o;
    adpb200_default_options(&o);
    o.pair_limit = ADPB200_PAIRS_TARGET;
    double *dA, *dB, *dC1, *dC2;
    cudaMalloc(&dA, A.size() * 8);
    cudaMalloc(&dB, B.size() * 8);
    cudaMalloc(&dC1, C0.size() * 8);
    cudaMalloc(&dC2, C0.size() * 8);
    int bad_total = 0;
    adpb200::PeerSlabs peers;
    if (adpb200::peer_slabs_create(peers, comm, 0, 1, 0, n, k, &o, st)) {
        std::fprintf(stderr, "peer_slabs_create: %s\n", adpb200_last_error());
        return 2;
    }
    const std::vector<double> B0 = B;
    for (int run = 0; run < 6; ++run) {
        const int poison = run & 1, fused = run >> 1;  // 0: all-gather, 1: in place, 2: pulled
        peers.pull = fused == 2;
        B = B0;
        if (poison) B[123] = std::nan("");
        cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dC1, C0.data(), C0.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dC2, C0.data(), C0.size() * 8, cudaMemcpyHostToDevice);
        int rc = adpb200::dgemm_dist_nccl(h, comm, 0, 1, 'N', m, m, n, k, 1.25, dA, m, dB, 0.5, dC1, m, &o, nullptr,
                                          st, fused ? &peers : nullptr);
        if (!rc) rc = adpb200_dgemm(h, 'N', 'N', m, n, k, 1.25, dA, m, dB, k, 0.5, dC2, m, &o, nullptr, st);
        cudaStreamSynchronize(st);
        if (rc) {
            std::fprintf(stderr, "rc %d: %s\n", rc, adpb200_last_error());
            return 3;
        }
        std::vector<double> c1(m * n), c2(m * n);
        cudaMemcpy(c1.data(), dC1, c1.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(c2.data(), dC2, c2.size() * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (size_t i = 0; i < c1.size(); ++i) {
            uint64_t x, y;
            std::memcpy(&x, &c1[i], 8);
            std::memcpy(&y, &c2[i], 8);
            const bool both_nan = c1[i] != c1[i] && c2[i] != c2[i];
            if (x != y && !both_nan) ++bad;
        }
        std::printf("%s%s: %d of %zu differ\n", fused == 2 ? "pulled " : (fused ? "fused " : ""),
                    poison ? "fallback" : "emulated", bad, c1.size());
        bad_total += bad;
    }
    adpb200::peer_slabs_destroy(peers);
    ncclCommDestroy(comm);
    adpb200_destroy(h);
    return bad_total ? 1 : 0;
}

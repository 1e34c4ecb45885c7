// Microbenchmark (not part of the product): sustained DPX __viaddmax_s16x2
// (SASS VIADDMNMX ... .S16x2) throughput on one B200 — the roofline denominator
// of the ESC kernel K2 (csrc/guard.cu esc_kernel), whose inner loop is this
// instruction fed from shared memory (2 per (i, j-pair, block)).
//
// 8 independent accumulator chains per thread, operands in registers, grid =
// resident CTAs; reports thread-level instructions per second and per SM clock
// (the SM clock from clock64 against %globaltimer on CTA 0). bench.py divides
// the live esc_kernel's instruction rate by this.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 dpx_peak.cu -o dpx_peak && ./dpx_peak
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

constexpr int kChains = 8;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// cycles[0] = SM clocks and cycles[1] = nanoseconds of CTA 0 (its SM's clock rate)
__global__ void __launch_bounds__(256) dpx_kernel(uint32_t seed, int iters, uint32_t* out, long long* cycles) {
    uint32_t z[kChains], a = seed ^ threadIdx.x, b = seed * 7u + blockIdx.x;
#pragma unroll
    for (int c = 0; c < kChains; ++c) z[c] = 0x80008000u + c;
    long long t0 = clock64();
    const unsigned long long g0 = gtimer();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int c = 0; c < kChains; ++c) z[c] = __viaddmax_s16x2(a + c, b, z[c]);
        a += 0x00010001u;
    }
    long long t1 = clock64();
    const unsigned long long g1 = gtimer();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc ^= z[c];
    if (acc == 0x12345678u) out[0] = acc;  // keep the chains live
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        cycles[0] = t1 - t0;
        cycles[1] = (long long)(g1 - g0);
    }
}

int main() {
    int dev = 0, sms = 0, per_sm = 0;
    cudaSetDevice(dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dpx_kernel, 256, 0);
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 16);
    const int grid = sms * per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // warm-up, then ~2 s of back-to-back launches
    const int iters = 20000;
    dpx_kernel<<<grid, 256>>>(1u, iters, out, cyc);
    cudaDeviceSynchronize();
    const int reps = 40;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) dpx_kernel<<<grid, 256>>>(r + 2u, iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    long long cyc_ns[2] = {0, 1};
    cudaMemcpy(cyc_ns, cyc, 16, cudaMemcpyDeviceToHost);
    const double instr = double(grid) * 256.0 * iters * 16.0 * kChains;  // per launch (thread-level)
    const double per_s = instr * reps / (ms * 1e-3);
    const double clock_hz = double(cyc_ns[0]) / (double(cyc_ns[1]) * 1e-9);  // the SM clock during the run
    const double per_clk_sm = per_s / (double(sms) * clock_hz);
    printf("{\"kernel\": \"dpx_peak __viaddmax_s16x2\", \"sms\": %d, \"ctas_per_sm\": %d, \"threads\": 256, "
           "\"chains\": %d, \"instr_per_s\": %.4e, \"instr_per_clk_per_sm\": %.2f, \"sm_clock_mhz\": %.0f, "
           "\"note\": \"thread-level VIADDMNMX.S16x2 instructions; each = 2 add+max of int16 pairs\", "
           "\"error\": \"%s\"}\n",
           sms, per_sm, kChains, per_s, per_clk_sm, clock_hz / 1e6,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}

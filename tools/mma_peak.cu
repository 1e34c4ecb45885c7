// Microbenchmark (not part of the product): sustained tcgen05.mma kind::i8
// throughput on one B200, operands resident in shared memory (no TMA), to
// measure (1) the INT8 dense tensor peak used as the roofline denominator of
// the slice GEMM and (2) how efficiently the slice-pair MMA schedule of
// igemm.cu (stacked B slices, mixed N) runs on the tensor pipe by itself.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include \
//        -I../paper_2511_13778_b200/csrc mma_peak.cu -o mma_peak && ./mma_peak
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "tc.cuh"

using namespace adpb200;

struct Op {
    uint32_t col, a_off, b_off, n;
};

__global__ void __launch_bounds__(128, 1) mma_loop(const Op* ops, int nops, int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ Op sops[64];
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 7);
    for (int i = threadIdx.x; i < nops; i += blockDim.x) sops[i] = ops[i];
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar, 1);
        tc::fence_barrier_init();
    }
    if (threadIdx.x / 32 == 1) tc::tmem_alloc(&tmem_slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        const uint32_t base = tc::smem_u32(smem);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            // 5 "stages" of 43 KB so consecutive k-blocks read different smem
            const uint32_t st = base + uint32_t(it % 3) * 43008u;
            for (int i = 0; i < nops; ++i) {
                const Op o = sops[i];
                tc::mma_i8(tmem + o.col, tc::smem_desc_sw32(st + o.a_off), tc::smem_desc_sw32(st + o.b_off),
                           tc::idesc_i8(128, o.n), it > 0 ? 1u : 0u);
            }
        }
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    if (threadIdx.x / 32 == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, 512);
    }
}

static double run(const char* name, const Op* hops, int nops, int iters, int nb_macs_per_iter_cols) {
    Op* dops;
    cudaMalloc(&dops, sizeof(Op) * nops);
    cudaMemcpy(dops, hops, sizeof(Op) * nops, cudaMemcpyHostToDevice);
    unsigned long long* dcyc;
    cudaMalloc(&dcyc, 148 * 8);
    const int smem = 160 * 1024 + 1024;
    cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_loop<<<148, 128, smem>>>(dops, nops, 10, dcyc);  // warm up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_loop<<<148, 128, smem>>>(dops, nops, iters, dcyc);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc[148];
    cudaMemcpy(cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
    double macs = 0;
    for (int i = 0; i < nops; ++i) macs += 128.0 * hops[i].n * 32.0;
    macs *= double(iters) * 148;
    double tops = 2.0 * macs / (ms * 1e-3) / 1e12;
    double cyc_per_iter = double(cyc[0]) / iters;
    double ideal = 0;
    for (int i = 0; i < nops; ++i) ideal += hops[i].n / 2.0;
    printf("{\"case\": \"%s\", \"err\": \"%s\", \"ms\": %.3f, \"int8_tops\": %.1f, \"cycles_per_iter\": %.1f, "
           "\"ideal_cycles_per_iter\": %.1f, \"efficiency\": %.3f}\n",
           name, cudaGetErrorString(err), ms, tops, cyc_per_iter, ideal, ideal / cyc_per_iter);
    cudaFree(dops);
    cudaFree(dcyc);
    return tops;
}

int main() {
    // 1) peak: back-to-back M=128 N=256 K=32 into 2 accumulators
    Op peak[2] = {{0, 0, 4096, 256}, {256, 0, 4096, 256}};
    run("peak_n256", peak, 2, 200000, 0);
    Op p128[2] = {{0, 0, 4096, 128}, {128, 0, 4096, 128}};
    run("n128", p128, 2, 200000, 0);
    Op p64[2] = {{0, 0, 4096, 64}, {64, 0, 4096, 64}};
    run("n64", p64, 2, 200000, 0);
    // 2) the slice-pair schedule of igemm<64> at s = 7, L = 7 (34 pairs)
    const int s = 7, L = 7, NB = 64, G = 4, BM = 128, KB = 32;
    Op sch[64];
    int n = 0;
    for (int da = 0; da <= (s - 1 < L ? s - 1 : L); ++da) {
        int nb = (s - 1 < L - da ? s - 1 : L - da) + 1;
        for (int db = 0; db < nb; db += G) {
            int cnt = nb - db < G ? nb - db : G;
            sch[n++] = Op{uint32_t((da + db) * NB), uint32_t(da * BM * KB), uint32_t(s * BM * KB + db * NB * KB),
                          uint32_t(cnt * NB)};
        }
    }
    run("schedule_s7_L7_nb64", sch, n, 20000, 0);
    return 0;
}

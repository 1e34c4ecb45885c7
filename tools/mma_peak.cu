// Microbenchmark (not part of the product): sustained tcgen05.mma kind::i8
// throughput on one B200 with operands resident in shared memory (no TMA, no
// epilogue). Measures (1) the dense INT8 tensor peak — the roofline
// denominator of the slice GEMM — with back-to-back M=128 N=256 K=32 MMAs,
// (2) the same for smaller N, (3) the slice-pair schedule of igemm<64> at
// s = 7, L = 7, and (4) the issue cost of a runtime (non-constant) MMA loop.
// MMAs are issued by a converged warp through elect.sync with compile-time
// descriptors, like the product kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include \
//        -I../paper_2511_13778_b200/csrc mma_peak.cu -o mma_peak && ./mma_peak
#include <cuda_runtime.h>
#include <stdio.h>

#include "tc.cuh"

using namespace adpb200;

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

struct Op {
    int col, a_off, b_off, n;
};

// 0: 2 x N=256; 1: 2 x N=128; 2: 2 x N=64; 3: the s=7 L=7 NB=64 schedule (11 MMAs, 34 pairs)
template <int CASE>
struct Ops;
template <>
struct Ops<0> {
    static constexpr int n = 2;
    static constexpr Op opv[2] = {{0, 0, 28672, 256}, {256, 4096, 28672, 256}};
    __host__ __device__ static constexpr Op op(int i) {
        constexpr Op t[2] = {{0, 0, 28672, 256}, {256, 4096, 28672, 256}};
        return t[i];
    }
};
template <>
struct Ops<1> {
    static constexpr int n = 2;
    static constexpr Op opv[2] = {{0, 0, 28672, 128}, {128, 4096, 28672, 128}};
    __host__ __device__ static constexpr Op op(int i) {
        constexpr Op t[2] = {{0, 0, 28672, 128}, {128, 4096, 28672, 128}};
        return t[i];
    }
};
template <>
struct Ops<2> {
    static constexpr int n = 2;
    static constexpr Op opv[2] = {{0, 0, 28672, 64}, {64, 4096, 28672, 64}};
    __host__ __device__ static constexpr Op op(int i) {
        constexpr Op t[2] = {{0, 0, 28672, 64}, {64, 4096, 28672, 64}};
        return t[i];
    }
};
template <>
struct Ops<3> {
    // (da, first db): N = 4 or fewer slices x 64
    static constexpr int n = 11;
    static constexpr Op opv[11] = {
        {0, 0, 28672, 256},          {256, 0, 28672 + 8192, 192},      {64, 4096, 28672, 256},
        {320, 4096, 28672 + 8192, 192}, {128, 8192, 28672, 256},       {384, 8192, 28672 + 8192, 128},
        {192, 12288, 28672, 256},    {448, 12288, 28672 + 8192, 64},   {256, 16384, 28672, 256},
        {320, 20480, 28672, 192},    {384, 24576, 28672, 128}};
    __host__ __device__ static constexpr Op op(int i) {
        constexpr Op t[11] = {
        {0, 0, 28672, 256},          {256, 0, 28672 + 8192, 192},      {64, 4096, 28672, 256},
        {320, 4096, 28672 + 8192, 192}, {128, 8192, 28672, 256},       {384, 8192, 28672 + 8192, 128},
        {192, 12288, 28672, 256},    {448, 12288, 28672 + 8192, 64},   {256, 16384, 28672, 256},
        {320, 20480, 28672, 192},    {384, 24576, 28672, 128}};
        return t[i];
    }
};

// Shared-memory write pressure next to the MMAs (tma_chunk > 0): warp 2 streams
// a global buffer into a separate smem ring with cp.async.bulk (the TMA's
// async-proxy write path, like the GEMM's producer) while warp 0 issues MMAs;
// the bytes it moved are reported through wbytes.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
                 : "memory");
}

template <int CASE>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, int runtime_ops, const Op* rt,
                                                   unsigned long long* cycles, int tma_chunk = 0,
                                                   const uint8_t* gsrc = nullptr, unsigned long long* wbytes = nullptr) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t wbar[3];
    __shared__ volatile int stop_flag;
    __shared__ Op sops[16];
    for (int i = threadIdx.x; i < 144 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 7);
    if (threadIdx.x < Ops<CASE>::n) sops[threadIdx.x] = rt[threadIdx.x];
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar, 1);
        for (int i = 0; i < 3; ++i) tc::mbar_init(&wbar[i], 1);
        stop_flag = 0;
        tc::fence_barrier_init();
    }
    if (threadIdx.x / 32 == 1) tc::tmem_alloc(&tmem_slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x < 32) {
        const uint32_t base = tc::smem_u32(smem);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t st = base + uint32_t(it & 1) * 65536u;  // alternate two "stages"
            const uint64_t d0 = tc::smem_desc_sw32(st);
            if (elect_one()) {
                if (runtime_ops) {
                    for (int i = 0; i < Ops<CASE>::n; ++i) {
                        const Op o = sops[i];
                        tc::mma_i8(tmem + o.col, d0 + (o.a_off >> 4), d0 + (o.b_off >> 4), tc::idesc_i8(128, o.n),
                                   1u);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < Ops<CASE>::n; ++i)
                        tc::mma_i8(tmem + Ops<CASE>::op(i).col, d0 + (Ops<CASE>::op(i).a_off >> 4),
                                   d0 + (Ops<CASE>::op(i).b_off >> 4), tc::idesc_i8(128, Ops<CASE>::op(i).n), 1u);
                }
            }
            __syncwarp();
        }
        if (elect_one()) tc::mma_commit(&bar);
        __syncwarp();
        tc::mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        if (threadIdx.x == 0) {
            cycles[blockIdx.x] = t1 - t0;
            stop_flag = 1;
        }
    } else if (threadIdx.x == 64 && tma_chunk > 0) {
        // three chunks in flight into [144 KiB, 144 KiB + 3 * tma_chunk)
        const uint32_t ring = tc::smem_u32(smem) + 144u * 1024u;
        unsigned long long moved = 0;
        uint32_t phase[3] = {0, 0, 0};
        const uint8_t* src = gsrc + size_t(blockIdx.x % 8) * (1u << 20);
        for (int i = 0; i < 3; ++i) {
            tc::mbar_expect_tx(&wbar[i], tma_chunk);
            bulk_g2s(ring + i * tma_chunk, src + i * tma_chunk, tma_chunk, tc::smem_u32(&wbar[i]));
        }
        for (int it = 0; !stop_flag; ++it) {
            const int i = it % 3;
            tc::mbar_wait(&wbar[i], phase[i]);
            phase[i] ^= 1;
            moved += tma_chunk;
            tc::mbar_expect_tx(&wbar[i], tma_chunk);
            bulk_g2s(ring + i * tma_chunk, src + ((it + 3) % 48) * tma_chunk, tma_chunk, tc::smem_u32(&wbar[i]));
        }
        for (int i = 0; i < 3; ++i) tc::mbar_wait(&wbar[i], phase[i]);
        wbytes[blockIdx.x] = moved;
    }
    __syncthreads();
    if (threadIdx.x / 32 == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, 512);
    }
}

template <int CASE>
static void run(const char* name, int iters, int runtime_ops, int tma_chunk = 0) {
    static uint8_t* gsrc = nullptr;
    static unsigned long long* wb = nullptr;
    if (!gsrc) {
        cudaMalloc(&gsrc, 8u << 20);
        cudaMemset(gsrc, 1, 8u << 20);
        cudaMalloc(&wb, 148 * 8);
    }
    Op* d;
    cudaMalloc(&d, sizeof(Op) * Ops<CASE>::n);
    cudaMemcpy(d, Ops<CASE>::opv, sizeof(Op) * Ops<CASE>::n, cudaMemcpyHostToDevice);
    unsigned long long* dcyc;
    cudaMalloc(&dcyc, 148 * 8);
    const int smem = 144 * 1024 + 3 * 16384 + 1024;
    cudaFuncSetAttribute(mma_loop<CASE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_loop<CASE><<<148, 128, smem>>>(100, runtime_ops, d, dcyc, tma_chunk, gsrc, wb);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_loop<CASE><<<148, 128, smem>>>(iters, runtime_ops, d, dcyc, tma_chunk, gsrc, wb);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc[148];
    cudaMemcpy(cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
    double macs = 0, ideal = 0;
    for (int i = 0; i < Ops<CASE>::n; ++i) {
        macs += 128.0 * Ops<CASE>::op(i).n * 32.0;
        ideal += Ops<CASE>::op(i).n / 2.0;
    }
    const double tops = 2.0 * macs * double(iters) * 148 / (ms * 1e-3) / 1e12;
    const double cpi = double(cyc[0]) / iters;
    unsigned long long wbh[148] = {};
    if (tma_chunk) cudaMemcpy(wbh, wb, sizeof(wbh), cudaMemcpyDeviceToHost);
    printf("{\"case\": \"%s\", \"err\": \"%s\", \"ms\": %.3f, \"int8_tops\": %.1f, \"cycles_per_iter\": %.1f, "
           "\"ideal_cycles_per_iter\": %.1f, \"efficiency\": %.3f, \"sm_clock_ghz\": %.3f, "
           "\"smem_write_B_per_clk\": %.1f}\n",
           name, cudaGetErrorString(err), ms, tops, cpi, ideal, ideal / cpi, double(cyc[0]) / (ms * 1e6),
           double(wbh[0]) / double(cyc[0]));
    cudaFree(d);
    cudaFree(dcyc);
}

int main(int argc, char** argv) {
    if (argc > 1) {  // sustained: ~4 s of back-to-back N=256 MMAs (power-capped steady state)
        run<0>("sustained_n256_static", 30000000, 0);
        return 0;
    }
    run<0>("peak_n256_static", 400000, 0);
    run<1>("n128_static", 400000, 0);
    run<2>("n64_static", 400000, 0);
    run<3>("schedule_s7_L7_nb64_static", 60000, 0);
    run<3>("schedule_s7_L7_nb64_runtime", 60000, 1);
    // the same schedule while a bulk-copy (TMA path) stream writes shared memory
    run<3>("schedule_s7_L7_nb64_with_bulk_writes_16k", 60000, 0, 16384);
    run<3>("schedule_s7_L7_nb64_with_bulk_writes_4k", 60000, 0, 4096);
    run<0>("n256_with_bulk_writes_16k", 400000, 0, 16384);
    return 0;
}

// Microbenchmark (not part of the product): latency of a dependent FP64 add
// chain on one thread, alone and fed from shared / global memory with the
// loads software-pipelined — the regime of the QR panel's reference-order sums.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(int n, double* out, unsigned long long* cyc, const double* g) {
    extern __shared__ double sm[];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 1e-3 * i;
    __syncthreads();
    if (threadIdx.x != 0) return;
    double acc = 0.0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, 1e-9);
    unsigned long long t1 = clock64();
    double acc2 = 0.0;
    for (int r = 0; r < 8192; r += 16) {
        double p[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) p[u] = __dmul_rn(sm[r + u], sm[r + u]);
#pragma unroll
        for (int u = 0; u < 16; ++u) acc2 = __dadd_rn(acc2, p[u]);
    }
    unsigned long long t2 = clock64();
    double acc3 = 0.0;
    for (int r = 0; r < 8192; r += 16) {
        double p[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) p[u] = __dmul_rn(g[r + u], g[r + u]);
#pragma unroll
        for (int u = 0; u < 16; ++u) acc3 = __dadd_rn(acc3, p[u]);
    }
    unsigned long long t3 = clock64();
    double acc4 = 0.0;
    for (int r = 0; r < 8192; r += 8) {
        double q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double d = __ddiv_rn(sm[r + u], 3.0);
            q[u] = __dmul_rn(d, d);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc4 = __dadd_rn(acc4, q[u]);
    }
    unsigned long long t4 = clock64();
    out[0] = acc + acc2 + acc3 + acc4;
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
}

int main() {
    double* out;
    double* g;
    unsigned long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&g, 8192 * 8);
    cudaMemset(g, 0, 8192 * 8);
    cudaMalloc(&cyc, 32);
    cudaFuncSetAttribute(chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const int n = 100000;
    chain<<<1, 256, 65536>>>(n, out, cyc, g);
    chain<<<1, 256, 65536>>>(n, out, cyc, g);
    unsigned long long h[4];
    cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("{\"dadd_chain_cycles_per_add\": %.2f, \"smem_fed_dot_cycles_per_elem\": %.2f, "
           "\"global_fed_dot_cycles_per_elem\": %.2f, \"ddiv_fed_sum_cycles_per_elem\": %.2f}\n",
           double(h[0]) / n, double(h[1]) / 8192, double(h[2]) / 8192, double(h[3]) / 8192);
    return 0;
}

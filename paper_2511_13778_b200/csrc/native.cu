// K6: the native FP64 fallback (native_gemm, proj/src/oracle.cpp:7-28).
//
// Every output is summed in ascending k with one rounding per multiply and
// one per add (sum = sum + a*b, no FMA — the reference build disables
// contraction, proj/CMakeLists.txt:16-18, and proj/tests/test_oracle.cpp:54-71
// pins it), then r = alpha*sum, and r = r + beta*c only when beta != 0. The
// result is therefore bitwise identical to the reference's fallback (NaN
// payloads aside: the GPU produces the canonical NaN).
//
// Register-tiled 64x64 CTA tiles, 4x4 outputs per thread, k staged through
// shared memory 16 at a time; the k loop is never split, so the summation
// order per output element is exactly the reference's.
#include "igemm.cuh"

namespace adpb200 {

namespace {

constexpr int kT = 64, kKT = 16;

__global__ void __launch_bounds__(256) native_kernel(LineView a, LineView b, double alpha, double beta,
                                                     const double* __restrict__ c_in, int64_t ldc_in,
                                                     double* __restrict__ c_out, int64_t ldc, const Plan* plan) {
    if (plan && plan->path != ADPB200_PATH_NATIVE) return;
    __shared__ double As[2][kKT][kT + 1];
    __shared__ double Bs[2][kKT][kT + 1];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t i0 = int64_t(blockIdx.x) * kT, j0 = int64_t(blockIdx.y) * kT;
    const int64_t K = a.len;

    auto load = [&](int buf, int64_t k0) {
        // A tile: 64 lines x 16 positions; B tile: 64 lines x 16 positions.
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int e = tid + q * 256;
            int li, kk;
            if (a.ls == 1) { li = e % kT; kk = e / kT; }
            else { kk = e % kKT; li = e / kKT; }
            int64_t gi = i0 + li, gk = k0 + kk;
            As[buf][kk][li] = (gi < a.lines && gk < K) ? a.ptr[gi * a.ls + gk * a.ps] : 0.0;
            int lj, kj;
            if (b.ls == 1) { lj = e % kT; kj = e / kT; }
            else { kj = e % kKT; lj = e / kKT; }
            int64_t gj = j0 + lj, gk2 = k0 + kj;
            Bs[buf][kj][lj] = (gj < b.lines && gk2 < K) ? b.ptr[gj * b.ls + gk2 * b.ps] : 0.0;
        }
    };

    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;

    const int64_t nk = (K + kKT - 1) / kKT;
    if (nk > 0) load(0, 0);
    __syncthreads();
    for (int64_t t = 0; t < nk; ++t) {
        const int buf = int(t & 1);
        if (t + 1 < nk) load(buf ^ 1, (t + 1) * kKT);
        const int kmax = (K - t * kKT) < kKT ? int(K - t * kKT) : kKT;
        for (int kk = 0; kk < kmax; ++kk) {  // ascending k, never reordered
            double av[4], bv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) av[r] = As[buf][kk][tx + 16 * r];
#pragma unroll
            for (int c = 0; c < 4; ++c) bv[c] = Bs[buf][kk][ty + 16 * c];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = __dadd_rn(acc[r][c], __dmul_rn(av[r], bv[c]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int64_t j = j0 + ty + 16 * c;
        if (j >= b.lines) continue;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t i = i0 + tx + 16 * r;
            if (i >= a.lines) continue;
            double v = __dmul_rn(alpha, acc[r][c]);
            if (beta != 0.0) v = __dadd_rn(v, __dmul_rn(beta, c_in[i + j * ldc_in]));
            c_out[i + j * ldc] = v;
        }
    }
}

}  // namespace

void launch_native(const LineView& a, const LineView& b, double alpha, double beta, const double* c_in,
                   int64_t ldc_in, double* c_out, int64_t ldc, const Plan* plan, cudaStream_t st, uint64_t* nlaunch) {
    if (a.lines == 0 || b.lines == 0) return;
    dim3 grid((unsigned)((a.lines + kT - 1) / kT), (unsigned)((b.lines + kT - 1) / kT));
    native_kernel<<<grid, 256, 0, st>>>(a, b, alpha, beta, c_in, ldc_in, c_out, ldc, plan);
    ++*nlaunch;
}

}  // namespace adpb200

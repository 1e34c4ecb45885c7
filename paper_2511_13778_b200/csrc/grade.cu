// Device grading tools: the double-double GEMM oracle and the error report.
//
// The reference grades a GEMM against exact_gemm (a superaccumulator,
// proj/src/oracle.cpp:55-75) on the CPU, which costs minutes at n >= 4096.
// The north star asks for "FP64-level error against a double-double oracle"
// at the headline sizes, so the GPU carries one:
//
//   dd_gemm_kernel   every output is Dot2 (Ogita, Rump & Oishi, "Accurate sum
//                    and dot product", SISC 2005): TwoProd via FMA, TwoSum of
//                    the running head, the low parts summed in a plain double;
//                    the result is as accurate as if computed in twice the
//                    working precision and then rounded:
//                      |ref - AB| <= eps |AB| + gamma_{2k}^2 (|A||B|)
//                    (eps = 2^-53). The same pass also sums (|A||B|)_ij, the
//                    denominator of the grading ratio (grading.cpp:108-123).
//   error_kernel     error_report (grading.cpp:67-90): componentwise relative
//                    errors |ref - c| / |ref| (entries with ref == 0 skipped and
//                    counted; diagonal entries compared against exact_diag when
//                    given, the Test-2 convention), plus the grading ratio
//                    |c - ref| / (2^-52 (|A||B|)_ij). Deterministic: fixed
//                    per-block partials, then one block folds them in order.
//
// Every FP64 operation is an explicitly rounded intrinsic (no contraction).
#include <math.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "igemm.cuh"

namespace adpb200 {

namespace {

constexpr int kT = 64, kKT = 16;

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
    s = __dadd_rn(a, b);
    const double z = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, z)), __dsub_rn(b, z));
}

// Dot2 per output over LineView operands (the native kernel's tiling, 4x4
// outputs per thread). out[i + j*ldo] = RN(head + tail), absab likewise.
__global__ void __launch_bounds__(256) dd_gemm_kernel(LineView a, LineView b, double* __restrict__ out,
                                                      double* __restrict__ absab, int64_t ldo) {
    __shared__ double As[2][kKT][kT + 1];
    __shared__ double Bs[2][kKT][kT + 1];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t i0 = int64_t(blockIdx.x) * kT, j0 = int64_t(blockIdx.y) * kT;
    const int64_t K = a.len;

    auto load = [&](int buf, int64_t k0) {
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

    double hi[4][4], lo[4][4], ab[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) hi[r][c] = lo[r][c] = ab[r][c] = 0.0;

    const int64_t nk = (K + kKT - 1) / kKT;
    if (nk > 0) load(0, 0);
    __syncthreads();
    for (int64_t t = 0; t < nk; ++t) {
        const int buf = int(t & 1);
        if (t + 1 < nk) load(buf ^ 1, (t + 1) * kKT);
#pragma unroll 4
        for (int kk = 0; kk < kKT; ++kk) {  // zero padding past K adds exact zeros
            double av[4], bv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) av[r] = As[buf][kk][tx + 16 * r];
#pragma unroll
            for (int c = 0; c < 4; ++c) bv[c] = Bs[buf][kk][ty + 16 * c];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const double p = __dmul_rn(av[r], bv[c]);
                    const double pe = __fma_rn(av[r], bv[c], -p);  // exact: p + pe = a*b
                    double s, se;
                    two_sum(hi[r][c], p, s, se);
                    hi[r][c] = s;
                    lo[r][c] = __dadd_rn(lo[r][c], __dadd_rn(se, pe));
                    ab[r][c] = __fma_rn(fabs(av[r]), fabs(bv[c]), ab[r][c]);
                }
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
            out[i + j * ldo] = __dadd_rn(hi[r][c], lo[r][c]);
            if (absab) absab[i + j * ldo] = ab[r][c];
        }
    }
}

constexpr int kErrBlocks = 1184;  // 8 x 148 SMs
constexpr int kErrThreads = 256;

// Partials per block: [max_rel, sum_rel, counted, skipped, max_ratio, sum_ratio, ratio_counted, pad]
__global__ void __launch_bounds__(kErrThreads) error_kernel(const double* __restrict__ c, const double* __restrict__ ref,
                                                            const double* __restrict__ absab, int64_t rows,
                                                            int64_t cols, double exact_diag, int use_diag,
                                                            double* __restrict__ partial) {
    double mx = 0.0, sum = 0.0, cnt = 0.0, skip = 0.0, rmx = 0.0, rsum = 0.0, rcnt = 0.0;
    const int64_t total = rows * cols;
    for (int64_t e = int64_t(blockIdx.x) * kErrThreads + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * kErrThreads) {
        const int64_t i = e / cols, j = e - i * cols;
        const double r = (use_diag && i == j) ? exact_diag : ref[e];
        const double v = c[e];
        if (r == 0.0) {
            skip += 1.0;
        } else {
            const double err = __ddiv_rn(fabs(__dsub_rn(r, v)), fabs(r));
            mx = fmax(mx, err);  // std::max(max_err, e) keeps max_err when e is NaN
            sum = __dadd_rn(sum, err);
            cnt += 1.0;
        }
        if (absab) {
            const double den = __dmul_rn(0x1p-52, absab[e]);
            if (den != 0.0) {
                const double g = __ddiv_rn(fabs(__dsub_rn(v, ref[e])), den);
                rmx = fmax(rmx, g);
                rsum = __dadd_rn(rsum, g);
                rcnt += 1.0;
            }
        }
    }
    __shared__ double red[7][kErrThreads];
    red[0][threadIdx.x] = mx;
    red[1][threadIdx.x] = sum;
    red[2][threadIdx.x] = cnt;
    red[3][threadIdx.x] = skip;
    red[4][threadIdx.x] = rmx;
    red[5][threadIdx.x] = rsum;
    red[6][threadIdx.x] = rcnt;
    __syncthreads();
    for (int w = kErrThreads / 2; w > 0; w /= 2) {
        if (threadIdx.x < w) {
            red[0][threadIdx.x] = fmax(red[0][threadIdx.x], red[0][threadIdx.x + w]);
            red[4][threadIdx.x] = fmax(red[4][threadIdx.x], red[4][threadIdx.x + w]);
#pragma unroll
            for (int f = 1; f < 7; ++f)
                if (f != 4) red[f][threadIdx.x] = __dadd_rn(red[f][threadIdx.x], red[f][threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x < 7) partial[blockIdx.x * 8 + threadIdx.x] = red[threadIdx.x][0];
}

// out[0..6] = max_rel, avg_rel, counted, skipped, max_ratio, avg_ratio, ratio_counted
__global__ void error_fold_kernel(const double* __restrict__ partial, int nblocks, double* __restrict__ out) {
    if (threadIdx.x != 0) return;
    double mx = 0.0, sum = 0.0, cnt = 0.0, skip = 0.0, rmx = 0.0, rsum = 0.0, rcnt = 0.0;
    for (int b = 0; b < nblocks; ++b) {
        const double* p = partial + b * 8;
        mx = fmax(mx, p[0]);
        sum = __dadd_rn(sum, p[1]);
        cnt = __dadd_rn(cnt, p[2]);
        skip = __dadd_rn(skip, p[3]);
        rmx = fmax(rmx, p[4]);
        rsum = __dadd_rn(rsum, p[5]);
        rcnt = __dadd_rn(rcnt, p[6]);
    }
    out[0] = mx;
    out[1] = cnt > 0.0 ? __ddiv_rn(sum, cnt) : 0.0;
    out[2] = cnt;
    out[3] = skip;
    out[4] = rmx;
    out[5] = rcnt > 0.0 ? __ddiv_rn(rsum, rcnt) : 0.0;
    out[6] = rcnt;
}

}  // namespace

void launch_dd_gemm(const LineView& a, const LineView& b, double* out, double* absab, int64_t ldo, cudaStream_t st,
                    uint64_t* nlaunch) {
    if (a.lines == 0 || b.lines == 0) return;
    dim3 grid((unsigned)((a.lines + kT - 1) / kT), (unsigned)((b.lines + kT - 1) / kT));
    dd_gemm_kernel<<<grid, 256, 0, st>>>(a, b, out, absab, ldo);
    ++*nlaunch;
}

size_t error_partial_bytes() { return size_t(kErrBlocks) * 8 * sizeof(double); }

void launch_error_report(const double* c, const double* ref, const double* absab, int64_t rows, int64_t cols,
                         double exact_diag, int use_diag, double* partial, double* out, cudaStream_t st,
                         uint64_t* nlaunch) {
    const int64_t total = rows * cols;
    int blocks = (int)((total + kErrThreads - 1) / kErrThreads);
    if (blocks > kErrBlocks) blocks = kErrBlocks;
    if (blocks < 1) blocks = 1;
    error_kernel<<<blocks, kErrThreads, 0, st>>>(c, ref, absab, rows, cols, exact_diag, use_diag, partial);
    error_fold_kernel<<<1, 32, 0, st>>>(partial, blocks, out);
    *nlaunch += 2;
}

}  // namespace adpb200

// ---- reproducible inputs on the device ---------------------------------------------
// xoshiro256++ with splitmix64 seeding (proj/include/ozadp/rng.hpp:11-54) and
// gen_uniform_rect (proj/src/grading.cpp:56-63): element e (row-major) is
// lo + (hi - lo) * u01 of the e-th draw. The state update of xoshiro256 is
// linear over GF(2), so the state after j*kRngChunk draws is J^j * s0 with
// J = T^kRngChunk, a 256 x 256 bit matrix built once by stepping the 256 basis
// states; every GPU thread then generates one chunk of kRngChunk draws. Same
// bits as the sequential generator.
namespace adpb200 {

namespace {

constexpr int64_t kRngChunk = 4096;

struct Xo {
    uint64_t s[4];
};

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

__host__ __device__ __forceinline__ uint64_t xo_next(Xo& r) {
    const uint64_t out = rotl64(r.s[0] + r.s[3], 23) + r.s[0];
    const uint64_t t = r.s[1] << 17;
    r.s[2] ^= r.s[0];
    r.s[3] ^= r.s[1];
    r.s[1] ^= r.s[2];
    r.s[0] ^= r.s[3];
    r.s[2] ^= t;
    r.s[3] = rotl64(r.s[3], 45);
    return out;
}

Xo xo_seed(uint64_t seed) {
    Xo r;
    uint64_t x = seed;
    for (auto& w : r.s) {
        x += 0x9e3779b97f4a7c15ULL;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        w = z ^ (z >> 31);
    }
    return r;
}

// J = T^kRngChunk as 256 column images: col[b] = J * e_b.
const std::vector<Xo>& jump_matrix() {
    static std::vector<Xo> cols;
    static std::once_flag once;
    std::call_once(once, [] {
        cols.resize(256);
        for (int b = 0; b < 256; ++b) {
            Xo r{};
            r.s[b / 64] = 1ull << (b % 64);
            for (int64_t i = 0; i < kRngChunk; ++i) xo_next(r);
            cols[b] = r;
        }
    });
    return cols;
}

Xo apply_jump(const std::vector<Xo>& J, const Xo& v) {
    Xo r{};
    for (int b = 0; b < 256; ++b)
        if ((v.s[b / 64] >> (b % 64)) & 1)
            for (int w = 0; w < 4; ++w) r.s[w] ^= J[b].s[w];
    return r;
}

__global__ void uniform_kernel(const Xo* __restrict__ starts, int64_t total, double lo, double hi,
                               double* __restrict__ out) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t e0 = c * kRngChunk;
    if (e0 >= total) return;
    Xo r = starts[c];
    const int64_t e1 = e0 + kRngChunk < total ? e0 + kRngChunk : total;
    const double w = __dsub_rn(hi, lo);
    for (int64_t e = e0; e < e1; ++e) {
        const double u = __dmul_rn(__dadd_rn(double(xo_next(r) >> 11), 0.5), 0x1p-53);
        out[e] = __dadd_rn(lo, __dmul_rn(w, u));
    }
}

__global__ void cyclic_kernel(const double* __restrict__ xl, const double* __restrict__ xr, int64_t n,
                              double* __restrict__ lhs, double* __restrict__ rhs) {
    const int64_t total = n * n;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / n, c = e - r * n;
        // lhs(k, i) = x_s 2^j_s and rhs(i, k) = x_s 2^-j_s with s = (i - k) mod n
        int64_t s = c - r;
        if (s < 0) s += n;
        lhs[e] = xl[s];
        int64_t s2 = r - c;  // rhs(r, c): i = r, k = c
        if (s2 < 0) s2 += n;
        rhs[e] = xr[s2];
    }
}

}  // namespace

int gen_uniform_device(int64_t rows, int64_t cols, uint64_t seed, double lo, double hi, double* out, cudaStream_t st,
                       uint64_t* nlaunch) {
    const int64_t total = rows * cols;
    if (total <= 0) return 0;
    const int64_t nch = (total + kRngChunk - 1) / kRngChunk;
    const std::vector<Xo>& J = jump_matrix();
    std::vector<Xo> starts(static_cast<size_t>(nch));
    starts[0] = xo_seed(seed);
    for (int64_t c = 1; c < nch; ++c) starts[size_t(c)] = apply_jump(J, starts[size_t(c - 1)]);
    Xo* d = nullptr;
    if (cudaMallocAsync(&d, size_t(nch) * sizeof(Xo), st) != cudaSuccess) return -1;
    if (cudaMemcpyAsync(d, starts.data(), size_t(nch) * sizeof(Xo), cudaMemcpyHostToDevice, st) != cudaSuccess)
        return -1;
    // the host vector must outlive the async copy
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    uniform_kernel<<<unsigned((nch + 127) / 128), 128, 0, st>>>(d, total, lo, hi, out);
    ++*nlaunch;
    cudaFreeAsync(d, st);
    return 0;
}

// gen_test2 (proj/src/grading.cpp:13-47): the x draws and exponents on the
// host (n values, sequential), the two n x n cyclic matrices on the device.
int gen_test2_device(int64_t n, int b, uint64_t seed, double* lhs, double* rhs, double* x_out, int32_t* j_out,
                     cudaStream_t st, uint64_t* nlaunch) {
    Xo r = xo_seed(seed);
    std::vector<double> x(static_cast<size_t>(n)), xl(static_cast<size_t>(n)), xr(static_cast<size_t>(n));
    const double delta = (2.0 * b) / double(n - 1);
    std::vector<int32_t> j(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) x[size_t(i)] = 1.0 + (double(xo_next(r) >> 11) + 0.5) * 0x1p-53;
    for (int64_t i = 0; i < n; ++i) j[size_t(i)] = b == 0 ? 0 : int(-b + llround(double(i) * delta));
    if (j.front() != -b || j.back() != b) return 1;
    for (int64_t i = 0; i < n; ++i) {
        xl[size_t(i)] = ldexp(x[size_t(i)], j[size_t(i)]);
        xr[size_t(i)] = ldexp(x[size_t(i)], -j[size_t(i)]);
    }
    if (x_out) memcpy(x_out, x.data(), size_t(n) * 8);
    if (j_out) memcpy(j_out, j.data(), size_t(n) * 4);
    double* d = nullptr;
    if (cudaMallocAsync(&d, size_t(2 * n) * 8, st) != cudaSuccess) return -1;
    if (cudaMemcpyAsync(d, xl.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(d + n, xr.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return -1;
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    cyclic_kernel<<<1184, 256, 0, st>>>(d, d + n, n, lhs, rhs);
    ++*nlaunch;
    cudaFreeAsync(d, st);
    return 0;
}

}  // namespace adpb200

// The reference's application caller: blocked Householder QR whose trailing
// updates run through the ADP GEMM (proj/src/qr.cpp:98-143, compact WY form,
// three adp_gemm per panel at :130-132).
//
// Device-resident and stream-ordered end to end. The level-2 panel work
// (make_reflector :26-47, apply_reflector :51-60, build_y :64-71, build_t
// :75-94) runs in ONE CTA per panel in the reference's exact operation order:
// every sum that the reference accumulates sequentially is accumulated
// sequentially by one thread (FP64 adds are not associative), with explicitly
// rounded intrinsics (the reference is built with -ffp-contract=off); only
// operations that are independent per element (the tail division, the
// per-column reflector applications, the z / T entries of one step) run in
// parallel. The three trailing-update products go through adpb200_adp_gemm
// (bitwise the reference's adp_gemm), so the factors, T blocks and traces are
// bitwise the reference's. materialize_q / qr_residual (:145-197) use the
// reference-order native GEMM and a sequential Frobenius sum.
#include <algorithm>
#include <vector>

#include "igemm.cuh"

namespace adpb200 {
namespace {

constexpr int kPanelThreads = 256;   // one CTA per panel; columns beyond 256 loop
constexpr size_t kPanelSmemMax = 192 * 1024;  // reflector column + squares in shared memory up to 12288 rows

// Sequential sums in the reference's order, with the loads software-pipelined
// (independent of the running sum) so one thread runs at FP64-add latency.
// sum_{r in [r0, r1)} x[r] * y[r] added onto `init` left to right.
__device__ __forceinline__ double seq_dot(double init, const double* __restrict__ x, const double* __restrict__ y,
                                          int64_t r0, int64_t r1) {
    // 16 products per chunk, the next chunk's loads issued before this chunk's adds:
    // ~32 loads in flight per thread hide the L2 latency of the column walk
    constexpr int kU = 16;
    double acc = init;
    int64_t r = r0;
    if (r + kU <= r1) {
        double xa[kU], ya[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            xa[u] = x[r + u];
            ya[u] = y[r + u];
        }
        for (; r + 2 * kU <= r1; r += kU) {
            double xb[kU], yb[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                xb[u] = x[r + kU + u];
                yb[u] = y[r + kU + u];
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) acc = __dadd_rn(acc, __dmul_rn(xa[u], ya[u]));
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                xa[u] = xb[u];
                ya[u] = yb[u];
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) acc = __dadd_rn(acc, __dmul_rn(xa[u], ya[u]));
        r += kU;
    }
    for (; r < r1; ++r) acc = __dadd_rn(acc, __dmul_rn(x[r], y[r]));
    return acc;
}

// ---- panel factorisation, one column step at a time across CTAs --------------------
// The panel f[p0:m, p0:p0+pw] is copied into P (column-major rows x pw). Column j's
// reflector is made by one CTA (its two sequential sums on two threads); then every
// later column of the panel is updated by its own CTA, which stages the reflector and
// the column in shared memory so that its one sequential dot runs at shared-memory
// latency. Every sum keeps the reference's order and rounding (make_reflector
// qr.cpp:26-47, apply_reflector :51-60); the parallelism is only across columns and
// across the element-independent divisions / updates.

__global__ void panel_load_kernel(const double* __restrict__ f, int64_t ld, int64_t p0, int64_t rows, int pw,
                                  double* __restrict__ P) {
    pdl_enter();
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * pw; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / pw, j = e - r * pw;
        P[j * rows + r] = f[(p0 + r) * ld + p0 + j];
    }
}

// make_reflector (qr.cpp:26-47) of panel column j (global `col`), whose values for
// rows [j, rows) are already in v; q2 is a rows-long scratch; tau[j] to global memory.
// Called by the whole CTA.
__device__ __forceinline__ void make_reflector_cta(double* __restrict__ col, double* v, double* q2, int64_t rows,
                                                   int j, double* __restrict__ tau) {
    const int tid = threadIdx.x, nth = blockDim.x;
    __shared__ double red_s[32];
    __shared__ double v0_s, beta_s, x0_s, tail_s;
    __shared__ int mode_s;
    __syncthreads();
    // column_norm's max (qr.cpp:15): exact and order-free, reduced in parallel
    double amax = 0.0;
    for (int64_t r = j + tid; r < rows; r += nth) {
        const double a = fabs(v[r]);
        amax = amax < a ? a : amax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double b = __shfl_xor_sync(0xffffffffu, amax, o);
        amax = amax < b ? b : amax;
    }
    if ((tid & 31) == 0) red_s[tid >> 5] = amax;
    __syncthreads();
    amax = red_s[0];
    for (int w = 1; w < (nth + 31) / 32; ++w) amax = amax < red_s[w] ? red_s[w] : amax;
    // the squares (f/amax)^2 of column_norm (qr.cpp:17-19) are element-independent:
    // divide in parallel (a division costs ~100 cycles on one thread), sum in order below
    if (amax != 0.0)
        for (int64_t r = j + tid; r < rows; r += nth) {
            const double q = __ddiv_rn(v[r], amax);
            q2[r] = __dmul_rn(q, q);
        }
    __syncthreads();
    // the two sequential sums run concurrently on two warps, each in reference order
    if (tid == 0) tail_s = seq_dot(0.0, v, v, j + 1, rows);  // tail_ss (qr.cpp:29)
    if (tid == 32 % nth) {
        double ss = 0.0;
        if (amax != 0.0) {
            int64_t r = j;
            for (; r + 16 <= rows; r += 16) {
                double b[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) b[u] = q2[r + u];
#pragma unroll
                for (int u = 0; u < 16; ++u) ss = __dadd_rn(ss, b[u]);
            }
            for (; r < rows; ++r) ss = __dadd_rn(ss, q2[r]);
        }
        beta_s = amax != 0.0 ? __dmul_rn(amax, __dsqrt_rn(ss)) : 0.0;
    }
    __syncthreads();
    if (tid == 0) {
        const double x0 = v[j], tail = tail_s;
        if (tail == 0.0) {
            mode_s = 0;
            if (x0 >= 0.0) {
                tau[j] = 0.0;
            } else {
                col[j] = -x0;
                tau[j] = 2.0;
            }
        } else {
            const double beta = beta_s;
            v0_s = x0 > 0.0 ? __ddiv_rn(-tail, __dadd_rn(x0, beta)) : __dsub_rn(x0, beta);
            x0_s = x0;
            mode_s = 1;
        }
    }
    __syncthreads();
    if (mode_s == 1) {
        const double v0 = v0_s;
        for (int64_t r = j + 1 + tid; r < rows; r += nth) col[r] = __ddiv_rn(v[r], v0);
        if (tid == 0) {
            col[j] = beta_s;
            tau[j] = __ddiv_rn(__dsub_rn(beta_s, x0_s), beta_s);
        }
    }
}

// make_reflector for panel column j as its own kernel (the first column of a panel, and
// the path for columns too long for shared memory). kSmem: the column lives in shared
// memory (a compile-time address space, so the sequential sums read it with LDS at
// shared-memory latency), else in the global scratch vglob.
template <bool kSmem>
__global__ void __launch_bounds__(kPanelThreads) reflector_kernel(double* __restrict__ P, int64_t rows, int j,
                                                                  double* __restrict__ tau,
                                                                  double* __restrict__ vglob) {
    pdl_enter();
    extern __shared__ double vsh[];
    double* v = kSmem ? vsh : vglob;
    double* col = P + int64_t(j) * rows;
    for (int64_t r = j + threadIdx.x; r < rows; r += blockDim.x) v[r] = col[r];
    make_reflector_cta(col, v, v + rows, rows, j, tau);
}

// apply_reflector (qr.cpp:51-60) of column j to panel column j + 1 + blockIdx.x
template <bool kStaged>
__global__ void __launch_bounds__(kPanelThreads) apply_kernel(double* __restrict__ P, int64_t rows, int j,
                                                              const double* __restrict__ tau) {
    pdl_enter();
    const double tj = tau[j];
    if (tj == 0.0) return;
    extern __shared__ double sh[];
    const int tid = threadIdx.x, nth = blockDim.x;
    const double* vcol = P + int64_t(j) * rows;
    double* dst = P + int64_t(j + 1 + blockIdx.x) * rows;
    if (kStaged) {
        for (int64_t r = j + tid; r < rows; r += nth) {
            sh[r] = vcol[r];
            sh[rows + r] = dst[r];
        }
        __syncthreads();
    }
    const double* sv = kStaged ? sh : vcol;
    const double* sd = kStaged ? sh + rows : dst;
    __shared__ double w_s, head_s;
    if (tid == 0) {
        const double dot = seq_dot(sd[j], sv, sd, j + 1, rows);
        const double w = __dmul_rn(tj, dot);
        w_s = w;
        head_s = __dsub_rn(sd[j], w);
    }
    __syncthreads();
    const double w = w_s;
    // element-independent update; with staging the new values go straight to P
    for (int64_t r = j + 1 + tid; r < rows; r += nth) dst[r] = __dsub_rn(sd[r], __dmul_rn(w, sv[r]));
    if (tid == 0) dst[j] = head_s;
}

// apply_reflector of column j to every later column, fused with the next step: CTA 0
// updates column j + 1 in shared memory as well and then makes its reflector
// (make_reflector of j + 1 needs exactly that column), so a panel takes one launch per
// column; the other CTAs' updates run meanwhile. Shared-memory (staged) path only.
__global__ void __launch_bounds__(kPanelThreads) apply_reflect_kernel(double* __restrict__ P, int64_t rows, int j,
                                                                      double* __restrict__ tau) {
    pdl_enter();
    const double tj = tau[j];
    const bool next = blockIdx.x == 0;  // this CTA owns column j + 1
    if (tj == 0.0 && !next) return;
    extern __shared__ double sh[];
    const int tid = threadIdx.x, nth = blockDim.x;
    const double* vcol = P + int64_t(j) * rows;
    double* dst = P + int64_t(j + 1 + blockIdx.x) * rows;
    double* sv = sh;
    double* sd = sh + rows;
    for (int64_t r = j + tid; r < rows; r += nth) {
        sv[r] = vcol[r];
        sd[r] = dst[r];
    }
    __syncthreads();
    if (tj != 0.0) {
        __shared__ double w_s, head_s;
        if (tid == 0) {
            const double dot = seq_dot(sd[j], sv, sd, j + 1, rows);
            const double w = __dmul_rn(tj, dot);
            w_s = w;
            head_s = __dsub_rn(sd[j], w);
        }
        __syncthreads();
        const double w = w_s;
        for (int64_t r = j + 1 + tid; r < rows; r += nth) {
            const double x = __dsub_rn(sd[r], __dmul_rn(w, sv[r]));
            dst[r] = x;
            if (next) sd[r] = x;
        }
        if (tid == 0) dst[j] = head_s;
    }
    if (!next) return;
    __syncthreads();
    // column j + 1's reflector from its updated values (sd), sv reused as the squares
    make_reflector_cta(dst, sd, sv, rows, j + 1, tau);
}

// write the panel back to f; build_y (qr.cpp:64-71)
__global__ void panel_store_kernel(const double* __restrict__ P, double* __restrict__ f, int64_t ld, int64_t p0,
                                   int64_t rows, int pw, double* __restrict__ y, double* __restrict__ yT) {
    pdl_enter();
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * pw; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / pw, j = e - r * pw;
        const double val = P[j * rows + r];
        f[(p0 + r) * ld + p0 + j] = val;
        const double yv = r == j ? 1.0 : (r > j ? val : 0.0);
        y[r * pw + j] = yv;
        yT[j * rows + r] = yv;
    }
}

// build_t's z (qr.cpp:79-85): z(i, j) = sum_{r >= j} y(r, i) y(r, j) for i < j, y(j, j) = 1
// first, then the tails; one CTA per j (column j staged in shared memory when it fits)
template <bool kStaged>
__global__ void __launch_bounds__(kPanelThreads) build_z_kernel(const double* __restrict__ P, int64_t rows, int pw,
                                                                double* __restrict__ z) {
    pdl_enter();
    extern __shared__ double sh[];
    const int j = blockIdx.x, tid = threadIdx.x, nth = blockDim.x;
    if (j == 0) return;
    if (kStaged) {
        for (int64_t r = j + tid; r < rows; r += nth) sh[r] = P[int64_t(j) * rows + r];
        __syncthreads();
    }
    const double* cj = kStaged ? sh : P + int64_t(j) * rows;
    for (int i = tid; i < j; i += nth) {
        const double* ci = P + int64_t(i) * rows;
        const double first = __dmul_rn(ci[j], 1.0);
        z[int64_t(i) * pw + j] = seq_dot(__dadd_rn(0.0, first), ci, cj, j + 1, rows);
    }
}

// build_t (qr.cpp:75-94): T(j,j) = tau_j, T(0:j, j) = -tau_j T(0:j,0:j) z(:, j); and T^T
template <bool kSmem>
__global__ void __launch_bounds__(kPanelThreads) build_t_kernel(const double* __restrict__ tau,
                                                                const double* __restrict__ z, int pw,
                                                                double* __restrict__ t, double* __restrict__ tT) {
    pdl_enter();
    // T (pw x pw) in shared memory when it fits, and z's column j staged per step: the
    // short sequential dots of the recursion then read LDS instead of global memory
    extern __shared__ double tsh[];
    double* T = kSmem ? tsh : t;
    double* zj = kSmem ? tsh + int64_t(pw) * pw : nullptr;
    const int tid = threadIdx.x, nth = blockDim.x;
    for (int64_t e = tid; e < int64_t(pw) * pw; e += nth) T[e] = 0.0;
    __syncthreads();
    for (int j = 0; j < pw; ++j) {
        if (kSmem) {
            for (int l = tid; l < j; l += nth) zj[l] = z[int64_t(l) * pw + j];
            __syncthreads();
        }
        if (tid == 0) T[j * pw + j] = tau[j];
        for (int i = tid; i < j; i += nth) {
            double dot = 0.0;
            for (int l = i; l < j; ++l)
                dot = __dadd_rn(dot, __dmul_rn(T[i * pw + l], kSmem ? zj[l] : z[int64_t(l) * pw + j]));
            T[i * pw + j] = __dmul_rn(-tau[j], dot);
        }
        __syncthreads();
    }
    for (int64_t e = tid; e < int64_t(pw) * pw; e += nth) {
        const int64_t i = e / pw, jj = e - i * pw;
        tT[jj * pw + i] = T[e];
        if (kSmem) t[e] = T[e];
    }
}

// dst (rows x cols, leading dimension ldd) = src (leading dimension lds)
__global__ void copy_block_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst, int64_t ldd,
                                  int64_t rows, int64_t cols) {
    pdl_enter();
    const int64_t total = rows * cols;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / cols, c = e - r * cols;
        dst[r * ldd + c] = src[r * lds + c];
    }
}

// dst (cols x rows) = transpose of src (rows x cols), both row-major compact
__global__ void transpose_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t rows, int64_t cols) {
    const int64_t total = rows * cols;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / cols, c = e - r * cols;
        dst[c * rows + r] = src[e];
    }
}

// build_y from the factors (materialize_q): y (rows x pw) unit lower trapezoid
__global__ void build_y_kernel(const double* __restrict__ fac, int64_t ld, int64_t m, int64_t p0, int pw,
                               double* __restrict__ y, double* __restrict__ yT) {
    const int64_t rows = m - p0;
    const int64_t total = rows * pw;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / pw, j = e - r * pw;
        const double v = r == j ? 1.0 : (r > j ? fac[(p0 + r) * ld + p0 + j] : 0.0);
        y[e] = v;
        yT[j * rows + r] = v;
    }
}

__global__ void eye_kernel(double* __restrict__ q, int64_t m, int64_t n) {
    const int64_t total = m * n;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e / n, j = e - i * n;
        q[e] = i == j ? 1.0 : 0.0;
    }
}

// upper_r (qr.cpp:175-181)
__global__ void upper_r_kernel(const double* __restrict__ fac, int64_t ld, int64_t n, double* __restrict__ r) {
    const int64_t total = n * n;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e / n, j = e - i * n;
        r[e] = j >= i ? fac[i * ld + j] : 0.0;
    }
}

// diff = a - b (elementwise); with b == nullptr, gram(i,i) -= 1 on a square matrix in place
__global__ void sub_kernel(double* __restrict__ a, const double* __restrict__ b, int64_t total, int64_t n_diag) {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        if (b) a[e] = __dsub_rn(a[e], b[e]);
        else if (e / n_diag == e % n_diag) a[e] = __dsub_rn(a[e], 1.0);
    }
}

// frobenius_norm (matrix.hpp:65-69): ONE sequential sum, like the reference.
// out[0] = ||d|| / ||a|| (||d|| when ||a|| == 0), out[1] = ||g||
__global__ void qr_norms_kernel(const double* __restrict__ d, const double* __restrict__ a, const double* __restrict__ g,
                                int64_t nda, int64_t ng, double* __restrict__ out) {
    auto frob = [](const double* x, int64_t cnt) {
        double s = 0.0;
        for (int64_t i = 0; i < cnt; ++i) s = __dadd_rn(s, __dmul_rn(x[i], x[i]));
        return __dsqrt_rn(s);
    };
    if (threadIdx.x == 0) {
        const double dn = frob(d, nda), an = frob(a, nda);
        out[0] = an == 0.0 ? dn : __ddiv_rn(dn, an);
    } else if (threadIdx.x == 32) {
        out[1] = frob(g, ng);
    }
}

unsigned grid_for(int64_t total) {
    int64_t b = (total + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, int64_t(num_sms()) * 16));
}

struct DevBuf {
    void* p = nullptr;
    cudaStream_t st;
    explicit DevBuf(cudaStream_t s) : st(s) {}
    double* alloc(size_t count) {
        if (cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(double), st) != cudaSuccess) p = nullptr;
        return static_cast<double*>(p);
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

}  // namespace

// ---- host orchestration (called from api.cu's C ABI) ------------------------------
int qr_geqrf(adpb200_handle h, int64_t m, int64_t n, int64_t panel, double* f, double* t_blocks, adpb200_trace* traces,
             const adpb200_options* opt, cudaStream_t st, uint64_t* nl) {
    const int64_t pwmax = std::min(panel, n);
    DevBuf bP(st), by(st), byT(st), bt(st), btT(st), bas(st), bw1(st), bw2(st), bup(st);
    double* P = bP.alloc(size_t(m) * pwmax);
    double* y = by.alloc(size_t(m) * pwmax);
    double* yT = byT.alloc(size_t(m) * pwmax);
    double* t = bt.alloc(size_t(pwmax) * pwmax);
    double* tT = btT.alloc(size_t(pwmax) * pwmax);
    double* as = bas.alloc(size_t(m) * (n - pwmax));
    double* w1 = bw1.alloc(size_t(pwmax) * (n - pwmax));
    double* w2 = bw2.alloc(size_t(pwmax) * (n - pwmax));
    double* up = bup.alloc(size_t(m) * (n - pwmax));
    if (!P || !y || !yT || !t || !tT || !as || !w1 || !w2 || !up) return 2;
    DevBuf bvg(st), btau(st), bz(st);
    double* vg = nullptr;
    if (2 * size_t(m) * sizeof(double) > kPanelSmemMax) {
        vg = bvg.alloc(2 * size_t(m));
        if (!vg) return 2;
    }
    double* tau = btau.alloc(size_t(pwmax));
    double* z = bz.alloc(size_t(pwmax) * pwmax);
    if (!tau || !z) return 2;
    static bool attr = [] {
        cudaFuncSetAttribute(reflector_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPanelSmemMax));
        cudaFuncSetAttribute(apply_reflect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPanelSmemMax));
        cudaFuncSetAttribute(build_z_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPanelSmemMax));
        cudaFuncSetAttribute(build_t_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPanelSmemMax));
        return true;
    }();
    (void)attr;
    int64_t p = 0;
    for (int64_t p0 = 0; p0 < n; p0 += panel, ++p) {
        const int pw = (int)std::min(panel, n - p0);
        const int64_t rows = m - p0, nt = n - p0 - pw;
        const int threads = kPanelThreads;
        // the reflector column (and, for the updates, the target column) in shared
        // memory when it fits: sequential sums at shared-memory latency
        const size_t vbytes = 2 * size_t(rows) * sizeof(double);
        const bool vsmem = vbytes <= kPanelSmemMax;
        launch_chain(panel_load_kernel, dim3(grid_for(rows * pw)), dim3(256), 0, st, f, n, p0, rows, pw, P);
        ++*nl;
        if (vsmem) {
            // one launch per column: update the later columns, make the next reflector
            launch_chain(reflector_kernel<true>, dim3(1), dim3(threads), vbytes, st, P, rows, 0, tau, nullptr);
            ++*nl;
            for (int j = 0; j + 1 < pw; ++j) {
                launch_chain(apply_reflect_kernel, dim3(unsigned(pw - j - 1)), dim3(threads), vbytes, st, P, rows, j, tau);
                ++*nl;
            }
        } else {
            for (int j = 0; j < pw; ++j) {
                launch_chain(reflector_kernel<false>, dim3(1), dim3(threads), 0, st, P, rows, j, tau, vg);
                ++*nl;
                if (j + 1 < pw) {
                    launch_chain(apply_kernel<false>, dim3(unsigned(pw - j - 1)), dim3(threads), 0, st, P, rows, j, tau);
                    ++*nl;
                }
            }
        }
        launch_chain(panel_store_kernel, dim3(grid_for(rows * pw)), dim3(256), 0, st, P, f, n, p0, rows, pw, y, yT);
        if (vsmem) launch_chain(build_z_kernel<true>, dim3(unsigned(pw)), dim3(threads), vbytes / 2, st, P, rows, pw, z);
        else launch_chain(build_z_kernel<false>, dim3(unsigned(pw)), dim3(threads), 0, st, P, rows, pw, z);
        const size_t tbytes = (size_t(pw) * pw + pw) * sizeof(double);
        if (tbytes <= kPanelSmemMax) launch_chain(build_t_kernel<true>, dim3(1), dim3(threads), tbytes, st, tau, z, pw, t, tT);
        else launch_chain(build_t_kernel<false>, dim3(1), dim3(threads), 0, st, tau, z, pw, t, tT);
        *nl += 3;
        launch_chain(copy_block_kernel, dim3(grid_for(int64_t(pw) * pw)), dim3(256), 0, st, t, pw, t_blocks + p * panel * panel, pw, pw, pw);
        ++*nl;
        if (nt > 0) {
            launch_chain(copy_block_kernel, dim3(grid_for(rows * nt)), dim3(256), 0, st, f + p0 * n + p0 + pw, n, as, nt, rows, nt);
            ++*nl;
        }
        // A_s -= Y T^T Y^T A_s, all three products dispatched (qr.cpp:127-132)
        int rc = adpb200_adp_gemm(h, pw, nt, rows, 1.0, yT, as, 0.0, nullptr, w1, opt, traces + 3 * p, st);
        if (!rc) rc = adpb200_adp_gemm(h, pw, nt, pw, 1.0, tT, w1, 0.0, nullptr, w2, opt, traces + 3 * p + 1, st);
        if (!rc) rc = adpb200_adp_gemm(h, rows, nt, pw, -1.0, y, w2, 1.0, as, up, opt, traces + 3 * p + 2, st);
        if (rc) return rc;
        if (nt > 0) {
            launch_chain(copy_block_kernel, dim3(grid_for(rows * nt)), dim3(256), 0, st, up, nt, f + p0 * n + p0 + pw, n, rows, nt);
            ++*nl;
        }
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int qr_materialize_q(adpb200_handle h, int64_t m, int64_t n, int64_t panel, const double* fac, const double* t_blocks,
                     double* q, cudaStream_t st, uint64_t* nl) {
    const int64_t pwmax = std::min(panel, n);
    DevBuf by(st), byT(st), bqs(st), bx1(st), bx2(st), bup(st);
    double* y = by.alloc(size_t(m) * pwmax);
    double* yT = byT.alloc(size_t(m) * pwmax);
    double* qs = bqs.alloc(size_t(m) * n);
    double* x1 = bx1.alloc(size_t(pwmax) * n);
    double* x2 = bx2.alloc(size_t(pwmax) * n);
    double* up = bup.alloc(size_t(m) * n);
    if (!y || !yT || !qs || !x1 || !x2 || !up) return 2;
    eye_kernel<<<grid_for(m * n), 256, 0, st>>>(q, m, n);
    ++*nl;
    const int64_t panels = (n + panel - 1) / panel;
    // Q = (I - Y_1 T_1 Y_1^T) ... (I - Y_K T_K Y_K^T) applied to thin I, rightmost first (qr.cpp:145-173)
    for (int64_t p = panels - 1; p >= 0; --p) {
        const int64_t p0 = p * panel;
        const int pw = (int)std::min(panel, n - p0);
        const int64_t rows = m - p0;
        build_y_kernel<<<grid_for(rows * pw), 256, 0, st>>>(fac, n, m, p0, pw, y, yT);
        copy_block_kernel<<<grid_for(rows * n), 256, 0, st>>>(q + p0 * n, n, qs, n, rows, n);
        *nl += 2;
        int rc = adpb200_native_gemm(h, yT, qs, pw, n, rows, 1.0, 0.0, nullptr, x1, st);
        if (!rc) {
            copy_block_kernel<<<grid_for(int64_t(pw) * pw), 256, 0, st>>>(t_blocks + p * panel * panel, pw, up, pw, pw,
                                                                         pw);
            ++*nl;
            rc = adpb200_native_gemm(h, up, x1, pw, n, pw, 1.0, 0.0, nullptr, x2, st);
        }
        if (!rc) rc = adpb200_native_gemm(h, y, x2, rows, n, pw, -1.0, 1.0, qs, up, st);
        if (rc) return rc;
        copy_block_kernel<<<grid_for(rows * n), 256, 0, st>>>(up, n, q + p0 * n, n, rows, n);
        ++*nl;
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int qr_residual(adpb200_handle h, int64_t m, int64_t n, int64_t panel, const double* a0, const double* fac,
                const double* t_blocks, double* out, cudaStream_t st, uint64_t* nl) {
    DevBuf bq(st), bqT(st), br(st), bd(st), bg(st);
    double* q = bq.alloc(size_t(m) * n);
    double* qT = bqT.alloc(size_t(m) * n);
    double* r = br.alloc(size_t(n) * n);
    double* d = bd.alloc(size_t(m) * n);
    double* g = bg.alloc(size_t(n) * n);
    if (!q || !qT || !r || !d || !g) return 2;
    int rc = qr_materialize_q(h, m, n, panel, fac, t_blocks, q, st, nl);
    if (rc) return rc;
    upper_r_kernel<<<grid_for(n * n), 256, 0, st>>>(fac, n, n, r);
    ++*nl;
    rc = adpb200_native_gemm(h, q, r, m, n, n, 1.0, 0.0, nullptr, d, st);  // prod = Q R
    if (rc) return rc;
    // diff = a0 - prod: d := a0 - d, computed as a copy of a0 minus prod
    copy_block_kernel<<<grid_for(m * n), 256, 0, st>>>(a0, n, qT, n, m, n);
    sub_kernel<<<grid_for(m * n), 256, 0, st>>>(qT, d, m * n, 0);
    *nl += 2;
    double* diff = qT;
    // gram = Q^T Q - I (the transpose goes into d, no longer needed)
    transpose_kernel<<<grid_for(m * n), 256, 0, st>>>(q, d, m, n);
    ++*nl;
    rc = adpb200_native_gemm(h, d, q, n, n, m, 1.0, 0.0, nullptr, g, st);
    if (rc) return rc;
    sub_kernel<<<grid_for(n * n), 256, 0, st>>>(g, nullptr, n * n, n);
    qr_norms_kernel<<<1, 64, 0, st>>>(diff, a0, g, m * n, n * n, out);
    *nl += 2;
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace adpb200

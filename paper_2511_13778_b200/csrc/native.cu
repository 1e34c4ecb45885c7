// K6: the native FP64 fallback (native_gemm, proj/src/oracle.cpp:7-28), two flavours.
//
// ADPB200_FALLBACK_REFERENCE (default) — bitwise the reference:
//   every output is summed in ascending k with one rounding per multiply and
//   one per add (sum = sum + a*b, no FMA — the reference build disables
//   contraction, proj/CMakeLists.txt:16-18, and proj/tests/test_oracle.cpp:54-71
//   pins it), then r = alpha*sum, and r = r + beta*c only when beta != 0
//   (NaN payloads aside: the GPU produces the canonical NaN). SIMT FP64:
//   64x64 CTA tiles, 4x4 outputs per thread, k staged through shared memory
//   16 at a time; the k loop is never split, so the summation order per
//   output element is exactly the reference's.
//
// ADPB200_FALLBACK_FAST — the FP64 tensor cores (DMMA, mma.sync m8n8k4.f64):
//   128x128 CTA tiles, 8 warps of 64x32, k staged 16 at a time through a
//   3-deep cp.async ring; fused multiply-adds in ascending k within each
//   output, so |C - AB| <= gamma_k |A||B| (+ the alpha/beta roundings) but not
//   the reference's bits. Opt-in (adpb200_options.fallback).
//
// Both kernels are persistent (grid = resident CTAs, tiles strided over it), so
// when the device plan says "emulated" the predicated launch costs one small
// wave that reads the plan and exits, not a full grid of tiles.
#include "igemm.cuh"
#include "tc.cuh"

namespace adpb200 {

namespace {

// ---- reference order (SIMT) ---------------------------------------------------------
// 128 x 128 CTA tiles, 16 x 16 threads with 8 x 8 outputs each (rows tx + 16 r, columns
// ty + 16 c): per k, 8 + 8 shared-memory reads feed 64 multiply-add pairs, so the FP64
// pipe (one DMUL and one DADD per term, no FMA), not shared memory, bounds the loop.
// k is staged 16 at a time through a 2-deep cp.async ring (zero-filled out of range);
// a full stage runs fully unrolled, the ragged last one term by term — always
// ascending k.
constexpr int kT = 128, kKT = 16, kTP = kT + 1;
constexpr size_t kNativeSmem = size_t(2) * 2 * kKT * kTP * sizeof(double);

__device__ __forceinline__ void cp_async8z(uint32_t dst, const double* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0));
}

template <bool kPeer>
__global__ void __launch_bounds__(256, 1) native_kernel(LineView a, LineView b, double alpha, double beta,
                                                        const double* __restrict__ c_in, int64_t ldc_in,
                                                        double* __restrict__ c_out, int64_t ldc, const Plan* plan,
                                                        PeerB pb) {
    pdl_enter();
    if (plan && plan->path != ADPB200_PATH_NATIVE) return;
    extern __shared__ __align__(16) double nsm[];
    // [buf][operand][k][line]
    auto tileA = [&](int buf) { return nsm + size_t(buf) * 2 * kKT * kTP; };
    auto tileB = [&](int buf) { return nsm + (size_t(buf) * 2 + 1) * kKT * kTP; };
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t K = a.len;
    const int64_t tiles_m = (a.lines + kT - 1) / kT, tiles_n = (b.lines + kT - 1) / kT;
    const int64_t nk = (K + kKT - 1) / kKT;

    for (int64_t tile = blockIdx.x; tile < tiles_m * tiles_n; tile += gridDim.x) {
        const int64_t i0 = (tile % tiles_m) * kT, j0 = (tile / tiles_m) * kT;
        auto load = [&](int buf, int64_t k0) {
            // 128 lines x 16 positions per operand, 8 elements per thread; lines innermost
            // when they are adjacent in memory, positions innermost otherwise
            const uint32_t sa = uint32_t(__cvta_generic_to_shared(tileA(buf)));
            const uint32_t sb = uint32_t(__cvta_generic_to_shared(tileB(buf)));
#pragma unroll
            for (int q = 0; q < kT * kKT / 256; ++q) {
                const int e = tid + q * 256;
                int li, kk;
                if (a.ls == 1) { li = e % kT; kk = e / kT; }
                else { kk = e % kKT; li = e / kKT; }
                const int64_t gi = i0 + li, gk = k0 + kk;
                const bool oka = gi < a.lines && gk < K;
                cp_async8z(sa + uint32_t(kk * kTP + li) * 8u, oka ? a.ptr + gi * a.ls + gk * a.ps : a.ptr, oka);
                int lj, kj;
                if (b.ls == 1) { lj = e % kT; kj = e / kT; }
                else { kj = e % kKT; lj = e / kKT; }
                const int64_t gj = j0 + lj, gk2 = k0 + kj;
                const bool okb = gj < b.lines && gk2 < K;
                const double* pbe = kPeer ? pb.at(gj, gk2, b.ls, b.ps) : b.ptr + gj * b.ls + gk2 * b.ps;
                cp_async8z(sb + uint32_t(kj * kTP + lj) * 8u, okb ? pbe : b.ptr, okb);
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };

        double acc[8][8];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;

        if (nk > 0) load(0, 0);
        for (int64_t t = 0; t < nk; ++t) {
            const int buf = int(t & 1);
            if (t + 1 < nk) {
                load(buf ^ 1, (t + 1) * kKT);
                asm volatile("cp.async.wait_group 1;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncthreads();  // stage t landed for every thread
            const double* As = tileA(buf);
            const double* Bs = tileB(buf);
            auto term = [&](int kk) {  // one k: ascending, never reordered
                double av[8], bv[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) av[r] = As[kk * kTP + tx + 16 * r];
#pragma unroll
                for (int c = 0; c < 8; ++c) bv[c] = Bs[kk * kTP + ty + 16 * c];
#pragma unroll
                for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[r][c] = __dadd_rn(acc[r][c], __dmul_rn(av[r], bv[c]));
            };
            const int kmax = (K - t * kKT) < kKT ? int(K - t * kKT) : kKT;
            if (kmax == kKT) {
#pragma unroll
                for (int kk = 0; kk < kKT; ++kk) term(kk);
            } else {
                for (int kk = 0; kk < kmax; ++kk) term(kk);
            }
            __syncthreads();  // stage t consumed before the copy into its buffer is issued
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int64_t j = j0 + ty + 16 * c;
            if (j >= b.lines) continue;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int64_t i = i0 + tx + 16 * r;
                if (i >= a.lines) continue;
                double v = __dmul_rn(alpha, acc[r][c]);
                if (beta != 0.0) v = __dadd_rn(v, __dmul_rn(beta, c_in[i + j * ldc_in]));
                c_out[i + j * ldc] = v;
            }
        }
    }
}

// ---- fast flavour: DMMA ---------------------------------------------------------------
constexpr int kDT = 128;       // CTA tile (lines of A) x (lines of B)
#ifndef ADPB200_DMMA_DK
#define ADPB200_DMMA_DK 16
#endif
#ifndef ADPB200_DMMA_STAGES
#define ADPB200_DMMA_STAGES 3
#endif
constexpr int kDK = ADPB200_DMMA_DK;  // k per stage
constexpr int kDStages = ADPB200_DMMA_STAGES;
constexpr int kPadL = kDT + 4;  // [k][line] rows: 132 doubles (== 4 mod 16: conflict-free fragment reads)
constexpr int kPadK = kDK + 4;  // [line][k] rows: kDK + 4 doubles (== 4 mod 16)
constexpr int kOpDoubles = (kDK * kPadL > kDT * kPadK) ? kDK * kPadL : kDT * kPadK;  // one operand, one stage
#ifndef ADPB200_DMMA_WARPS
#define ADPB200_DMMA_WARPS 8
#endif
constexpr int kDmmaWarps = ADPB200_DMMA_WARPS;
constexpr int kGroupTiles = 8;  // raster: CTA tiles along m per group (B tiles stay in L2)
constexpr size_t kDmmaSmem = size_t(kDStages) * 2 * kOpDoubles * sizeof(double);

__device__ __forceinline__ void cp_async8(uint32_t dst, const double* src, bool valid) {
    // src-size 0 zero-fills (out-of-range rows / k)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// One operand's tile (128 lines x 16 k) of one stage: `line_major` layout S[k][line]
// when the lines are contiguous in memory (ls == 1), else S[line][k].
template <bool kLineMajor, int kThreads, bool kPeer = false>
struct OpTile {
    static constexpr bool line_major = kLineMajor;
    const double* ptr;
    int64_t lines, len, ls, ps;
    PeerB pb;  // kPeer: element (line, k) in the ranks' slabs
    __device__ __forceinline__ void load(uint32_t sdst, int64_t l0, int64_t k0, int tid) const {
#pragma unroll
        for (int q = 0; q < kDT * kDK / kThreads; ++q) {
            const int e = tid + q * kThreads;
            int li, kk;
            uint32_t off;
            if (line_major) {
                li = e % kDT;
                kk = e / kDT;
                off = uint32_t(kk * kPadL + li);
            } else {
                kk = e % kDK;
                li = e / kDK;
                off = uint32_t(li * kPadK + kk);
            }
            const int64_t gl = l0 + li, gk = k0 + kk;
            const bool ok = gl < lines && gk < len;
            const double* e_ptr = kPeer ? pb.at(gl, gk, ls, ps) : ptr + gl * ls + gk * ps;
            cp_async8(sdst + off * 8u, ok ? e_ptr : ptr, ok);
        }
    }
    __device__ __forceinline__ double frag(const double* s, int line, int k) const {
        return line_major ? s[k * kPadL + line] : s[line * kPadK + k];
    }
};

// kWarps = 8: warp tiles of 64 x 32 (2 x 4 warps, 2 per scheduler); kWarps = 16:
// 32 x 32 (4 x 4 warps, 4 per scheduler, half the accumulator registers each).
template <bool kAL, bool kBL, int kWarps>
__global__ void __launch_bounds__(kWarps * 32, 1) dmma_kernel(LineView a, LineView b, double alpha, double beta,
                                                              const double* __restrict__ c_in, int64_t ldc_in,
                                                              double* __restrict__ c_out, int64_t ldc,
                                                              const Plan* plan) {
    pdl_enter();
    if (plan && plan->path != ADPB200_PATH_NATIVE) return;
    constexpr int kThreads = kWarps * 32;
    constexpr int kWarpsM = kWarps == 8 ? 2 : 4, kWarpsN = 4;
    constexpr int kMI = kDT / kWarpsM / 8, kNI = kDT / kWarpsN / 8;  // 8x8 fragments per warp
    extern __shared__ __align__(16) double dsm[];
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int wm = warp % kWarpsM, wn = warp / kWarpsM;  // warp tile: lines [8 kMI wm, +8 kMI) of A x [8 kNI wn, +8 kNI) of B
    const OpTile<kAL, kThreads> ta{a.ptr, a.lines, a.len, a.ls, a.ps, PeerB{}};
    const OpTile<kBL, kThreads> tb{b.ptr, b.lines, b.len, b.ls, b.ps, PeerB{}};
    const int64_t K = a.len;
    const int64_t tiles_m = (a.lines + kDT - 1) / kDT, tiles_n = (b.lines + kDT - 1) / kDT;
    const int64_t nk = (K + kDK - 1) / kDK;
    const uint32_t s0 = uint32_t(__cvta_generic_to_shared(dsm));
    auto sa = [&](int st) { return dsm + size_t(st) * 2 * kOpDoubles; };
    auto sb = [&](int st) { return dsm + size_t(st) * 2 * kOpDoubles + kOpDoubles; };
    auto sa_u = [&](int st) { return s0 + uint32_t(st) * 2u * kOpDoubles * 8u; };
    auto sb_u = [&](int st) { return s0 + (uint32_t(st) * 2u + 1u) * kOpDoubles * 8u; };
    const int fr = lane / 4, fk = lane % 4;  // fragment row (line) and k of this lane

    for (int64_t tile = blockIdx.x; tile < tiles_m * tiles_n; tile += gridDim.x) {
        // grouped raster: kGroupTiles m-tiles share each B tile while it is L2-resident
        const int64_t group = int64_t(kGroupTiles) * tiles_n;
        const int64_t first_m = (tile / group) * kGroupTiles;
        const int64_t gm = tiles_m - first_m < kGroupTiles ? tiles_m - first_m : kGroupTiles;
        const int64_t local = tile % group;
        const int64_t i0 = (first_m + local % gm) * kDT, j0 = (local / gm) * kDT;

        double acc[kMI][kNI][2];
#pragma unroll
        for (int mi = 0; mi < kMI; ++mi)
#pragma unroll
            for (int ni = 0; ni < kNI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

#pragma unroll
        for (int st = 0; st < kDStages - 1; ++st) {
            if (st < nk) {
                ta.load(sa_u(st), i0, int64_t(st) * kDK, tid);
                tb.load(sb_u(st), j0, int64_t(st) * kDK, tid);
            }
            cp_async_commit();
        }
        // stage indices tracked incrementally (no 64-bit modulo in the loop)
        int st_cur = 0, st_next = kDStages - 1;
        for (int64_t t = 0; t < nk; ++t) {
            cp_async_wait<kDStages - 2>();
            __syncthreads();  // stage t visible to all; stage t-1 fully consumed
            const int64_t tn = t + kDStages - 1;
            if (tn < nk) {
                ta.load(sa_u(st_next), i0, tn * kDK, tid);
                tb.load(sb_u(st_next), j0, tn * kDK, tid);
            }
            cp_async_commit();
            const double* As = sa(st_cur);
            const double* Bs = sb(st_cur);
            st_cur = st_cur + 1 == kDStages ? 0 : st_cur + 1;
            st_next = st_next + 1 == kDStages ? 0 : st_next + 1;
#pragma unroll
            for (int kk = 0; kk < kDK; kk += 4) {
                double af[kMI], bf[kNI];
#pragma unroll
                for (int mi = 0; mi < kMI; ++mi) af[mi] = ta.frag(As, wm * kMI * 8 + mi * 8 + fr, kk + fk);
#pragma unroll
                for (int ni = 0; ni < kNI; ++ni) bf[ni] = tb.frag(Bs, wn * kNI * 8 + ni * 8 + fr, kk + fk);
#pragma unroll
                for (int mi = 0; mi < kMI; ++mi)
#pragma unroll
                    for (int ni = 0; ni < kNI; ++ni) dmma(acc[mi][ni], af[mi], bf[ni]);
            }
        }
        cp_async_wait<0>();
        __syncthreads();  // the next tile's prologue overwrites stages 0..1
        // C fragment: line i = 8 mi + lane/4 of A, lines j = 8 ni + 2 (lane%4) + {0, 1} of B
#pragma unroll
        for (int ni = 0; ni < kNI; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t j = j0 + wn * kNI * 8 + ni * 8 + 2 * fk + h;
                if (j >= b.lines) continue;
#pragma unroll
                for (int mi = 0; mi < kMI; ++mi) {
                    const int64_t i = i0 + wm * kMI * 8 + mi * 8 + fr;
                    if (i >= a.lines) continue;
                    double v = __dmul_rn(alpha, acc[mi][ni][h]);
                    if (beta != 0.0) v = __dadd_rn(v, __dmul_rn(beta, c_in[i + j * ldc_in]));
                    c_out[i + j * ldc] = v;
                }
            }
    }
}

// ---- fast flavour, warp-specialised: producers and consumers on mbarriers ---------------
// 4 producer warps issue the cp.async copies of a stage and publish it on its `full`
// mbarrier once they have landed (wait_group + a release arrive); 8 consumer warps (the
// same 64 x 32 DMMA tiles) wait on `full`, compute, and release the stage on
// `empty`. No CTA-wide barrier in the k loop, so a scheduler's two consumer warps
// are never held back by the slowest warp of another scheduler, and the copy
// issue work leaves the consumer warps. Registers: setmaxnreg 56 / 224.
#ifndef ADPB200_DMMA_WS_STAGES
#define ADPB200_DMMA_WS_STAGES 4
#endif
constexpr int kWsStages = ADPB200_DMMA_WS_STAGES;
constexpr int kWsProd = 4, kWsCons = 8, kWsThreads = (kWsProd + kWsCons) * 32;
constexpr size_t kWsHeader = 128;  // 2 * kWsStages mbarriers
constexpr size_t kDmmaWsSmem = kWsHeader + size_t(kWsStages) * 2 * kOpDoubles * sizeof(double);
static_assert(2 * kWsStages * 8 <= kWsHeader && kWsStages >= 3, "mbarrier header; kLag = stages - 2 >= 1");

template <bool kAL, bool kBL, bool kPeer>
__global__ void __launch_bounds__(kWsThreads, 1) dmma_ws_kernel(LineView a, LineView b, double alpha, double beta,
                                                                const double* __restrict__ c_in, int64_t ldc_in,
                                                                double* __restrict__ c_out, int64_t ldc,
                                                                const Plan* plan, PeerB pb) {
    pdl_enter();
    if (plan && plan->path != ADPB200_PATH_NATIVE) return;
    extern __shared__ __align__(128) unsigned char dws[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dws);
    uint64_t* empty = full + kWsStages;
    double* ops = reinterpret_cast<double*>(dws + kWsHeader);
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    if (tid == 0) {
        for (int st = 0; st < kWsStages; ++st) {
            tc::mbar_init(&full[st], kWsProd * 32);
            tc::mbar_init(&empty[st], kWsCons);
        }
        tc::fence_barrier_init();
    }
    __syncthreads();
    const int64_t K = a.len;
    const int64_t tiles_m = (a.lines + kDT - 1) / kDT, tiles_n = (b.lines + kDT - 1) / kDT;
    const int64_t nk = (K + kDK - 1) / kDK;
    auto coords = [&](int64_t tile, int64_t& i0, int64_t& j0) {
        const int64_t group = int64_t(kGroupTiles) * tiles_n;
        const int64_t first_m = (tile / group) * kGroupTiles;
        const int64_t gm = tiles_m - first_m < kGroupTiles ? tiles_m - first_m : kGroupTiles;
        const int64_t local = tile % group;
        i0 = (first_m + local % gm) * kDT;
        j0 = (local / gm) * kDT;
    };
    if (warp < kWsProd) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::);
        const OpTile<kAL, kWsProd * 32> ta{a.ptr, a.lines, a.len, a.ls, a.ps, pb};
        const OpTile<kBL, kWsProd * 32, kPeer> tb{b.ptr, b.lines, b.len, b.ls, b.ps, pb};
        const uint32_t s0 = tc::smem_u32(ops);
        int st = 0;
        uint32_t ph = 0;
        // A stage is published kLag stages after its copies were issued: the thread waits
        // for that commit group (cp.async.wait_group) and arrives on `full` with release
        // semantics, so the consumers' acquire-wait orders their reads after the copies.
        // kLag + 1 stages stay in flight per producer thread (kLag < kWsStages).
        constexpr int kLag = kWsStages - 2;
        int sig = 0;         // next stage to publish
        int64_t owed = 0;    // issued, not yet published
        for (int64_t tile = blockIdx.x; tile < tiles_m * tiles_n; tile += gridDim.x) {
            int64_t i0, j0;
            coords(tile, i0, j0);
            for (int64_t t = 0; t < nk; ++t) {
                tc::mbar_wait(&empty[st], ph ^ 1);
                const uint32_t sa = s0 + uint32_t(st) * 2u * kOpDoubles * 8u;
                ta.load(sa, i0, t * kDK, tid);
                tb.load(sa + kOpDoubles * 8u, j0, t * kDK, tid);
                asm volatile("cp.async.commit_group;\n" ::: "memory");
                if (++owed > kLag) {
                    asm volatile("cp.async.wait_group %0;\n" ::"n"(kLag) : "memory");
                    tc::mbar_arrive(&full[sig]);
                    sig = sig + 1 == kWsStages ? 0 : sig + 1;
                    --owed;
                }
                if (++st == kWsStages) {
                    st = 0;
                    ph ^= 1;
                }
            }
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        for (; owed > 0; --owed) {
            tc::mbar_arrive(&full[sig]);
            sig = sig + 1 == kWsStages ? 0 : sig + 1;
        }
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::);
    const int cw = warp - kWsProd;
    const int wm = cw % 2, wn = cw / 2;  // warp tile: lines [64 wm, +64) of A x [32 wn, +32) of B
    const OpTile<kAL, kWsProd * 32> ta{a.ptr, a.lines, a.len, a.ls, a.ps, pb};
    const OpTile<kBL, kWsProd * 32, kPeer> tb{b.ptr, b.lines, b.len, b.ls, b.ps, pb};
    const int fr = lane / 4, fk = lane % 4;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t tile = blockIdx.x; tile < tiles_m * tiles_n; tile += gridDim.x) {
        int64_t i0, j0;
        coords(tile, i0, j0);
        double acc[8][4][2];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        for (int64_t t = 0; t < nk; ++t) {
            tc::mbar_wait(&full[st], ph);
            const double* As = ops + size_t(st) * 2 * kOpDoubles;
            const double* Bs = As + kOpDoubles;
#pragma unroll
            for (int kk = 0; kk < kDK; kk += 4) {
                double af[8], bf[4];
#pragma unroll
                for (int mi = 0; mi < 8; ++mi) af[mi] = ta.frag(As, wm * 64 + mi * 8 + fr, kk + fk);
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) bf[ni] = tb.frag(Bs, wn * 32 + ni * 8 + fr, kk + fk);
#pragma unroll
                for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], af[mi], bf[ni]);
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&empty[st]);
            if (++st == kWsStages) {
                st = 0;
                ph ^= 1;
            }
        }
        // C fragment: line i = 8 mi + lane/4 of A, lines j = 8 ni + 2 (lane%4) + {0, 1} of B
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t j = j0 + wn * 32 + ni * 8 + 2 * fk + h;
                if (j >= b.lines) continue;
#pragma unroll
                for (int mi = 0; mi < 8; ++mi) {
                    const int64_t i = i0 + wm * 64 + mi * 8 + fr;
                    if (i >= a.lines) continue;
                    double v = __dmul_rn(alpha, acc[mi][ni][h]);
                    if (beta != 0.0) v = __dadd_rn(v, __dmul_rn(beta, c_in[i + j * ldc_in]));
                    c_out[i + j * ldc] = v;
                }
            }
    }
}

int resident_grid(const void* fn, int threads, size_t smem, int64_t tiles) {
    static int sms = 0;
    if (!sms) sms = num_sms();
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const int64_t cap = int64_t(sms) * per_sm;
    return int(tiles < cap ? tiles : cap);
}

}  // namespace

void launch_native(const LineView& a, const LineView& b, double alpha, double beta, const double* c_in,
                   int64_t ldc_in, double* c_out, int64_t ldc, const Plan* plan, cudaStream_t st, uint64_t* nlaunch,
                   int flavour, const PeerB* peer) {
    if (a.lines == 0 || b.lines == 0) return;
    const bool use_peer = peer && peer->world > 0;
    const PeerB pb = use_peer ? *peer : PeerB{};
    using Fn = void (*)(LineView, LineView, double, double, const double*, int64_t, double*, int64_t, const Plan*,
                        PeerB);
#ifndef ADPB200_DMMA_WS
#define ADPB200_DMMA_WS 1
#endif
    if (flavour == ADPB200_FALLBACK_FAST && (ADPB200_DMMA_WS || use_peer)) {
        // [peer][A lines adjacent][B lines adjacent]
        static const Fn fns[8] = {dmma_ws_kernel<false, false, false>, dmma_ws_kernel<false, true, false>,
                                  dmma_ws_kernel<true, false, false>,  dmma_ws_kernel<true, true, false>,
                                  dmma_ws_kernel<false, false, true>,  dmma_ws_kernel<false, true, true>,
                                  dmma_ws_kernel<true, false, true>,   dmma_ws_kernel<true, true, true>};
        static bool attr = false;
        if (!attr) {
            for (Fn f : fns)
                cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kDmmaWsSmem));
            attr = true;
        }
        const Fn fn = fns[(use_peer ? 4 : 0) + (a.ls == 1 ? 2 : 0) + (b.ls == 1 ? 1 : 0)];
        const int64_t tiles = ((a.lines + kDT - 1) / kDT) * ((b.lines + kDT - 1) / kDT);
        const int grid = resident_grid(reinterpret_cast<const void*>(fn), kWsThreads, kDmmaWsSmem, tiles);
        launch_chain(fn, dim3(grid), dim3(kWsThreads), kDmmaWsSmem, st, a, b, alpha, beta, c_in, ldc_in, c_out, ldc, plan, pb);
    } else if (flavour == ADPB200_FALLBACK_FAST) {
        // operand layouts in shared memory follow the contiguous direction in HBM
        using Fn0 = void (*)(LineView, LineView, double, double, const double*, int64_t, double*, int64_t,
                             const Plan*);
        static const Fn0 fns[4] = {dmma_kernel<false, false, kDmmaWarps>, dmma_kernel<false, true, kDmmaWarps>,
                                   dmma_kernel<true, false, kDmmaWarps>, dmma_kernel<true, true, kDmmaWarps>};
        static bool attr = false;
        if (!attr) {
            for (Fn0 f : fns)
                cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kDmmaSmem));
            attr = true;
        }
        const Fn0 fn = fns[(a.ls == 1 ? 2 : 0) + (b.ls == 1 ? 1 : 0)];
        const int64_t tiles = ((a.lines + kDT - 1) / kDT) * ((b.lines + kDT - 1) / kDT);
        const int grid = resident_grid(reinterpret_cast<const void*>(fn), kDmmaWarps * 32, kDmmaSmem, tiles);
        launch_chain(fn, dim3(grid), dim3(kDmmaWarps * 32), kDmmaSmem, st, a, b, alpha, beta, c_in, ldc_in, c_out, ldc, plan);
    } else {
        static const Fn fns[2] = {native_kernel<false>, native_kernel<true>};
        static bool attr = false;
        if (!attr) {
            for (Fn f : fns)
                cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kNativeSmem));
            attr = true;
        }
        const Fn fn = fns[use_peer ? 1 : 0];
        const int64_t tiles = ((a.lines + kT - 1) / kT) * ((b.lines + kT - 1) / kT);
        const int grid = resident_grid(reinterpret_cast<const void*>(fn), 256, kNativeSmem, tiles);
        launch_chain(fn, dim3(grid), dim3(256), kNativeSmem, st, a, b, alpha, beta, c_in, ldc_in, c_out, ldc, plan, pb);
    }
    ++*nlaunch;
}

}  // namespace adpb200

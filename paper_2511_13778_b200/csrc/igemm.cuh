#pragma once
#include <cuda.h>

#include "guard.cuh"

namespace adpb200 {

constexpr int kGemmSmemBytes = 227 * 1024;
// Exact partial sums of one tile between k-chunks: NL limbs x NB x 128 rows
// (max over the variants: 2 x 64 x 128 x 8 B).
constexpr size_t kPartialBytesPerCta = 131072;

// Internal problem: C(i, j) = sum_l A(i, l) B(l, j), i < M (A-lines), j < N
// (B-lines), both operands sliced K-major into planes [slice][line][pitch].
constexpr int kMaxPeers = 8;  // ranks whose slab records one fused GEMM can read
constexpr int64_t kDistFlagBytes = 256;  // fused path's ready / consumed flags at the end of a slab buffer

struct GemmArgs {
    const Plan* plan;
    int64_t M, N, K;
    const int32_t* scale_a;  // E per A-line
    const int32_t* scale_b;  // E per B-line
    double alpha, beta;
    double* c_out;           // C(i, j) at c_out[i + j*ldc]
    int64_t ldc;
    const double* c_in;      // read iff beta != 0 (may alias c_out)
    int64_t ldc_in;
    uint64_t* partial;       // multi-chunk exact partial sums, kPartialBytesPerCta per CTA
    int64_t* dump;           // stage export: acc[(i*N + j)*ndump + D] += diagonal D
    int ndump;
    int smem_bytes;
    int debug;  // timing diagnostics only (ADPB200_DEBUG): 1 skip MMAs, 2 skip epilogue math
    int64_t mt_begin, mt_end;  // 128-row m-tile range to compute (mt_end 0 = all)
    int64_t nt_begin, nt_end;  // NB-column n-tile range to compute (nt_end 0 = all)
    int32_t* zero_flag;        // certified ESC: no C; set to 1 if any (i, j) has a zero diagonal-0 count
    uint32_t* fold_out;        // deferred rounding (NB 64, one k-chunk): the folded words go to
                               // fold_out[word][col][row] (M x N per word) instead of C
    // fused all-gather -> GEMM (multi-GPU phase 7): B planes and scales read in place
    // from every rank's slab record over peer memory; rank r owns columns
    // [r*peer_nr, (r+1)*peer_nr), tiled on its own (partial last tile per rank)
    int peer_world;            // 0: B from planes_b; else the number of ranks whose tiles run
    int64_t peer_nr;
    const int32_t* peer_scale[kMaxPeers];
    int peer_rank[kMaxPeers];  // global rank of each of those entries (its column offset)
    int pdl_early;             // trigger the dependent launch at kernel entry (else at exit)
};

// Fused peer variant of launch_igemm: B from world slab records ([scale int32 x nr |
// pad to hdr][cap planes of nkb x nr x 32 B], peer_slabs[r] = rank r's record as
// mapped in this process, or nullptr to skip rank r's columns), nsl planes each.
// Launches every variant (one does work).
int launch_igemm_peer(const int8_t* planes_a, int64_t slots_a, int64_t nkb, int cap, const int8_t* const* peer_slabs,
                      int world, int64_t nr, int64_t hdr, int nsl, const GemmArgs& g, cudaStream_t st,
                      uint64_t* nlaunch);

// nb in {64, 32, 16, 8}; the kernel returns immediately unless plan->variant == nb.
// planes_a / planes_b: blocked, pre-swizzled slice planes (cap planes of nkb
// k-blocks of slots_a / slots_b line slots, slots a multiple of 4).
int launch_igemm(int nb, const int8_t* planes_a, const int8_t* planes_b, int64_t slots_a, int64_t slots_b,
                 int64_t nkb, int cap, const GemmArgs& g, cudaStream_t st, uint64_t* nlaunch);

// Deferred rounding: C from the folded words the GEMM left in fold (4 planes of M x N
// uint32, column-major); predicated on the plan (variant 64, one k-chunk), like the GEMM.
void launch_round_folded(const Plan* plan, const uint32_t* fold, int64_t M, int64_t N, const int32_t* scale_a,
                         const int32_t* scale_b, double alpha, double beta, const double* c_in, int64_t ldc_in,
                         double* c_out, int64_t ldc, cudaStream_t st, uint64_t* nlaunch);

// recompose (igemm.cpp:99-127): acc = m x n x ndiag int64 element-major, row-major out.
void launch_recompose(const int64_t* acc, int64_t m, int64_t n, int ndiag, const int32_t* row_scale,
                      const int32_t* col_scale, double alpha, double beta, const double* c_in, double* out,
                      cudaStream_t st, uint64_t* nlaunch);

// K6: native FP64 fallback. flavour ADPB200_FALLBACK_REFERENCE: the reference's
// summation order (ascending k, separate multiply and add: oracle.cpp:7-28), bitwise;
// ADPB200_FALLBACK_FAST: FP64 tensor cores (DMMA). Runs iff the plan says native (or
// always when plan == nullptr); persistent grids, so a skipped launch is one small wave.
// B spread over the ranks' slab buffers (fused multi-GPU fallback): column j lives in
// p[j / nr] at column j % nr, each slab compact column-major (k x nr, leading dimension k).
struct PeerB {
    const double* p[kMaxPeers];
    int64_t nr;
    int world;  // 0: B is the LineView's own pointer
    __device__ __forceinline__ const double* at(int64_t j, int64_t kpos, int64_t ls, int64_t ps) const {
        const int64_t r = j / nr;
        return p[r] + (j - r * nr) * ls + kpos * ps;
    }
};

// pb (optional): B's columns read from the ranks' slabs instead of b.ptr (b.ls / b.ps
// then describe one slab).
void launch_native(const LineView& a, const LineView& b, double alpha, double beta, const double* c_in,
                   int64_t ldc_in, double* c_out, int64_t ldc, const Plan* plan, cudaStream_t st, uint64_t* nlaunch,
                   int flavour = ADPB200_FALLBACK_REFERENCE, const PeerB* pb = nullptr);
int num_sms();

// Grading tools (grade.cu): Dot2 double-double GEMM oracle out[i + j*ldo]
// (+ (|A||B|)_ij when absab != nullptr), and error_report on row-major
// rows x cols results: out[0..6] = max_rel, avg_rel, counted, skipped,
// max_ratio, avg_ratio, ratio_counted (device doubles).
void launch_dd_gemm(const LineView& a, const LineView& b, double* out, double* absab, int64_t ldo, cudaStream_t st,
                    uint64_t* nlaunch);
size_t error_partial_bytes();
void launch_error_report(const double* c, const double* ref, const double* absab, int64_t rows, int64_t cols,
                         double exact_diag, int use_diag, double* partial, double* out, cudaStream_t st,
                         uint64_t* nlaunch);
// Reproducible inputs (grade.cu): gen_uniform_rect (grading.cpp:56-63) on the
// device via xoshiro256++ jump-ahead, gen_test2 (grading.cpp:13-47). 0 ok,
// 1 contract (endpoint rounding), -1 CUDA error.
int gen_uniform_device(int64_t rows, int64_t cols, uint64_t seed, double lo, double hi, double* out, cudaStream_t st,
                       uint64_t* nlaunch);
int gen_test2_device(int64_t n, int b, uint64_t seed, double* lhs, double* rhs, double* x_out, int32_t* j_out,
                     cudaStream_t st, uint64_t* nlaunch);
// QR caller (qr.cu): blocked Householder QR with ADP trailing updates, Q and residuals.
int qr_geqrf(adpb200_handle h, int64_t m, int64_t n, int64_t panel, double* f, double* t_blocks, adpb200_trace* traces,
             const adpb200_options* opt, cudaStream_t st, uint64_t* nl);
int qr_materialize_q(adpb200_handle h, int64_t m, int64_t n, int64_t panel, const double* fac, const double* t_blocks,
                     double* q, cudaStream_t st, uint64_t* nl);
int qr_residual(adpb200_handle h, int64_t m, int64_t n, int64_t panel, const double* a0, const double* fac,
                const double* t_blocks, double* out, cudaStream_t st, uint64_t* nl);

}  // namespace adpb200

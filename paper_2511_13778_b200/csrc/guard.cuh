#pragma once
#include "common.cuh"

namespace adpb200 {

int num_sms();

// K1: fused Inf/NaN/-0 counts + per-(line, block) exponent max/min + line max.
// transposed = 1 stores the block stats block-major ([block][line], what the
// ESC kernel consumes); 0 the reference's line-major [line][block].
// tstride: line stride of the transposed layout (0 = v.lines), so a range of lines
// can write into a larger block-major array.
void launch_stats(const LineView& v, int64_t block_len, int32_t* bmax, int32_t* bmin, int32_t* line_max,
                  unsigned long long* counts, int32_t* exc_flag, int exc_bit, int transposed, cudaStream_t st,
                  uint64_t* nlaunch, int64_t tstride = 0, int skip_line_max = 0);
// Statistics of A (exc bit 1) and B (exc bit 2), same K and block length, transposed
// layout (line stride = lines): one launch in the column-major N,N case
// (ADPB200_STATS_PAIR, default 1), else two; the line maxima are left to
// launch_line_max_t_pair.
void launch_stats_pair(const LineView& va, int32_t* amax, int32_t* amin, unsigned long long* acounts,
                       const LineView& vb, int32_t* bmax, int32_t* bmin, unsigned long long* bcounts,
                       int64_t block_len, int32_t* exc_flag, cudaStream_t st, uint64_t* nlaunch);
// The line maxima of two transposed statistics arrays (A's and B's, lines x blocks
// each, line stride = lines) in one launch, for launch_stats(..., skip_line_max = 1).
void launch_line_max_t_pair(const int32_t* amaxT, int64_t alines, int32_t* aline, const int32_t* bmaxT,
                            int64_t blines, int32_t* bline, int64_t blocks, cudaStream_t st, uint64_t* nlaunch);
void launch_scan(const double* a, int64_t count, unsigned long long* counts, int32_t* exc, cudaStream_t st,
                 uint64_t* nlaunch);
// K2: coarsened ESC over block-major stats (atomicMax into esc_out, which must start at 0).
// B stats may come as column slabs of b_nr lines, slab r's record starting at
// r * b_rec int32 (bmax/bmin/bline pointers at their offsets inside record 0);
// b_nr = 0: one slab of all n lines. a_stride: line stride of the A stats (0 = m),
// so a range of A-lines of a larger block-major array can be passed.
void launch_esc(const int32_t* amax, const int32_t* amin, const int32_t* aline, const int32_t* bmax,
                const int32_t* bmin, const int32_t* bline, int64_t m, int64_t n, int64_t t, const Plan* plan,
                int32_t* esc_out, int32_t* ran_flag, cudaStream_t st, uint64_t* nlaunch, int64_t b_nr = 0,
                int64_t b_rec = 0, int64_t a_stride = 0);

// Multi-GPU B-distributed path: copy all-gathered slab records
// ([scale int32 x nr | pad to hdr][nsl planes of nkb x nr x 32 B]) into the
// GEMM's blocked plane layout (global line = r * nr + local) and scale_b.
// (`world` records starting with rank r_first.)
void launch_gather_planes(const int8_t* recs, int64_t rec_bytes, int64_t hdr, int world, int64_t nr, int64_t nkb,
                          int nsl, int8_t* planes, int64_t slots, int64_t plane_stride, int32_t* scale,
                          cudaStream_t st, uint64_t* nlaunch, int r_first = 0);
void launch_esc_finish(int32_t* out, int target_bits, cudaStream_t st, uint64_t* nlaunch);
// esc_exact (esc.cpp:61-87) stage export: A m x k and B k x n row-major; exponent
// fields ea (m*k) / eb (k*n) and maxima rmax (m) / cmax (n) are scratch; exc |= 1 on
// Inf/NaN; out[0] = max(0, max span) (must start at 0).
void launch_esc_exact(const double* A, const double* B, int64_t m, int64_t n, int64_t k, int32_t* ea, int32_t* eb,
                      int32_t* rmax, int32_t* cmax, int32_t* exc, int32_t* out, cudaStream_t st, uint64_t* nlaunch);
void launch_transpose_i32(const int32_t* src, int64_t lines, int64_t blocks, int32_t* dst, cudaStream_t st,
                          uint64_t* nlaunch);
// swap_ab: the internal operands are the user's B (A-lines) and A (B-lines).
void launch_decide(Plan* plan, const adpb200_options& opt, int64_t m, int64_t n, int64_t k, int esc_expected,
                   int swap_ab, adpb200_trace* trace, cudaStream_t st, uint64_t* nlaunch, int defer = 0);

// Stage exports: a fixed emulation plan (slices s, pair policy) without guardrails.
void launch_set_plan(Plan* plan, int s, int pair_limit, int64_t k, cudaStream_t st, uint64_t* nlaunch);

// K3: slicing into K-major int8 planes [slice][line][pitch] + per-line scale E.
// slices_fixed > 0 overrides the plan (stage exports); otherwise the kernel
// reads s / nsl from the plan and does nothing unless the path is emulated.
// plane_cap bounds nsl (sizes the transpose tile of the strided variant).
// blocked = 1: plane d is [k-block of 32][line][32 B] (the GEMM's TMA layout),
// zero-filled up to the next multiple of 32 positions; 0: [line][pitch].
void launch_slice(const LineView& v, const int32_t* line_max, int8_t* planes, int64_t pitch, int64_t plane_stride,
                  int blocked, int32_t* scale, const Plan* plan, int slices_fixed, int plane_cap, cudaStream_t st,
                  uint64_t* nlaunch, int indicator = 0);
// Slicing of both operands (same plan and blocking): one launch when the layouts
// allow it (ADPB200_SLICE_PAIR, default 1), else two launch_slice calls.
struct SliceOperand {
    LineView v;
    const int32_t* line_max;
    int8_t* planes;
    int64_t pitch, plane_stride;
    int32_t* scale;
};
void launch_slice_pair(const SliceOperand& A, const SliceOperand& B, int blocked, const Plan* plan, int slices_fixed,
                       int plane_cap, cudaStream_t st, uint64_t* nlaunch);

// Certified ESC (adpb200_options.esc_method): prep turns the coarsened result in
// `plan` into the indicator-GEMM plan `rplan` (path kPathDone when there is
// nothing to certify); finish lowers plan->esc_raw to 2*delta+1 when no
// (i, j) count came out zero.
// force = 1 (multi-GPU phases) arms rplan whatever this rank's coarsened result;
// max_planes (1 or 2) bounds the indicator planes per operand (= certificate levels).
void launch_certify_prep(const Plan* plan, Plan* rplan, int target_bits, int64_t k, cudaStream_t st,
                         uint64_t* nlaunch, int force = 0, int max_planes = 2);
// Indicator planes per operand a forced (multi-GPU) certificate uses.
inline int certify_planes(int target_bits) {
    return (certify_delta(target_bits, 0) >= 0 ? 1 : 0) + (certify_delta(target_bits, 1) >= 0 ? 1 : 0);
}
void launch_certify_finish(Plan* plan, const Plan* rplan, int target_bits, cudaStream_t st, uint64_t* nlaunch);
// Multi-GPU exchange block {exceptional | kXchgCertFail, esc_raw}: export before the
// max-allreduce, import after it (the certificate applied when no rank failed it).
void launch_dist_export(const Plan* plan, const Plan* rplan, int32_t* xchg, int certified, cudaStream_t st,
                        uint64_t* nlaunch);
void launch_dist_import(Plan* plan, const int32_t* xchg, int target_bits, int certified, cudaStream_t st,
                        uint64_t* nlaunch);

}  // namespace adpb200

/* adpb200 — B200-native (sm_100a) Automatic Dynamic Precision emulated DGEMM.
 *
 * C ABI of the drop-in for the reference's ADP GEMM path
 * (ozadp::adp_gemm, /root/reference/proj/include/ozadp/adp.hpp:84-87,
 *  impl proj/src/adp.cpp:139-178). Plain pointers and sizes only; every
 * matrix pointer is a DEVICE pointer; every call is stream-ordered and never
 * synchronises the host (the ADP decision lives in device memory).
 *
 * Return codes mirror the reference CLI's exit codes
 * (proj/tools/ozadp_main.cpp:235-244): 0 ok, 2 runtime/usage error
 * (CUDA failure, bad handle), 3 contract violation (the cases where the
 * reference throws std::invalid_argument: bad config, shape mismatch,
 * beta != 0 without C). No C++ exception crosses this boundary.
 */
#ifndef ADPB200_H
#define ADPB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADPB200_OK 0
#define ADPB200_ERR_RUNTIME 2
#define ADPB200_ERR_CONTRACT 3

/* AdpMode (adp.hpp:16) */
#define ADPB200_MODE_AUTO 0
#define ADPB200_MODE_EMULATE 1 /* ForceEmulate: forced_slices */
#define ADPB200_MODE_NATIVE 2  /* ForceNative */

/* AdpPath / AdpReason (adp.hpp:35-45), same numbering */
#define ADPB200_PATH_EMULATED 0
#define ADPB200_PATH_NATIVE 1
#define ADPB200_REASON_OK 0
#define ADPB200_REASON_FORCED 1
#define ADPB200_REASON_EXCEPTIONAL 2
#define ADPB200_REASON_ESC_TOO_LARGE 3
#define ADPB200_REASON_TOO_SMALL 4
#define ADPB200_REASON_COST_MODEL 5

/* Slice-pair policy (igemm.hpp:11-18).
 *   ADPB200_PAIRS_FULL   : all s^2 pairs — what adp_gemm uses (adp.cpp:172);
 *                          output bitwise equal to the reference.
 *   ADPB200_PAIRS_TARGET : pairs with d_a + d_b <= s only, i.e. the pairs
 *                          below the target precision are skipped (the north
 *                          star's fast path); = DiagonalTruncated(limit = s).
 *   >= 0                 : DiagonalTruncated(limit) exactly. */
#define ADPB200_PAIRS_FULL (-1)
#define ADPB200_PAIRS_TARGET (-2)

/* Native-fallback flavour. */
#define ADPB200_FALLBACK_REFERENCE 0 /* ascending-k, separate mul/add: bitwise native_gemm */
#define ADPB200_FALLBACK_FAST 1      /* FP64 tensor cores (DMMA m8n8k4), fused multiply-adds:
                                        |C - AB| <= gamma_k |A||B| (+ alpha/beta roundings),
                                        not the reference's bits; opt-in */

typedef struct adpb200_options {
    /* ozadp::AdpConfig (adp.hpp:18-33), same meaning and defaults */
    int32_t target_bits;   /* 53 */
    int32_t max_slices;    /* 18, valid [7, 32] */
    int64_t esc_block_len; /* 256 */
    int64_t min_dim;       /* 256 */
    int32_t mode;          /* ADPB200_MODE_* */
    int32_t forced_slices; /* 7 */
    double cost_ratio;     /* 512 */
    int64_t chunk_len;     /* 65536; validated like GemmParams (igemm.cpp:10-16) */
    /* extensions */
    int32_t pair_limit;        /* ADPB200_PAIRS_FULL (default) / _TARGET / >= 0 */
    int32_t guardrails_forced; /* 1: MODE_EMULATE still runs the scan+ESC+decide
                                  guardrails (the paper's "ADP forced to 55 bits",
                                  PAPER.md:734-757); the slice count stays pinned to
                                  forced_slices, exceptional inputs still fall back */
    int32_t fallback;          /* ADPB200_FALLBACK_* */
    int32_t esc_method;        /* ADPB200_ESC_COARSENED (default: the reference's esc_coarsened)
                                  or ADPB200_ESC_CERTIFIED: when the coarsened ESC asks for more
                                  than the minimum slice count s0 = ceil((target_bits+2)/8), an
                                  INT8 tensor-core GEMM of exponent indicator planes checks
                                  whether every (i,j) has, among the first min(k, 512)
                                  positions, a product within 2*delta bits of
                                  rowmax_i + colmax_j (delta the largest with 2*delta+1 <= the
                                  ESC s0 tolerates); if so esc_bits = 2*delta+1 (an upper bound
                                  of esc_exact, esc.cpp:61-87), else the coarsened value stays.
                                  Honoured by every entry point: the multi-GPU phases run the
                                  indicator GEMM on the local rows against the gathered column
                                  indicators and max-reduce its verdict with the ESC. */
    int32_t rounding;          /* ADPB200_ROUND_*: where the NB = 64 slice GEMM rounds the exact
                                  sums to FP64 — inside its epilogue (FUSED) or in a separate
                                  HBM pass over parked folded words (DEFERRED, 12 B of workspace
                                  per element of C; pays off for short k over a large C). AUTO
                                  defers for k <= 1536 and m*n >= 2^24 (env ADPB200_DEFER_ROUND
                                  = 0/1 overrides AUTO). Bitwise the same C either way. */
    int32_t reserved[3];
} adpb200_options;

#define ADPB200_ROUND_AUTO 0
#define ADPB200_ROUND_FUSED 1
#define ADPB200_ROUND_DEFERRED 2

#define ADPB200_ESC_COARSENED 0
#define ADPB200_ESC_CERTIFIED 1

/* AdpTrace (adp.hpp:57-67) + decision details; written to DEVICE memory by
 * the pipeline (stream-ordered). -1 encodes JSON null. */
typedef struct adpb200_trace {
    int32_t path;       /* ADPB200_PATH_* */
    int32_t reason;     /* ADPB200_REASON_* */
    int32_t esc_bits;   /* -1 when ESC never ran */
    int32_t slices;     /* -1 unless emulated */
    int32_t pair_limit; /* largest admitted d_a+d_b actually computed (-1 if native) */
    int32_t pairs;      /* slice pairs computed per output element */
    double modeled_cost_ratio;
    uint64_t nan_a, inf_a, negzero_a; /* ScanReport (fpbits.hpp:78-83) */
    uint64_t nan_b, inf_b, negzero_b;
    int64_t m, n, k;
    int32_t gemm_variant; /* columns per diagonal accumulator of the tcgen05 kernel */
    int32_t k_chunks;     /* int32 TMEM accumulation chunks along k */
    int32_t rounding_deferred; /* 1: C was rounded by the separate pass (adpb200_options.rounding) */
    int32_t reserved_t;
} adpb200_trace;

typedef struct adpb200_context* adpb200_handle;

void adpb200_default_options(adpb200_options* opt);
/* AdpConfig::validate (adp.cpp:15-28): 0 or ADPB200_ERR_CONTRACT */
int adpb200_validate_options(const adpb200_options* opt);
const char* adpb200_status_string(int status);
/* last error message of the calling thread (empty when none) */
const char* adpb200_last_error(void);
/* library version string; also proves the .so loads without a GPU */
const char* adpb200_version(void);

int adpb200_create(adpb200_handle* handle, int device);
int adpb200_destroy(adpb200_handle handle);

/* ---- the drop-in entry points ------------------------------------------------ */

/* BLAS DGEMM: C = alpha*op(A)*op(B) + beta*C, column-major, trans in
 * {'N','n','T','t','C','c'}. beta == 0 never reads C (BLAS / reference
 * convention, oracle.cpp:23). trace may be NULL. */
int adpb200_dgemm(adpb200_handle handle, char transa, char transb, int64_t m, int64_t n, int64_t k,
                  double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                  double beta, double* C, int64_t ldc, const adpb200_options* opt,
                  adpb200_trace* trace, void* stream);

/* ozadp::adp_gemm semantics on row-major device buffers (MatrixF64 layout):
 * out = alpha*A*B + beta*c_in, A m x k, B k x n. c_in may be NULL iff beta == 0
 * and may alias out. Bitwise equal to the reference for the same options. */
int adpb200_adp_gemm(adpb200_handle handle, int64_t m, int64_t n, int64_t k, double alpha,
                     const double* A, const double* B, double beta, const double* c_in,
                     double* out, const adpb200_options* opt, adpb200_trace* trace,
                     void* stream);

/* Host-buffer variants (A, B, C, trace in HOST memory; page-locked buffers
 * recommended): the end-to-end path the reference's value-returning adp_gemm
 * corresponds to; returns when C is on the host. The PCIe transfer overlaps
 * the computation: op(A) goes first, op(B) follows in column chunks on a
 * second stream, and each chunk's exponent stats, ESC contribution, slicing
 * and GEMM columns run as soon as it lands with a speculated slice count (the
 * handle's last decision), its C columns going straight back. The real ADP
 * decision is still made on the device from all the data; when it differs
 * from the speculation the predicated stages recompute C. Results are bitwise
 * those of adpb200_dgemm / adpb200_adp_gemm on device copies. */
int adpb200_dgemm_host(adpb200_handle handle, char transa, char transb, int64_t m, int64_t n, int64_t k,
                       double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                       double beta, double* C, int64_t ldc, const adpb200_options* opt,
                       adpb200_trace* trace, void* stream);
int adpb200_adp_gemm_host(adpb200_handle handle, int64_t m, int64_t n, int64_t k, double alpha,
                          const double* A, const double* B, double beta, const double* c_in,
                          double* out, const adpb200_options* opt, adpb200_trace* trace,
                          void* stream);

/* Row-block partition across ranks (one process per GPU): this rank owns rows
 * [r0, r0+m) of C / op(A) of a global m_global x n x k product and all of
 * op(B). phase 1 runs the guardrails (scan, exponent stats, ESC) on the local
 * rows and writes {exceptional, esc_bits} to xchg (device int32[2]); the caller
 * max-allreduces xchg over the ranks (e.g. ncclAllReduce(ncclMax, ncclInt32)
 * on the same stream); phase 2 consumes the reduced xchg, decides with the
 * global dimensions and computes the local rows. Same s and decision on every
 * rank, so C is bit-identical to the single-GPU result. */
int adpb200_dgemm_rows(adpb200_handle handle, int phase, int64_t m_global, char transa, char transb,
                       int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
                       const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                       const adpb200_options* opt, adpb200_trace* trace, int32_t* xchg, void* stream);

/* B-distributed row partition (the north star's multi-GPU layout): rank r
 * of `world` owns rows [r0, r0+m) of op(A) and C (all n columns) and the
 * column slab r of B: k x (n/world), column-major, leading dimension k.
 * n/world must be a multiple of 8. Four stream-ordered phases; the caller runs
 * the collectives between them (NCCL over NVLink; sizes from
 * adpb200_dist_sizes, out[0..3] = bstats record int32 count, slab header
 * bytes, bytes per slab plane, slab capacity bytes):
 *   phase 1  exponent stats of the A rows and of the B slab -> bstats_local
 *            (record int32[out[0]])            -> all-gather into bstats_all
 *   phase 2  ESC of the local rows against every B column -> xchg (int32[2])
 *                                              -> max-allreduce xchg
 *            (esc_method = ADPB200_ESC_CERTIFIED: the bstats record also holds
 *            the slab's indicator plane, phase 2 certifies the local rows
 *            against every column and sets bit 8 of xchg[0] when some (i, j)
 *            fails; phase 3 applies the certificate only if no rank set it,
 *            so the decision equals the single-GPU one)
 *   phase 3  decision with the global dimensions; slice the A rows; slice the
 *            B slab into `slab` = [scale | planes]. The caller copies xchg to
 *            the host and calls adpb200_dist_decision -> nsl planes:
 *              nsl > 0: all-gather the first out[1] + nsl*out[2] bytes of slab
 *              nsl = 0 (native fallback): all-gather the FP64 B slabs (= B)
 *   phase 4  gathered records -> the GEMM's plane layout, tcgen05 GEMM of the
 *            local rows (or the native GEMM against the gathered B).
 * Overlapped alternative to phase 4 (the plane all-gather runs while the GEMM
 * tiles that need only this rank's own B columns compute):
 *   phase 5  gathered = this rank's own slab record (`slab`): place it and run
 *            the GEMM n-tiles inside columns [rank*n/world, (rank+1)*n/world)
 *            (no-op when nsl = 0) — issue it, then wait for the all-gather;
 *   phase 6  gathered = all records: place them and run every other n-tile
 *            (or, when nsl = 0, the native GEMM against the gathered B).
 * Fused alternative to phases 4-6 (no plane all-gather at all, nsl > 0 only):
 *   phase 7  gathered = HOST array of `world` device pointers, entry r = rank
 *            r's `slab` buffer as mapped in this process (cudaIpcOpenMemHandle
 *            or peer access over NVLink; entry `rank` = the local slab). The
 *            GEMM's TMA loads read each rank's B planes in place, tile by tile
 *            (rank r's columns tiled on their own), and the epilogue reads the
 *            scales from the record headers. Every rank must be past phase 3
 *            before any rank starts phase 7, and slabs must stay untouched
 *            until every rank has finished it (two barriers). world <= 8.
 *            A null entry skips that rank's columns: one launch per rank, each
 *            after a pull of that rank's record into local memory
 *            (adpb200_copy_async on a copy stream), pipelines the transfer of
 *            rank r+1's planes with the GEMM of rank r's columns.
 *            nsl = 0 (host-sync-free form): the plane count and the path stay on
 *            the device. Every GEMM variant and the native fallback are launched
 *            predicated on the plan; the fallback reads B's FP64 columns from the
 *            ranks' slab buffers, where phase 8 put them.
 *   phase 8  (fused form, right after phase 3) on the native fallback only (device
 *            decided): copy this rank's FP64 B slab into `slab`.
 * Host-sync-free fused sequence per call (no host read, no host barrier): wait
 * until every peer's "consumed" flag of this slab buffer reaches epoch-1, phase 3,
 * phase 8, write the own "ready" flag = epoch, wait until every peer's "ready" flag
 * reaches epoch, phase 7 with nsl = 0, write the own "consumed" flag = epoch —
 * the flags are the last bytes of each slab buffer (adpb200_dist_flag_offset),
 * written and waited on by the streams themselves (adpb200_stream_write_flag /
 * adpb200_stream_wait_geq, CUDA stream memory operations, also across processes
 * on IPC mappings), epoch = 1, 2, ... per buffer.
 * Same decision and slice count on every rank: the assembled C is
 * bit-identical to the single-GPU adpb200_dgemm('N'/transa, 'N'). */
int adpb200_dist_sizes(int64_t n, int64_t k, int world, const adpb200_options* opt, int64_t out[4]);
/* Byte offset of a slab buffer's flag (which = 0 ready, 1 consumed) for a buffer of
 * slab_bytes (= adpb200_dist_sizes out[3]). */
int64_t adpb200_dist_flag_offset(int64_t slab_bytes, int which);
/* Stream-ordered 32-bit flags (CUDA stream memory operations): the stream waits until
 * *flag >= value; the stream writes *flag = value after its prior work. flag may be
 * an IPC / peer mapping. */
int adpb200_stream_wait_geq(const void* flag, uint32_t value, void* stream);
int adpb200_stream_write_flag(void* flag, uint32_t value, void* stream);
/* Slab buffers for phase 7, shared between the ranks' processes over CUDA IPC
 * (NVLink peer mappings): alloc exports a cudaMalloc'd buffer's 64-byte handle,
 * open maps a peer's handle (lazy peer access), close / free release them. */
int adpb200_ipc_alloc(int device, int64_t bytes, void** ptr, uint8_t handle[64]);
int adpb200_ipc_open(int device, const uint8_t handle[64], void** ptr);
int adpb200_ipc_close(void* ptr);
int adpb200_ipc_free(void* ptr);
/* Stream-ordered copy between any device pointers of this process, incl. IPC-mapped
 * peer buffers (the copy engines pull over NVLink). */
int adpb200_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* decide() on the reduced xchg (host copy): out = path, slices, nsl (planes to
 * gather; 0 on the native path), GEMM variant. */
int adpb200_dist_decision(const adpb200_options* opt, const int32_t xchg[2], int64_t m_global,
                          int64_t n, int64_t k, int32_t out[4]);
int adpb200_dgemm_dist(adpb200_handle handle, int phase, int64_t m_global, int world, int rank, char transa,
                       int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
                       const double* B_slab, double beta, double* C, int64_t ldc,
                       const adpb200_options* opt, adpb200_trace* trace, int32_t* bstats_local,
                       const int32_t* bstats_all, int32_t* xchg, int8_t* slab,
                       const void* gathered, int nsl, void* stream);

/* ---- stage exports (parity surface; row-major device buffers) --------------- */

/* decide() (adp.cpp:46-96) evaluated on the HOST by the same code the
 * device decision kernel runs. esc_bits = what the ESC provider returns.
 * out[0..4] = path, reason, slices, provider_called, esc_bits(-1 if not). */
int adpb200_decide_host(int exc_a, int exc_b, int64_t m, int64_t n, int64_t k, int esc_bits,
                        const adpb200_options* opt, int32_t out[5], double* cost_ratio);

/* scan_matrix (fpbits.cpp:5-24): counts[0..2] nan/inf/-0 (device uint64) */
int adpb200_scan(adpb200_handle handle, const double* A, int64_t count, uint64_t* counts,
                 void* stream);
/* block_exponent_stats (fpbits.cpp:26-73); orient 0 ByRow, 1 ByCol.
 * max_exp/min_exp: lines x blocks int32, line_max: lines int32 (device).
 * exceptional (device int32, may be NULL) is set to 1 on Inf/NaN. */
int adpb200_block_stats(adpb200_handle handle, const double* A, int64_t rows, int64_t cols,
                        int orient, int64_t block_len, int32_t* max_exp, int32_t* min_exp,
                        int32_t* line_max, int32_t* exceptional, void* stream);
/* esc_coarsened (esc.cpp:89-117) on device stats; out[0..2] = esc_bits,
 * window_bits, slices_required (device int32). */
int adpb200_esc_coarsened(adpb200_handle handle, const int32_t* a_max, const int32_t* a_min,
                          const int32_t* a_line, const int32_t* b_max, const int32_t* b_min,
                          const int32_t* b_line, int64_t m, int64_t n, int64_t blocks,
                          int target_bits, int32_t* out, void* stream);
/* esc_exact (esc.cpp:61-87), the O(mnk) ESC the reference's tests use as the
 * coarsened ESC's oracle, as a DPX max-plus kernel: A m x k and B k x n
 * row-major; out (device int32[3]) = {esc_bits, window_bits, slices_required};
 * *exceptional (device int32) = 1 on Inf/NaN input (the reference throws
 * std::domain_error; out is then meaningless). */
int adpb200_esc_exact(adpb200_handle handle, const double* A, const double* B, int64_t m, int64_t n,
                      int64_t k, int target_bits, int32_t* out, int32_t* exceptional, void* stream);
/* decompose (slicing.cpp:90-136): digits = slices planes of lines x len int8
 * (plane-major, each plane line-major = K-major), scale_exp: lines int32. */
int adpb200_decompose(adpb200_handle handle, const double* A, int64_t rows, int64_t cols,
                      int orient, int slices, int8_t* digits, int32_t* scale_exp, void* stream);
/* slice_pair_mm (igemm.cpp:38-97) computed on the tcgen05 INT8 tensor cores:
 * acc = m x n x (2s-1) int64 element-major (DiagonalAccumulators layout,
 * igemm.hpp:34-47). pair_limit: ADPB200_PAIRS_FULL or >= 0. */
int adpb200_slice_pair_mm(adpb200_handle handle, const double* A, const double* B, int64_t m,
                          int64_t n, int64_t k, int slices, int pair_limit, int64_t* acc,
                          void* stream);
/* recompose (igemm.cpp:99-127): out (m x n row-major FP64) from the diagonal
 * accumulators of slice_pair_mm (2*slices-1 per element) and the decompose scales
 * (row_scale: m, col_scale: n): S = sum_D acc_D 2^(8(dmax-D)) exactly, one RNE
 * rounding of S 2^(row+col-14-8 dmax), r = alpha v (+ beta C, C read iff beta != 0). */
int adpb200_recompose(adpb200_handle handle, const int64_t* acc, int64_t m, int64_t n, int slices,
                      const int32_t* row_scale, const int32_t* col_scale, double alpha, double beta,
                      const double* c_in, double* out, void* stream);
/* emulated_gemm (igemm.cpp:129-137): fixed slices, no guardrails. */
int adpb200_emulated_gemm(adpb200_handle handle, const double* A, const double* B, int64_t m,
                          int64_t n, int64_t k, double alpha, double beta, const double* c_in,
                          double* out, int slices, int pair_limit, void* stream);
/* native_gemm (oracle.cpp:7-28): ascending-k, separate multiply/add. */
int adpb200_native_gemm(adpb200_handle handle, const double* A, const double* B, int64_t m,
                        int64_t n, int64_t k, double alpha, double beta, const double* c_in,
                        double* out, void* stream);

/* ---- grading tools (device) ---------------------------------------------------
 * The reference grades against exact_gemm (oracle.cpp:55-75, CPU
 * superaccumulator). On the device: a double-double (Dot2: TwoProd by FMA +
 * TwoSum) GEMM oracle, as accurate as a twice-working-precision product
 * rounded once: |ref - AB| <= 2^-53 |AB| + gamma_2k^2 (|A||B|). Row-major
 * (MatrixF64) layout like adpb200_adp_gemm. absab (nullable) receives the
 * plain FP64 sum of |a||b|, the grading-ratio denominator (grading.cpp:108-123). */
int adpb200_dd_gemm(adpb200_handle handle, int64_t m, int64_t n, int64_t k, const double* A,
                    const double* B, double* ref, double* absab, void* stream);
/* error_report (grading.cpp:67-90) on rows x cols row-major device matrices:
 * componentwise |ref - C| / |ref| (ref == 0 skipped and counted; with
 * use_exact_diag, diagonal entries compare against exact_diag, the Test-2
 * convention) and, when absab != NULL, the grading ratio
 * |C - ref| / (2^-52 (|A||B|)_ij). out (device double[7]) = max_rel,
 * avg_rel, counted, skipped, max_ratio, avg_ratio, ratio_counted.
 * Deterministic (fixed-order reduction). */
int adpb200_error_report(adpb200_handle handle, int64_t rows, int64_t cols, const double* C,
                         const double* ref, const double* absab, double exact_diag,
                         int use_exact_diag, double* out, void* stream);

/* gen_uniform_rect (grading.cpp:56-63): row-major rows x cols uniform(lo, hi)
 * from xoshiro256++ (rng.hpp:11-54), generated on the device (jump-ahead per
 * 4096-draw chunk); bitwise the reference's matrix for the same seed. */
int adpb200_gen_uniform_rect(adpb200_handle handle, int64_t rows, int64_t cols, uint64_t seed,
                             double lo, double hi, double* out, void* stream);
/* gen_test2 (grading.cpp:13-47): the adversarial exponent-span pair, n x n
 * row-major lhs / rhs on the device; x (host double[n]) and j (host
 * int32[n]) optional. Synchronises the stream once (host vectors). */
int adpb200_gen_test2(adpb200_handle handle, int64_t n, int b, uint64_t seed, double* lhs,
                      double* rhs, double* x, int32_t* j, void* stream);

/* ---- the reference's application caller: blocked Householder QR ----------------
 * geqrf_blocked (qr.cpp:98-143): A (row-major m x n device, m >= n >= 1) is
 * overwritten by the factors (R in the upper triangle, unit-diagonal reflector
 * tails below); t_blocks (device, ceil(n/panel) slots of panel*panel doubles)
 * receives each panel's upper-triangular T, packed pw x pw at the slot start;
 * traces (device, 3 per panel) the dispatch of every trailing-update GEMM
 * (W = Y^T A_s, W = T^T W, A_s -= Y W, all through adpb200_adp_gemm with opt).
 * Panel factorisation in the reference's operation order on the device:
 * factors, T and traces are bitwise the reference's. panel <= 1024. */
int adpb200_geqrf_blocked(adpb200_handle handle, int64_t m, int64_t n, int64_t panel, double* A,
                          double* t_blocks, adpb200_trace* traces, const adpb200_options* opt,
                          void* stream);
/* materialize_q (qr.cpp:145-173): thin Q (m x n, row-major device). */
int adpb200_qr_materialize_q(adpb200_handle handle, int64_t m, int64_t n, int64_t panel,
                             const double* factors, const double* t_blocks, double* Q, void* stream);
/* qr_residual (qr.cpp:183-197): out (device double[2]) = |A0 - QR|_F / |A0|_F,
 * |I - Q^T Q|_F, with the reference-order native GEMM and sequential norms. */
int adpb200_qr_residual(adpb200_handle handle, int64_t m, int64_t n, int64_t panel, const double* A0,
                        const double* factors, const double* t_blocks, double* out, void* stream);

/* Kernel launches issued by this handle since creation (all kernels are ours). */
uint64_t adpb200_launch_count(adpb200_handle handle);
/* bytes of device workspace the handle currently owns (grows on demand, never shrinks) */
uint64_t adpb200_workspace_bytes(adpb200_handle handle);

/* Stage timing with CUDA events on the caller's stream (no effect on results).
 * Stages: 0 scan+stats (K1), 1 ESC (K2), 2 decide, 3 slicing (K3),
 * 4 tcgen05 GEMM + epilogue (K4/K5), 5 native fallback (K6).
 * enable(max_calls) records the next max_calls pipeline calls (0 disables);
 * read() waits for them and returns ms[call*6 + stage], then resets. */
#define ADPB200_PROFILE_STAGES 6
int adpb200_profile_enable(adpb200_handle handle, int max_calls);
int adpb200_profile_read(adpb200_handle handle, float* ms, int* ncalls);

#ifdef __cplusplus
}
#endif
#endif /* ADPB200_H */

/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the ADP emulated DGEMM path.
 *
 * A plain-C restatement of the reference algorithm (ozadp, /root/reference/proj)
 * used exclusively by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the CHECKER. The product (paper_2511_13778_b200/) never
 * links, loads or calls it. Pinned against the reference itself (oracle/_ref,
 * built from the reference sources by oracle/Makefile) and against the golden
 * vectors of the reference's own tests (tests/golden/, tests/test_oracle_*.py).
 *
 * Conventions: matrices are dense row-major like ozadp::MatrixF64
 * (proj/include/ozadp/matrix.hpp:12-43). orient 0 = ByRow (lines are rows),
 * 1 = ByCol (lines are columns). Return codes: 0 ok, 3 contract violation
 * (std::invalid_argument / std::domain_error in the reference).
 */
#ifndef ADP_ORACLE_H
#define ADP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OZ_NEG_SENTINEL (-1000000) /* proj/include/ozadp/fpbits.hpp:22 */
#define OZ_MAX_SLICES 32           /* proj/include/ozadp/slicing.hpp:11 */

/* --- inputs (proj/include/ozadp/rng.hpp:11-54, proj/src/grading.cpp:13-63) --- */
void oz_gen_uniform_rect(int64_t rows, int64_t cols, uint64_t seed, double lo, double hi,
                         double* out);
int oz_gen_test2(int64_t n, int b, uint64_t seed, double* lhs, double* rhs);

/* --- guardrails (proj/src/fpbits.cpp, proj/src/esc.cpp) --- */
int oz_effective_exponent_bits(uint64_t bits);
void oz_scan(const double* a, int64_t count, uint64_t counts[3], int* exceptional);
int oz_block_stats(const double* a, int64_t rows, int64_t cols, int orient, int64_t block_len,
                   int32_t* max_exp, int32_t* min_exp, int32_t* line_max);
int oz_required_slices(int target_bits, int esc_bits);
/* out[0..2] = esc_bits, window_bits, slices_required */
int oz_esc_coarsened(const int32_t* a_max, const int32_t* a_min, const int32_t* a_line,
                     const int32_t* b_max, const int32_t* b_min, const int32_t* b_line,
                     int64_t m, int64_t n, int64_t blocks, int target_bits, int out[3]);
int oz_esc_exact(const double* a, const double* b, int64_t m, int64_t n, int64_t k,
                 int target_bits, int out[3]);

/* --- dispatcher (proj/src/adp.cpp:15-96) --- */
typedef struct oz_config {
    int target_bits;       /* 53 */
    int64_t esc_block_len; /* 256 */
    int max_slices;        /* 18 */
    int64_t min_dim;       /* 256 */
    int mode;              /* 0 auto, 1 force emulate, 2 force native */
    int forced_slices;     /* 7 */
    double cost_ratio;     /* 512 */
    int64_t chunk_len;     /* 65536 */
} oz_config;
void oz_config_default(oz_config* c);
int oz_config_validate(const oz_config* c);
/* esc_bits < 0 means "not computed"; the provider is modelled by passing the
 * value it would return (esc_in) and counting whether decide() asked for it.
 * out: path (0 emulated, 1 native), reason (AdpReason order), slices,
 * provider_called, esc_bits (-1 when not consulted). */
int oz_decide(int exc_a, int exc_b, int64_t m, int64_t n, int64_t k, int esc_in,
              const oz_config* c, int out[5], double* cost_ratio);

/* --- emulation (proj/src/slicing.cpp, proj/src/igemm.cpp) --- */
void oz_extract_digits(double v, int32_t scale_exp, int slices, int32_t* lead, uint8_t* sub);
void oz_element_digits(double v, int32_t scale_exp, int slices, int8_t* out);
/* digits: slices planes of lines*len (plane-major, line-major inside a plane) */
int oz_decompose(const double* a, int64_t rows, int64_t cols, int orient, int slices,
                 int8_t* digits, int32_t* scale_exp);
/* acc: m*n*(2s-1) int64, element-major; limit < 0 = Full pair set */
int oz_slice_pair_mm(const int8_t* sa, const int8_t* sb, int64_t m, int64_t n, int64_t k,
                     int slices, int limit, int64_t* acc);
/* one element: exact sum of acc[0..ndiag) at weights 2^(8(ndiag-1-d)), times 2^exp2, RNE */
double oz_fold_round(const int64_t* acc, int ndiag, long exp2);
int oz_recompose(const int64_t* acc, int64_t m, int64_t n, int slices, const int32_t* row_scale,
                 const int32_t* col_scale, double alpha, double beta, const double* c,
                 double* out);
int oz_emulated_gemm(const double* a, const double* b, int64_t m, int64_t n, int64_t k,
                     double alpha, double beta, const double* c, int slices, int limit,
                     double* out);

/* --- fallback + exact oracle (proj/src/oracle.cpp) --- */
int oz_native_gemm(const double* a, const double* b, int64_t m, int64_t n, int64_t k,
                   double alpha, double beta, const double* c, double* out);
int oz_exact_gemm(const double* a, const double* b, int64_t m, int64_t n, int64_t k,
                  double* out);

/* --- whole entry point (proj/src/adp.cpp:139-178) ---
 * trace: path, reason, esc_bits(-1 null), slices(-1 null), scan counts a[3], b[3] */
int oz_adp_gemm(const double* a, const double* b, int64_t m, int64_t n, int64_t k, double alpha,
                double beta, const double* c, const oz_config* cfg, double* out,
                int64_t trace[10], double* cost_ratio);

#ifdef __cplusplus
}
#endif
#endif

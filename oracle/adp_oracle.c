/* TEST INFRASTRUCTURE ONLY — CPU oracle for the ADP emulated DGEMM path.
 * See adp_oracle.h. Compiled with -ffp-contract=off so that every FP64
 * multiply and add rounds separately, like the reference build
 * (proj/CMakeLists.txt:16-18). Each function cites the reference lines it
 * restates.
 */
#include "adp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static uint64_t f64_bits(double v) {
    uint64_t b;
    memcpy(&b, &v, 8);
    return b;
}
static int raw_exp(uint64_t bits) { return (int)((bits >> 52) & 0x7ff); }
static const uint64_t kMant = (((uint64_t)1) << 52) - 1;

/* ------------------------------------------------------------------------ */
/* xoshiro256++ / splitmix64 (proj/include/ozadp/rng.hpp:11-54)              */
typedef struct { uint64_t s[4]; } xoshiro;
static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
static uint64_t splitmix64(uint64_t* x) {
    *x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static void xo_seed(xoshiro* r, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&x);
}
static uint64_t xo_next(xoshiro* r) {
    uint64_t* s = r->s;
    uint64_t res = rotl(s[0] + s[3], 23) + s[0];
    uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return res;
}
/* open interval (0,1): rng.hpp:37 */
static double xo_u01(xoshiro* r) { return ((double)(xo_next(r) >> 11) + 0.5) * 0x1p-53; }

/* grading.cpp:56-63 */
void oz_gen_uniform_rect(int64_t rows, int64_t cols, uint64_t seed, double lo, double hi,
                         double* out) {
    xoshiro r;
    xo_seed(&r, seed);
    for (int64_t i = 0; i < rows * cols; ++i) {
        double u = xo_u01(&r);
        out[i] = lo + (hi - lo) * u;
    }
}

/* grading.cpp:13-47 */
int oz_gen_test2(int64_t n, int b, uint64_t seed, double* lhs, double* rhs) {
    if (n < 2 || b < 0 || b > 1022) return 3;
    double delta = (2.0 * b) / (double)(n - 1);
    xoshiro r;
    xo_seed(&r, seed);
    double* x = (double*)malloc(sizeof(double) * (size_t)n);
    int* j = (int*)malloc(sizeof(int) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) x[i] = 1.0 + xo_u01(&r);
    for (int64_t i = 0; i < n; ++i) j[i] = b == 0 ? 0 : (int)(-b + llround((double)i * delta));
    int rc = (j[0] == -b && j[n - 1] == b) ? 0 : 3;
    for (int64_t kk = 0; kk < n && rc == 0; ++kk) {
        for (int64_t i = 0; i < n; ++i) {
            int64_t s = i >= kk ? i - kk : i + n - kk;
            lhs[kk * n + i] = ldexp(x[s], j[s]);
            rhs[i * n + kk] = ldexp(x[s], -j[s]);
        }
    }
    free(x);
    free(j);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* fpbits (proj/include/ozadp/fpbits.hpp:34-48, proj/src/fpbits.cpp)         */
int oz_effective_exponent_bits(uint64_t bits) {
    int e = raw_exp(bits);
    if (e != 0) return e - 1023;
    uint64_t mant = bits & kMant;
    return (63 - __builtin_clzll(mant)) - 1074;
}
static uint64_t normalized_mantissa(uint64_t bits) {
    int e = raw_exp(bits);
    uint64_t mant = bits & kMant;
    if (e != 0) return mant | (((uint64_t)1) << 52);
    return mant << (52 - (63 - __builtin_clzll(mant)));
}

/* fpbits.cpp:5-24 */
void oz_scan(const double* a, int64_t count, uint64_t counts[3], int* exceptional) {
    uint64_t nans = 0, infs = 0, negz = 0;
    for (int64_t i = 0; i < count; ++i) {
        uint64_t bits = f64_bits(a[i]);
        int e = raw_exp(bits);
        uint64_t mant = bits & kMant;
        if (e == 0x7ff) {
            if (mant) ++nans;
            else ++infs;
        } else if (e == 0 && mant == 0 && (bits >> 63)) {
            ++negz;
        }
    }
    counts[0] = nans;
    counts[1] = infs;
    counts[2] = negz;
    *exceptional = (nans + infs) > 0;
}

/* fpbits.cpp:26-73. Element (line,pos) of a row-major rows x cols matrix. */
int oz_block_stats(const double* a, int64_t rows, int64_t cols, int orient, int64_t block_len,
                   int32_t* max_exp, int32_t* min_exp, int32_t* line_max) {
    if (block_len < 1) return 3;
    int64_t lines = orient ? cols : rows, len = orient ? rows : cols;
    int64_t blocks = len == 0 ? 0 : (len + block_len - 1) / block_len;
    int64_t ls = orient ? 1 : cols, ps = orient ? cols : 1;
    int exc = 0;
#pragma omp parallel for schedule(static) reduction(|| : exc)
    for (int64_t line = 0; line < lines; ++line) {
        int32_t lmax = OZ_NEG_SENTINEL;
        for (int64_t blk = 0; blk < blocks; ++blk) {
            int64_t lo = blk * block_len, hi = lo + block_len < len ? lo + block_len : len;
            int32_t bmax = OZ_NEG_SENTINEL, bmin = -OZ_NEG_SENTINEL;
            for (int64_t pos = lo; pos < hi; ++pos) {
                uint64_t bits = f64_bits(a[line * ls + pos * ps]);
                if (raw_exp(bits) == 0x7ff) {
                    exc = 1;
                    continue;
                }
                if ((bits << 1) == 0) continue;
                int32_t e = oz_effective_exponent_bits(bits);
                if (e > bmax) bmax = e;
                if (e < bmin) bmin = e;
            }
            max_exp[line * blocks + blk] = bmax != OZ_NEG_SENTINEL ? bmax : OZ_NEG_SENTINEL;
            min_exp[line * blocks + blk] = bmax != OZ_NEG_SENTINEL ? bmin : OZ_NEG_SENTINEL;
            if (bmax != OZ_NEG_SENTINEL && bmax > lmax) lmax = bmax;
        }
        line_max[line] = lmax;
    }
    return exc ? 3 : 0;
}

/* esc.cpp:8-12 */
int oz_required_slices(int target_bits, int esc_bits) { return (target_bits + esc_bits + 2 + 7) / 8; }

/* esc.cpp:89-117 */
int oz_esc_coarsened(const int32_t* a_max, const int32_t* a_min, const int32_t* a_line,
                     const int32_t* b_max, const int32_t* b_min, const int32_t* b_line,
                     int64_t m, int64_t n, int64_t t, int target_bits, int out[3]) {
    int esc = 0;
#pragma omp parallel for schedule(static) reduction(max : esc)
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            int32_t z = OZ_NEG_SENTINEL;
            for (int64_t blk = 0; blk < t; ++blk) {
                int32_t amax = a_max[i * t + blk];
                if (amax == OZ_NEG_SENTINEL) continue;
                int32_t bmax = b_max[j * t + blk];
                if (bmax == OZ_NEG_SENTINEL) continue;
                int32_t c1 = amax + b_min[j * t + blk], c2 = a_min[i * t + blk] + bmax;
                int32_t cand = c1 > c2 ? c1 : c2;
                if (cand > z) z = cand;
            }
            if (z == OZ_NEG_SENTINEL) continue;
            int span = a_line[i] + b_line[j] - z + 1;
            if (span > esc) esc = span;
        }
    }
    out[0] = esc;
    out[1] = target_bits + esc;
    out[2] = oz_required_slices(target_bits, esc);
    return 0;
}

/* esc.cpp:27-87 */
int oz_esc_exact(const double* a, const double* b, int64_t m, int64_t n, int64_t k,
                 int target_bits, int out[3]) {
    int32_t* ea = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m * k + 1));
    int32_t* eb = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * k + 1));
    int32_t* ra = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
    int32_t* cb = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int exc = 0;
    for (int64_t i = 0; i < m; ++i) {
        ra[i] = OZ_NEG_SENTINEL;
        for (int64_t l = 0; l < k; ++l) {
            uint64_t bits = f64_bits(a[i * k + l]);
            ea[i * k + l] = OZ_NEG_SENTINEL;
            if (raw_exp(bits) == 0x7ff) { exc = 1; continue; }
            if ((bits << 1) == 0) continue;
            int32_t e = oz_effective_exponent_bits(bits);
            ea[i * k + l] = e;
            if (e > ra[i]) ra[i] = e;
        }
    }
    for (int64_t j = 0; j < n; ++j) {
        cb[j] = OZ_NEG_SENTINEL;
        for (int64_t l = 0; l < k; ++l) {
            uint64_t bits = f64_bits(b[l * n + j]);
            eb[j * k + l] = OZ_NEG_SENTINEL;
            if (raw_exp(bits) == 0x7ff) { exc = 1; continue; }
            if ((bits << 1) == 0) continue;
            int32_t e = oz_effective_exponent_bits(bits);
            eb[j * k + l] = e;
            if (e > cb[j]) cb[j] = e;
        }
    }
    int esc = 0;
    if (!exc) {
#pragma omp parallel for schedule(static) reduction(max : esc)
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < n; ++j) {
                int32_t z = OZ_NEG_SENTINEL;
                for (int64_t l = 0; l < k; ++l) {
                    if (ea[i * k + l] == OZ_NEG_SENTINEL || eb[j * k + l] == OZ_NEG_SENTINEL) continue;
                    int32_t s = ea[i * k + l] + eb[j * k + l];
                    if (s > z) z = s;
                }
                if (z == OZ_NEG_SENTINEL) continue;
                int span = ra[i] + cb[j] - z + 1;
                if (span > esc) esc = span;
            }
    }
    free(ea); free(eb); free(ra); free(cb);
    if (exc) return 3;
    out[0] = esc;
    out[1] = target_bits + esc;
    out[2] = oz_required_slices(target_bits, esc);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* dispatcher (proj/src/adp.cpp:15-28, 46-96; defaults adp.hpp:18-33)        */
void oz_config_default(oz_config* c) {
    c->target_bits = 53;
    c->esc_block_len = 256;
    c->max_slices = 18;
    c->min_dim = 256;
    c->mode = 0;
    c->forced_slices = 7;
    c->cost_ratio = 512.0;
    c->chunk_len = 65536;
}

int oz_config_validate(const oz_config* c) {
    if (!(c->target_bits >= 1 && c->target_bits <= 1024)) return 3;
    if (!(c->esc_block_len >= 1)) return 3;
    if (!(c->max_slices >= 7 && c->max_slices <= OZ_MAX_SLICES)) return 3;
    if (!(c->min_dim >= 1)) return 3;
    if (!(c->cost_ratio > 0.0)) return 3;
    if (c->mode == 1 && !(c->forced_slices >= 1 && c->forced_slices <= OZ_MAX_SLICES)) return 3;
    if (!(c->chunk_len >= 1 && c->chunk_len * 16384 < (((int64_t)1) << 31))) return 3;
    return 0;
}

int oz_decide(int exc_a, int exc_b, int64_t m, int64_t n, int64_t k, int esc_in,
              const oz_config* c, int out[5], double* cost_ratio) {
    if (oz_config_validate(c)) return 3;
    out[3] = 0;
    out[4] = -1;
    *cost_ratio = 0.0;
    if (c->mode == 2) { out[0] = 1; out[1] = 1; out[2] = 0; return 0; }      /* Forced */
    if (exc_a || exc_b) { out[0] = 1; out[1] = 2; out[2] = 0; return 0; }   /* Exceptional */
    if (c->mode == 1) { out[0] = 0; out[1] = 1; out[2] = c->forced_slices; return 0; }
    int64_t mn = m < n ? m : n;
    mn = mn < k ? mn : k;
    if (mn < c->min_dim) { out[0] = 1; out[1] = 4; out[2] = 0; return 0; }  /* TooSmall */
    out[3] = 1;
    out[4] = esc_in;
    int s_req = oz_required_slices(c->target_bits, esc_in);
    if (s_req > c->max_slices) { out[0] = 1; out[1] = 3; out[2] = 0; return 0; } /* EscTooLarge */
    double mnk = (double)m * (double)n * (double)k;
    double s = (double)s_req;
    double estimator = (double)m * (double)k + (double)k * (double)n;
    *cost_ratio = (s * s * mnk / c->cost_ratio + estimator) / mnk;
    if (*cost_ratio >= 1.0) { out[0] = 1; out[1] = 5; out[2] = 0; return 0; } /* CostModel */
    out[0] = 0;
    out[1] = 0;
    out[2] = s_req;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* slicing (proj/src/slicing.cpp:11-136)                                     */
static uint32_t byte_window(uint64_t x, long a) {
    if (a >= 64 || a <= -8) return 0;
    if (a >= 0) return (uint32_t)(x >> a) & 0xffu;
    return (uint32_t)(x << -a) & 0xffu;
}

/* slicing.cpp:20-48 */
void oz_extract_digits(double v, int32_t scale_exp, int slices, int32_t* lead, uint8_t* sub) {
    uint64_t bits = f64_bits(v);
    if ((bits << 1) == 0) {
        *lead = 0;
        for (int d = 1; d < slices; ++d) sub[d - 1] = 0;
        return;
    }
    int neg = (bits >> 63) != 0;
    uint64_t M = normalized_mantissa(bits);
    int e = oz_effective_exponent_bits(bits);
    long sh = 45 + (long)scale_exp - e;
    if (!neg) {
        *lead = sh < 64 ? (int32_t)(M >> sh) : 0;
        for (int d = 1; d < slices; ++d) sub[d - 1] = (uint8_t)byte_window(M, sh - 8 * d);
    } else {
        uint64_t Mm1 = M - 1;
        *lead = sh < 64 ? -(int32_t)(Mm1 >> sh) - 1 : -1;
        for (int d = 1; d < slices; ++d) {
            long a = sh - 8 * d;
            uint32_t mask = a >= 0 ? 0xffu : (a <= -8 ? 0u : (0xffu << -a) & 0xffu);
            sub[d - 1] = (uint8_t)(~byte_window(Mm1, a) & mask);
        }
    }
}

/* slicing.cpp:50-66: extract, then remap least-significant first with carry */
void oz_element_digits(double v, int32_t scale_exp, int slices, int8_t* out) {
    int32_t lead;
    uint8_t sub[OZ_MAX_SLICES];
    oz_extract_digits(v, scale_exp, slices, &lead, sub);
    int carry = 0;
    for (int d = slices - 1; d >= 1; --d) {
        int c = sub[d - 1] + carry;
        if (c <= 127) { out[d] = (int8_t)c; carry = 0; }
        else { out[d] = (int8_t)(c - 256); carry = 1; }
    }
    out[0] = (int8_t)(lead + carry);
}

/* slicing.cpp:90-136 */
int oz_decompose(const double* a, int64_t rows, int64_t cols, int orient, int slices,
                 int8_t* digits, int32_t* scale_exp) {
    if (slices < 1 || slices > OZ_MAX_SLICES) return 3;
    int64_t lines = orient ? cols : rows, len = orient ? rows : cols;
    int64_t ls = orient ? 1 : cols, ps = orient ? cols : 1;
    int64_t plane = lines * len;
    memset(digits, 0, (size_t)(plane * slices));
    int exc = 0;
#pragma omp parallel for schedule(static) reduction(|| : exc)
    for (int64_t line = 0; line < lines; ++line) {
        scale_exp[line] = 0;
        int32_t lmax = OZ_NEG_SENTINEL;
        for (int64_t pos = 0; pos < len; ++pos) {
            uint64_t bits = f64_bits(a[line * ls + pos * ps]);
            if (raw_exp(bits) == 0x7ff) { exc = 1; continue; }
            if ((bits << 1) == 0) continue;
            int32_t e = oz_effective_exponent_bits(bits);
            if (e > lmax) lmax = e;
        }
        if (lmax == OZ_NEG_SENTINEL) continue;
        int32_t E = lmax + 2;
        scale_exp[line] = E;
        int8_t dig[OZ_MAX_SLICES];
        for (int64_t pos = 0; pos < len; ++pos) {
            double v = a[line * ls + pos * ps];
            if (v == 0.0) continue;
            oz_element_digits(v, E, slices, dig);
            for (int d = 0; d < slices; ++d) digits[d * plane + line * len + pos] = dig[d];
        }
    }
    return exc ? 3 : 0;
}

/* ------------------------------------------------------------------------ */
/* integer contraction (proj/src/igemm.cpp:38-97). Every sum is an exact     */
/* integer, so the chunked int32/int64 schedule of the reference is         */
/* irrelevant to the result; 64-bit sums are used directly.                  */
int oz_slice_pair_mm(const int8_t* sa, const int8_t* sb, int64_t m, int64_t n, int64_t k,
                     int s, int limit, int64_t* acc) {
    int diag = 2 * s - 1;
    memset(acc, 0, sizeof(int64_t) * (size_t)(m * n * diag));
    if (m == 0 || n == 0) return 0;
#pragma omp parallel for schedule(dynamic) collapse(2)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j)
            for (int da = 0; da < s; ++da)
                for (int db = 0; db < s; ++db) {
                    int d = da + db;
                    if (limit >= 0 && d > limit) continue;
                    const int8_t* pa = sa + (int64_t)da * m * k + i * k;
                    const int8_t* pb = sb + (int64_t)db * n * k + j * k;
                    int64_t tot = 0;
                    for (int64_t base = 0; base < k; base += 65536) {
                        int64_t end = base + 65536 < k ? base + 65536 : k;
                        int32_t s32 = 0;
                        for (int64_t l = base; l < end; ++l) s32 += (int32_t)pa[l] * (int32_t)pb[l];
                        tot += s32;
                    }
                    acc[(i * n + j) * diag + d] += tot;
                }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* exact rounding (proj/include/ozadp/exactsum.hpp:50-74, 98-158)            */
/* Restated on a little-endian array of 64-bit limbs holding a magnitude.    */
static uint64_t field(const uint64_t* l, int nl, long lo, long hi) {
    if (hi < lo) return 0;
    if (lo < 0) {
        if (hi < 0) return 0;
        return field(l, nl, 0, hi) << (-lo);
    }
    long q = lo >> 6;
    int r = (int)(lo & 63);
    uint64_t v = 0;
    if (q < nl) {
        v = l[q] >> r;
        if (r != 0 && q + 1 < nl) v |= l[q + 1] << (64 - r);
    }
    int width = (int)(hi - lo + 1);
    return width >= 64 ? v : (v & ((((uint64_t)1) << width) - 1));
}
static int any_below(const uint64_t* l, int nl, long idx) {
    if (idx <= 0) return 0;
    long q = idx >> 6;
    int r = (int)(idx & 63);
    for (long i = 0; i < q && i < nl; ++i)
        if (l[i]) return 1;
    if (r != 0 && q < nl && (l[q] & ((((uint64_t)1) << r) - 1))) return 1;
    return 0;
}
static double round_mag(const uint64_t* l, int nl, long exp2, int negative) {
    long top = -1;
    for (int i = nl - 1; i >= 0; --i)
        if (l[i]) { top = (long)i * 64 + (63 - __builtin_clzll(l[i])); break; }
    if (top < 0) return 0.0;
    long e = top + exp2;
    long p = e >= -1022 ? top - 52 : -1074 - exp2;
    uint64_t mm = field(l, nl, p, top);
    int rnd = p - 1 >= 0 && p - 1 <= top && ((l[(p - 1) >> 6] >> ((p - 1) & 63)) & 1);
    int sticky = any_below(l, nl, p - 1);
    if (rnd && (sticky || (mm & 1))) {
        ++mm;
        if (mm == (((uint64_t)1) << 53)) { mm >>= 1; ++p; }
    }
    double r = ldexp((double)mm, (int)(p + exp2));
    return negative ? -r : r;
}

#define WL 12 /* 768-bit two's complement, exactsum.hpp:98-101 */
static void wide_add_shifted(uint64_t* limb, int64_t v, int shift) {
    if (v == 0) return;
    int q = shift >> 6, r = shift & 63;
    u128 a = ((u128)(uint64_t)v) << r;
    uint64_t sext = v < 0 ? ~(uint64_t)0 : 0;
    uint64_t lo = (uint64_t)a;
    uint64_t hi = r == 0 ? sext : ((uint64_t)(a >> 64) | (sext << r));
    u128 t = (u128)limb[q] + lo;
    limb[q] = (uint64_t)t;
    uint64_t carry = (uint64_t)(t >> 64);
    if (q + 1 < WL) {
        t = (u128)limb[q + 1] + hi + carry;
        limb[q + 1] = (uint64_t)t;
        carry = (uint64_t)(t >> 64);
    }
    for (int i = q + 2; i < WL; ++i) {
        t = (u128)limb[i] + sext + carry;
        limb[i] = (uint64_t)t;
        carry = (uint64_t)(t >> 64);
    }
}
static double wide_to_double(const uint64_t* limb, long exp2) {
    uint64_t mag[WL];
    int neg = (limb[WL - 1] >> 63) != 0;
    if (neg) {
        uint64_t carry = 1;
        for (int i = 0; i < WL; ++i) {
            u128 t = (u128)(~limb[i]) + carry;
            mag[i] = (uint64_t)t;
            carry = (uint64_t)(t >> 64);
        }
    } else {
        memcpy(mag, limb, sizeof(mag));
    }
    return round_mag(mag, WL, exp2, neg);
}

double oz_fold_round(const int64_t* acc, int ndiag, long exp2) {
    uint64_t limb[WL] = {0};
    for (int d = 0; d < ndiag; ++d) wide_add_shifted(limb, acc[d], 8 * (ndiag - 1 - d));
    return wide_to_double(limb, exp2);
}

/* igemm.cpp:99-127 */
int oz_recompose(const int64_t* acc, int64_t m, int64_t n, int s, const int32_t* rs,
                 const int32_t* cs, double alpha, double beta, const double* c, double* out) {
    if (beta != 0.0 && !c) return 3;
    int diag = 2 * s - 1, dmax = diag - 1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            long exp2 = (long)rs[i] + cs[j] - 14 - 8 * (long)dmax;
            double v = oz_fold_round(acc + (i * n + j) * diag, diag, exp2);
            double r = alpha * v;
            if (beta != 0.0) r = r + beta * c[i * n + j];
            out[i * n + j] = r;
        }
    return 0;
}

/* igemm.cpp:129-137 */
int oz_emulated_gemm(const double* a, const double* b, int64_t m, int64_t n, int64_t k,
                     double alpha, double beta, const double* c, int slices, int limit,
                     double* out) {
    if (slices < 1 || slices > OZ_MAX_SLICES) return 3;
    if (beta != 0.0 && !c) return 3;
    int8_t* sa = (int8_t*)malloc((size_t)(slices * m * k + 1));
    int8_t* sb = (int8_t*)malloc((size_t)(slices * n * k + 1));
    int32_t* ra = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
    int32_t* cb = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int64_t* acc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m * n * (2 * slices - 1) + 1));
    int rc = oz_decompose(a, m, k, 0, slices, sa, ra);
    if (!rc) rc = oz_decompose(b, k, n, 1, slices, sb, cb);
    if (!rc) rc = oz_slice_pair_mm(sa, sb, m, n, k, slices, limit, acc);
    if (!rc) rc = oz_recompose(acc, m, n, slices, ra, cb, alpha, beta, c, out);
    free(sa); free(sb); free(ra); free(cb); free(acc);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* oracle.cpp:7-28: ascending k, separate multiply and add (no contraction)  */
int oz_native_gemm(const double* a, const double* b, int64_t m, int64_t n, int64_t k,
                   double alpha, double beta, const double* c, double* out) {
    if (beta != 0.0 && !c) return 3;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double sum = 0.0;
            for (int64_t l = 0; l < k; ++l) {
                double p = a[i * k + l] * b[l * n + j];
                sum = sum + p;
            }
            double r = alpha * sum;
            if (beta != 0.0) r = r + beta * c[i * n + j];
            out[i * n + j] = r;
        }
    return 0;
}

/* oracle.cpp:55-75: exact dot products in a fixed-point accumulator wide   */
/* enough for every finite FP64 product (weights 2^-2300 .. 2^2300), one RNE */
#define XL 72
#define XBASE (-2300L)
static void xacc_add(uint64_t* acc, double x, double y) {
    uint64_t bx = f64_bits(x), by = f64_bits(y);
    if ((bx << 1) == 0 || (by << 1) == 0) return;
    u128 p = (u128)normalized_mantissa(bx) * normalized_mantissa(by);
    long w = (long)oz_effective_exponent_bits(bx) + oz_effective_exponent_bits(by) - 104 - XBASE;
    int neg = ((bx ^ by) >> 63) != 0;
    /* add/subtract p << w into the two's complement limb array */
    int q = (int)(w >> 6), r = (int)(w & 63);
    uint64_t part[3];
    part[0] = (uint64_t)(p << r);
    part[1] = r ? (uint64_t)(p >> (64 - r)) : (uint64_t)(p >> 64);
    part[2] = r ? (uint64_t)((p >> 64) >> (64 - r)) : 0;
    if (!neg) {
        uint64_t carry = 0;
        for (int i = q; i < XL; ++i) {
            uint64_t addv = i - q < 3 ? part[i - q] : 0;
            u128 t = (u128)acc[i] + addv + carry;
            acc[i] = (uint64_t)t;
            carry = (uint64_t)(t >> 64);
            if (i - q >= 2 && carry == 0) break;
        }
    } else {
        uint64_t borrow = 0;
        for (int i = q; i < XL; ++i) {
            uint64_t subv = i - q < 3 ? part[i - q] : 0;
            u128 t = (u128)acc[i] - subv - borrow;
            acc[i] = (uint64_t)t;
            borrow = (uint64_t)(t >> 64) ? 1 : 0;
            if (i - q >= 2 && borrow == 0) break;
        }
    }
}
int oz_exact_gemm(const double* a, const double* b, int64_t m, int64_t n, int64_t k,
                  double* out) {
    for (int64_t i = 0; i < m * k; ++i)
        if (raw_exp(f64_bits(a[i])) == 0x7ff) return 3;
    for (int64_t i = 0; i < k * n; ++i)
        if (raw_exp(f64_bits(b[i])) == 0x7ff) return 3;
#pragma omp parallel for schedule(static) collapse(2)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            uint64_t acc[XL];
            memset(acc, 0, sizeof(acc));
            for (int64_t l = 0; l < k; ++l) xacc_add(acc, a[i * k + l], b[l * n + j]);
            int neg = (acc[XL - 1] >> 63) != 0;
            if (neg) {
                uint64_t carry = 1;
                for (int t = 0; t < XL; ++t) {
                    u128 s = (u128)(~acc[t]) + carry;
                    acc[t] = (uint64_t)s;
                    carry = (uint64_t)(s >> 64);
                }
            }
            out[i * n + j] = round_mag(acc, XL, XBASE, neg);
        }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* adp_gemm (proj/src/adp.cpp:139-178)                                       */
int oz_adp_gemm(const double* a, const double* b, int64_t m, int64_t n, int64_t k, double alpha,
                double beta, const double* c, const oz_config* cfg, double* out,
                int64_t trace[10], double* cost_ratio) {
    if (oz_config_validate(cfg)) return 3;
    if (beta != 0.0 && !c) return 3;
    uint64_t ca[3] = {0, 0, 0}, cb[3] = {0, 0, 0};
    int ea = 0, eb = 0;
    if (cfg->mode != 2) {
        oz_scan(a, m * k, ca, &ea);
        oz_scan(b, k * n, cb, &eb);
    }
    /* the ESC provider, evaluated only if decide() reaches it */
    int esc_in = 0, dec[5];
    int64_t mn = m < n ? m : n;
    mn = mn < k ? mn : k;
    int needs_esc = cfg->mode == 0 && !ea && !eb && mn >= cfg->min_dim;
    if (needs_esc) {
        int64_t t = (k + cfg->esc_block_len - 1) / cfg->esc_block_len;
        int32_t* amax = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m * t + 1));
        int32_t* amin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m * t + 1));
        int32_t* alin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m + 1));
        int32_t* bmax = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * t + 1));
        int32_t* bmin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * t + 1));
        int32_t* blin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
        int e3[3];
        oz_block_stats(a, m, k, 0, cfg->esc_block_len, amax, amin, alin);
        oz_block_stats(b, k, n, 1, cfg->esc_block_len, bmax, bmin, blin);
        oz_esc_coarsened(amax, amin, alin, bmax, bmin, blin, m, n, t, cfg->target_bits, e3);
        esc_in = e3[0];
        free(amax); free(amin); free(alin); free(bmax); free(bmin); free(blin);
    }
    oz_decide(ea, eb, m, n, k, esc_in, cfg, dec, cost_ratio);
    trace[0] = dec[0];
    trace[1] = dec[1];
    trace[2] = dec[3] ? dec[4] : -1;
    trace[3] = dec[0] == 0 ? dec[2] : -1;
    for (int i = 0; i < 3; ++i) { trace[4 + i] = (int64_t)ca[i]; trace[7 + i] = (int64_t)cb[i]; }
    if (dec[0] == 0) return oz_emulated_gemm(a, b, m, n, k, alpha, beta, c, dec[2], -1, out);
    return oz_native_gemm(a, b, m, n, k, alpha, beta, c, out);
}

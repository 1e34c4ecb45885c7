// K3: unsigned-integer slicing of FP64 lines into signed int8 digit planes
// (decompose / element_digits / extract_digits / remap_digits,
//  proj/src/slicing.cpp:20-136).
//
// Each line is scaled by E = line_max + 2 (0 for all-zero lines); element v
// becomes the floor fixed-point integer U = floor(v * 2^(7 + 8(s-1) - E)),
// whose base-256 digits (lead signed, the rest unsigned) are exactly the
// reference's extract_digits chain. The reference's least-significant-first
// remap (c > 127 -> c - 256, carry 1) equals adding 0x80 to every sub-leading
// byte: with X = U + 0x8080...80 (s-1 bytes), digit 0 is byte s-1 of X read
// as int8 and digit d >= 1 is byte s-1-d of X xor 0x80. So every plane byte
// is a byte of X: s <= 8 needs one 64-bit integer per element, s <= 16 a
// 128-bit one, s in [17, 32] takes the per-digit restatement of the
// reference. The slice count is a compile-time constant of the inner loop
// (dispatched once per CTA from the device plan), so byte selection is
// static.
//
// Output layouts: "blocked" (the GEMM's TMA layout) stores plane d as
// [k-block of 32][line slot][32 bytes], PRE-SWIZZLED with the UMMA 32-byte
// K-major pattern (16-byte half index ^= bit 2 of the line), so a GEMM stage
// is a plain linear copy of contiguous 4 KiB runs that TMA moves with
// 128-byte requests; "pitched" (stage export) is the reference's plane-major
// [line][len].
//
// HBM-bound: 8 B read + nsl B written per element (+4 B per line).
#include <type_traits>

#include "guard.cuh"

namespace adpb200 {

namespace {

typedef unsigned __int128 u128;
typedef __int128 i128;

template <int S>
struct Word {
    typedef typename std::conditional<(S <= 8), uint64_t, u128>::type T;
};

template <int S>
__device__ __forceinline__ typename Word<S>::T slice_const() {
    typedef typename Word<S>::T T;
    T C = 0;
#pragma unroll
    for (int j = 0; j < S - 1; ++j) C |= T(0x80) << (8 * j);
    return C;
}

// X = floor(v * 2^(7 + 8(S-1) - E)) + 0x80..80 (S <= 16)
template <int S>
__device__ __forceinline__ typename Word<S>::T slice_word(uint64_t bits, int E) {
    typedef typename Word<S>::T T;
    const T C = slice_const<S>();
    if constexpr (S <= 8) {
        // normal numbers, branch-free: with x = M * 2^9 (< 2^62) the net right
        // shift t = st + 9 = (E + 1077 - 8(S-1)) - biased_exp is >= 0 because
        // st >= 47 - 8(S-1) >= -9; floor(-x / 2^t) = ~((x - 1) >> t).
        const uint32_t ex = uint32_t(bits >> 52) & 0x7ffu;
        if (ex != 0) {
            const uint64_t neg = bits >> 63;
            const uint64_t x = ((bits & 0xFFFFFFFFFFFFFull) | (1ull << 52)) << 9;
            int t = E + 1077 - 8 * (S - 1) - int(ex);
            t = t < 63 ? t : 63;  // (x - neg) < 2^62: a shift of 63 already gives 0
            const uint64_t q = (x - neg) >> t;
            return (q ^ (0ull - neg)) + C;
        }
    }
    if ((bits << 1) == 0) return C;
    const bool neg = (bits >> 63) != 0;
    const uint64_t M = norm_mant(bits);
    const int e = eff_exp(bits);
    const int st = 45 + E - e - 8 * (S - 1);  // net right shift of the 53-bit mantissa
    T U;
    if (st >= 0) {
        const uint64_t q = st >= 64 ? 0ull : ((neg ? M - 1 : M) >> st);
        U = neg ? ~T(q) : T(q);  // floor(-M 2^-st) = ~((M-1) >> st)
    } else {
        const T w = T(M) << (-st);  // exact: -st <= 8(S-1) - 47
        U = neg ? T(0) - w : w;
    }
    return U + C;
}

// The same words for 16 elements through the FP64 pipe: U = floor(v * 2^p),
// p = 7 + 8(S-1) - E, is one exact multiply by a power of two (|v 2^p| < 2^(8S-2)
// cannot overflow, and p >= 0 cannot lose bits) and one round-toward--inf
// conversion. Zeros (either sign) give U = 0 like the integer path. Taken when
// 0 <= p <= 1023 (lines whose maximum exponent is below 8S, i.e. every line of
// data scaled anywhere near 1) and all 16 elements are finite; otherwise the
// caller runs slice_word.
template <int S>
__device__ __forceinline__ bool fast_words(const uint64_t (&bits)[16], int E, uint64_t (&X)[16]) {
    // p >= 0: v 2^p is exact for every finite v (normal or not, no underflow), so
    // the only per-element test is "finite": the largest exponent field < 2047
    const int p = 7 + 8 * (S - 1) - E;
    if (p < 0 || p > 1023) return false;
    uint32_t exmax = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) exmax = max(exmax, uint32_t(bits[q] >> 32) & 0x7ff00000u);
    if (exmax == 0x7ff00000u) return false;
    const double sc = __longlong_as_double(int64_t(p + 1023) << 52);
    const uint64_t C = slice_const<S>();
#pragma unroll
    for (int q = 0; q < 16; ++q)
        X[q] = uint64_t(__double2ll_rd(__dmul_rn(__longlong_as_double(int64_t(bits[q])), sc))) + C;
    return true;
}

// S in 9..16, 8 elements, through the FP64 pipe as well: with f = |v| 2^(p-64) (exact,
// p >= 64), H = floor(f), r = f - H (exact for f >= 0) and L = floor(r 2^64) (r 2^64 is
// exact), |v| 2^p = H 2^64 + L + frac; U = H:L for v >= 0, and for v < 0 floor gives
// -(H:L) when frac = 0, else -(H:L) - 1 = ~(H:L). Taken when 64 <= p <= 1087 and all 8
// elements are finite; otherwise the caller runs slice_word.
template <int S>
__device__ __forceinline__ bool fast_words_w(const uint64_t* bits, int E, uint32_t (&W)[8][4]) {
    const int p = 7 + 8 * (S - 1) - E;
    if (p < 64 || p > 64 + 1023) return false;
    uint32_t exmax = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) exmax = max(exmax, uint32_t(bits[q] >> 32) & 0x7ff00000u);
    if (exmax == 0x7ff00000u) return false;
    const double sc = __longlong_as_double(int64_t(p - 64 + 1023) << 52);
    const u128 C = slice_const<S>();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const double f = __dmul_rn(__longlong_as_double(int64_t(bits[q] & 0x7fffffffffffffffull)), sc);
        const double hd = floor(f);
        const double ld = __dmul_rn(__dsub_rn(f, hd), 18446744073709551616.0);  // r 2^64
        const double lf = floor(ld);
        u128 U = (u128(uint64_t(hd)) << 64) | u128(uint64_t(lf));
        if (bits[q] >> 63) U = lf != ld ? ~U : u128(0) - U;
        const u128 X = U + C;
#pragma unroll
        for (int i = 0; i < 4; ++i) W[q][i] = uint32_t(X >> (32 * i));
    }
    return true;
}

// Every plane's bytes of 8 elements X[0..7] (S <= 8) into w[d][o], w[d][o + 1].
// Bytes j and j + 1 (j even) of X live in the same 32-bit half, so one byte
// permute per element pair serves two planes: t = (x_j, y_j, x_j+1, y_j+1), then
// two permutes per plane merge the four pairs (0.5 permutes per plane byte).
template <int S>
__device__ __forceinline__ void pack_planes(const uint64_t* X, uint32_t (&w)[S][4], int o) {
#pragma unroll
    for (int j = 0; j < S; j += 2) {
        uint32_t h[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) h[q] = j < 4 ? uint32_t(X[q]) : uint32_t(X[q] >> 32);
        const uint32_t b = uint32_t(j & 3);
        const int d = S - 1 - j;  // plane of byte j; byte j + 1 is plane d - 1
        if (j + 1 < S) {
            const uint32_t sel = b | ((4 + b) << 4) | ((b + 1) << 8) | ((5 + b) << 12);
            const uint32_t t0 = __byte_perm(h[0], h[1], sel), t1 = __byte_perm(h[2], h[3], sel);
            const uint32_t t2 = __byte_perm(h[4], h[5], sel), t3 = __byte_perm(h[6], h[7], sel);
            w[d][o] = __byte_perm(t0, t1, 0x5410);
            w[d][o + 1] = __byte_perm(t2, t3, 0x5410);
            const uint32_t f = d - 1 != 0 ? 0x80808080u : 0u;  // sub-leading digits: byte ^ 0x80
            w[d - 1][o] = __byte_perm(t0, t1, 0x7632) ^ f;
            w[d - 1][o + 1] = __byte_perm(t2, t3, 0x7632) ^ f;
        } else {  // the top byte alone (odd S): the lead digit, plane 0
            const uint32_t sel = b | ((4 + b) << 4);
            w[d][o] = __byte_perm(__byte_perm(h[0], h[1], sel), __byte_perm(h[2], h[3], sel), 0x5410);
            w[d][o + 1] = __byte_perm(__byte_perm(h[4], h[5], sel), __byte_perm(h[6], h[7], sel), 0x5410);
        }
        if (d != 0) {
            w[d][o] ^= 0x80808080u;
            w[d][o + 1] ^= 0x80808080u;
        }
    }
}

// The same for S in 9..16 from four 32-bit words per element (byte j of X in word j/4).
template <int S>
__device__ __forceinline__ void pack_planes_w(const uint32_t (&W)[8][4], uint32_t (&w)[S][2]) {
#pragma unroll
    for (int j = 0; j < S; j += 2) {
        uint32_t h[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) h[q] = W[q][j >> 2];
        const uint32_t b = uint32_t(j & 3);
        const int d = S - 1 - j;
        if (j + 1 < S) {
            const uint32_t sel = b | ((4 + b) << 4) | ((b + 1) << 8) | ((5 + b) << 12);
            const uint32_t t0 = __byte_perm(h[0], h[1], sel), t1 = __byte_perm(h[2], h[3], sel);
            const uint32_t t2 = __byte_perm(h[4], h[5], sel), t3 = __byte_perm(h[6], h[7], sel);
            const uint32_t f = d - 1 != 0 ? 0x80808080u : 0u;
            w[d][0] = __byte_perm(t0, t1, 0x5410) ^ (d != 0 ? 0x80808080u : 0u);
            w[d][1] = __byte_perm(t2, t3, 0x5410) ^ (d != 0 ? 0x80808080u : 0u);
            w[d - 1][0] = __byte_perm(t0, t1, 0x7632) ^ f;
            w[d - 1][1] = __byte_perm(t2, t3, 0x7632) ^ f;
        } else {
            const uint32_t sel = b | ((4 + b) << 4);
            w[d][0] = __byte_perm(__byte_perm(h[0], h[1], sel), __byte_perm(h[2], h[3], sel), 0x5410);
            w[d][1] = __byte_perm(__byte_perm(h[4], h[5], sel), __byte_perm(h[6], h[7], sel), 0x5410);
            if (d != 0) {
                w[d][0] ^= 0x80808080u;
                w[d][1] ^= 0x80808080u;
            }
        }
    }
}

// Reference-form restatement for any s <= 32 (slicing.cpp:11-66).
__device__ __forceinline__ uint32_t byte_window(uint64_t x, int a) {
    if (a >= 64 || a <= -8) return 0;
    if (a >= 0) return uint32_t(x >> a) & 0xffu;
    return uint32_t(x << -a) & 0xffu;
}
__device__ void slice_digits_slow(uint64_t bits, int E, int s, int8_t* out) {
    if ((bits << 1) == 0) {
        for (int d = 0; d < s; ++d) out[d] = 0;
        return;
    }
    const bool neg = (bits >> 63) != 0;
    const uint64_t M = norm_mant(bits);
    const int e = eff_exp(bits);
    const int sh = 45 + E - e;
    int32_t lead;
    uint8_t sub[kMaxSlices];
    if (!neg) {
        lead = sh < 64 ? int32_t(M >> sh) : 0;
        for (int d = 1; d < s; ++d) sub[d - 1] = uint8_t(byte_window(M, sh - 8 * d));
    } else {
        const uint64_t Mm1 = M - 1;
        lead = sh < 64 ? -int32_t(Mm1 >> sh) - 1 : -1;
        for (int d = 1; d < s; ++d) {
            int a = sh - 8 * d;
            uint32_t mask = a >= 0 ? 0xffu : (a <= -8 ? 0u : (0xffu << -a) & 0xffu);
            sub[d - 1] = uint8_t(~byte_window(Mm1, a) & mask);
        }
    }
    int carry = 0;
    for (int d = s - 1; d >= 1; --d) {
        int c = sub[d - 1] + carry;
        if (c <= 127) {
            out[d] = int8_t(c);
            carry = 0;
        } else {
            out[d] = int8_t(c - 256);
            carry = 1;
        }
    }
    out[0] = int8_t(lead + carry);
}

struct SliceArgs {
    LineView v;
    const int32_t* line_max;
    int8_t* planes;
    int64_t pitch;         // pitched: bytes between lines; blocked: line slots per k-block
    int64_t plane_stride;  // bytes between planes
    int blocked;           // 1: [d][kb][line][32]
    int32_t* scale;
    const Plan* plan;
    int slices_fixed;
    int indicator;         // certified ESC: plan->nsl planes of (e >= line_max - delta) bytes,
                           // delta = plan->aux (plane 0) / plan->aux2 (plane 1)
    int plane_cap;         // planes the buffer holds (> 0): digit planes past it are not stored
};

// Certified-ESC indicator bytes of 8 elements: 1 where the element is finite,
// nonzero and its effective exponent is within delta of the line maximum.
__device__ __forceinline__ void indicator_bytes(const uint64_t* bits, int lm, int delta, uint32_t& lo, uint32_t& hi) {
    lo = hi = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint64_t b = bits[q];
        const bool on = (b << 1) != 0 && ((b >> 52) & 0x7ff) != 0x7ff && eff_exp(b) >= lm - delta;
        if (q < 4) lo |= uint32_t(on) << (8 * q);
        else hi |= uint32_t(on) << (8 * (q - 4));
    }
}

// byte offset of (d, line, pos) inside the planes
__device__ __forceinline__ int64_t plane_off(const SliceArgs& a, int d, int64_t line, int64_t pos) {
    if (a.blocked)  // SW32: the 16-byte half of a 32-byte row flips on bit 2 of the row (line)
        return int64_t(d) * a.plane_stride + ((pos >> 5) * a.pitch + line) * 32 + ((pos & 31) ^ ((line & 4) << 2));
    return int64_t(d) * a.plane_stride + line * a.pitch + pos;
}

__device__ __forceinline__ bool resolve(const SliceArgs& a, int& s, int& nsl) {
    if (a.slices_fixed > 0) {
        s = a.slices_fixed;
        nsl = s;
    } else {
        if (a.plan->path != ADPB200_PATH_EMULATED) return false;
        s = a.plan->slices;
        nsl = a.plan->nsl;
    }
    // a fixed s with a pair limit L only uses planes 0..L (the buffer holds L + 1)
    if (!a.indicator && a.plane_cap > 0 && nsl > a.plane_cap) nsl = a.plane_cap;
    return true;
}

// Plane d's bytes of positions p0 .. p0 + nvalid - 1 (p0 a multiple of 16, so in
// the blocked layout they sit in one 16-byte half-row): one 128-bit store when
// all 16 are there and the address allows it, byte stores otherwise.
__device__ __forceinline__ void put16(const SliceArgs& a, int d, int64_t line, int64_t p0, int nvalid, uint32_t w0,
                                      uint32_t w1, uint32_t w2, uint32_t w3) {
    int8_t* out = a.planes + plane_off(a, d, line, p0);
    if (nvalid >= 16 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
        *reinterpret_cast<uint4*>(out) = make_uint4(w0, w1, w2, w3);
        return;
    }
    const uint64_t lo = uint64_t(w0) | (uint64_t(w1) << 32), hi = uint64_t(w2) | (uint64_t(w3) << 32);
    for (int q = 0; q < nvalid && q < 16; ++q) out[q] = int8_t((q < 8 ? lo : hi) >> (8 * (q & 7)));
}
// the same for 8 positions (p0 a multiple of 8)
__device__ __forceinline__ void put8(const SliceArgs& a, int d, int64_t line, int64_t p0, int nvalid, uint32_t lo,
                                     uint32_t hi) {
    int8_t* out = a.planes + plane_off(a, d, line, p0);
    if (nvalid >= 8 && (reinterpret_cast<uintptr_t>(out) & 7) == 0) {
        *reinterpret_cast<uint2*>(out) = make_uint2(lo, hi);
        return;
    }
    const uint64_t w = uint64_t(lo) | (uint64_t(hi) << 32);
    for (int q = 0; q < nvalid && q < 8; ++q) out[q] = int8_t(w >> (8 * q));
}

// All planes of 16 consecutive positions of one line (nvalid of them inside the
// plane span). S = 0: the certified-ESC indicator planes; S <= 8: one 64-bit
// word per element, one 128-bit store per plane; S <= 16: 128-bit words, two
// halves of 8; S = 32: the reference-form restatement per element.
template <int S>
__device__ __forceinline__ void emit16(const SliceArgs& a, int nsl, const uint64_t (&bits)[16], int E, int lm,
                                       int64_t line, int64_t p0, int nvalid) {
    if constexpr (S == 0) {
        for (int d = 0; d < nsl; ++d) {
            const int delta = d == 0 ? a.plan->aux : a.plan->aux2;
            uint32_t w0, w1, w2, w3;
            indicator_bytes(bits, lm, delta, w0, w1);
            indicator_bytes(bits + 8, lm, delta, w2, w3);
            put16(a, d, line, p0, nvalid, w0, w1, w2, w3);
        }
    } else if constexpr (S <= 8) {
        uint64_t X[16];
        if (!fast_words<S>(bits, E, X)) {
#pragma unroll
            for (int q = 0; q < 16; ++q) X[q] = slice_word<S>(bits[q], E);
        }
        uint32_t w[S][4];  // plane d: bytes of positions 0-3, 4-7, 8-11, 12-15
        pack_planes<S>(X, w, 0);
        pack_planes<S>(X + 8, w, 2);
        // plane d's 16 bytes sit at base + d * plane_stride: one address, one alignment test
        int8_t* out = a.planes + plane_off(a, 0, line, p0);
        const bool v16 = nvalid >= 16 && ((reinterpret_cast<uintptr_t>(out) | uintptr_t(a.plane_stride)) & 15) == 0;
        if (v16 && nsl == S) {  // the hot path: straight-line 128-bit stores
#pragma unroll
            for (int d = 0; d < S; ++d) {
                *reinterpret_cast<uint4*>(out) = make_uint4(w[d][0], w[d][1], w[d][2], w[d][3]);
                out += a.plane_stride;
            }
        } else {
#pragma unroll
            for (int d = 0; d < S; ++d) {
                if (d >= nsl) break;
                if (v16) {
                    *reinterpret_cast<uint4*>(out) = make_uint4(w[d][0], w[d][1], w[d][2], w[d][3]);
                } else {
                    const uint64_t lo = uint64_t(w[d][0]) | (uint64_t(w[d][1]) << 32);
                    const uint64_t hi = uint64_t(w[d][2]) | (uint64_t(w[d][3]) << 32);
                    for (int q = 0; q < nvalid && q < 16; ++q) out[q] = int8_t((q < 8 ? lo : hi) >> (8 * (q & 7)));
                }
                out += a.plane_stride;
            }
        }
    } else if constexpr (S <= 16) {
        // two halves of 8 elements: 128-bit words, split into four 32-bit words each and
        // gathered into the planes with the same paired byte permutes as S <= 8; one
        // 16-byte store per plane once both halves are packed
        auto half_words = [&](int h, uint32_t (&wh)[S][2]) {
            uint32_t W[8][4];
            if (!fast_words_w<S>(bits + 8 * h, E, W)) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const u128 X = slice_word<S>(bits[8 * h + q], E);
#pragma unroll
                    for (int i = 0; i < 4; ++i) W[q][i] = uint32_t(X >> (32 * i));
                }
            }
            pack_planes_w<S>(W, wh);
        };
        int8_t* out = a.planes + plane_off(a, 0, line, p0);
        if constexpr (S > 12) {
            // (more planes than registers for both halves: 8-byte stores per half)
            const bool v8 = ((reinterpret_cast<uintptr_t>(out) | uintptr_t(a.plane_stride)) & 7) == 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (8 * h >= nvalid) break;
                uint32_t wh[S][2];
                half_words(h, wh);
                const int nv = nvalid - 8 * h;
                int8_t* o = out + 8 * h;
#pragma unroll
                for (int d = 0; d < S; ++d) {
                    if (d >= nsl) break;
                    if (v8 && nv >= 8) {
                        *reinterpret_cast<uint2*>(o) = make_uint2(wh[d][0], wh[d][1]);
                    } else {
                        const uint64_t x = uint64_t(wh[d][0]) | (uint64_t(wh[d][1]) << 32);
                        for (int q = 0; q < nv && q < 8; ++q) o[q] = int8_t(x >> (8 * q));
                    }
                    o += a.plane_stride;
                }
            }
            return;
        }
        uint32_t w[S][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t wh[S][2];
            half_words(h, wh);
#pragma unroll
            for (int d = 0; d < S; ++d) {
                w[d][2 * h] = wh[d][0];
                w[d][2 * h + 1] = wh[d][1];
            }
        }
        const bool v16 = nvalid >= 16 && ((reinterpret_cast<uintptr_t>(out) | uintptr_t(a.plane_stride)) & 15) == 0;
#pragma unroll
        for (int d = 0; d < S; ++d) {
            if (d >= nsl) break;
            if (v16) {
                *reinterpret_cast<uint4*>(out) = make_uint4(w[d][0], w[d][1], w[d][2], w[d][3]);
            } else {
                const uint64_t lo = uint64_t(w[d][0]) | (uint64_t(w[d][1]) << 32);
                const uint64_t hi = uint64_t(w[d][2]) | (uint64_t(w[d][3]) << 32);
                for (int q = 0; q < nvalid && q < 16; ++q) out[q] = int8_t((q < 8 ? lo : hi) >> (8 * (q & 7)));
            }
            out += a.plane_stride;
        }
    } else {
        int8_t dig[kMaxSlices];
        const int s = a.slices_fixed > 0 ? a.slices_fixed : a.plan->slices;
        for (int q = 0; q < nvalid && q < 16; ++q) {
            slice_digits_slow(bits[q], E, s, dig);
            for (int d = 0; d < nsl; ++d) a.planes[plane_off(a, d, line, p0 + q)] = dig[d];
        }
    }
}

// ---- the staged tile pipeline ------------------------------------------------------------
// A CTA owns tiles of 4096 elements (32 KiB of FP64): rows variant (positions
// contiguous, ps == 1) 32 lines x 128 positions, cols variant (any strides; lines
// adjacent when ls == 1) 128 lines x one k-block of 32 positions. Tiles are
// copied HBM -> shared memory with cp.async in fully coalesced 16-byte chunks
// (8 B per element when the addresses do not allow 16), kStages deep, so the
// copies of the next tiles are in flight while the current one is sliced.
// Out-of-range elements are zero-filled by the copy (src-size 0). Each thread
// then slices 16 consecutive positions of one line out of shared memory and
// stores one 16-byte chunk per plane: per plane a warp writes 4 x 128 B (rows)
// or 512 contiguous bytes (cols) of the blocked layout. Consecutive tiles walk
// the lines first, so the CTAs in flight fill whole k-blocks.
constexpr int kRowsLines = 32, kRowsPos = 128;  // rows tile
constexpr int kColsLines = 128, kColsPos = 32;  // cols tile
constexpr int kTileElems = 4096;
#ifndef ADPB200_SLICE_STAGES
#define ADPB200_SLICE_STAGES 2
#endif
constexpr int kStages = ADPB200_SLICE_STAGES;
constexpr size_t kSliceSmem = size_t(kStages) * kTileElems * 8;

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp8(uint32_t dst, const void* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// rows stage: [line 32][16-byte chunk 64], chunk c of a line stored at c ^ ((c >> 3) & 7),
// so the 8 lanes of a quarter-warp reading chunk 8g + q (g = 0..7) hit 8 distinct bank groups
__device__ __forceinline__ int rows_chunk(int c) { return c ^ ((c >> 3) & 7); }

// Tile coordinates (line tile, position tile), walked lines first; a thread
// advances them by gridDim.x tiles with one add and one carry (no 64-bit divisions).
struct TileIdx {
    int64_t lt, pt;
};

template <bool kRows, bool kVec>
struct Tiler {
    static constexpr int kL = kRows ? kRowsLines : kColsLines;
    static constexpr int kP = kRows ? kRowsPos : kColsPos;
    const SliceArgs& a;
    int64_t nlt, npt, glt, gpt;  // tiles along lines / positions; the CTA count as (lines, positions) step
    int64_t cta;
    __device__ __forceinline__ Tiler(const SliceArgs& a_, int64_t span, int cta_, int nctas) : a(a_), cta(cta_) {
        nlt = (a.v.lines + kL - 1) / kL;
        npt = (span + kP - 1) / kP;
        gpt = int64_t(nctas) / nlt;
        glt = int64_t(nctas) - gpt * nlt;
    }
    __device__ __forceinline__ TileIdx first() const {
        const int64_t pt = cta / nlt;
        return TileIdx{cta - pt * nlt, pt};
    }
    __device__ __forceinline__ void step(TileIdx& t) const {
        t.lt += glt;
        t.pt += gpt;
        if (t.lt >= nlt) {
            t.lt -= nlt;
            ++t.pt;
        }
    }
    __device__ __forceinline__ bool valid(const TileIdx& t) const { return t.pt < npt; }
    // issue the copies of tile t into the stage at shared address s
    __device__ __forceinline__ void issue(const TileIdx& t, uint32_t s) const {
        const int64_t l0 = t.lt * kL, p0 = t.pt * kP;
        const int tid = threadIdx.x;
        if (kVec) {
            // 2048 chunks of 16 B (two elements adjacent in memory), 8 per thread:
            // chunk column c = tid % 64 fixed, rows r = tid / 64 + 4 i
            const int c = tid & 63, r0 = tid >> 6;
            // (the per-chunk test is one 32-bit compare against what is left of the tile)
            if (kRows) {  // a warp: 32 consecutive chunks (512 B) of one line
                const int64_t pos = p0 + 2 * c;
                const int bytes = pos < a.v.len ? (pos + 1 < a.v.len ? 16 : 8) : 0;
                const int64_t left64 = a.v.lines - (l0 + r0);
                const int left = left64 < 32 ? int(left64) : 32;
                const double* src = a.v.ptr + (l0 + r0) * a.v.ls + pos;
                const int64_t dl = 4 * a.v.ls;
                const uint32_t dst = s + uint32_t(r0 * 64 + rows_chunk(c)) * 16u;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int nb = 4 * i < left ? bytes : 0;
                    cp16(dst + i * (4u * 64u * 16u), nb ? src : a.v.ptr, nb);
                    src += dl;
                }
            } else {      // a warp: 64 adjacent lines at one position (512 contiguous bytes)
                const int64_t line = l0 + 2 * c;
                const int bytes = line < a.v.lines ? (line + 1 < a.v.lines ? 16 : 8) : 0;
                const int64_t left64 = a.v.len - (p0 + r0);
                const int left = left64 < 32 ? int(left64) : 32;
                const double* src = a.v.ptr + line + (p0 + r0) * a.v.ps;
                const int64_t dp = 4 * a.v.ps;
                const uint32_t dst = s + uint32_t(r0 * kColsLines + 2 * c) * 8u;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int nb = 4 * i < left ? bytes : 0;
                    cp16(dst + i * (4u * kColsLines * 8u), nb ? src : a.v.ptr, nb);
                    src += dp;
                }
            }
        } else {
            // 4096 elements of 8 B, 16 per thread, any strides
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int e = tid + 256 * i;
                int64_t line, pos;
                uint32_t off;
                if (kRows) {
                    const int r = e >> 7, q = e & 127;
                    line = l0 + r;
                    pos = p0 + q;
                    off = uint32_t(r * 64 + rows_chunk(q >> 1)) * 16u + uint32_t(q & 1) * 8u;
                } else {
                    const int r = e >> 7, l = e & 127;
                    line = l0 + l;
                    pos = p0 + r;
                    off = uint32_t(r * kColsLines + l) * 8u;
                }
                const bool ok = line < a.v.lines && pos < a.v.len;
                cp8(s + off, ok ? a.v.ptr + line * a.v.ls + pos * a.v.ps : a.v.ptr, ok ? 8 : 0);
            }
        }
    }
    // this thread's line and first position inside a tile
    __device__ __forceinline__ void mine(int& lsub, int& psub) const {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (kRows) {
            lsub = warp * 4 + (lane >> 3);
            psub = (lane & 7) * 16;
        } else {
            lsub = warp * 16 + (lane >> 1);
            psub = (lane & 1) * 16;
        }
    }
    // its 16 elements out of a stage
    __device__ __forceinline__ void read(const char* stage, int lsub, int psub, uint64_t (&bits)[16]) const {
        if (kRows) {
            const int c0 = psub >> 1;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint4 v = *reinterpret_cast<const uint4*>(stage + (lsub * 64 + rows_chunk(c0 + q)) * 16);
                bits[2 * q] = uint64_t(v.x) | (uint64_t(v.y) << 32);
                bits[2 * q + 1] = uint64_t(v.z) | (uint64_t(v.w) << 32);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 16; ++q)
                bits[q] = *reinterpret_cast<const uint64_t*>(stage + ((psub + q) * kColsLines + lsub) * 8);
        }
    }
};

template <int S, bool kRows, bool kVec>
__device__ __forceinline__ void staged_body(const SliceArgs& a, int nsl, int64_t span, char* smem, int cta,
                                            int nctas) {
    const Tiler<kRows, kVec> T(a, span, cta, nctas);
    const uint32_t s0 = uint32_t(__cvta_generic_to_shared(smem));
    int lsub, psub;
    T.mine(lsub, psub);
    TileIdx cur = T.first(), ahead = cur;
#pragma unroll
    for (int st = 0; st < kStages - 1; ++st) {
        if (T.valid(ahead)) T.issue(ahead, s0 + uint32_t(st) * kTileElems * 8u);
        cp_commit();
        T.step(ahead);
    }
    for (int it = 0; T.valid(cur); T.step(cur), ++it) {
        // keep kStages - 1 tiles in flight: the copy of iteration it + kStages - 1
        if (T.valid(ahead)) T.issue(ahead, s0 + uint32_t((it + kStages - 1) % kStages) * kTileElems * 8u);
        cp_commit();
        T.step(ahead);
        cp_wait<kStages - 1>();
        __syncthreads();  // every thread's copies of this tile have landed
        const int64_t line = cur.lt * T.kL + lsub, pos = cur.pt * T.kP + psub;
        if (line < a.v.lines && pos < span) {
            uint64_t bits[16];
            T.read(smem + size_t(it % kStages) * kTileElems * 8, lsub, psub, bits);
            const int lm = a.line_max[line];
            const int E = lm == kNegSentinel ? 0 : lm + 2;
            if (pos == 0 && a.scale) a.scale[line] = E;
            const int nvalid = span - pos < 16 ? int(span - pos) : 16;
            emit16<S>(a, nsl, bits, E, lm, line, pos, nvalid);
        }
        __syncthreads();  // the stage is free for the copy issued next iteration
    }
    cp_wait<0>();
}

// one operand's slicing by CTAs cta = 0..nctas-1 of the grid
template <bool kRows, bool kVec>
__device__ __forceinline__ void slice_operand(const SliceArgs& a, char* smem, int cta, int nctas) {
    int s, nsl;
    if (!resolve(a, s, nsl)) return;
    // blocked planes are zero-filled up to the 32-byte k-block
    const int64_t span = a.blocked ? (a.v.len + 31) / 32 * 32 : a.v.len;
    if (a.indicator) {
        staged_body<0, kRows, kVec>(a, nsl, span, smem, cta, nctas);
        return;
    }
    switch (s) {
#define ADPB200_SLICE_CASE(S) \
    case S: staged_body<S, kRows, kVec>(a, nsl, span, smem, cta, nctas); break;
        ADPB200_SLICE_CASE(1) ADPB200_SLICE_CASE(2) ADPB200_SLICE_CASE(3) ADPB200_SLICE_CASE(4)
        ADPB200_SLICE_CASE(5) ADPB200_SLICE_CASE(6) ADPB200_SLICE_CASE(7) ADPB200_SLICE_CASE(8)
        ADPB200_SLICE_CASE(9) ADPB200_SLICE_CASE(10) ADPB200_SLICE_CASE(11) ADPB200_SLICE_CASE(12)
        ADPB200_SLICE_CASE(13) ADPB200_SLICE_CASE(14) ADPB200_SLICE_CASE(15) ADPB200_SLICE_CASE(16)
#undef ADPB200_SLICE_CASE
        default: staged_body<32, kRows, kVec>(a, nsl, span, smem, cta, nctas); break;
    }
}

template <bool kRows, bool kVec>
__global__ void __launch_bounds__(256, 3) slice_kernel(SliceArgs a) {
    pdl_enter();
    extern __shared__ __align__(16) char smem[];
    slice_operand<kRows, kVec>(a, smem, blockIdx.x, gridDim.x);
}

// Both operands in one launch (the common layout: A-lines with adjacent lines,
// B-lines contiguous): CTAs [0, grid_a) slice A, the rest B. At small sizes one
// operand alone does not fill the SMs' slots and the second launch is one more
// kernel boundary on the call's critical path.
__global__ void __launch_bounds__(256, 3) slice_pair_kernel(SliceArgs a, SliceArgs b, int grid_a) {
    pdl_enter();
    extern __shared__ __align__(16) char smem[];
    if (int(blockIdx.x) < grid_a) slice_operand<false, true>(a, smem, blockIdx.x, grid_a);
    else slice_operand<true, true>(b, smem, int(blockIdx.x) - grid_a, int(gridDim.x) - grid_a);
}

using SliceFn = void (*)(SliceArgs);

// resident CTAs per SM of a slicing kernel (the grids are persistent)
int resident(SliceFn fn) {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kSliceSmem));
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, kSliceSmem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    return per_sm;
}

}  // namespace

namespace {
struct SlicePrep {
    SliceArgs a;
    int which;      // 0 cols, 1 cols 16-byte, 2 rows, 3 rows 16-byte
    int64_t tiles;  // 0: nothing to do
};

const SliceFn kSliceFns[4] = {slice_kernel<false, false>, slice_kernel<false, true>, slice_kernel<true, false>,
                              slice_kernel<true, true>};

int slice_resident(int which) {  // which 4 = the paired kernel
    static int res[5] = {0, 0, 0, 0, 0};
    if (!res[0]) {
        for (int i = 0; i < 4; ++i) res[i] = resident(kSliceFns[i]);
        cudaFuncSetAttribute(reinterpret_cast<const void*>(slice_pair_kernel),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSliceSmem));
        int per_sm = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, slice_pair_kernel, 256, kSliceSmem) !=
                cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
        res[4] = per_sm;
    }
    return res[which];
}

SlicePrep prep_slice(const LineView& v, const int32_t* line_max, int8_t* planes, int64_t pitch, int64_t plane_stride,
                     int blocked, int32_t* scale, const Plan* plan, int slices_fixed, int indicator, int plane_cap) {
    SlicePrep p{
        SliceArgs{v, line_max, planes, pitch, plane_stride, blocked, scale, plan, slices_fixed, indicator, plane_cap},
        0, 0};
    const int64_t span = blocked ? (v.len + 31) / 32 * 32 : v.len;
    if (v.lines == 0 || span == 0) return p;
    const bool aligned = (reinterpret_cast<uintptr_t>(v.ptr) & 15) == 0;
    if (v.ps == 1 || v.len == 1) {
        if (v.lines == 1) p.a.v.ls = 0;
        p.which = 2 + ((aligned && (p.a.v.ls & 1) == 0) ? 1 : 0);  // 16-byte chunks need even line starts
        p.tiles = (v.lines + kRowsLines - 1) / kRowsLines * ((span + kRowsPos - 1) / kRowsPos);
    } else {
        p.which = (aligned && v.ls == 1 && (v.ps & 1) == 0) ? 1 : 0;  // two adjacent lines per 16-byte chunk
        p.tiles = (v.lines + kColsLines - 1) / kColsLines * ((span + kColsPos - 1) / kColsPos);
    }
    return p;
}

void launch_prepped(const SlicePrep& p, cudaStream_t st, uint64_t* nlaunch) {
    if (!p.tiles) return;
    const int64_t cap = int64_t(num_sms()) * slice_resident(p.which);
    const int grid = int(p.tiles < cap ? p.tiles : cap);
    launch_chain(kSliceFns[p.which], dim3(grid), dim3(256), kSliceSmem, st, p.a);
    ++*nlaunch;
}
}  // namespace

void launch_slice(const LineView& v, const int32_t* line_max, int8_t* planes, int64_t pitch, int64_t plane_stride,
                  int blocked, int32_t* scale, const Plan* plan, int slices_fixed, int plane_cap, cudaStream_t st,
                  uint64_t* nlaunch, int indicator) {
    launch_prepped(
        prep_slice(v, line_max, planes, pitch, plane_stride, blocked, scale, plan, slices_fixed, indicator, plane_cap),
        st, nlaunch);
}

void launch_slice_pair(const SliceOperand& A, const SliceOperand& B, int blocked, const Plan* plan, int slices_fixed,
                       int plane_cap, cudaStream_t st, uint64_t* nlaunch) {
    const SlicePrep pa = prep_slice(A.v, A.line_max, A.planes, A.pitch, A.plane_stride, blocked, A.scale, plan,
                                    slices_fixed, 0, plane_cap);
    const SlicePrep pb = prep_slice(B.v, B.line_max, B.planes, B.pitch, B.plane_stride, blocked, B.scale, plan,
                                    slices_fixed, 0, plane_cap);
    static const bool paired = [] {
        const char* e = getenv("ADPB200_SLICE_PAIR");
        return !e || atoi(e) != 0;
    }();
    if (!paired || !pa.tiles || !pb.tiles || pa.which != 1 || pb.which != 3) {
        launch_prepped(pa, st, nlaunch);
        launch_prepped(pb, st, nlaunch);
        return;
    }
    // split the persistent grid in proportion to the tiles (each part at least one CTA)
    const int64_t cap = int64_t(num_sms()) * slice_resident(4);
    int64_t ga = pa.tiles, gb = pb.tiles;
    if (ga + gb > cap) {
        ga = (cap * pa.tiles + (pa.tiles + pb.tiles) / 2) / (pa.tiles + pb.tiles);
        ga = ga < 1 ? 1 : (ga > cap - 1 ? cap - 1 : ga);
        gb = cap - ga;
        if (ga > pa.tiles) ga = pa.tiles;
        if (gb > pb.tiles) gb = pb.tiles;
    }
    launch_chain(slice_pair_kernel, dim3(unsigned(ga + gb)), dim3(256), kSliceSmem, st, pa.a, pb.a, int(ga));
    ++*nlaunch;
}

namespace {

// One 16-byte chunk per thread: (rank, plane, k-block, local line, half).
__global__ void gather_planes_kernel(const int8_t* __restrict__ recs, int64_t rec_bytes, int64_t hdr, int world,
                                     int r_first, int64_t nr, int64_t nkb, int nsl, int8_t* __restrict__ planes,
                                     int64_t slots, int64_t plane_stride, int32_t* __restrict__ scale) {
    const int64_t per_rank = int64_t(nsl) * nkb * nr * 2;
    const int64_t total = per_rank * world;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / per_rank;
        int64_t x = e - r * per_rank;
        const int64_t half = x & 1;
        x >>= 1;
        const int64_t jl = x % nr;
        x /= nr;
        const int64_t kb = x % nkb;
        const int64_t d = x / nkb;
        const uint4 v = *reinterpret_cast<const uint4*>(recs + r * rec_bytes + hdr + ((d * nkb + kb) * nr + jl) * 32 +
                                                        half * 16);
        *reinterpret_cast<uint4*>(planes + d * plane_stride + (kb * slots + (r_first + r) * nr + jl) * 32 + half * 16) =
            v;
    }
    const int64_t ns = int64_t(world) * nr;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < ns; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / nr;
        scale[r_first * nr + e] = reinterpret_cast<const int32_t*>(recs + r * rec_bytes)[e - r * nr];
    }
}

}  // namespace

void launch_gather_planes(const int8_t* recs, int64_t rec_bytes, int64_t hdr, int world, int64_t nr, int64_t nkb,
                          int nsl, int8_t* planes, int64_t slots, int64_t plane_stride, int32_t* scale,
                          cudaStream_t st, uint64_t* nlaunch, int r_first) {
    if (world <= 0 || nr <= 0) return;
    gather_planes_kernel<<<num_sms() * 8, 256, 0, st>>>(recs, rec_bytes, hdr, world, r_first, nr, nkb, nsl, planes,
                                                        slots, plane_stride, scale);
    ++*nlaunch;
}

}  // namespace adpb200

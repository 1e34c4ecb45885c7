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

// byte j of X as stored in plane d = S-1-j
template <int S>
__device__ __forceinline__ uint32_t plane_byte(typename Word<S>::T X, int d) {
    const uint32_t b = uint32_t(X >> (8 * (S - 1 - d))) & 0xffu;
    return d == 0 ? b : (b ^ 0x80u);
}

// Plane d's bytes of 8 consecutive elements, packed into two words with
// byte permutes (d is a compile-time constant after unrolling).
template <int S>
__device__ __forceinline__ void pack_plane(const typename Word<S>::T (&X)[8], int d, uint32_t& lo, uint32_t& hi) {
    if constexpr (S <= 8) {
        const int j = S - 1 - d;  // byte of X
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = j < 4 ? uint32_t(X[q]) : uint32_t(X[q] >> 32);
        const uint32_t b = uint32_t(j & 3);
        const uint32_t sel = b | ((4 + b) << 4);  // byte b of x -> byte 0, byte b of y -> byte 1
        lo = __byte_perm(__byte_perm(w[0], w[1], sel), __byte_perm(w[2], w[3], sel), 0x5410);
        hi = __byte_perm(__byte_perm(w[4], w[5], sel), __byte_perm(w[6], w[7], sel), 0x5410);
        if (d != 0) {
            lo ^= 0x80808080u;
            hi ^= 0x80808080u;
        }
    } else {
        lo = hi = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            lo |= plane_byte<S>(X[q], d) << (8 * q);
            hi |= plane_byte<S>(X[q + 4], d) << (8 * q);
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
};

// Certified-ESC indicator bytes of 8 elements: 1 where the element is finite,
// nonzero and its effective exponent is within delta of the line maximum.
__device__ __forceinline__ void indicator_bytes(const uint64_t (&bits)[8], int lm, int delta, uint32_t& lo,
                                                uint32_t& hi) {
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
        return true;
    }
    if (a.plan->path != ADPB200_PATH_EMULATED) return false;
    s = a.plan->slices;
    nsl = a.plan->nsl;
    return true;
}

// ---- lines contiguous (ps == 1): a thread slices 8 consecutive positions ----------
template <int S, bool kVec>
__device__ __forceinline__ void rows_body(const SliceArgs& a, int nsl, int64_t groups, int64_t span) {
    // A warp covers 4 lines x 64 positions (lane = 8 x line + group): per plane it
    // stores two full 128-byte rows of the blocked layout (4 adjacent line slots x
    // 32 B) and reads 4 runs of 512 B. Fewer than 4 lines: one line per warp.
    const bool quad = a.v.lines >= 4;
    const int64_t gw = (groups + 7) / 8;
    const int64_t tasks = quad ? (a.v.lines + 3) / 4 * gw * 32 : a.v.lines * groups;
    auto decode = [&](int64_t task, int64_t& line, int64_t& g) {
        if (quad) {
            const int64_t wt = task >> 5;
            const int lane = int(task & 31);
            line = (wt / gw) * 4 + (lane >> 3);
            g = (wt % gw) * 8 + (lane & 7);
            return line < a.v.lines && g < groups;
        }
        line = task / groups;
        g = task - line * groups;
        return true;
    };
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    // the next task's 64 bytes are requested before this task is sliced and
    // stored: two loads in flight per thread keep HBM busier
    auto load = [&](int64_t task, uint64_t (&bits)[8]) {
        int64_t line, g;
        if (!decode(task, line, g)) return;
        const int64_t p0 = g * 8;
        const double* lp = a.v.ptr + line * a.v.ls;
        if (kVec && p0 + 8 <= a.v.len) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double2 d2 = __ldg(reinterpret_cast<const double2*>(lp + p0) + q);
                bits[2 * q] = __double_as_longlong(d2.x);
                bits[2 * q + 1] = __double_as_longlong(d2.y);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
                bits[q] = p0 + q < a.v.len ? __double_as_longlong(__ldg(lp + p0 + q)) : 0ull;
        }
    };
    int64_t task = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint64_t cur[8];
    if (task < tasks) load(task, cur);
    for (; task < tasks; task += stride) {
        uint64_t nxt[8];
        if (task + stride < tasks) load(task + stride, nxt);
        int64_t line, g;
        if (!decode(task, line, g)) {
#pragma unroll
            for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
            continue;
        }
        const int lm = a.line_max[line];
        const int E = lm == kNegSentinel ? 0 : lm + 2;
        if (g == 0 && a.scale) a.scale[line] = E;
        const int64_t p0 = g * 8;
        const int nvalid = span - p0 < 8 ? int(span - p0) : 8;
        if constexpr (S == 0) {
            for (int d = 0; d < nsl; ++d) {
                uint32_t lo, hi;
                indicator_bytes(cur, lm, d == 0 ? a.plan->aux : a.plan->aux2, lo, hi);
                int8_t* out = a.planes + plane_off(a, d, line, p0);
                if (kVec && nvalid == 8) {
                    *reinterpret_cast<uint2*>(out) = make_uint2(lo, hi);
                } else {
                    const uint64_t w = uint64_t(lo) | (uint64_t(hi) << 32);
                    for (int q = 0; q < nvalid; ++q) out[q] = int8_t(w >> (8 * q));
                }
            }
        } else if constexpr (S <= 16) {
            typename Word<S>::T X[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) X[q] = slice_word<S>(cur[q], E);
#pragma unroll
            for (int d = 0; d < S; ++d) {
                if (d >= nsl) break;
                uint32_t lo, hi;
                pack_plane<S>(X, d, lo, hi);
                int8_t* out = a.planes + plane_off(a, d, line, p0);
                if (kVec && nvalid == 8) {
                    *reinterpret_cast<uint2*>(out) = make_uint2(lo, hi);
                } else {
                    const uint64_t w = uint64_t(lo) | (uint64_t(hi) << 32);
                    for (int q = 0; q < nvalid; ++q) out[q] = int8_t(w >> (8 * q));
                }
            }
        } else {
            int8_t dig[kMaxSlices];
            const int s = a.slices_fixed > 0 ? a.slices_fixed : a.plan->slices;
            for (int q = 0; q < nvalid; ++q) {
                slice_digits_slow(cur[q], E, s, dig);
                for (int d = 0; d < nsl; ++d) a.planes[plane_off(a, d, line, p0 + q)] = dig[d];
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
    }
}

template <bool kVec>
__global__ void __launch_bounds__(256, 3) slice_rows_kernel(SliceArgs a) {
    int s, nsl;
    if (!resolve(a, s, nsl)) return;
    // blocked planes are zero-filled up to the 32-byte k-block
    const int64_t span = a.blocked ? (a.v.len + 31) / 32 * 32 : a.v.len;
    const int64_t groups = (span + 7) / 8;
    if (a.indicator) {
        rows_body<0, kVec>(a, nsl, groups, span);
        return;
    }
    switch (s) {
#define ADPB200_ROWS_CASE(S) \
    case S: rows_body<S, kVec>(a, nsl, groups, span); break;
        ADPB200_ROWS_CASE(1) ADPB200_ROWS_CASE(2) ADPB200_ROWS_CASE(3) ADPB200_ROWS_CASE(4)
        ADPB200_ROWS_CASE(5) ADPB200_ROWS_CASE(6) ADPB200_ROWS_CASE(7) ADPB200_ROWS_CASE(8)
        ADPB200_ROWS_CASE(9) ADPB200_ROWS_CASE(10) ADPB200_ROWS_CASE(11) ADPB200_ROWS_CASE(12)
        ADPB200_ROWS_CASE(13) ADPB200_ROWS_CASE(14) ADPB200_ROWS_CASE(15) ADPB200_ROWS_CASE(16)
#undef ADPB200_ROWS_CASE
        default: rows_body<32, kVec>(a, nsl, groups, span); break;
    }
}

// ---- lines adjacent (ls == 1), positions strided: 64 lines x 32 positions ---------
// The FP64 tile is transposed through shared memory (loads coalesced across
// lines, 16.6 KiB per CTA whatever s is); each thread then slices 8
// consecutive positions of one line exactly like the contiguous variant, so a
// warp stores 8 lines x 32 B = one contiguous 256-byte run per plane in the
// blocked layout.
constexpr int kTL = 64, kTP = 32, kTPad = kTL + 1;

template <int S>
__device__ __forceinline__ void cols_body(const SliceArgs& a, int nsl, const uint64_t (&bits)[8], int E,
                                          int64_t line, int64_t p0, int nvalid) {
    if constexpr (S <= 16) {
        typename Word<S>::T X[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) X[q] = slice_word<S>(bits[q], E);
#pragma unroll
        for (int d = 0; d < S; ++d) {
            if (d >= nsl) break;
            uint32_t lo, hi;
            pack_plane<S>(X, d, lo, hi);
            int8_t* out = a.planes + plane_off(a, d, line, p0);
            if (nvalid == 8 && (reinterpret_cast<uintptr_t>(out) & 7) == 0) {
                *reinterpret_cast<uint2*>(out) = make_uint2(lo, hi);
            } else {
                const uint64_t w = uint64_t(lo) | (uint64_t(hi) << 32);
                for (int q = 0; q < nvalid; ++q) a.planes[plane_off(a, d, line, p0 + q)] = int8_t(w >> (8 * q));
            }
        }
    } else {
        int8_t dig[kMaxSlices];
        const int s = a.slices_fixed > 0 ? a.slices_fixed : a.plan->slices;
        for (int q = 0; q < nvalid; ++q) {
            slice_digits_slow(bits[q], E, s, dig);
            for (int d = 0; d < nsl; ++d) a.planes[plane_off(a, d, line, p0 + q)] = dig[d];
        }
    }
}

__global__ void __launch_bounds__(256) slice_cols_kernel(SliceArgs a) {
    int s, nsl;
    if (!resolve(a, s, nsl)) return;
    __shared__ uint64_t tile[kTP][kTPad];
    const int64_t line0 = int64_t(blockIdx.x) * kTL;
    const int64_t pos0 = int64_t(blockIdx.y) * kTP;
    {
        const int tl = threadIdx.x % kTL, tp = threadIdx.x / kTL;  // 4 position rows per pass
        const int64_t line = line0 + tl;
        uint64_t v[kTP / 4];
#pragma unroll
        for (int i = 0; i < kTP / 4; ++i) {
            const int64_t pos = pos0 + tp + 4 * i;
            v[i] = (line < a.v.lines && pos < a.v.len) ? __double_as_longlong(__ldg(a.v.ptr + line + pos * a.v.ps))
                                                        : 0ull;
        }
#pragma unroll
        for (int i = 0; i < kTP / 4; ++i) tile[tp + 4 * i][tl] = v[i];
    }
    __syncthreads();
    const int ol = threadIdx.x / 4, og = threadIdx.x % 4;  // line, group of 8 positions
    const int64_t line = line0 + ol;
    if (line >= a.v.lines) return;
    const int lm = a.line_max[line];
    const int E = lm == kNegSentinel ? 0 : lm + 2;
    if (blockIdx.y == 0 && og == 0 && a.scale) a.scale[line] = E;
    const int64_t span = a.blocked ? (a.v.len + 31) / 32 * 32 : a.v.len;
    const int64_t p0 = pos0 + og * 8;
    if (p0 >= span) return;
    const int nvalid = span - p0 < 8 ? int(span - p0) : 8;
    uint64_t bits[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) bits[q] = tile[og * 8 + q][ol];
    if (a.indicator) {
        for (int d = 0; d < nsl; ++d) {
            uint32_t lo, hi;
            indicator_bytes(bits, lm, d == 0 ? a.plan->aux : a.plan->aux2, lo, hi);
            const uint64_t w = uint64_t(lo) | (uint64_t(hi) << 32);
            int8_t* out = a.planes + plane_off(a, d, line, p0);
            if (nvalid == 8 && (reinterpret_cast<uintptr_t>(out) & 7) == 0)
                *reinterpret_cast<uint2*>(out) = make_uint2(lo, hi);
            else
                for (int q = 0; q < nvalid; ++q) a.planes[plane_off(a, d, line, p0 + q)] = int8_t(w >> (8 * q));
        }
        return;
    }
    switch (s) {
#define ADPB200_COLS_CASE(S) \
    case S: cols_body<S>(a, nsl, bits, E, line, p0, nvalid); break;
        ADPB200_COLS_CASE(1) ADPB200_COLS_CASE(2) ADPB200_COLS_CASE(3) ADPB200_COLS_CASE(4)
        ADPB200_COLS_CASE(5) ADPB200_COLS_CASE(6) ADPB200_COLS_CASE(7) ADPB200_COLS_CASE(8)
        ADPB200_COLS_CASE(9) ADPB200_COLS_CASE(10) ADPB200_COLS_CASE(11) ADPB200_COLS_CASE(12)
        ADPB200_COLS_CASE(13) ADPB200_COLS_CASE(14) ADPB200_COLS_CASE(15) ADPB200_COLS_CASE(16)
#undef ADPB200_COLS_CASE
        default: cols_body<32>(a, nsl, bits, E, line, p0, nvalid); break;
    }
}

}  // namespace

void launch_slice(const LineView& v, const int32_t* line_max, int8_t* planes, int64_t pitch, int64_t plane_stride,
                  int blocked, int32_t* scale, const Plan* plan, int slices_fixed, int plane_cap, cudaStream_t st,
                  uint64_t* nlaunch, int indicator) {
    if (v.lines == 0) return;
    SliceArgs a{v, line_max, planes, pitch, plane_stride, blocked, scale, plan, slices_fixed, indicator};
    const bool rows = v.ps == 1 || v.lines == 1 || v.len == 0;
    if (rows) {
        if (a.v.lines == 1) a.v.ls = 0;
        const int64_t span = blocked ? (v.len + 31) / 32 * 32 : v.len;
        int64_t groups = (span + 7) / 8;
        if (groups == 0) groups = 1;
        int64_t tasks = v.lines * groups;
        int64_t want = (tasks + 255) / 256;
        int grid = (int)(want < int64_t(num_sms()) * 16 ? want : int64_t(num_sms()) * 16);
        if (grid < 1) grid = 1;
        const bool vec = ((reinterpret_cast<uintptr_t>(v.ptr) & 15) == 0) && ((v.ls & 1) == 0 || v.lines == 1) &&
                         (blocked || (((pitch & 7) == 0) && ((plane_stride & 7) == 0))) &&
                         ((reinterpret_cast<uintptr_t>(planes) & 7) == 0);
        if (vec) slice_rows_kernel<true><<<grid, 256, 0, st>>>(a);
        else slice_rows_kernel<false><<<grid, 256, 0, st>>>(a);
    } else {
        const int64_t span = blocked ? (v.len + 31) / 32 * 32 : v.len;
        dim3 grid((unsigned)((v.lines + kTL - 1) / kTL), (unsigned)((span + kTP - 1) / kTP));
        slice_cols_kernel<<<grid, 256, 0, st>>>(a);
    }
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

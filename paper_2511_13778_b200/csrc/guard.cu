// Guardrail kernels of the ADP pipeline (K1 scan + exponent statistics,
// K2 coarsened ESC max-plus reduction, the single-thread decision writer).
//
//   K1  scan_matrix + block_exponent_stats   proj/src/fpbits.cpp:5-73
//   K2  esc_coarsened + required_slices       proj/src/esc.cpp:8-12, 89-117
//   D   decide                                proj/src/adp.cpp:46-96
//
// K1 is HBM-bound: one pass over the operand, 8 B/element read, (2*t + 1)*4
// B/line written. It fuses the Inf/NaN/-0 counts, the per-(line, block)
// max/min effective exponents and (via a tiny second kernel) the line maxima
// that both ESC and slicing need.
#include "guard.cuh"

namespace adpb200 {

namespace {

__device__ __forceinline__ void classify(uint64_t bits, int& nan, int& inf, int& negz, bool& finite_nz,
                                         int& e) {
    int ex = raw_exp(bits);
    uint64_t mant = bits & 0xFFFFFFFFFFFFFull;
    finite_nz = false;
    if (ex == 0x7ff) {
        if (mant) ++nan;
        else ++inf;
        return;
    }
    if ((bits << 1) == 0) {
        if (bits >> 63) ++negz;
        return;
    }
    finite_nz = true;
    e = eff_exp(bits);
}

// Exponent statistics of N elements. Fast path (three instructions per element):
// when every element is a finite, normal nonzero number, the effective exponent is
// the biased exponent field - 1023, so the field's max / min over the group are
// the block's; otherwise (a zero, subnormal, Inf or NaN is present) classify() runs
// per element, exactly as before.
template <int N>
__device__ __forceinline__ void stats_group(const uint64_t (&bb)[N], int& nan, int& inf, int& negz, int& bmax,
                                            int& bmin) {
    uint32_t mx = 0, mn = 0xffffffffu;
#pragma unroll
    for (int q = 0; q < N; ++q) {
        const uint32_t f = uint32_t(bb[q] >> 32) & 0x7ff00000u;
        mx = max(mx, f);
        mn = min(mn, f);
    }
    if (mn != 0 && mx != 0x7ff00000u) {
        bmax = max(bmax, int(mx >> 20) - 1023);
        bmin = min(bmin, int(mn >> 20) - 1023);
        return;
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
        bool fnz;
        int e = 0;
        classify(bb[q], nan, inf, negz, fnz, e);
        if (fnz) {
            bmax = max(bmax, e);
            bmin = min(bmin, e);
        }
    }
}

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void flush_counts(int nan, int inf, int negz, unsigned long long* counts,
                                             int32_t* exc_flag, int exc_bit) {
    nan = warp_sum(nan);
    inf = warp_sum(inf);
    negz = warp_sum(negz);
    if ((threadIdx.x & 31) == 0) {
        if (nan) atomicAdd(&counts[0], (unsigned long long)nan);
        if (inf) atomicAdd(&counts[1], (unsigned long long)inf);
        if (negz) atomicAdd(&counts[2], (unsigned long long)negz);
        if ((nan || inf) && exc_flag) atomicOr(exc_flag, exc_bit);
    }
}

// Lines contiguous (ps == 1): one warp per (line, block); lanes stride the
// block so every load instruction is a coalesced 256 B request.
struct StatsArgs {
    LineView v;
    int64_t block_len, blocks;
    int32_t* bmax_out;
    int32_t* bmin_out;
    unsigned long long* counts;
    int32_t* exc_flag;
    int exc_bit, transposed;
    int64_t tstride;
    int groups;  // cols variant only
};

// rows variant run by CTAs cta = 0..nctas-1
__device__ __forceinline__ void stats_rows_body(const StatsArgs& A, int64_t cta, int64_t nctas) {
    const LineView& v = A.v;
    const int64_t block_len = A.block_len, blocks = A.blocks, tstride = A.tstride;
    int32_t* __restrict__ bmax_out = A.bmax_out;
    int32_t* __restrict__ bmin_out = A.bmin_out;
    const int transposed = A.transposed;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (cta * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (nctas * blockDim.x) >> 5;
    int nan = 0, inf = 0, negz = 0;
    const int64_t tasks = v.lines * blocks;
    for (int64_t task = warp; task < tasks; task += nwarps) {
        const int64_t line = task / blocks, blk = task - line * blocks;
        const int64_t lo = blk * block_len;
        const int64_t hi = lo + block_len < v.len ? lo + block_len : v.len;
        const double* lp = v.ptr + line * v.ls;
        int bmax = kNegSentinel, bmin = -kNegSentinel;
        int64_t pos = lo + lane;
        // 8 (then 4) independent loads in flight per lane
        for (; pos + 224 < hi; pos += 256) {
            uint64_t bb[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) bb[q] = __double_as_longlong(__ldg(lp + pos + 32 * q));
            stats_group(bb, nan, inf, negz, bmax, bmin);
        }
        for (; pos + 96 < hi; pos += 128) {
            uint64_t bb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) bb[q] = __double_as_longlong(__ldg(lp + pos + 32 * q));
            stats_group(bb, nan, inf, negz, bmax, bmin);
        }
        for (; pos < hi; pos += 32) {
            bool fnz;
            int e = 0;
            classify(__double_as_longlong(__ldg(lp + pos)), nan, inf, negz, fnz, e);
            if (fnz) {
                bmax = max(bmax, e);
                bmin = min(bmin, e);
            }
        }
        bmax = warp_max(bmax);
        bmin = warp_min(bmin);
        if (lane == 0) {
            bool any = bmax != kNegSentinel;
            const int64_t o = transposed ? blk * tstride + line : task;
            bmax_out[o] = any ? bmax : kNegSentinel;
            bmin_out[o] = any ? bmin : kNegSentinel;
        }
    }
    flush_counts(nan, inf, negz, A.counts, A.exc_flag, A.exc_bit);
}

__global__ void __launch_bounds__(256) stats_rows_kernel(StatsArgs A) {
    pdl_enter();
    stats_rows_body(A, blockIdx.x, gridDim.x);
}

// Lines adjacent (ls == 1): one thread per (line, block); a warp covers 32
// consecutive lines so each load is a coalesced 256 B request.
// cols variant as CTA (bx, by) of a gx x gy grid
__device__ __forceinline__ void stats_cols_body(const StatsArgs& A, int64_t bx, int64_t by, int64_t gy) {
    const LineView& v = A.v;
    const int64_t block_len = A.block_len, blocks = A.blocks, tstride = A.tstride;
    int32_t* __restrict__ bmax_out = A.bmax_out;
    int32_t* __restrict__ bmin_out = A.bmin_out;
    const int transposed = A.transposed, groups = A.groups;
    // 256 / groups adjacent lines x `groups` position groups per CTA: a warp loads a
    // 256-byte coalesced row across 32 lines, and a block's positions are split over
    // the groups (combined through shared memory) when the matrix is too small to
    // fill the SMs with one thread per (line, block)
    __shared__ int smax[8][256], smin[8][256];
    int nan = 0, inf = 0, negz = 0;
    const int width = 256 / groups;
    const int li = threadIdx.x % width, grp = threadIdx.x / width;
    const int64_t line = bx * width + li;
    const int64_t per = (block_len + groups - 1) / groups;
    for (int64_t blk = by; blk < blocks; blk += gy) {
        int bmax = kNegSentinel, bmin = -kNegSentinel;
        if (line < v.lines) {
            const int64_t b0 = blk * block_len, b1 = b0 + block_len < v.len ? b0 + block_len : v.len;
            const int64_t lo = b0 + grp * per;
            const int64_t hi = lo + per < b1 ? lo + per : b1;
            const double* p = v.ptr + line;
            int64_t pos = lo;
            for (; pos + 7 < hi; pos += 8) {
                uint64_t bb[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) bb[q] = __double_as_longlong(__ldg(p + (pos + q) * v.ps));
                stats_group(bb, nan, inf, negz, bmax, bmin);
            }
            for (; pos + 3 < hi; pos += 4) {
                uint64_t bb[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) bb[q] = __double_as_longlong(__ldg(p + (pos + q) * v.ps));
                stats_group(bb, nan, inf, negz, bmax, bmin);
            }
            for (; pos < hi; ++pos) {
                bool fnz;
                int e = 0;
                classify(__double_as_longlong(__ldg(p + pos * v.ps)), nan, inf, negz, fnz, e);
                if (fnz) {
                    bmax = max(bmax, e);
                    bmin = min(bmin, e);
                }
            }
        }
        if (groups > 1) {
            smax[grp][li] = bmax;
            smin[grp][li] = bmin;
            __syncthreads();
        }
        if (grp == 0 && line < v.lines) {
            for (int g = 1; g < groups; ++g) {
                bmax = max(bmax, smax[g][li]);
                bmin = min(bmin, smin[g][li]);
            }
            const bool any = bmax != kNegSentinel;
            const int64_t o = transposed ? blk * tstride + line : line * blocks + blk;
            bmax_out[o] = any ? bmax : kNegSentinel;
            bmin_out[o] = any ? bmin : kNegSentinel;
        }
        if (groups > 1) __syncthreads();
    }
    flush_counts(nan, inf, negz, A.counts, A.exc_flag, A.exc_bit);
}

__global__ void __launch_bounds__(256) stats_cols_kernel(StatsArgs A) {
    pdl_enter();
    stats_cols_body(A, blockIdx.x, blockIdx.y, gridDim.y);
}

// Both operands' statistics in one launch (A-lines adjacent, B-lines contiguous: the
// column-major N,N case): CTAs [0, gx*gy) run A's cols grid, the rest B's rows grid.
__global__ void __launch_bounds__(256) stats_pair_kernel(StatsArgs A, int gx, int gy, StatsArgs B) {
    pdl_enter();
    const int64_t ncols = int64_t(gx) * gy, id = blockIdx.x;
    if (id < ncols) stats_cols_body(A, id % gx, id / gx, gy);
    else stats_rows_body(B, id - ncols, int64_t(gridDim.x) - ncols);
}

// line_max[line] = max over the line's block maxima (sentinel is the minimum,
// so all-zero blocks drop out and all-zero lines stay sentinel).
__global__ void line_max_t_kernel(const int32_t* __restrict__ bmaxT, int64_t lines, int64_t blocks, int64_t stride,
                                  int32_t* __restrict__ line_max) {
    pdl_enter();
    const int64_t line = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (line >= lines) return;
    int mx = kNegSentinel;
    for (int64_t b = 0; b < blocks; ++b) mx = max(mx, bmaxT[b * stride + line]);
    line_max[line] = mx;
}

// line_max_t_kernel over A's lines then B's (threads [0, alines) then [alines, alines + blines))
__global__ void line_max_t_pair_kernel(const int32_t* __restrict__ amaxT, int64_t alines, int32_t* __restrict__ aline,
                                       const int32_t* __restrict__ bmaxT, int64_t blines, int32_t* __restrict__ bline,
                                       int64_t blocks) {
    pdl_enter();
    int64_t line = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int32_t* src = amaxT;
    int32_t* out = aline;
    int64_t stride = alines;
    if (line >= alines) {
        line -= alines;
        if (line >= blines) return;
        src = bmaxT;
        out = bline;
        stride = blines;
    }
    int mx = kNegSentinel;
    for (int64_t b = 0; b < blocks; ++b) mx = max(mx, src[b * stride + line]);
    out[line] = mx;
}

__global__ void line_max_kernel(const int32_t* __restrict__ bmax, int64_t lines, int64_t blocks,
                                int32_t* __restrict__ line_max) {
    pdl_enter();
    const int64_t line = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (line >= lines) return;
    int mx = kNegSentinel;
    for (int64_t b = lane; b < blocks; b += 32) mx = max(mx, bmax[line * blocks + b]);
    mx = warp_max(mx);
    if (lane == 0) line_max[line] = mx;
}

// Plain scan (stage export): counts only.
__global__ void scan_kernel(const double* __restrict__ a, int64_t count, unsigned long long* counts,
                            int32_t* exc_flag) {
    int nan = 0, inf = 0, negz = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x) {
        bool fnz;
        int e = 0;
        classify(__double_as_longlong(__ldg(a + i)), nan, inf, negz, fnz, e);
    }
    flush_counts(nan, inf, negz, counts, exc_flag, 1);
}

// ---- K2: coarsened ESC as a max-plus product over blocks --------------------------
// z_ij = max_t max(Amax_it + Bmin_jt, Amin_it + Bmax_jt); span = lA_i + lB_j - z + 1.
// The block stats arrive block-major ([t][line]) so each smem stage is a
// straight coalesced copy. Exponents live in [-1074, 1023] and are packed two
// per 32-bit word (int16x2); the reference's kNegSentinel becomes -16384. Any
// sum involving a sentinel is <= -16384 + 1023 < -2148 <= every real sum, and
// -16384 + -16384 = -32768 does not wrap, so sentinel blocks can never win a
// max and z stays <= -15361 exactly when the reference's z stays kNegSentinel
// (structurally zero dot product) — the exact same maximum, with no
// per-block branches. DPX __viaddmax_s16x2 fuses add + max for two (i, j)
// pairs per instruction.
constexpr int kEscBI = 64, kEscBJ = 128;       // CTA tile (16 x 16 threads, 4 x 8 per thread)
constexpr int kEscTB = 32;                     // blocks staged per smem round
constexpr int kS16 = -16384;

__device__ __forceinline__ uint32_t pack2(int lo, int hi) {
    return (uint32_t(lo) & 0xffffu) | (uint32_t(hi) << 16);
}
__device__ __forceinline__ int to16(int v) { return v == kNegSentinel ? kS16 : v; }

__global__ void __launch_bounds__(256, 4) esc_kernel(const int32_t* __restrict__ amaxT,
                                                  const int32_t* __restrict__ aminT,
                                                  const int32_t* __restrict__ aline,
                                                  const int32_t* __restrict__ bmaxT,
                                                  const int32_t* __restrict__ bminT,
                                                  const int32_t* __restrict__ bline, int64_t m, int64_t n,
                                                  int64_t t, int64_t nr, int64_t rec, int64_t astride,
                                                  const Plan* plan, int32_t* esc_out, int32_t* ran_flag) {
    pdl_enter();
    if (plan && plan->exc) return;  // exceptional inputs never reach the ESC (adp.cpp:58-62)
    // A words hold (a, a); B words hold (b_j, b_j+1) for the thread's j pairs
    __shared__ __align__(16) uint32_t sAmx[kEscTB][kEscBI];
    __shared__ __align__(16) uint32_t sAmn[kEscTB][kEscBI];
    __shared__ __align__(16) uint32_t sBmx[kEscTB][kEscBJ / 2];
    __shared__ __align__(16) uint32_t sBmn[kEscTB][kEscBJ / 2];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    // A CTA owns one 128-column j tile and walks the 64-row i tiles it.y, it.y + grid.y, ...
    // (persistent in i: the B side — offsets, and for t <= kEscTB the staged B stats —
    // is set up once per CTA, which is what short k, e.g. C5b's t = 4, spends its time on)
    const int64_t j0 = int64_t(blockIdx.x) * kEscBJ;
    const int64_t tiles_m = (m + kEscBI - 1) / kEscBI;
    // B stats of column slabs of nr lines, one record of `rec` int32 per slab (the
    // all-gathered layout of the B-distributed path; nr = n: one slab): the offset of
    // column j0 + jj minus gt * nr, computed once per CTA (no division in the loops)
    __shared__ int64_t sBoff[kEscBJ];
    __shared__ int sBound, sStop;
#ifndef ADPB200_ESC_PRUNE
#define ADPB200_ESC_PRUNE 1
#endif
    // the pruning probe's give-up flag, read under the barrier below (see kProbeGiveUp)
    constexpr int kProbeGiveUp = 128;
    if (threadIdx.x == 0)
        sStop = !ADPB200_ESC_PRUNE ||
                (plan && *reinterpret_cast<const volatile int32_t*>(&plan->esc_probe_fail) >= kProbeGiveUp);
    if (threadIdx.x < kEscBJ) {
        const int64_t gj = j0 + threadIdx.x;
        const int64_t r = gj / nr;
        sBoff[threadIdx.x] = r * rec + (gj - r * nr);
    }
    __syncthreads();
    const bool probe = sStop == 0;
    // staging roles, fixed per thread: one A line (or one B column pair), every 4th block
    const int sl = threadIdx.x % 64, st0 = threadIdx.x / 64;
    const bool b_ok0 = j0 + 2 * sl < n, b_ok1 = j0 + 2 * sl + 1 < n;
    const int64_t bo0 = sBoff[2 * sl], bo1 = sBoff[2 * sl + 1];
    const bool b_resident = t <= kEscTB;  // one staged round holds every block of B
    bool b_staged = false;
    auto stage_b = [&](int tt, int64_t gt) {
        const bool tok = gt < t;
        const int64_t go = gt * nr;
        sBmx[tt][sl] = pack2(b_ok0 && tok ? to16(bmaxT[bo0 + go]) : kS16, b_ok1 && tok ? to16(bmaxT[bo1 + go]) : kS16);
        sBmn[tt][sl] = pack2(b_ok0 && tok ? to16(bminT[bo0 + go]) : kS16, b_ok1 && tok ? to16(bminT[bo1 + go]) : kS16);
    };
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && ran_flag) *ran_flag = 1;
    for (int64_t it = blockIdx.y; it < tiles_m; it += gridDim.y) {
        const int64_t i0 = it * kEscBI;
        const int64_t ga = i0 + sl;
        const bool a_ok = ga < m;
        const int32_t* pamx = amaxT + ga;
        const int32_t* pamn = aminT + ga;
        uint32_t z[4][4];  // [i][j pair]
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) z[a][b] = 0x80008000u;
        auto stage_a = [&](int tt, int64_t gt) {
            const bool tok = gt < t;
            const int vx = a_ok && tok ? to16(pamx[gt * astride]) : kS16;
            const int vn = a_ok && tok ? to16(pamn[gt * astride]) : kS16;
            sAmx[tt][sl] = pack2(vx, vx);
            sAmn[tt][sl] = pack2(vn, vn);
        };
        auto step = [&](int tt) {
            const uint4 a_mx = *reinterpret_cast<const uint4*>(&sAmx[tt][ty * 4]);
            const uint4 a_mn = *reinterpret_cast<const uint4*>(&sAmn[tt][ty * 4]);
            const uint4 b_mx = *reinterpret_cast<const uint4*>(&sBmx[tt][tx * 4]);
            const uint4 b_mn = *reinterpret_cast<const uint4*>(&sBmn[tt][tx * 4]);
            const uint32_t amx[4] = {a_mx.x, a_mx.y, a_mx.z, a_mx.w};
            const uint32_t amn[4] = {a_mn.x, a_mn.y, a_mn.z, a_mn.w};
            const uint32_t bmx[4] = {b_mx.x, b_mx.y, b_mx.z, b_mx.w};
            const uint32_t bmn[4] = {b_mn.x, b_mn.y, b_mn.z, b_mn.w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    z[a][b] = __viaddmax_s16x2(amx[a], bmn[b], z[a][b]);
                    z[a][b] = __viaddmax_s16x2(amn[a], bmx[b], z[a][b]);
                }
        };
        // spans, two j per int16x2 word: la + lb + 1 - z in [-4193, 4195] for real
        // exponents; z <= -8000 (structurally zero dot product, or a padded row /
        // column) is masked to -32768 so it never wins the max.
        // max over this thread's pairs of la + lb + 1 - z, dead pairs (z <= -8000) as
        // `dead_as` (the line maxima are re-read per call rather than held in registers
        // across the max-plus loop)
        auto span_max = [&](uint32_t dead_as) {
            uint32_t lbp[4], lap[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int jj = 2 * (tx * 4 + b);
                const int l0 = j0 + jj < n ? bline[sBoff[jj]] : 0, l1 = j0 + jj + 1 < n ? bline[sBoff[jj + 1]] : 0;
                lbp[b] = pack2(l0 + 1, l1 + 1);
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int64_t gi = i0 + ty * 4 + a;
                const int la = gi < m ? aline[gi] : 0;
                lap[a] = pack2(la, la);
            }
            const uint32_t lim = pack2(-8000, -8000);
            uint32_t best = pack2(-32768, -32768);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const uint32_t span = __vsub2(__vadd2(lap[a], lbp[b]), z[a][b]);
                    const uint32_t dead = __vcmples2(z[a][b], lim);  // 0xffff per half where z <= -8000
                    best = __vmaxs2(best, (span & ~dead) | (dead_as & dead));
                }
            return max(int(int16_t(best & 0xffffu)), int(int16_t(best >> 16)));
        };
        // Tile pruning (exact). z only grows as blocks are added, so la + lb + 1 - z over
        // the blocks seen so far bounds every final span from above -- for pairs whose z
        // is already live (> -8000; a dead pair may still come alive, so it bounds
        // nothing). When that bound is <= the running maximum already published to
        // esc_out (by other tiles), no span of this tile can raise it and the tile stops:
        // the result is the reference's max over every (i, j). Checked after block 0
        // and after every staged round; narrow exponent ranges (every block of every
        // line alike) stop after one block.
        // The block-0 probe costs each tile a serial staging + reduction latency (~17 % of
        // the kernel when no tile can stop), so it gives up once kProbeGiveUp probes have
        // failed against an already published maximum (plan->esc_probe_fail; probes that
        // found nothing published yet, as in the first wave, do not count).
        auto prunable = [&](bool count) {
            if (threadIdx.x == 0) sBound = -32768;
            __syncthreads();
            const int bnd = warp_max(span_max(0x7fff7fffu));
            if ((threadIdx.x & 31) == 0) atomicMax(&sBound, bnd);
            __syncthreads();
            // one thread reads the running maximum, so the whole CTA takes the same branch
            if (threadIdx.x == 0) {
                const int published = *reinterpret_cast<volatile int32_t*>(esc_out);
                sStop = sBound <= published;
                if (count && !sStop && published > 0 && plan)
                    atomicAdd(&const_cast<Plan*>(plan)->esc_probe_fail, 1);
            }
            __syncthreads();
            return sStop != 0;
        };
        bool pruned = false;
        if (probe) {
            __syncthreads();  // the previous tile's reads of the stage are done
            if (st0 == 0) {
                stage_a(0, 0);
                if (!b_resident || !b_staged) stage_b(0, 0);
            }
            __syncthreads();
            step(0);
            pruned = prunable(true);
        }
        for (int64_t tb = 0; tb < t && !pruned; tb += kEscTB) {
            // only the blocks that exist are staged and stepped (short k, e.g. 4 blocks at
            // k = 1024, would otherwise spend 7/8 of the max-plus on sentinel padding)
            const int tcount = t - tb < kEscTB ? int(t - tb) : kEscTB;
            __syncthreads();
            for (int tt = st0; tt < tcount; tt += 4) {
                stage_a(tt, tb + tt);
                if (!b_resident || !b_staged) stage_b(tt, tb + tt);
            }
            __syncthreads();
            b_staged = true;
            if (tcount == kEscTB) {
#pragma unroll 4
                for (int tt = 0; tt < kEscTB; ++tt) step(tt);
            } else {
#pragma unroll 4
                for (int tt = 0; tt < tcount; ++tt) step(tt);
            }
            if (ADPB200_ESC_PRUNE && tb + kEscTB < t && prunable(false)) pruned = true;
        }
        if (!pruned) {
            // publish this tile's maximum now, so the CTAs' later tiles prune against it
            const int esc = warp_max(max(span_max(0x80008000u), 0));
            if ((threadIdx.x & 31) == 0 && esc > 0) atomicMax(esc_out, esc);
        }
    }
}

// [lines][blocks] -> [blocks][lines] (stage export of esc_coarsened, which
// takes the reference's line-major stats).
__global__ void transpose_i32_kernel(const int32_t* __restrict__ src, int64_t lines, int64_t blocks,
                                     int32_t* __restrict__ dst) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= lines * blocks) return;
    const int64_t line = i / blocks, b = i - line * blocks;
    dst[b * lines + line] = src[i];
}

// Finalise a standalone esc_coarsened export: out = {esc, target+esc, slices}.
__global__ void esc_finish_kernel(int32_t* out, int target_bits) {
    int esc = out[0];
    out[1] = target_bits + esc;
    out[2] = required_slices(target_bits, esc);
}

// ---- the decision kernel (one thread) ---------------------------------------------
__global__ void decide_kernel(Plan* plan, adpb200_options opt, int64_t m, int64_t n, int64_t k,
                              int esc_expected, int swap_ab, adpb200_trace* trace, int defer) {
    pdl_enter();
    Plan& p = *plan;
    DecideInput in;
    in.exc_a = p.exc & 1;
    in.exc_b = (p.exc >> 1) & 1;
    in.m = m;
    in.n = n;
    in.k = k;
    in.esc_bits = p.esc_raw;
    DecideOutput d = decide(in, opt);
    // Extension (H7): guardrails ran although the slice count is pinned.
    if (opt.mode == ADPB200_MODE_EMULATE && opt.guardrails_forced && d.path == ADPB200_PATH_EMULATED &&
        esc_expected && p.esc_ran) {
        d.esc_bits = p.esc_raw;
    }
    p.path = d.path;
    p.reason = d.reason;
    p.esc_bits = d.esc_bits;
    p.cost = d.cost;
    p.slices = d.path == ADPB200_PATH_EMULATED ? d.slices : 0;
    p.variant = 0;
    p.L = -1;
    p.nsl = 0;
    p.pairs = 0;
    p.kchunk = 0;
    p.nchunks = 0;
    if (d.path == ADPB200_PATH_EMULATED) fill_emulation_plan(p, d.slices, opt.pair_limit, k);
    if (trace) {
        adpb200_trace t;
        t.path = d.path;
        t.reason = d.reason;
        t.esc_bits = d.esc_bits;
        t.slices = d.path == ADPB200_PATH_EMULATED ? d.slices : -1;
        t.pair_limit = p.L;
        t.pairs = p.pairs;
        t.modeled_cost_ratio = d.cost;
        const int ia = swap_ab ? 3 : 0, ib = swap_ab ? 0 : 3;  // user A/B vs internal A/B
        t.nan_a = p.counts[ia + 0];
        t.inf_a = p.counts[ia + 1];
        t.negzero_a = p.counts[ia + 2];
        t.nan_b = p.counts[ib + 0];
        t.inf_b = p.counts[ib + 1];
        t.negzero_b = p.counts[ib + 2];
        t.m = m;
        t.n = n;
        t.k = k;
        t.gemm_variant = p.variant;
        t.k_chunks = p.nchunks;
        // the separate rounding pass runs exactly when the NB = 64 variant works on one k-chunk
        t.rounding_deferred = defer && d.path == ADPB200_PATH_EMULATED && p.variant == 64 && p.nchunks == 1;
        t.reserved_t = 0;
        *trace = t;
    }
}

}  // namespace

// ---- launchers ------------------------------------------------------------------
namespace {
thread_local bool t_pdl_call = true;
}
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("ADPB200_PDL");
        return !e || atoi(e) != 0;
    }();
    return on && t_pdl_call;
}
PdlScope::PdlScope(int64_t m, int64_t n, int64_t k) : prev(t_pdl_call) {
    static const double max_mnk = [] {
        const char* e = getenv("ADPB200_PDL_MAX_LOG2_MNK");
        const int lg = e ? atoi(e) : 35;
        return lg >= 62 ? 1e300 : double(int64_t(1) << (lg < 0 ? 0 : lg));
    }();
    t_pdl_call = double(m) * double(n) * double(k) <= max_mnk;
}
PdlScope::~PdlScope() { t_pdl_call = prev; }

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

namespace {
// grid of one operand's statistics kernel: rows (1-D, gx CTAs) or cols (gx x gy)
struct StatsPlan {
    StatsArgs args;
    bool rows;
    int gx, gy;
};

StatsPlan plan_stats(const LineView& v, int64_t block_len, int64_t blocks, int32_t* bmax, int32_t* bmin,
                     unsigned long long* counts, int32_t* exc_flag, int exc_bit, int transposed, int64_t tstride) {
    StatsPlan p{StatsArgs{v, block_len, blocks, bmax, bmin, counts, exc_flag, exc_bit, transposed, tstride, 1}, false,
                1, 1};
    if (v.ps == 1 || v.lines == 1) {
        // lines of a single row-major line: ps may be anything when len == 1
        if (v.lines == 1) p.args.v.ls = 0;
        p.rows = true;
        const int64_t want = (v.lines * blocks + 7) / 8;
        const int64_t grid = want < int64_t(num_sms()) * 16 ? want : int64_t(num_sms()) * 16;
        p.gx = int(grid < 1 ? 1 : grid);
    } else {
        // position groups per (line, block): enough threads to fill the SMs (one group at 8192^2)
        int groups = 1;
        while (groups < 8 && v.lines * blocks * groups < int64_t(num_sms()) * 1024) groups *= 2;
        const int width = 256 / groups;
        p.args.groups = groups;
        p.gx = int((v.lines + width - 1) / width);
        p.gy = int(blocks < 65535 ? blocks : 65535);
    }
    return p;
}

void launch_planned(const StatsPlan& p, cudaStream_t st) {
    if (p.rows) launch_chain(stats_rows_kernel, dim3(p.gx), dim3(256), 0, st, p.args);
    else launch_chain(stats_cols_kernel, dim3(p.gx, p.gy), dim3(256), 0, st, p.args);
}
}  // namespace

void launch_stats(const LineView& v, int64_t block_len, int32_t* bmax, int32_t* bmin, int32_t* line_max,
                  unsigned long long* counts, int32_t* exc_flag, int exc_bit, int transposed, cudaStream_t st,
                  uint64_t* nlaunch, int64_t tstride, int skip_line_max) {
    const int64_t blocks = v.len == 0 ? 0 : (v.len + block_len - 1) / block_len;
    if (tstride <= 0) tstride = v.lines;
    if (v.lines == 0) return;
    if (blocks > 0) {
        launch_planned(plan_stats(v, block_len, blocks, bmax, bmin, counts, exc_flag, exc_bit, transposed, tstride),
                       st);
        ++*nlaunch;
    }
    if (skip_line_max) return;
    if (transposed) {
        launch_chain(line_max_t_kernel, dim3((unsigned)((v.lines + 255) / 256)), dim3(256), 0, st, bmax, v.lines, blocks, tstride,
                                                                               line_max);
    } else {
        int lgrid = (int)((v.lines * 32 + 255) / 256);
        launch_chain(line_max_kernel, dim3(lgrid), dim3(256), 0, st, bmax, v.lines, blocks, line_max);
    }
    ++*nlaunch;
}

void launch_stats_pair(const LineView& va, int32_t* amax, int32_t* amin, unsigned long long* acounts,
                       const LineView& vb, int32_t* bmax, int32_t* bmin, unsigned long long* bcounts,
                       int64_t block_len, int32_t* exc_flag, cudaStream_t st, uint64_t* nlaunch) {
    const int64_t blocks = va.len == 0 ? 0 : (va.len + block_len - 1) / block_len;
    if (va.lines == 0 || vb.lines == 0 || blocks == 0) return;
    const StatsPlan pa = plan_stats(va, block_len, blocks, amax, amin, acounts, exc_flag, 1, 1, va.lines);
    const StatsPlan pb = plan_stats(vb, block_len, blocks, bmax, bmin, bcounts, exc_flag, 2, 1, vb.lines);
    static const bool paired = [] {
        const char* e = getenv("ADPB200_STATS_PAIR");
        return !e || atoi(e) != 0;
    }();
    if (paired && !pa.rows && pb.rows) {
        launch_chain(stats_pair_kernel, dim3(unsigned(int64_t(pa.gx) * pa.gy + pb.gx)), dim3(256), 0, st, pa.args,
                     pa.gx, pa.gy, pb.args);
        ++*nlaunch;
    } else {
        launch_planned(pa, st);
        launch_planned(pb, st);
        *nlaunch += 2;
    }
}

void launch_line_max_t_pair(const int32_t* amaxT, int64_t alines, int32_t* aline, const int32_t* bmaxT,
                            int64_t blines, int32_t* bline, int64_t blocks, cudaStream_t st, uint64_t* nlaunch) {
    const int64_t lines = alines + blines;
    if (lines == 0) return;
    launch_chain(line_max_t_pair_kernel, dim3((unsigned)((lines + 255) / 256)), dim3(256), 0, st, amaxT, alines, aline,
                 bmaxT, blines, bline, blocks);
    ++*nlaunch;
}

void launch_scan(const double* a, int64_t count, unsigned long long* counts, int32_t* exc, cudaStream_t st,
                 uint64_t* nlaunch) {
    if (count == 0) return;
    int64_t want = (count + 255) / 256;
    int grid = (int)(want < int64_t(num_sms()) * 8 ? want : int64_t(num_sms()) * 8);
    scan_kernel<<<grid, 256, 0, st>>>(a, count, counts, exc);
    ++*nlaunch;
}

void launch_esc(const int32_t* amax, const int32_t* amin, const int32_t* aline, const int32_t* bmax,
                const int32_t* bmin, const int32_t* bline, int64_t m, int64_t n, int64_t t, const Plan* plan,
                int32_t* esc_out, int32_t* ran_flag, cudaStream_t st, uint64_t* nlaunch, int64_t b_nr,
                int64_t b_rec, int64_t a_stride) {
    if (m == 0 || n == 0) return;
    if (b_nr <= 0) b_nr = n;
    if (a_stride <= 0) a_stride = m;
    // short k (every block staged in one round, B resident): persistent in i, about two
    // waves of CTAs (4 resident per SM) each walking i tiles; longer k: one CTA per tile,
    // which balances the irregular work tile pruning leaves better than a static walk
    const int64_t gx = (n + kEscBJ - 1) / kEscBJ, tiles_m = (m + kEscBI - 1) / kEscBI;
    int64_t gy = t <= kEscTB ? int64_t(num_sms()) * 8 / gx : tiles_m;
    gy = gy < 1 ? 1 : (gy > tiles_m ? tiles_m : gy);
    dim3 grid((unsigned)gx, (unsigned)(gy < 65535 ? gy : 65535));
    launch_chain(esc_kernel, grid, dim3(256), 0, st, amax, amin, aline, bmax, bmin, bline, m, n, t, b_nr, b_rec, a_stride, plan,
                                     esc_out, ran_flag);
    ++*nlaunch;
}

void launch_transpose_i32(const int32_t* src, int64_t lines, int64_t blocks, int32_t* dst, cudaStream_t st,
                          uint64_t* nlaunch) {
    if (lines * blocks == 0) return;
    transpose_i32_kernel<<<(unsigned)((lines * blocks + 255) / 256), 256, 0, st>>>(src, lines, blocks, dst);
    ++*nlaunch;
}

void launch_esc_finish(int32_t* out, int target_bits, cudaStream_t st, uint64_t* nlaunch) {
    esc_finish_kernel<<<1, 1, 0, st>>>(out, target_bits);
    ++*nlaunch;
}

__global__ void set_plan_kernel(Plan* plan, int s, int pair_limit, int64_t k) {
    Plan p = *plan;
    p.reason = ADPB200_REASON_FORCED;
    p.esc_bits = -1;
    fill_emulation_plan(p, s, pair_limit, k);
    *plan = p;
}

void launch_set_plan(Plan* plan, int s, int pair_limit, int64_t k, cudaStream_t st, uint64_t* nlaunch) {
    set_plan_kernel<<<1, 1, 0, st>>>(plan, s, pair_limit, k);
    ++*nlaunch;
}

// ---- certified ESC ----------------------------------------------------------------
// s0 = required_slices(target_bits, 0) is the fewest slices any input can get;
// s0 + l slices tolerate esc <= e_l = 8 (s0 + l) - target_bits - 2. If some
// position l has e(a_il) >= rowmax_i - delta and e(b_lj) >= colmax_j - delta,
// the exact largest product exponent z_ij (esc.cpp:61-87) is >= rowmax_i +
// colmax_j - 2 delta, so span_ij <= 2 delta + 1; delta_l = (e_l - 1) / 2
// (certify_delta) makes that span fit s0 + l slices. The "some l" test for every
// (i, j) is an INT8 GEMM of 0/1 planes: one plane per operand for one level, two
// (level 0, level 1) when the coarsened ESC asks for more than s0 + 1 slices;
// the two-plane GEMM's diagonals 0 and 2 hold the two levels' counts.
__global__ void certify_prep_kernel(const Plan* plan, Plan* rplan, int target_bits, int64_t k, int force,
                                    int max_planes) {
    Plan r{};
    r.path = kPathDone;
    const int d0 = certify_delta(target_bits, 0), d1 = certify_delta(target_bits, 1);
    const int coarse = plan->esc_raw;
    const bool ok = force || (plan->esc_ran && plan->exc == 0);
    // levels worth testing: force (multi-GPU) tests both, the outcome combines later
    const bool l0 = ok && d0 >= 0 && (force || coarse > 2 * d0 + 1);
    const bool l1 = ok && d1 >= 0 && (force || coarse > 2 * d1 + 1) && (max_planes >= 2 || !l0);
    if ((l0 || l1) && k > 0 && k <= (int64_t(1) << 30)) {
        const int planes = (l0 && l1) ? 2 : 1;
        r.path = ADPB200_PATH_EMULATED;
        r.slices = planes;
        r.L = 2 * (planes - 1);  // pairs d_a + d_b <= L: (0,0) [+ (0,1), (1,0), (1,1)]
        r.nsl = planes;
        r.pairs = planes * planes;
        r.variant = 64;
        r.kchunk = int32_t((k + 31) / 32 * 32);  // counts <= k: one int32 chunk
        r.nchunks = 1;
        r.aux = l0 ? d0 : d1;
        r.aux2 = d1;
        r.lvl0 = l0 ? 0 : 1;
        r.exc = 0;  // the GEMM's zero-count flags: bit 0 plane-0 level, bit 1 plane-1 level
    }
    *rplan = r;
}

// outcome v of an armed certificate plan (0, 1 or 2 as in certified_esc)
__device__ __forceinline__ int certify_outcome(const Plan* rplan) {
    if (rplan->path != ADPB200_PATH_EMULATED) return 2;
    if (!(rplan->exc & 1)) return rplan->lvl0;
    if (rplan->nsl == 2 && !(rplan->exc & 2)) return 1;
    return 2;
}

__global__ void certify_finish_kernel(Plan* plan, const Plan* rplan, int target_bits) {
    if (rplan->path == ADPB200_PATH_EMULATED)
        plan->esc_raw = certified_esc(plan->esc_raw, certify_outcome(rplan), target_bits);
}

__global__ void dist_export_kernel(const Plan* plan, const Plan* rplan, int32_t* xchg, int certified) {
    int32_t x0 = plan->exc;
    // (an unarmed certificate plan or an exceptional rank reports v = 2)
    if (certified) x0 |= int32_t(plan->exc != 0 ? 2 : certify_outcome(rplan)) << kXchgCertShift;
    xchg[0] = x0;
    xchg[1] = plan->esc_raw;
}

__global__ void dist_import_kernel(Plan* plan, const int32_t* xchg, int target_bits, int certified) {
    const int32_t x0 = xchg[0];
    plan->exc = x0 & 3;
    plan->esc_raw = xchg[1];
    if (certified) plan->esc_raw = certified_esc(plan->esc_raw, (x0 >> kXchgCertShift) & 3, target_bits);
}

void launch_certify_prep(const Plan* plan, Plan* rplan, int target_bits, int64_t k, cudaStream_t st,
                         uint64_t* nlaunch, int force, int max_planes) {
    certify_prep_kernel<<<1, 1, 0, st>>>(plan, rplan, target_bits, k, force, max_planes);
    ++*nlaunch;
}

void launch_certify_finish(Plan* plan, const Plan* rplan, int target_bits, cudaStream_t st, uint64_t* nlaunch) {
    certify_finish_kernel<<<1, 1, 0, st>>>(plan, rplan, target_bits);
    ++*nlaunch;
}

void launch_dist_export(const Plan* plan, const Plan* rplan, int32_t* xchg, int certified, cudaStream_t st,
                        uint64_t* nlaunch) {
    dist_export_kernel<<<1, 1, 0, st>>>(plan, rplan, xchg, certified);
    ++*nlaunch;
}

void launch_dist_import(Plan* plan, const int32_t* xchg, int target_bits, int certified, cudaStream_t st,
                        uint64_t* nlaunch) {
    dist_import_kernel<<<1, 1, 0, st>>>(plan, xchg, target_bits, certified);
    ++*nlaunch;
}

void launch_decide(Plan* plan, const adpb200_options& opt, int64_t m, int64_t n, int64_t k, int esc_expected,
                   int swap_ab, adpb200_trace* trace, cudaStream_t st, uint64_t* nlaunch, int defer) {
    launch_chain(decide_kernel, dim3(1), dim3(1), 0, st, plan, opt, m, n, k, esc_expected, swap_ab, trace, defer);
    ++*nlaunch;
}

// ---- esc_exact stage export (esc.cpp:26-87) ---------------------------------------
namespace {
constexpr int32_t kExactSentinel = -(1 << 28);  // zeros: two of them still sum above INT_MIN

// exponent field of a row-major rows x cols matrix (zeros -> sentinel), exceptional flag
__global__ void exp_field_kernel(const double* __restrict__ a, int64_t count, int32_t* __restrict__ e,
                                 int32_t* exc) {
    bool bad = false;
    for (int64_t x = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; x < count; x += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t b = __double_as_longlong(__ldg(a + x));
        if (((b >> 52) & 0x7ff) == 0x7ff) {
            bad = true;
            e[x] = kExactSentinel;
        } else {
            e[x] = (b << 1) == 0 ? kExactSentinel : eff_exp(b);
        }
    }
    if (bad) atomicOr(exc, 1);
}

// line maxima: rows of e (stride_line = cols, stride_pos = 1) or columns (1, cols)
__global__ void exp_line_max_kernel(const int32_t* __restrict__ e, int64_t lines, int64_t len, int64_t s_line,
                                    int64_t s_pos, int32_t* __restrict__ out) {
    const int64_t line = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (line >= lines) return;
    int32_t mx = kExactSentinel;
    for (int64_t p = 0; p < len; ++p) mx = max(mx, e[line * s_line + p * s_pos]);
    out[line] = mx;
}

// z_ij = max_l ea[i][l] + eb[l][j] (DPX add-max), 64 x 64 outputs per CTA, 4 x 4 per thread;
// span_ij = rowmax_i + colmax_j - z_ij + 1 over the (i, j) with a nonzero product
__global__ void __launch_bounds__(256) esc_exact_kernel(const int32_t* __restrict__ ea, const int32_t* __restrict__ eb,
                                                        const int32_t* __restrict__ rmax,
                                                        const int32_t* __restrict__ cmax, int64_t m, int64_t n,
                                                        int64_t k, int32_t* out) {
    __shared__ int32_t As[32][65];
    __shared__ int32_t Bs[32][64];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t i0 = int64_t(blockIdx.y) * 64, j0 = int64_t(blockIdx.x) * 64;
    int32_t z[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) z[a][b] = 2 * kExactSentinel;
    for (int64_t l0 = 0; l0 < k; l0 += 32) {
        for (int t = threadIdx.x; t < 64 * 32; t += 256) {
            const int r = t / 32, c = t % 32;  // A tile: row r, position c (coalesced along positions)
            const int64_t gi = i0 + r, gl = l0 + c;
            As[c][r] = (gi < m && gl < k) ? ea[gi * k + gl] : kExactSentinel;
            const int br = t / 64, bc = t % 64;  // B tile: position br, column bc
            const int64_t bl = l0 + br, bj = j0 + bc;
            Bs[br][bc] = (bl < k && bj < n) ? eb[bl * n + bj] : kExactSentinel;
        }
        __syncthreads();
#pragma unroll 8
        for (int c = 0; c < 32; ++c) {
            int32_t av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = As[c][ty * 4 + a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = Bs[c][tx * 4 + b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) z[a][b] = __viaddmax_s32(av[a], bv[b], z[a][b]);
        }
        __syncthreads();
    }
    int32_t esc = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t gi = i0 + ty * 4 + a, gj = j0 + tx * 4 + b;
            if (gi < m && gj < n && z[a][b] > kExactSentinel / 2) esc = max(esc, rmax[gi] + cmax[gj] - z[a][b] + 1);
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) esc = max(esc, __shfl_xor_sync(0xffffffffu, esc, o));
    if ((threadIdx.x & 31) == 0 && esc > 0) atomicMax(out, esc);
}
}  // namespace

void launch_esc_exact(const double* A, const double* B, int64_t m, int64_t n, int64_t k, int32_t* ea, int32_t* eb,
                      int32_t* rmax, int32_t* cmax, int32_t* exc, int32_t* out, cudaStream_t st, uint64_t* nlaunch) {
    auto grid_for = [](int64_t count) {
        const int64_t want = (count + 255) / 256;
        return int(want < int64_t(num_sms()) * 16 ? (want > 0 ? want : 1) : int64_t(num_sms()) * 16);
    };
    exp_field_kernel<<<grid_for(m * k), 256, 0, st>>>(A, m * k, ea, exc);
    exp_field_kernel<<<grid_for(k * n), 256, 0, st>>>(B, k * n, eb, exc);
    exp_line_max_kernel<<<unsigned((m + 255) / 256 > 0 ? (m + 255) / 256 : 1), 256, 0, st>>>(ea, m, k, k, 1, rmax);
    exp_line_max_kernel<<<unsigned((n + 255) / 256 > 0 ? (n + 255) / 256 : 1), 256, 0, st>>>(eb, n, k, 1, n, cmax);
    *nlaunch += 4;
    if (m > 0 && n > 0 && k > 0) {
        dim3 grid(unsigned((n + 63) / 64), unsigned((m + 63) / 64));
        esc_exact_kernel<<<grid, 256, 0, st>>>(ea, eb, rmax, cmax, m, n, k, out);
        ++*nlaunch;
    }
}

}  // namespace adpb200

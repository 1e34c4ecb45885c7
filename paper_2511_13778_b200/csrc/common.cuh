// Shared definitions of the adpb200 pipeline (device plan, operand views,
// FP64 bit helpers, the host+device decision function).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "adpb200.h"

namespace adpb200 {

constexpr int32_t kNegSentinel = -1000000;  // fpbits.hpp:22
constexpr int kMaxSlices = 32;              // slicing.hpp:11

// A matrix seen as `lines` lines of `len` elements: element (line, pos) is at
// ptr[line*ls + pos*ps]. A-lines are rows of op(A), B-lines columns of op(B);
// both are K-long, which is the orientation the slice planes are stored in.
struct LineView {
    const double* ptr;
    int64_t lines, len;
    int64_t ls, ps;
};

// Internal path value (never reported): the work of the plan is already done
// (the streamed host path's speculation matched the decision).
constexpr int32_t kPathDone = 7;

// Device-resident plan: filled by the guardrail kernels and the decision
// kernel, read by every later kernel (no host round trip).
struct Plan {
    // written by the scan/stats kernels
    unsigned long long counts[6];  // nan/inf/-0 of A, then B
    int32_t exc;                   // bit0 A exceptional, bit1 B exceptional
    int32_t esc_raw;               // max span over (i,j), >= 0 (atomicMax)
    int32_t esc_ran;               // ESC kernel executed
    // written by the decision kernel
    int32_t path;      // ADPB200_PATH_*
    int32_t reason;    // ADPB200_REASON_*
    int32_t esc_bits;  // -1 if not computed
    int32_t slices;    // s
    int32_t L;         // largest diagonal index accumulated (d_a + d_b <= L)
    int32_t nsl;       // slices that take part: min(s, L+1)
    int32_t pairs;     // admitted (d_a, d_b) pairs
    int32_t variant;   // GEMM variant: columns per diagonal (64/32/16), 0 = none
    int32_t kchunk;    // k elements per int32 accumulation chunk
    int32_t nchunks;
    double cost;
    int32_t aux;   // certified-ESC plan: indicator threshold delta of plane 0
    int32_t aux2;  //   ... of plane 1 (two-level plans)
    int32_t lvl0;  //   certificate level plane 0 stands for (0, or 1 when level 0 cannot help)
    int32_t esc_probe_fail;  // ESC tiles whose block-0 pruning probe failed against a published maximum
};

// ---- programmatic dependent launch (PDL) along the per-call kernel chain ----
// Every chain kernel starts with pdl_enter(): griddepcontrol.wait blocks until
// the previous kernel of the stream has completed and its writes are visible
// (a no-op for a kernel launched without the attribute), then
// launch_dependents lets the next kernel's CTAs be scheduled on the slots this
// grid leaves free. Since each kernel waits before touching memory, the order
// of effects is the plain stream order; what the overlap removes is the launch
// gap between consecutive kernels (10 per call), which dominates calls below
// ~2048^3. The trigger only fires once every CTA of this grid has executed it,
// so waiting dependents can never take the slots of CTAs not yet started.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
    pdl_wait();
    pdl_trigger();
}

bool pdl_enabled();  // ADPB200_PDL (default 1) and the calling thread's per-call choice
// Per-call choice (thread-local, default on): a pipeline call turns PDL off above
// mnk = 2^35 (ADPB200_PDL_MAX_LOG2_MNK), where the launch gaps are hidden anyway and
// the overlap measured 0.7 % slower at 8192^3 (lower clock at the same power cap).
struct PdlScope {
    bool prev;
    PdlScope(int64_t m, int64_t n, int64_t k);
    ~PdlScope();
};

// launch a chain kernel (one that begins with pdl_enter) with the PDL attribute
template <typename... KArgs, typename... Args>
inline cudaError_t launch_chain(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

struct DecideInput {
    int32_t exc_a, exc_b;
    int64_t m, n, k;
    int32_t esc_bits;  // value the ESC provider returns (only consulted when reached)
};

struct DecideOutput {
    int32_t path, reason, slices, provider_called, esc_bits;
    double cost;
};

__host__ __device__ inline int required_slices(int target_bits, int esc_bits) {
    return (target_bits + esc_bits + 2 + 7) / 8;  // esc.cpp:8-12
}

// decide() (adp.cpp:46-96): identical gate order and FP64 cost model. Every
// FP64 operation is written as an explicitly rounded intrinsic on the device
// (no FMA contraction, matching -ffp-contract=off of the reference build).
// Certified ESC (adpb200_options.esc_method): the indicator threshold delta of
// certificate level l, which targets s0 + l slices (s0 = required_slices(
// target_bits, 0), the fewest any input gets): 2 delta + 1 is the largest ESC
// s0 + l slices tolerate (-1: that level cannot help).
__host__ __device__ inline int certify_delta(int target_bits, int level = 0) {
    const int s = (target_bits + 2 + 7) / 8 + level;
    const int e = 8 * s - target_bits - 2;
    return e >= 1 ? (e - 1) / 2 : -1;
}
// The certified ESC from the coarsened one and the certificate outcome v:
// 0 = level 0 holds for every (i, j), 1 = only level 1 does, 2 = neither.
__host__ __device__ inline int certified_esc(int coarse, int v, int target_bits) {
    const int d0 = certify_delta(target_bits, 0), d1 = certify_delta(target_bits, 1);
    if (v == 0 && d0 >= 0 && coarse > 2 * d0 + 1) return 2 * d0 + 1;
    if (v <= 1 && d1 >= 0 && coarse > 2 * d1 + 1) return 2 * d1 + 1;
    return coarse;
}
// Multi-GPU exchange word 0 (max-reduced): exceptional bits 0-1, and with the
// certified ESC the rank's outcome v in bits 8-9 (max over ranks = the global
// outcome; an exceptional rank reports v = 2, so the maximum also keeps its
// exceptional bits).
constexpr int kXchgCertShift = 8;
constexpr int32_t kXchgCertFail = 2 << kXchgCertShift;

__host__ __device__ inline DecideOutput decide(const DecideInput& in, const adpb200_options& c) {
    DecideOutput d{ADPB200_PATH_NATIVE, ADPB200_REASON_OK, 0, 0, -1, 0.0};
    if (c.mode == ADPB200_MODE_NATIVE) {
        d.reason = ADPB200_REASON_FORCED;
        return d;
    }
    if (in.exc_a || in.exc_b) {
        d.reason = ADPB200_REASON_EXCEPTIONAL;
        return d;
    }
    if (c.mode == ADPB200_MODE_EMULATE) {
        d.path = ADPB200_PATH_EMULATED;
        d.reason = ADPB200_REASON_FORCED;
        d.slices = c.forced_slices;
        return d;
    }
    int64_t mn = in.m < in.n ? in.m : in.n;
    mn = mn < in.k ? mn : in.k;
    if (mn < c.min_dim) {
        d.reason = ADPB200_REASON_TOO_SMALL;
        return d;
    }
    d.provider_called = 1;
    d.esc_bits = in.esc_bits;
    int s_req = required_slices(c.target_bits, in.esc_bits);
    if (s_req > c.max_slices) {
        d.reason = ADPB200_REASON_ESC_TOO_LARGE;
        return d;
    }
#ifdef __CUDA_ARCH__
    double mnk = __dmul_rn(__dmul_rn((double)in.m, (double)in.n), (double)in.k);
    double s = (double)s_req;
    double est = __dadd_rn(__dmul_rn((double)in.m, (double)in.k), __dmul_rn((double)in.k, (double)in.n));
    d.cost = __ddiv_rn(__dadd_rn(__ddiv_rn(__dmul_rn(__dmul_rn(s, s), mnk), c.cost_ratio), est), mnk);
#else
    volatile double mnk = (double)in.m * (double)in.n;
    mnk = mnk * (double)in.k;
    double s = (double)s_req;
    volatile double t1 = (double)in.m * (double)in.k;
    volatile double t2 = (double)in.k * (double)in.n;
    volatile double est = t1 + t2;
    volatile double ss = s * s;
    volatile double num = ss * mnk;
    num = num / c.cost_ratio;
    num = num + est;
    d.cost = num / mnk;
#endif
    if (d.cost >= 1.0) {
        d.reason = ADPB200_REASON_COST_MODEL;
        return d;
    }
    d.path = ADPB200_PATH_EMULATED;
    d.reason = ADPB200_REASON_OK;
    d.slices = s_req;
    return d;
}

// ---- FP64 bit helpers (fpbits.hpp:34-48) ------------------------------------------
__device__ __forceinline__ int raw_exp(uint64_t b) { return (int)((b >> 52) & 0x7ff); }
__device__ __forceinline__ int eff_exp(uint64_t b) {
    int e = raw_exp(b);
    if (e != 0) return e - 1023;
    return (63 - __clzll((long long)(b & 0xFFFFFFFFFFFFFull))) - 1074;
}
__device__ __forceinline__ uint64_t norm_mant(uint64_t b) {
    int e = raw_exp(b);
    uint64_t mant = b & 0xFFFFFFFFFFFFFull;
    if (e != 0) return mant | (1ull << 52);
    return mant << (52 - (63 - __clzll((long long)mant)));
}

// Number of admitted pairs and the largest per-diagonal pair count for
// slice count s and diagonal limit L (d_a + d_b <= L, 0 <= d_a, d_b < s).
__host__ __device__ inline void pair_stats(int s, int L, int* pairs, int* max_per_diag) {
    int p = 0, mx = 0;
    for (int D = 0; D <= L; ++D) {
        int lo = D - (s - 1) > 0 ? D - (s - 1) : 0;
        int hi = D < s - 1 ? D : s - 1;
        int c = hi >= lo ? hi - lo + 1 : 0;
        p += c;
        if (c > mx) mx = c;
    }
    *pairs = p;
    *max_per_diag = mx;
}

// k elements one int32 TMEM accumulator can absorb without wrapping: every
// product is bounded by 128*128 = 2^14 (igemm.hpp:24-29), a diagonal sums at
// most max_per_diag products per k. Rounded down to the 32-byte k-block.
__host__ __device__ inline int64_t int32_kchunk(int max_per_diag) {
    int64_t c = ((int64_t(1) << 31) - 1) / (int64_t(max_per_diag) * 16384);
    return (c / 32) * 32;
}

// Fill the emulation part of the plan for slice count s and the requested
// pair policy (ADPB200_PAIRS_FULL / _TARGET / limit >= 0).
__host__ __device__ inline void fill_emulation_plan(Plan& p, int s, int pair_limit, int64_t k) {
    int L = 2 * s - 2;
    if (pair_limit == ADPB200_PAIRS_TARGET) L = s < L ? s : L;
    else if (pair_limit >= 0) L = pair_limit < L ? pair_limit : L;
    p.path = ADPB200_PATH_EMULATED;
    p.slices = s;
    p.L = L;
    p.nsl = s < L + 1 ? s : L + 1;
    int pairs, mpd;
    pair_stats(s, L, &pairs, &mpd);
    p.pairs = pairs;
    const int ndiag = L + 1;
    // columns per diagonal accumulator so that ndiag * variant <= 512 TMEM columns
    p.variant = ndiag <= 8 ? 64 : (ndiag <= 10 ? 48 : (ndiag <= 16 ? 32 : (ndiag <= 32 ? 16 : 8)));
    const int64_t kc = int32_kchunk(mpd);
    p.kchunk = (int32_t)kc;
    p.nchunks = k == 0 ? 0 : (int32_t)((k + kc - 1) / kc);
}

}  // namespace adpb200

// adpb200_nccl.hpp — the B-distributed multi-GPU ADP DGEMM driven from C++ with
// NCCL (one process or thread per GPU, one ncclComm_t per rank), the native
// counterpart of paper_2511_13778_b200/dist.py. Header-only; link libadpb200.so,
// the CUDA runtime and libnccl.
//
// Rank r owns rows [r0, r0+m) of op(A) and C (column-major, ld lda / ldc) and
// the B column slab r: k x (n/world), column-major, leading dimension k
// (n/world a multiple of 8). The collectives run on the caller's stream
// (statistics all-gather, decision max-allreduce) and on a second stream for
// the B-plane all-gather, which overlaps the GEMM of the rank's own columns
// (phases 5/6 of adpb200_dgemm_dist). One 8-byte host read of the reduced
// decision input sizes that all-gather. Every rank takes the same decision:
// the assembled C is bit-identical to one GPU's adpb200_dgemm.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "adpb200.h"

namespace adpb200 {

namespace nccl_detail {
inline int cu(cudaError_t e) { return e == cudaSuccess ? ADPB200_OK : ADPB200_ERR_RUNTIME; }
inline int nc(ncclResult_t r) { return r == ncclSuccess ? ADPB200_OK : ADPB200_ERR_RUNTIME; }
}  // namespace nccl_detail

// Slab buffers for the fused phase 7 (the GEMM reads every rank's B planes in
// place over NVLink): two per rank (calls alternate, see dist.py PeerSlabs),
// shared once per communicator through CUDA IPC handles all-gathered over NCCL.
struct PeerSlabs {
    int world = 0, rank = 0, device = 0, calls = 0;
    bool pull = false;           // copy engines pull each peer's record under the GEMM (phase 7 per rank)
    void* own[2] = {nullptr, nullptr};
    std::vector<void*> ptrs[2];  // entry r: rank r's buffer in this process
    uint32_t epoch[2] = {0, 0};  // uses of each buffer so far (the in-place path's flag values)
};

inline int peer_slabs_create(PeerSlabs& ps, ncclComm_t comm, int rank, int world, int device, int64_t n, int64_t k,
                             const adpb200_options* opt, cudaStream_t st) {
    using namespace nccl_detail;
    int64_t sz[4];
    int rc = adpb200_dist_sizes(n, k, world, opt, sz);
    if (rc) return rc;
    ps.world = world;
    ps.rank = rank;
    ps.device = device;
    std::vector<uint8_t> mine(128), all(size_t(128) * world);
    for (int b = 0; b < 2 && !rc; ++b) rc = adpb200_ipc_alloc(device, sz[3], &ps.own[b], mine.data() + 64 * b);
    uint8_t* dbuf = nullptr;
    if (!rc) rc = cu(cudaMalloc(&dbuf, all.size()));
    if (!rc) rc = cu(cudaMemcpyAsync(dbuf + 128 * rank, mine.data(), 128, cudaMemcpyHostToDevice, st));
    if (!rc) rc = nc(ncclAllGather(dbuf + 128 * rank, dbuf, 128, ncclUint8, comm, st));
    if (!rc) rc = cu(cudaMemcpyAsync(all.data(), dbuf, all.size(), cudaMemcpyDeviceToHost, st));
    if (!rc) rc = cu(cudaStreamSynchronize(st));
    if (dbuf) cudaFree(dbuf);
    for (int b = 0; b < 2 && !rc; ++b) {
        ps.ptrs[b].assign(world, nullptr);
        for (int r = 0; r < world && !rc; ++r) {
            if (r == rank) ps.ptrs[b][r] = ps.own[b];
            else rc = adpb200_ipc_open(device, all.data() + 128 * r + 64 * b, &ps.ptrs[b][r]);
        }
    }
    return rc;
}

inline void peer_slabs_destroy(PeerSlabs& ps) {
    cudaDeviceSynchronize();
    for (int b = 0; b < 2; ++b) {
        for (int r = 0; r < int(ps.ptrs[b].size()); ++r)
            if (r != ps.rank && ps.ptrs[b][r]) adpb200_ipc_close(ps.ptrs[b][r]);
        if (ps.own[b]) adpb200_ipc_free(ps.own[b]);
        ps.own[b] = nullptr;
        ps.ptrs[b].clear();
    }
}

// Returns an adpb200 status (0 ok, 2 runtime incl. CUDA/NCCL failures, 3 contract).
// peers (optional, from peer_slabs_create for this n, k): the fused phase 7 — no
// plane all-gather. In place (default): no host read and no host barrier — the
// streams order the ranks through the slab buffers' ready / consumed flags (CUDA
// stream memory operations on the IPC mappings) and the device plan decides between
// the GEMM and the native fallback (phase 8 / phase 7 with nsl = 0). Pulled
// (peers->pull): one 8-byte host read sizes the copies, then a barrier.
inline int dgemm_dist_nccl(adpb200_handle h, ncclComm_t comm, int rank, int world, char transa, int64_t m_global,
                           int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
                           const double* B_slab, double beta, double* C, int64_t ldc, const adpb200_options* opt,
                           adpb200_trace* trace_dev, cudaStream_t st, PeerSlabs* peers = nullptr) {
    using namespace nccl_detail;
    int64_t sz[4];
    int rc = adpb200_dist_sizes(n, k, world, opt, sz);
    if (rc) return rc;
    const int64_t nrec = sz[0], hdr = sz[1], plane_bytes = sz[2], cap_bytes = sz[3];
    int32_t *bl = nullptr, *ba = nullptr, *xchg = nullptr;
    int8_t *slab = nullptr, *gathered = nullptr;
    double* bfull = nullptr;
    cudaStream_t comm_st = nullptr;
    cudaEvent_t ev_slab = nullptr, ev_gather = nullptr;
    int32_t xh[2] = {0, 0};
    int32_t dec[4] = {0, 0, 0, 0};
    auto phase = [&](int p, const void* g, int nsl) {
        return adpb200_dgemm_dist(h, p, m_global, world, rank, transa, m, n, k, alpha, A, lda, B_slab, beta, C, ldc,
                                  opt, trace_dev, bl, ba, xchg, slab, g, nsl, st);
    };
    const int buf = peers ? peers->calls++ % 2 : 0;
    const std::vector<void*>* pp = peers ? &peers->ptrs[buf] : nullptr;
    const bool in_place = pp && !peers->pull;
    rc = cu(cudaMallocAsync(&bl, size_t(nrec) * 4, st));
    if (!rc) rc = cu(cudaMallocAsync(&ba, size_t(nrec) * 4 * world, st));
    if (!rc) rc = cu(cudaMallocAsync(&xchg, 8, st));
    if (pp) slab = static_cast<int8_t*>((*pp)[rank]);
    else if (!rc) rc = cu(cudaMallocAsync(&slab, size_t(cap_bytes), st));
    if (!rc) rc = cu(cudaMemsetAsync(xchg, 0, 8, st));
    // 1: exponent statistics of the A rows and the B slab; all-gather the slab records
    if (!rc) rc = phase(1, nullptr, 0);
    if (!rc) rc = nc(ncclAllGather(bl, ba, size_t(nrec), ncclInt32, comm, st));
    // 2: ESC of the local rows against every column; max-allreduce {exceptional, esc}
    if (!rc) rc = phase(2, nullptr, 0);
    if (!rc) rc = nc(ncclAllReduce(xchg, xchg, 2, ncclInt32, ncclMax, comm, st));
    if (in_place) {
        // host-sync-free fused path: slice into this buffer only after every peer has
        // finished reading it (its previous use), publish it, wait for every peer's
        // slab, run the device-decided phase 7, then release this call's slabs
        const uint32_t e = ++peers->epoch[buf];
        const int64_t off_ready = adpb200_dist_flag_offset(cap_bytes, 0);
        const int64_t off_used = adpb200_dist_flag_offset(cap_bytes, 1);
        for (int r = 0; r < world && !rc; ++r)
            if (r != rank) rc = adpb200_stream_wait_geq(static_cast<char*>((*pp)[r]) + off_used, e - 1, st);
        if (!rc) rc = phase(3, nullptr, 0);
        if (!rc) rc = phase(8, nullptr, 0);
        if (!rc) rc = adpb200_stream_write_flag(slab + off_ready, e, st);
        for (int r = 0; r < world && !rc; ++r)
            if (r != rank) rc = adpb200_stream_wait_geq(static_cast<char*>((*pp)[r]) + off_ready, e, st);
        if (!rc) rc = phase(7, pp->data(), 0);
        if (!rc) rc = adpb200_stream_write_flag(slab + off_used, e, st);
        if (bl) cudaFreeAsync(bl, st);
        if (ba) cudaFreeAsync(ba, st);
        if (xchg) cudaFreeAsync(xchg, st);
        return rc;
    }
    // 3: decision, slicing; the host learns how many planes travel
    if (!rc) rc = phase(3, nullptr, 0);
    if (!rc) rc = cu(cudaMemcpyAsync(xh, xchg, 8, cudaMemcpyDeviceToHost, st));
    if (!rc) rc = cu(cudaStreamSynchronize(st));
    if (!rc) rc = adpb200_dist_decision(opt, xh, m_global, n, k, dec);
    const int nsl = dec[2];
    if (!rc && nsl > 0 && pp) {
        // pulled: every rank's slab is sliced (the host sync above) once this barrier passes
        rc = nc(ncclAllReduce(xchg, xchg, 1, ncclInt32, ncclMax, comm, st));
        if (!rc) rc = cu(cudaStreamSynchronize(st));
        if (!rc) {
            // own columns first, then rank by rank: the copy engines pull rank r's record
            // into local memory on a side stream while the GEMM of the previous rank runs
            const int64_t rec = hdr + int64_t(nsl) * plane_bytes;
            std::vector<cudaEvent_t> ready(world, nullptr);
            rc = cu(cudaMallocAsync(&gathered, size_t(rec) * world, st));
            if (!rc) rc = cu(cudaStreamCreateWithFlags(&comm_st, cudaStreamNonBlocking));
            if (!rc) rc = cu(cudaEventCreateWithFlags(&ev_slab, cudaEventDisableTiming));
            if (!rc) rc = cu(cudaEventRecord(ev_slab, st));
            if (!rc) rc = cu(cudaStreamWaitEvent(comm_st, ev_slab, 0));
            for (int j = 1; j < world && !rc; ++j) {
                const int r = (rank + j) % world;
                rc = adpb200_copy_async(gathered + int64_t(r) * rec, (*pp)[r], rec, comm_st);
                if (!rc) rc = cu(cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming));
                if (!rc) rc = cu(cudaEventRecord(ready[r], comm_st));
            }
            std::vector<const void*> one(world, nullptr);
            for (int j = 0; j < world && !rc; ++j) {
                const int r = (rank + j) % world;
                std::fill(one.begin(), one.end(), nullptr);
                one[r] = r == rank ? (*pp)[r] : static_cast<const void*>(gathered + int64_t(r) * rec);
                if (r != rank) rc = cu(cudaStreamWaitEvent(st, ready[r], 0));
                if (!rc) rc = phase(7, one.data(), nsl);
            }
            for (cudaEvent_t e : ready)
                if (e) cudaEventDestroy(e);
        }
    } else if (!rc && nsl > 0) {
        // B planes all-gathered on a second stream while this rank's own columns compute
        const int64_t rec = hdr + int64_t(nsl) * plane_bytes;
        rc = cu(cudaMallocAsync(&gathered, size_t(rec) * world, st));
        if (!rc) rc = cu(cudaStreamCreateWithFlags(&comm_st, cudaStreamNonBlocking));
        if (!rc) rc = cu(cudaEventCreateWithFlags(&ev_slab, cudaEventDisableTiming));
        if (!rc) rc = cu(cudaEventCreateWithFlags(&ev_gather, cudaEventDisableTiming));
        if (!rc) rc = cu(cudaEventRecord(ev_slab, st));
        if (!rc) rc = cu(cudaStreamWaitEvent(comm_st, ev_slab, 0));
        if (!rc) rc = nc(ncclAllGather(slab, gathered, size_t(rec), ncclInt8, comm, comm_st));
        if (!rc) rc = cu(cudaEventRecord(ev_gather, comm_st));
        if (!rc) rc = phase(5, slab, nsl);
        if (!rc) rc = cu(cudaStreamWaitEvent(st, ev_gather, 0));
        if (!rc) rc = phase(6, gathered, nsl);
    } else if (!rc) {
        // native fallback: every rank needs all of B in FP64 (the slabs concatenate to B, ld = k)
        rc = cu(cudaMallocAsync(&bfull, size_t(k) * size_t(n) * 8, st));
        if (!rc) rc = nc(ncclAllGather(B_slab, bfull, size_t(k) * size_t(n / world), ncclFloat64, comm, st));
        if (!rc) rc = phase(6, bfull, 0);
    }
    // stream-ordered frees; the events / side stream are released once their work is done
    if (bl) cudaFreeAsync(bl, st);
    if (ba) cudaFreeAsync(ba, st);
    if (xchg) cudaFreeAsync(xchg, st);
    if (slab && !pp) cudaFreeAsync(slab, st);
    if (gathered) cudaFreeAsync(gathered, st);
    if (bfull) cudaFreeAsync(bfull, st);
    if (comm_st) {
        cudaStreamSynchronize(comm_st);
        cudaStreamDestroy(comm_st);
    }
    if (ev_slab) cudaEventDestroy(ev_slab);
    if (ev_gather) cudaEventDestroy(ev_gather);
    return rc;
}

}  // namespace adpb200

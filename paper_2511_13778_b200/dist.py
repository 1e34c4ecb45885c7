"""Row-block partition of one large DGEMM across the GPUs of a node.

One process per GPU (torch.distributed, NCCL over NVLink). Rank r owns the
rows rows_of(r) of op(A) and C. Two layouts of B:

* dgemm_rows: every rank holds all of op(B). The only exchange is the ADP
  decision input, a max-allreduce of {exceptional, esc_bits} (two int32)
  between the guardrail and compute phases of adpb200_dgemm_rows.
* dgemm_dist: rank r holds the column slab cols_of(r) of B. The B exponent
  statistics are all-gathered (so each rank's ESC covers every column), the
  decision input is max-allreduced, and each rank's B slice planes (int8,
  s/8 of the FP64 bytes) are all-gathered before the tcgen05 GEMM — or, on
  the native fallback, the FP64 B slabs themselves.

Every rank takes the same decision with the same slice count, so the
assembled C is bit-identical to the single-GPU result.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from ._lib import check, lib
from .adp import AdpConfig, Handle, _ptr, _stream


def rows_of(rank: int, world: int, m: int, align: int = 128) -> Tuple[int, int]:
    """[start, stop) of rank's row block: contiguous, multiples of `align`
    rows (the GEMM's M tile) except possibly the last, as even as possible."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    tiles = (m + align - 1) // align
    base, extra = divmod(tiles, world)
    t0 = rank * base + min(rank, extra)
    t1 = t0 + base + (1 if rank < extra else 0)
    return min(m, t0 * align), min(m, t1 * align)


def reduce_xchg(xchg: torch.Tensor, group=None) -> None:
    """Max-reduce the guardrail exchange block over the ranks (in place)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if dist.get_backend(group) == "gloo" and xchg.is_cuda:
            t = xchg.cpu()
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            xchg.copy_(t)
        else:
            dist.all_reduce(xchg, op=dist.ReduceOp.MAX, group=group)


def dgemm_rows(transa: str, transb: str, m_global: int, m: int, n: int, k: int, alpha: float, A: torch.Tensor,
               lda: int, B: torch.Tensor, ldb: int, beta: float, C_: torch.Tensor, ldc: int,
               config: Optional[AdpConfig] = None, handle: Optional[Handle] = None, group=None,
               trace: Optional[torch.Tensor] = None, xchg: Optional[torch.Tensor] = None) -> None:
    """This rank's share of a row-partitioned ADP DGEMM (column-major storage
    of the local block: C_ is m x n with leading dimension ldc). Stream
    ordered end to end; the allreduce runs on NCCL's stream, ordered against
    the current stream by torch."""
    config = config or AdpConfig()
    dev = C_.device
    handle = handle or Handle.default(dev.index)
    if xchg is None:
        xchg = torch.zeros(2, dtype=torch.int32, device=dev)
    o = config.to_c()
    args = (m_global, transa.encode()[:1], transb.encode()[:1], m, n, k, float(alpha), _ptr(A), lda, _ptr(B), ldb,
            float(beta), _ptr(C_), ldc, C.byref(o), None if trace is None else C.c_void_p(trace.data_ptr()),
            C.c_void_p(xchg.data_ptr()), _stream(dev))
    check(lib().adpb200_dgemm_rows(handle.h, 1, *args))
    reduce_xchg(xchg, group)
    check(lib().adpb200_dgemm_rows(handle.h, 2, *args))


# ---- B distributed by column slabs, slice planes all-gathered ---------------------
def cols_of(rank: int, world: int, n: int) -> Tuple[int, int]:
    """[start, stop) of rank's B column slab (equal slabs; n/world must be a multiple of 8)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if n % world or (n // world) % 8:
        raise ValueError("cols_of: n must split into equal slabs of a multiple of 8 columns")
    nr = n // world
    return rank * nr, (rank + 1) * nr


def dist_sizes(n: int, k: int, world: int, config: Optional[AdpConfig] = None):
    """(bstats record int32 count, slab header bytes, bytes per slab plane, slab capacity bytes)."""
    o = (config or AdpConfig()).to_c()
    out = (C.c_int64 * 4)()
    check(lib().adpb200_dist_sizes(n, k, world, C.byref(o), out))
    return tuple(int(x) for x in out)


def dist_decision(xchg_host, m_global: int, n: int, k: int, config: Optional[AdpConfig] = None):
    """decide() on the reduced exchange block: (path, slices, nsl planes to gather, GEMM variant)."""
    o = (config or AdpConfig()).to_c()
    x = (C.c_int32 * 2)(int(xchg_host[0]), int(xchg_host[1]))
    out = (C.c_int32 * 4)()
    check(lib().adpb200_dist_decision(C.byref(o), x, m_global, n, k, out))
    return tuple(int(v) for v in out)


class LazyDecision:
    """(path, slices, nsl) of a dist call whose host never read the decision (the
    fused in-place path): computed from the reduced exchange block on first access,
    which synchronises with the device then."""

    def __init__(self, xchg: torch.Tensor, m_global: int, n: int, k: int, config: AdpConfig):
        self._args = (xchg, m_global, n, k, config)
        self._value = None

    def value(self) -> Tuple[int, int, int]:
        if self._value is None:
            xchg, m_global, n, k, config = self._args
            self._value = dist_decision(xchg.cpu().tolist(), m_global, n, k, config)[:3]
        return self._value

    def __getitem__(self, i):
        return self.value()[i]

    def __iter__(self):
        return iter(self.value())

    def __len__(self):
        return 3

    def __eq__(self, other):
        return tuple(self.value()) == tuple(other)

    def __repr__(self):
        return f"LazyDecision{tuple(self.value())}"


def flag_ptr(slab_ptr: int, slab_bytes: int, which: int) -> int:
    """Address of a slab buffer's fused-path flag (which = 0 ready, 1 consumed)."""
    return int(slab_ptr) + int(lib().adpb200_dist_flag_offset(slab_bytes, which))


def dgemm_dist_steps(world: int, transa: str, m_global: int, m: int, n: int, k: int, alpha: float,
                     A: torch.Tensor, lda: int, B_slab: torch.Tensor, beta: float, C_: torch.Tensor, ldc: int,
                     config: Optional[AdpConfig] = None, handle: Optional[Handle] = None,
                     trace: Optional[torch.Tensor] = None, rank: int = 0, overlap: bool = True,
                     slab_ptrs: Optional[Sequence[int]] = None, pull: bool = False, epoch: int = 1):
    """The B-distributed ADP DGEMM of one rank as a generator of collective
    requests, so that the same orchestration runs under torch.distributed
    (dgemm_dist) and under a single-process multi-rank driver (the tests):

        ("all_gather", out, inp)   out = concatenation over ranks of inp
        ("all_gather_async", out, inp)  the same, started without waiting
        ("wait",)                  wait for the pending asynchronous all-gather
        ("all_reduce_max", t)      t = elementwise max over ranks (in place)

    With overlap (default) the B-plane all-gather runs while the GEMM tiles that
    need only this rank's own B columns compute (phases 5 and 6).

    With slab_ptrs (every rank's slab buffer as mapped in this process, entry
    `rank` its own: PeerSlabs over CUDA IPC, or zeroed buffers of one device in
    the tests) there is no plane all-gather: the fused phase 7 GEMM reads the B
    planes of every rank in place over peer memory, with no host read and no
    host barrier — the streams order the ranks through each buffer's ready /
    consumed flags (`epoch` = this buffer's use count, 1, 2, ...; see
    adpb200.h) and the device plan picks the GEMM or the native fallback:
        ("device_barrier",)        a no-op for real ranks (the flags order them);
                                   the virtual-rank driver enqueues every rank's
                                   phase 3 before any rank's wait
    With pull=True the copy engines pull each peer's record into local memory
    on a side stream while the GEMM of the previous rank's columns runs (one
    phase-7 launch per rank, own columns first; after one 8-byte host read and
        ("barrier",)               every rank past its phase 3 (slab sliced)
    ): the transfer overlaps the math rank by rank and the GEMM reads local,
    L2-cached planes.

    Rank owns rows of op(A) / C (column-major local block, ldc) and the B
    column slab B_slab (k x n/world column-major, compact: a (n/world, k)
    row-major torch tensor). Stream-ordered except, on the all-gather and pull
    paths, one 8-byte host read of the reduced decision input (it sizes the
    transfer). Returns (path, slices, nsl) — lazily on the in-place fused path."""
    config = config or AdpConfig()
    dev = C_.device
    handle = handle or Handle.default(dev.index)
    o = config.to_c()
    nrec, hdr, plane_bytes, cap_bytes = dist_sizes(n, k, world, config)
    bl = torch.empty(nrec, dtype=torch.int32, device=dev)
    ba = torch.empty(nrec * world, dtype=torch.int32, device=dev)
    xchg = torch.zeros(2, dtype=torch.int32, device=dev)
    fused = slab_ptrs is not None
    slab = None if fused else torch.empty(cap_bytes, dtype=torch.int8, device=dev)
    slab_p = C.c_void_p(int(slab_ptrs[rank])) if fused else _ptr(slab)
    st = _stream(dev)
    tr = None if trace is None else C.c_void_p(trace.data_ptr())

    def phase(p, gathered=None, nsl=0):
        check(lib().adpb200_dgemm_dist(handle.h, p, m_global, world, rank, transa.encode()[:1], m, n, k, float(alpha),
                                       _ptr(A), lda, _ptr(B_slab), float(beta), _ptr(C_), ldc, C.byref(o), tr,
                                       _ptr(bl), _ptr(ba), _ptr(xchg), slab_p, gathered, int(nsl), st))

    phase(1)
    yield ("all_gather", ba, bl)
    phase(2)
    yield ("all_reduce_max", xchg)
    if fused and not pull:
        # in place, host-sync free: slice into this buffer once every peer has finished
        # reading its previous use, publish it, wait for every peer's, GEMM (or native
        # fallback) on the device's decision, release
        ldev = lib()
        for r in range(world):
            if r != rank:
                check(ldev.adpb200_stream_wait_geq(C.c_void_p(flag_ptr(slab_ptrs[r], cap_bytes, 1)), epoch - 1, st))
        phase(3)
        phase(8)
        check(ldev.adpb200_stream_write_flag(C.c_void_p(flag_ptr(slab_ptrs[rank], cap_bytes, 0)), epoch, st))
        yield ("device_barrier",)
        for r in range(world):
            if r != rank:
                check(ldev.adpb200_stream_wait_geq(C.c_void_p(flag_ptr(slab_ptrs[r], cap_bytes, 0)), epoch, st))
        ptrs = (C.c_void_p * world)(*[int(p) for p in slab_ptrs])
        phase(7, C.cast(ptrs, C.c_void_p), 0)
        check(ldev.adpb200_stream_write_flag(C.c_void_p(flag_ptr(slab_ptrs[rank], cap_bytes, 1)), epoch, st))
        return LazyDecision(xchg, m_global, n, k, config)
    phase(3)
    path, s, nsl, _ = dist_decision(xchg.cpu().tolist(), m_global, n, k, config)  # (syncs: slab sliced)
    if nsl > 0 and fused:  # pulled
        yield ("barrier",)
        rec = hdr + nsl * plane_bytes
        staging = torch.empty(rec * world, dtype=torch.int8, device=dev)
        cur = torch.cuda.current_stream(dev)
        side = torch.cuda.Stream(dev)
        staging.record_stream(side)
        side.wait_stream(cur)
        order = [(rank + j) % world for j in range(world)]
        ready = {}
        with torch.cuda.stream(side):
            for r in order[1:]:
                check(lib().adpb200_copy_async(C.c_void_p(staging.data_ptr() + r * rec), C.c_void_p(int(slab_ptrs[r])),
                                               rec, C.c_void_p(side.cuda_stream)))
                ready[r] = torch.cuda.Event()
                ready[r].record(side)
        for r in order:
            ptrs = (C.c_void_p * world)()
            if r == rank:
                ptrs[r] = int(slab_ptrs[r])
            else:
                cur.wait_event(ready[r])
                ptrs[r] = staging.data_ptr() + r * rec
            phase(7, C.cast(ptrs, C.c_void_p), nsl)
        return (path, s, nsl)
    if nsl > 0:
        rec = hdr + nsl * plane_bytes
        gathered = torch.empty(rec * world, dtype=torch.int8, device=dev)
        if overlap:
            yield ("all_gather_async", gathered, slab[:rec])
            phase(5, C.c_void_p(slab.data_ptr()), nsl)     # own columns while the planes travel
            yield ("wait",)
            phase(6, C.c_void_p(gathered.data_ptr()), nsl)
            return (path, s, nsl)
        yield ("all_gather", gathered, slab[:rec])
    else:
        gathered = torch.empty((n, k), dtype=torch.float64, device=dev)  # column-major B, ldb = k
        yield ("all_gather", gathered.view(-1), B_slab.reshape(-1))
    phase(4, C.c_void_p(gathered.data_ptr()), nsl)
    return (path, s, nsl)


def dgemm_dist(transa: str, m_global: int, m: int, n: int, k: int, alpha: float, A: torch.Tensor, lda: int,
               B_slab: torch.Tensor, beta: float, C_: torch.Tensor, ldc: int, config: Optional[AdpConfig] = None,
               handle: Optional[Handle] = None, group=None, trace: Optional[torch.Tensor] = None,
               peers: Optional["PeerSlabs"] = None, pull: bool = False):
    """This rank's share of a row-partitioned ADP DGEMM with B distributed by
    column slabs: exponent stats and B slice planes all-gathered, the ADP
    decision input max-allreduced, all over NCCL (torch.distributed). With
    `peers` (a PeerSlabs for this n, k) the plane all-gather is replaced by
    the fused phase 7: the GEMM reads every rank's planes over NVLink (pull=True:
    the copy engines pull them rank by rank while the GEMM runs on local copies)."""
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    slab_ptrs, epoch = peers.next_with_epoch() if peers is not None else (None, 1)
    gen = dgemm_dist_steps(world, transa, m_global, m, n, k, alpha, A, lda, B_slab, beta, C_, ldc, config, handle,
                           trace, rank=rank, slab_ptrs=slab_ptrs, pull=pull, epoch=epoch)
    return drive_collectives(gen, world, group)


class PeerSlabs:
    """Slab record buffers for the fused phase 7, shared over CUDA IPC: each rank
    cudaMallocs two (calls alternate between them, so a rank slicing call i+2 can
    never overwrite planes a peer still reads for call i: every rank passes call
    i+1's barrier only after its own call-i GEMM has completed), exports the IPC
    handles, all-gathers them (torch.distributed, CPU objects) and maps its
    peers' buffers (lazy NVLink peer access). `next()` -> the pointer list of
    the buffer for the next call, entry r = rank r's buffer in this process."""

    def __init__(self, n: int, k: int, config: Optional[AdpConfig] = None, group=None, device: int = 0):
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self.device = device
        _, _, _, cap_bytes = dist_sizes(n, k, self.world, config)
        self.own, self.opened, self.ptrs = [], [], []
        self.group = group
        # every step is agreed on by all ranks, so a failure on one rank raises on all
        # of them (no rank is left waiting in a collective the others never enter)
        handles, err = [], None
        try:
            for _ in range(2):
                p, h = C.c_void_p(), (C.c_uint8 * 64)()
                check(lib().adpb200_ipc_alloc(device, cap_bytes, C.byref(p), h))
                self.own.append(p.value)
                handles.append(bytes(h))
        except Exception as e:  # noqa: BLE001 — reported on every rank below
            err = f"rank {self.rank}: {e}"
        allh = self._gather(None if err else handles, err)
        try:
            for b in range(2):
                row = []
                for r in range(self.world):
                    if r == self.rank:
                        row.append(self.own[b])
                        continue
                    p = C.c_void_p()
                    check(lib().adpb200_ipc_open(device, (C.c_uint8 * 64).from_buffer_copy(allh[r][b]),
                                                 C.byref(p)))
                    self.opened.append(p.value)
                    row.append(p.value)
                self.ptrs.append(row)
        except Exception as e:  # noqa: BLE001
            err = f"rank {self.rank}: {e}"
        self._gather(err is None, err)
        self.calls = 0

    def _gather(self, item, err):
        """all_gather_object of `item`; raises on every rank if any rank reported an error."""
        got = [(item, err)]
        if self.world > 1:
            got = [None] * self.world
            dist.all_gather_object(got, (item, err), group=self.group)
        errs = [e for _, e in got if e]
        if errs:
            self.close()
            raise RuntimeError("PeerSlabs: " + "; ".join(errs))
        return [x for x, _ in got]

    def next(self):
        return self.next_with_epoch()[0]

    def next_with_epoch(self):
        """(pointer list, epoch) for the next call: buffers alternate, and the epoch
        counts the uses of that buffer (the value its flags take, 1, 2, ...)."""
        b = self.calls % 2
        self.calls += 1
        return self.ptrs[b], self.calls // 2 + (self.calls % 2)

    def close(self) -> None:
        torch.cuda.synchronize(self.device)
        for p in getattr(self, "opened", []):
            lib().adpb200_ipc_close(C.c_void_p(p))
        for p in getattr(self, "own", []):
            lib().adpb200_ipc_free(C.c_void_p(p))
        self.opened, self.own, self.ptrs = [], [], []


def drive_collectives(gen, world: int, group=None):
    """Run a dgemm_dist_steps-style generator, serving its collective requests
    with torch.distributed (NCCL on GPUs, gloo in the CPU tests). Returns the
    generator's return value."""
    pending = None
    try:
        req = next(gen)
        while True:
            if req[0] in ("all_gather", "all_gather_async"):
                asy = req[0] == "all_gather_async"
                if world > 1 and dist.get_backend(group) == "gloo":
                    # (gloo: staged through host memory when the buffers live on a GPU)
                    src = req[2].contiguous().view(-1)
                    out = req[1].view(-1)
                    parts = [torch.empty_like(src, device="cpu") for _ in range(world)]
                    dist.all_gather(parts, src.cpu(), group=group)
                    out.copy_(torch.cat(parts))
                elif world > 1:
                    # async: NCCL's stream waits for the inputs; the caller's stream only waits at "wait"
                    work = dist.all_gather_into_tensor(req[1], req[2].contiguous(), group=group, async_op=asy)
                    if asy:
                        pending = work
                else:
                    req[1].copy_(req[2].reshape(req[1].shape))
            elif req[0] == "wait":
                if pending is not None:
                    pending.wait()
                    pending = None
            elif req[0] == "all_reduce_max":
                reduce_xchg(req[1], group)
            elif req[0] == "barrier":
                if world > 1:
                    dist.barrier(group=group)
            elif req[0] == "device_barrier":
                pass  # the streams' flags order the ranks
            else:
                raise ValueError(f"unknown collective request {req[0]!r}")
            req = next(gen)
    except StopIteration as fin:
        return fin.value

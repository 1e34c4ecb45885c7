"""CPU (gloo, world_size 2): the host logic of the multi-GPU row partition.

* rows_of() tiles [0, m) exactly, in 128-row multiples, balanced;
* the guardrail exchange block {exceptional, esc_bits} is max-reduced so
  every rank reaches the same ADP decision (paper_2511_13778_b200/dist.py);
* decide() evaluated on the reduced block is identical on every rank.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_13778_b200 import AdpConfig, decide
    from paper_2511_13778_b200.dist import reduce_xchg, rows_of

    m = 8192 * world + 77
    r0, r1 = rows_of(rank, world, m)
    # each rank saw different local guardrail results
    local = {0: [0, 3], 1: [1, 9]}[rank]
    x = torch.tensor(local, dtype=torch.int32)
    reduce_xchg(x)
    d = decide(bool(x[0] & 1), bool(x[0] & 2), m, 8192, 8192, int(x[1]), AdpConfig())
    d_ok = decide(False, False, m, 8192, 8192, int(x[1]), AdpConfig())
    results[rank] = (r0, r1, x.tolist(), d, d_ok)
    dist.destroy_process_group()


def test_row_partition_and_decision_exchange():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    (a0, a1, xa, da, oka), (b0, b1, xb, db, okb) = results[0], results[1]
    assert (a0, a1) == (0, 8320) and (b0, b1) == (8320, 16461)
    assert xa == xb == [1, 9]                     # max over ranks
    assert da == db and da[1] == "exceptional_values"   # one rank's NaN sends every rank to the fallback
    assert oka == okb and oka[0] == "emulated" and oka[2] == 8


@pytest.mark.parametrize("world,m", [(1, 5), (2, 129), (4, 8192), (8, 32768), (8, 1000), (3, 128)])
def test_rows_of_covers_exactly(world, m):
    from paper_2511_13778_b200.dist import rows_of

    spans = [rows_of(r, world, m) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == m
    for (s0, e0), (s1, e1) in zip(spans, spans[1:]):
        assert e0 == s1 and s0 <= e0
    for s, e in spans[:-1]:
        assert s % 128 == 0 and e % 128 == 0


# ---- B-distributed path: host logic ---------------------------------------------------
def test_cols_of_and_contract():
    from paper_2511_13778_b200.dist import cols_of

    assert [cols_of(r, 4, 512) for r in range(4)] == [(0, 128), (128, 256), (256, 384), (384, 512)]
    with pytest.raises(ValueError):
        cols_of(0, 3, 512)      # unequal slabs
    with pytest.raises(ValueError):
        cols_of(0, 8, 8 * 12)   # slab not a multiple of 8


def test_dist_sizes():
    from paper_2511_13778_b200 import AdpConfig
    from paper_2511_13778_b200.dist import dist_sizes

    nrec, hdr, plane, cap = dist_sizes(8192, 8192, 8)
    nr, t = 1024, 32
    assert nrec == 2 * t * nr + nr and hdr == 4096 and plane == 8192 * nr
    # auto mode: max_slices planes (or the FP64 slab, whichever is larger) + the fused path's flags
    assert cap == max(hdr + 18 * plane, nr * 8192 * 8) + 256
    assert dist_sizes(8192, 100, 8, AdpConfig(mode=1, forced_slices=7))[3] == 1024 * 4 + 7 * 128 * 1024 + 256
    assert dist_sizes(8192, 100, 8, AdpConfig(mode=1, forced_slices=5))[3] == 1024 * 100 * 8 + 256
    with pytest.raises(ValueError):
        dist_sizes(100, 100, 8)


def test_dist_decision_matches_decide():
    from paper_2511_13778_b200 import AdpConfig, PAIRS_TARGET, decide
    from paper_2511_13778_b200.dist import dist_decision

    for cfg in (AdpConfig(), AdpConfig(pair_limit=PAIRS_TARGET), AdpConfig(mode=1, forced_slices=9)):
        for exc, esc in [(0, 1), (0, 8), (0, 11), (0, 48), (1, 3), (2, 0), (3, 5)]:
            path, s, nsl, var = dist_decision([exc, esc], 8192, 8192, 8192, cfg)
            d = decide(bool(exc & 1), bool(exc & 2), 8192, 8192, 8192, esc, cfg)
            assert (path == 0) == (d[0] == "emulated")
            assert s == (d[2] if d[0] == "emulated" else 0)
            assert (nsl > 0) == (path == 0) and nsl <= max(s, 0)
    # the fast policy gathers s planes, the variant follows the diagonal count
    assert dist_decision([0, 1], 8192, 8192, 8192, AdpConfig(pair_limit=PAIRS_TARGET)) == (0, 7, 7, 64)
    assert dist_decision([0, 8], 8192, 8192, 8192, AdpConfig(pair_limit=PAIRS_TARGET)) == (0, 8, 8, 48)
    # certified ESC: applied unless some rank flagged a zero count (256); exceptional still wins
    cc = AdpConfig(pair_limit=PAIRS_TARGET, esc_method="certified")
    assert dist_decision([0, 8], 8192, 8192, 8192, cc) == (0, 7, 7, 64)
    assert dist_decision([256, 8], 8192, 8192, 8192, cc) == (0, 8, 8, 48)
    assert dist_decision([257, 8], 8192, 8192, 8192, cc)[0] == 1
    assert dist_decision([0, 8], 100, 8192, 8192, cc) == (1, 0, 0, 0)  # too small: no ESC, no certificate
    # two certificate levels in bits 8-9 (max over ranks): v = 0 level 0 held, 1 only level 1, 2 neither
    assert dist_decision([0, 12], 8192, 8192, 8192, cc)[1] == 7
    assert dist_decision([1 << 8, 12], 8192, 8192, 8192, cc)[1] == 8
    assert dist_decision([2 << 8, 12], 8192, 8192, 8192, cc)[1] == 9
    assert dist_decision([2 << 8, 12], 8192, 8192, 8192, AdpConfig(pair_limit=PAIRS_TARGET))[1] == 9


def _collective_worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_13778_b200.dist import drive_collectives

    def fake_rank_steps():
        # the request sequence of dgemm_dist_steps on one rank, CPU tensors
        bl = torch.arange(6, dtype=torch.int32) + 10 * rank
        ba = torch.empty(6 * world, dtype=torch.int32)
        yield ("all_gather", ba, bl)
        x = torch.tensor([rank & 1, 3 + 4 * rank], dtype=torch.int32)
        yield ("all_reduce_max", x)
        slab = torch.full((16,), rank + 1, dtype=torch.int8)
        g = torch.empty(8 * world, dtype=torch.int8)
        yield ("all_gather_async", g, slab[:8])
        yield ("wait",)
        return ba.tolist(), x.tolist(), g.tolist()

    results[rank] = drive_collectives(fake_rank_steps(), world)
    dist.destroy_process_group()


def test_drive_collectives_gloo():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_collective_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for r in range(world):
        ba, x, g = results[r]
        assert ba == list(range(6)) + [10 + i for i in range(6)]
        assert x == [1, 7]
        assert g == [1] * 8 + [2] * 8


def test_peer_slabs_epochs_alternate_buffers():
    """PeerSlabs.next_with_epoch: buffers alternate per call and the epoch counts the
    uses of the chosen buffer (the fused path's flag values)."""
    from paper_2511_13778_b200.dist import PeerSlabs

    ps = object.__new__(PeerSlabs)  # no IPC: only the call bookkeeping
    ps.ptrs, ps.calls = [["b0"], ["b1"]], 0
    got = [ps.next_with_epoch() for _ in range(5)]
    assert [p[0] for p, _ in got] == ["b0", "b1", "b0", "b1", "b0"]
    assert [e for _, e in got] == [1, 1, 2, 2, 3]


def test_flag_offsets_and_lazy_decision():
    import torch

    from paper_2511_13778_b200 import AdpConfig
    from paper_2511_13778_b200.dist import LazyDecision, dist_decision, dist_sizes, flag_ptr

    cap = dist_sizes(1024, 512, 4)[3]
    assert flag_ptr(1000, cap, 0) == 1000 + cap - 256 and flag_ptr(1000, cap, 1) == 1000 + cap - 128
    xchg = torch.tensor([0, 3], dtype=torch.int32)  # no exception, esc 3
    lazy = LazyDecision(xchg, 4096, 1024, 512, AdpConfig())
    want = dist_decision([0, 3], 4096, 1024, 512, AdpConfig())[:3]
    assert tuple(lazy) == want and lazy == want and lazy[0] == want[0] and len(lazy) == 3

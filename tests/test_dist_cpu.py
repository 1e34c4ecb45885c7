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

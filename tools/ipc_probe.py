"""Two processes on one GPU sharing slab records over CUDA IPC (gloo for the
small collectives): time dgemm_dist with the fused phase 7 (in place) and the
pulled variant at a given size. Usage: python tools/ipc_probe.py [n] [mode ...]"""
import json
import os
import socket
import sys
import time

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, port, n, modes):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_13778_b200 as adp
    from paper_2511_13778_b200.dist import PeerSlabs, cols_of, dgemm_dist, rows_of

    cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)
    m = n
    r0, r1 = rows_of(rank, world, m)
    c0, c1 = cols_of(rank, world, n)
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    A = torch.rand((n, m), generator=g, device="cuda", dtype=torch.float64)[:, r0:r1].contiguous() + 1
    B = torch.rand((n, n), generator=g, device="cuda", dtype=torch.float64)[c0:c1].contiguous() + 1
    C = torch.zeros((n, r1 - r0), device="cuda", dtype=torch.float64)
    peers = PeerSlabs(n, n, cfg)
    out = {}
    for mode in modes:
        kw = {} if mode == "allgather" else {"peers": peers, "pull": mode == "pull"}
        ts = []
        for _ in range(3):
            torch.distributed.barrier()
            torch.cuda.synchronize()
            t0 = time.time()
            dgemm_dist("N", m, r1 - r0, n, n, 1.0, A, r1 - r0, B, 0.0, C, r1 - r0, cfg, **kw)
            torch.cuda.synchronize()
            ts.append(time.time() - t0)
        out[mode] = [round(t * 1e3, 2) for t in ts]
    if rank == 0:
        print(json.dumps({"n": n, "ms": out}), flush=True)
    torch.distributed.barrier()
    peers.close()
    torch.distributed.destroy_process_group()


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    modes = sys.argv[2:] or ["pull", "fused"]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(worker, args=(2, port, n, modes), nprocs=2, start_method="spawn")

"""The fused phase 7 across real processes: two ranks (gloo for the small
collectives, both on cuda:0 — this pool's boxes have one GPU) share their slab
buffers through CUDA IPC (PeerSlabs: cudaIpcGetMemHandle / OpenMemHandle, the
same calls that map NVLink peers on a multi-GPU node), and each rank's GEMM
reads the other's B planes in place. The assembled C must equal one GPU's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu

M, N, K = 700, 512, 900


def _operands():
    g = torch.Generator()
    g.manual_seed(21)
    A = torch.rand((K, M), generator=g, dtype=torch.float64) * 2 - 1   # column-major m x k
    B = torch.rand((N, K), generator=g, dtype=torch.float64) * 2 - 1   # column-major k x n
    return A, B


def _worker(rank, world, port, esc, out_dir, pull):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2511_13778_b200 as adp
    from paper_2511_13778_b200.dist import PeerSlabs, cols_of, dgemm_dist, rows_of

    cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET, esc_method=esc)
    A, B = _operands()
    r0, r1 = rows_of(rank, world, M)
    c0, c1 = cols_of(rank, world, N)
    Ab = A[:, r0:r1].contiguous().cuda()
    Bs = B[c0:c1].contiguous().cuda()
    Cb = torch.zeros((N, r1 - r0), dtype=torch.float64, device="cuda")
    peers = PeerSlabs(N, K, cfg)
    outs = []
    for _ in range(3):  # both buffers of the double buffer, then the first again
        res = dgemm_dist("N", M, r1 - r0, N, K, 1.0, Ab, r1 - r0, Bs, 0.0, Cb, r1 - r0, cfg, peers=peers, pull=pull)
        torch.cuda.synchronize()
        outs.append(Cb.cpu().clone())
    torch.distributed.barrier()
    peers.close()
    np.save(os.path.join(out_dir, f"r{rank}.npy"), torch.stack(outs).numpy())
    np.save(os.path.join(out_dir, f"res{rank}.npy"), np.array(res))
    torch.distributed.destroy_process_group()


@pytest.mark.parametrize("esc,pull", [("coarsened", False), ("certified", False), ("coarsened", True)])
def test_fused_phase7_over_cuda_ipc(gpu, tmp_path, esc, pull):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    mp.start_processes(_worker, args=(world, port, esc, str(tmp_path), pull), nprocs=world, start_method="spawn")
    A, B = _operands()
    ref = torch.zeros((N, M), dtype=torch.float64, device="cuda")
    gpu.dgemm("N", "N", M, N, K, 1.0, A.cuda(), M, B.cuda(), K, 0.0, ref, M,
              gpu.AdpConfig(pair_limit=gpu.PAIRS_TARGET, esc_method=esc))
    ref = ref.cpu().numpy()
    from paper_2511_13778_b200.dist import rows_of

    for r in range(world):
        r0, r1 = rows_of(r, world, M)
        got = np.load(os.path.join(str(tmp_path), f"r{r}.npy"))
        res = np.load(os.path.join(str(tmp_path), f"res{r}.npy"))
        assert res[0] == 0 and res[2] > 0  # emulated, planes read over IPC
        for c in got:
            assert np.array_equal(c.view(np.uint64), ref[:, r0:r1].view(np.uint64))

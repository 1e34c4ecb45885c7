"""GPU (one device, several virtual ranks): the B-distributed multi-GPU path.

Each virtual rank has its own handle (workspace) and runs the real
orchestration (dist.dgemm_dist_steps); the collectives it requests are served
by hand across the ranks (concatenation / elementwise max), exactly what
NCCL all-gather / all-reduce(MAX) produce. The assembled C must be
bit-identical to the single-GPU adpb200_dgemm.
"""
import numpy as np
import pytest
import torch

from conftest import assert_bitwise

pytestmark = pytest.mark.gpu


def run_virtual(gens):
    reqs = [next(g) for g in gens]
    results = [None] * len(gens)
    while True:
        kind = reqs[0][0]
        assert all(r[0] == kind for r in reqs), "ranks diverged"
        if kind in ("wait", "barrier", "device_barrier"):
            pass
        elif kind in ("all_gather", "all_gather_async"):
            cat = torch.cat([r[2].reshape(-1) for r in reqs])
            for r in reqs:
                r[1].view(-1).copy_(cat)
        else:
            mx = torch.stack([r[1] for r in reqs]).amax(0)
            for r in reqs:
                r[1].copy_(mx)
        nxt = []
        for i, g in enumerate(gens):
            try:
                nxt.append(next(g))
            except StopIteration as fin:
                results[i] = fin.value
        if all(x is not None for x in results):
            return results
        assert len(nxt) == len(gens), "ranks finished at different steps"
        reqs = nxt


def dist_case(gpu, world, m, n, k, cfg, transa="N", alpha=1.0, beta=0.0, poison=None, lo=-1.0, seed=3,
              overlap=True, zero_row=None, fused=False, mutate=None, pull=False):
    from paper_2511_13778_b200 import Handle
    from paper_2511_13778_b200.dist import cols_of, dgemm_dist_steps, rows_of

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    # column-major storage: A (m x k) -> tensor (k, m); op(A) = A^T for 'T': A stored k x m -> tensor (m, k)
    Ast = torch.rand((k, m) if transa == "N" else (m, k), generator=g, device="cuda", dtype=torch.float64)
    Ast = Ast * (1.0 - lo) + lo
    Bt = torch.rand((n, k), generator=g, device="cuda", dtype=torch.float64) * (1.0 - lo) + lo  # B k x n col-major
    Ct = torch.rand((n, m), generator=g, device="cuda", dtype=torch.float64)
    if poison is not None:
        Bt[poison] = float("nan")
    if mutate is not None:
        mutate(Ast, Bt)
    if zero_row is not None:  # row i of op(A) all zeros
        if transa == "N":
            Ast[:, zero_row] = 0.0
        else:
            Ast[zero_row, :] = 0.0
    ref = Ct.clone()
    lda = m if transa == "N" else k
    gpu.dgemm(transa, "N", m, n, k, alpha, Ast, lda, Bt, k, beta, ref, m, cfg)
    gens, blocks = [], []
    slab_ptrs = None
    if fused:  # the fused phase 7: every rank's slab buffer, read in place by all ranks' GEMMs
        from paper_2511_13778_b200.dist import dist_sizes

        cap_bytes = dist_sizes(n, k, world, cfg)[3]
        # zeroed: the in-place path's ready / consumed flags at each buffer's end start at 0
        slabs = [torch.zeros(cap_bytes, dtype=torch.int8, device="cuda") for _ in range(world)]
        slab_ptrs = [t.data_ptr() for t in slabs]
    for r in range(world):
        r0, r1 = rows_of(r, world, m)
        c0, c1 = cols_of(r, world, n)
        mr = r1 - r0
        Ab = (Ast[:, r0:r1] if transa == "N" else Ast[r0:r1, :]).contiguous()
        lda_r = max(mr, 1) if transa == "N" else k
        Bs = Bt[c0:c1].contiguous()
        Cb = Ct[:, r0:r1].contiguous()
        blocks.append(Cb)
        gens.append(dgemm_dist_steps(world, transa, m, mr, n, k, alpha, Ab, lda_r, Bs, beta, Cb, max(mr, 1), cfg,
                                     Handle(0), rank=r, overlap=overlap, slab_ptrs=slab_ptrs, pull=pull))
    res = run_virtual(gens)
    torch.cuda.synchronize()
    assembled = torch.cat(blocks, dim=1)
    return assembled, ref, res


@pytest.mark.parametrize("world,m,n,k,policy", [(2, 640, 384, 512, "full"), (4, 1000, 512, 768, "target"),
                                                (2, 300, 256, 2048, "target"), (8, 1024, 1024, 1024, "full")])
def test_dist_bit_identical(gpu, world, m, n, k, policy):
    cfg = gpu.AdpConfig(pair_limit=gpu.PAIRS_TARGET if policy == "target" else gpu.PAIRS_FULL)
    got, ref, res = dist_case(gpu, world, m, n, k, cfg, alpha=-1.25, beta=0.5)
    path, s, nsl = res[0]
    assert all(r == res[0] for r in res)
    assert path == 0 and s >= 7 and nsl == s
    assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), nan_equiv=False)


@pytest.mark.parametrize("world,n", [(4, 4 * 40), (8, 8 * 24), (2, 2 * 200)])
def test_dist_overlap_ragged_slabs(gpu, world, n):
    """Slabs that are not multiples of the GEMM's NB: tiles straddling two ranks'
    columns are left to phase 6; C still bit-identical, with and without overlap."""
    for cfg in (gpu.AdpConfig(min_dim=8), gpu.AdpConfig(min_dim=8, pair_limit=gpu.PAIRS_TARGET)):
        for overlap in (True, False):
            got, ref, res = dist_case(gpu, world, 512, n, 640, cfg, overlap=overlap)
            assert res[0][0] == 0
            assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), nan_equiv=False)


def test_dist_transposed_a_and_wide_span(gpu):
    cfg = gpu.AdpConfig()
    got, ref, res = dist_case(gpu, 4, 768, 512, 640, cfg, transa="T", lo=1.0)
    assert res[0][0] == 0
    assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), nan_equiv=False)


def test_dist_nan_in_one_slab_falls_back_everywhere(gpu):
    """A NaN in rank 1's B slab: the max-allreduced exceptional flag sends
    every rank to the native path, which all-gathers the FP64 B slabs."""
    cfg = gpu.AdpConfig()
    n = 512
    got, ref, res = dist_case(gpu, 4, 700, n, 600, cfg, poison=(n // 4 + 3, 17))
    assert all(r[0] == 1 and r[2] == 0 for r in res)
    assert_bitwise(got.cpu().numpy(), ref.cpu().numpy())


def test_dist_forced_and_native_modes(gpu):
    for cfg in (gpu.AdpConfig(mode=gpu.AdpMode.ForceEmulate, forced_slices=9, pair_limit=gpu.PAIRS_TARGET),
                gpu.AdpConfig(mode=gpu.AdpMode.ForceNative)):
        got, ref, res = dist_case(gpu, 2, 512, 256, 512, cfg)
        assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), nan_equiv=False)



@pytest.mark.parametrize("world,m,n,k", [(2, 640, 384, 512), (4, 1000, 512, 768), (3, 900, 384, 1536)])
def test_dist_certified_esc(gpu, world, m, n, k):
    """Certified ESC across ranks: B indicator planes travel with the slab stats,
    each rank certifies its rows, the fail flag rides the max-allreduce; the
    decision and C equal the single-GPU certified dgemm bitwise."""
    cfg = gpu.AdpConfig(pair_limit=gpu.PAIRS_TARGET, esc_method="certified")
    got, ref, res = dist_case(gpu, world, m, n, k, cfg, alpha=0.75, beta=-0.5)
    assert all(r == res[0] for r in res)
    assert res[0][0] == 0 and res[0][1] == 7
    assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), nan_equiv=False)
    # one zero row on the last rank: its certificate fails, so every rank keeps the coarsened s
    got, ref, res = dist_case(gpu, world, m, n, k, cfg, zero_row=m - 2)
    assert all(r == res[0] for r in res)
    assert res[0][0] == 0 and res[0][1] > 7
    assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), nan_equiv=False)
    # a wide exponent range: level 0 fails somewhere, level 1 (s0 + 1 = 8 slices) holds everywhere
    def widen(Ast, Bt):
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        Ast.mul_(torch.exp2(torch.randint(-40, 40, Ast.shape, generator=g, device="cuda").double()))

    got, ref, res = dist_case(gpu, world, m, n, k, cfg, mutate=widen)
    assert all(r == res[0] for r in res)
    assert res[0][0] == 0 and res[0][1] == 8
    assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), nan_equiv=False)
    for fused in (True,):
        got, ref, res = dist_case(gpu, world, m, n, k, cfg, mutate=widen, fused=fused)
        assert res[0][1] == 8
        assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), nan_equiv=False)
    # NaN in a slab: native everywhere
    got, ref, res = dist_case(gpu, world, m, n, k, cfg, poison=(n // world + 1, 5))
    assert all(r[0] == 1 for r in res)
    assert_bitwise(got.cpu().numpy(), ref.cpu().numpy())


@pytest.mark.parametrize("world,m,n,k,cfgname", [(2, 640, 384, 512, "full"), (4, 1000, 512, 768, "target"),
                                                 (8, 1024, 1024, 1024, "target"), (3, 700, 3 * 200, 900, "target"),
                                                 (4, 512, 4 * 40, 640, "certified"), (2, 520, 2 * 104, 1100, "u12")])
def test_dist_fused_peer_gemm(gpu, world, m, n, k, cfgname):
    """Phase 7: no plane all-gather; the GEMM's TMA loads read each rank's slab
    planes in place (here: buffers of one device standing in for the NVLink
    peer mappings) with every rank's columns tiled on their own, including
    slabs that are not a multiple of the variant's NB (partial last tile per
    rank) and the 48-column variant (s = 8). C bit-identical to one GPU."""
    cfg = {"full": gpu.AdpConfig(min_dim=8), "target": gpu.AdpConfig(min_dim=8, pair_limit=gpu.PAIRS_TARGET),
           "certified": gpu.AdpConfig(min_dim=8, pair_limit=gpu.PAIRS_TARGET, esc_method="certified"),
           "u12": gpu.AdpConfig(min_dim=8, pair_limit=gpu.PAIRS_TARGET)}[cfgname]
    for pull in (False, True):  # in place / pulled rank by rank into local copies
        got, ref, res = dist_case(gpu, world, m, n, k, cfg, alpha=-0.5, beta=1.25, fused=True, pull=pull,
                                  lo=1.0 if cfgname == "u12" else -1.0)
        assert all(r == res[0] for r in res)
        assert res[0][0] == 0
        assert_bitwise(got.cpu().numpy(), ref.cpu().numpy(), nan_equiv=False)
    # NaN in one slab: native fallback everywhere — in place (device-decided), each rank's
    # native GEMM reads the FP64 slabs the peers copied into their buffers (phase 8); pulled,
    # the host sees the decision and all-gathers FP64 B
    for pull in (False, True):
        got, ref, res = dist_case(gpu, world, m, n, k, cfg, poison=(n // world + 1, 3), fused=True, pull=pull)
        assert all(r[0] == 1 for r in res)
        assert_bitwise(got.cpu().numpy(), ref.cpu().numpy())
    for flavour in ("fast",):  # the DMMA flavour reads the peers' slabs too (within its bound)
        fcfg = gpu.AdpConfig(min_dim=8, pair_limit=gpu.PAIRS_TARGET, fallback=flavour)
        got, ref, res = dist_case(gpu, world, m, n, k, fcfg, poison=(n // world + 1, 3), fused=True)
        assert all(r[0] == 1 for r in res)
        g, rf = got.cpu().numpy(), ref.cpu().numpy()
        fin = np.isfinite(rf)
        assert np.array_equal(np.isnan(g), np.isnan(rf))
        assert np.allclose(g[fin], rf[fin], rtol=1e-12, atol=1e-12)


def test_dist_fused_in_place_reuses_buffers_across_calls(gpu):
    """The host-sync-free fused path over several calls: two slab buffers alternate
    (epochs 1, 1, 2, 2), every call's slicing waits on the peers' "consumed" flag of
    the buffer's previous use and its GEMM on their "ready" flags. Each call changes
    the operands (and the third one poisons B, so the native fallback reads the peers'
    FP64 slabs); every assembled C must equal one GPU's."""
    from paper_2511_13778_b200 import Handle
    from paper_2511_13778_b200.dist import cols_of, dgemm_dist_steps, dist_sizes, rows_of

    world, m, n, k = 3, 700, 3 * 128, 900
    cfg = gpu.AdpConfig(min_dim=8, pair_limit=gpu.PAIRS_TARGET)
    cap = dist_sizes(n, k, world, cfg)[3]
    bufs = [[torch.zeros(cap, dtype=torch.int8, device="cuda") for _ in range(world)] for _ in range(2)]
    handles = [Handle(0) for _ in range(world)]
    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    for call in range(4):
        Ast = torch.rand((k, m), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
        Bt = torch.rand((n, k), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
        if call == 2:
            Bt[n // world + 5, 17] = float("nan")
        ref = torch.zeros((n, m), device="cuda", dtype=torch.float64)
        gpu.dgemm("N", "N", m, n, k, 1.0, Ast, m, Bt, k, 0.0, ref, m, cfg)
        slab_ptrs = [t.data_ptr() for t in bufs[call % 2]]
        gens, blocks = [], []
        for r in range(world):
            r0, r1 = rows_of(r, world, m)
            c0, c1 = cols_of(r, world, n)
            Cb = torch.zeros((n, r1 - r0), device="cuda", dtype=torch.float64)
            blocks.append(Cb)
            gens.append(dgemm_dist_steps(world, "N", m, r1 - r0, n, k, 1.0, Ast[:, r0:r1].contiguous(), r1 - r0,
                                         Bt[c0:c1].contiguous(), 0.0, Cb, r1 - r0, cfg, handles[r], rank=r,
                                         slab_ptrs=slab_ptrs, epoch=call // 2 + 1))
        res = run_virtual(gens)
        torch.cuda.synchronize()
        assert all(x[0] == (1 if call == 2 else 0) for x in res)
        assert_bitwise(torch.cat(blocks, dim=1).cpu().numpy(), ref.cpu().numpy())
    # the flags record the last epoch of each buffer
    from paper_2511_13778_b200.dist import flag_ptr

    for b in range(2):
        for r in range(world):
            t = bufs[b][r]
            for which in (0, 1):
                off = flag_ptr(t.data_ptr(), cap, which) - t.data_ptr()
                assert int(t[off:off + 4].view(torch.int32).item()) == 2

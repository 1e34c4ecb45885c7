#!/usr/bin/env python3
"""bench.py — ADP emulated DGEMM on B200 (effective FP64 TFLOP/s, 2mnk/t).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1)

Workload (BASELINE.json configs[1], the headline metric): ADP DGEMM
8192^3 per GPU, synthetic U(1,2) operands (seeded), column-major NN through
the C-ABI drop-in adpb200_dgemm with the ADP guardrails live (scan, ESC,
decision on device): ESC picks s = 7 slices = the 55-bit window, and the
slice pairs below the target precision are skipped (d_a + d_b <= s). For
N > 1 the rows of A/C are partitioned (weak scaling: 8192 rows per GPU,
B replicated) and the ADP decision inputs are max-allreduced over NCCL.

The timed region follows a 2 s soak, so `value` is the power-capped steady
state (`value_burst`: 5 steps right after the warm-up). The JSON line also
reports native FP64 (cuBLAS via torch.matmul) on the same GPU, the ADP overhead
against fixed-slice emulation, the U[-1,1] (s = 8) and bitwise-reference (all
s^2 pairs) variants, BASELINE configs 2 (U[-1,1]) and 5, the native-fallback
flavours on an input with a NaN (config 3), config 4 (32768^3) row-partitioned
over the N ranks beside the same problem on one GPU (`strong_c4`), the
per-stage times, the rooflines of the slice GEMM (INT8 tensor peak) and of the
ESC (measured DPX peak), and the reference CPU implementation timed on this
host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NOMINAL = 8192


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=150)  # ~2 s timed: enough nvidia-smi samples under load
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--size", type=int, default=NOMINAL, help="m_per_gpu = n = k")
    p.add_argument("--config", choices=["c2", "c4"], default="c2",
                   help="c2: the headline (8192^3 per GPU, weak scaling); c4: BASELINE config 4, 32768^3 U[-1,1] "
                        "row-partitioned over the GPUs (strong scaling; side measurements skipped)")
    p.add_argument("--esc", choices=["coarsened", "certified"], default="coarsened",
                   help="ESC method of the timed calls: the reference's coarsened ESC (default) or the "
                        "certified ESC option (single-GPU paths)")
    p.add_argument("--dist", choices=["fused", "pull", "allgather"], default="allgather",
                   help="N > 1: allgather (default: each plane byte crosses NVLink once, NCCL; one 8-byte host "
                        "read per call sizes it) = NCCL all-gather of the B planes overlapped with the "
                        "own-column GEMM (phases 5/6); fused = the GEMM reads every rank's B planes in place "
                        "over NVLink (CUDA IPC peer mappings, phase 7), ordered by stream-side flags with no "
                        "host read or barrier; pull = the copy engines pull each peer's planes while the GEMM "
                        "of the previous rank's columns runs (phase 7 per rank). fused / pull are not yet timed "
                        "on an NVLink node")
    p.add_argument("--quick", action="store_true", help="skip the side measurements")
    p.add_argument("--soak", type=float, default=2.0,
                   help="seconds of untimed steps between the warm-up and the timed region, so the timed region "
                        "runs at the power-capped steady state (value_burst: 5 steps right after the warm-up)")
    p.add_argument("--c4-size", type=int, default=32768,
                   help="strong_c4 side measurement: m = n = k (BASELINE config 4 is 32768; smaller only for "
                        "plumbing checks); 0 skips it")
    p.add_argument("--c4-dist", choices=["rows", "allgather"], default="rows",
                   help="strong_c4 partition: rows = every rank holds B and slices it (one 8-byte stream-ordered "
                        "max-allreduce per call, no host sync); allgather = B column slabs, slice planes "
                        "all-gathered over NCCL")
    p.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def cpu_model() -> str:
    """The host CPU model (the CPU baseline's hardware, like `lscpu`)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu=timestamp,{self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def stop(self, t0, t1):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [s for (t, s) in self.samples if t0 - 0.2 <= t <= t1 + 0.2] or [s for _, s in self.samples[-5:]]
        sm, mx, reasons, pw = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            parts = [x.strip() for x in r.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
            try:
                pw.append(float(parts[7]))
            except (ValueError, IndexError):
                pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(pw) if pw else None}


# ---------------------------------------------------------------------------------
def reference_arm(args):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    built from /root/reference sources) of adp_gemm, on a bounded sample of the
    same workload per step, all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    from oracle.oracle import Oracle, available

    kind = "reference" if available("reference") else "port"
    orc = Oracle(kind)
    cores = os.cpu_count() or 1
    rs, cs, k = 256, 2048, args.size  # a 256 x 2048 block of C, full k: same decision path (min dim 256)
    # the reference's own generator (gen_uniform_rect, xoshiro256++), U(1,2), seeds 1 and 2
    a = orc.gen_uniform_rect(rs, k, 1, 1.0, 2.0)
    b = orc.gen_uniform_rect(k, cs, 2, 1.0, 2.0)
    # keep the whole --steps K --warmup W run within ~2.5 minutes: one probe call sizes
    # the column count of the sample (multiples of 256, at least 256)
    t0 = time.perf_counter()
    if kind == "reference":
        orc.time_call(1, a, b)
    else:
        orc.adp_gemm(a, b)
    probe = time.perf_counter() - t0
    budget = 150.0 / max(1, args.warmup + args.steps)
    if probe > budget:
        cs = max(256, int(cs * budget / probe) // 256 * 256)
        b = np.ascontiguousarray(b[:, :cs])
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if kind == "reference":
            orc.time_call(1, a, b)
        else:
            orc.adp_gemm(a, b)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    value = 2.0 * rs * cs * k / t / 1e12
    line = {
        "impl": "reference", "metric": "effective FP64 TFLOP/s (2mnk/t) of ADP DGEMM, 55-bit, 8192^3",
        "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic U(1,2): the reference's gen_uniform_rect (xoshiro256++) seeds 1, 2",
        "config": {"workload": f"reference adp_gemm (CPU, OpenMP) on a {rs}x{cs}x{k} block of the "
                               f"{args.size}^3 ADP DGEMM", "sample_m": rs, "sample_n": cs, "k": k},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "cpu": cpu_model(), "kind": kind,
                         "sample": f"{rs}x{cs}x{k} block of C per step"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(A_host_rows, B_host, k):
    """The reference CPU path on a bounded sample (rank 0, N=1 only)."""
    from oracle.oracle import Oracle, available

    kind = "reference" if available("reference") else "port"
    orc = Oracle(kind)
    cores = os.cpu_count() or 1
    a, b = A_host_rows, B_host
    t0 = time.perf_counter()
    if kind == "reference":
        dt = orc.time_call(1, a, b)
    else:
        orc.adp_gemm(a, b)
        dt = time.perf_counter() - t0
    m, n = a.shape[0], b.shape[1]
    return {"value": 2.0 * m * n * k / dt / 1e12, "unit": "TFLOP/s", "cores": cores, "cpu": cpu_model(), "kind": kind,
            "sample": f"reference adp_gemm on a {m}x{n}x{k} block of the same operands ({dt:.1f} s)"}


# ---------------------------------------------------------------------------------
def strong_c4(args, adp, grading, dev, world, rank, handle, timed, dist):
    """BASELINE config 4 (m = n = k = 32768, U[-1,1], coarsened ESC -> s = 8): the
    row-partitioned call over the N ranks, and the same problem on one GPU (each
    rank alone, max over ranks); speedup = single / partitioned."""
    import torch

    from paper_2511_13778_b200.dist import cols_of, dgemm_dist, dgemm_rows, rows_of

    n = k = mg = args.c4_size
    cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET)
    flops = 2.0 * mg * n * k
    out = {"m": mg, "n": n, "k": k, "unit": "TFLOP/s", "data": "U[-1,1], gen_uniform_rect seeds 1, 2",
           "partition": args.c4_dist if world > 1 else "single GPU"}
    if os.environ.get("ADPB200_BENCH_SHARED_GPU") == "1":
        out["note"] = "plumbing check: all ranks share cuda:0, so neither time is a scaling measurement"
    torch.cuda.empty_cache()
    # one GPU, the whole problem (column-major NN)
    At = grading.gen_uniform_rect(k, mg, 1, -1.0, 1.0, dev.index)
    Bt = grading.gen_uniform_rect(n, k, 2, -1.0, 1.0, dev.index)
    Ct = torch.empty((n, mg), device=dev, dtype=torch.float64)

    def one():
        adp.dgemm("N", "N", mg, n, k, 1.0, At, mg, Bt, k, 0.0, Ct, mg, cfg, handle)

    t1 = timed(one, 2, 1)
    _, tr = adp.adp_gemm(At.t(), Bt.t(), config=cfg, handle=handle)  # the decision of this problem
    out.update({"one_gpu_value": flops / (t1 * 1e-3) / 1e12, "one_gpu_ms": t1, "slices": tr.slices,
                "esc_bits": tr.esc_bits, "pairs": tr.pairs})
    del Ct
    if world == 1:
        out["value"], out["ms_per_step"], out["speedup_vs_1gpu"] = out["one_gpu_value"], t1, 1.0
        return out
    r0, r1 = rows_of(rank, world, mg)
    ml = r1 - r0
    Al = At[:, r0:r1].contiguous()                 # this rank's rows of A (column-major, lda = ml)
    Cl = torch.empty((n, ml), device=dev, dtype=torch.float64)
    if args.c4_dist == "rows":
        xchg = torch.zeros(2, dtype=torch.int32, device=dev)

        def part():
            xchg.zero_()
            dgemm_rows("N", "N", mg, ml, n, k, 1.0, Al, ml, Bt, k, 0.0, Cl, ml, cfg, handle, xchg=xchg)
    else:
        c0, c1 = cols_of(rank, world, n)
        Bs = Bt[c0:c1].contiguous()

        def part():
            dgemm_dist("N", mg, ml, n, k, 1.0, Al, ml, Bs, 0.0, Cl, ml, cfg, handle)
    del At
    tN = timed(part, 3, 1)
    out.update({"value": flops / (tN * 1e-3) / 1e12, "ms_per_step": tN, "speedup_vs_1gpu": t1 / tN,
                "rows_per_rank": ml})
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2511_13778_b200 as adp
    from paper_2511_13778_b200 import _lib
    from paper_2511_13778_b200.dist import cols_of, dgemm_dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shared = os.environ.get("ADPB200_BENCH_SHARED_GPU") == "1"  # plumbing check only: all ranks on cuda:0, gloo
    if world > 1:
        if shared:
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    c4 = args.config == "c4"
    if c4:
        from paper_2511_13778_b200.dist import rows_of

        n = k = m_global = 32768       # BASELINE config 4 (strong scaling: rows partitioned)
        r0, r1 = rows_of(rank, world, m_global)
        m = r1 - r0
        lo = -1.0
        args.quick = True
    else:
        n = k = args.size
        m = args.size                  # rows per GPU (weak scaling)
        m_global = m * world
        lo = 1.0
    handle = adp.Handle.default(dev.index)

    # synthetic operands, column-major storage (torch row-major of the transpose),
    # filled in storage order by the reference's generator (gen_uniform_rect,
    # xoshiro256++, grading.cpp:56-63) drawn on the device
    from paper_2511_13778_b200 import grading

    At = grading.gen_uniform_rect(k, m, 1 + 1000 * rank, lo, 2.0 if lo > 0 else 1.0, dev.index)  # A: m x k col-major
    Bt = grading.gen_uniform_rect(n, k, 2, lo, 2.0 if lo > 0 else 1.0, dev.index)               # B: k x n col-major
    if world > 1:
        # B distributed by column slabs: this rank keeps columns cols_of(rank) only
        c0, c1 = cols_of(rank, world, n)
        Bt = Bt[c0:c1].contiguous()
    Ct = torch.zeros((n, m), device=dev, dtype=torch.float64)                  # C: m x n col-major
    cfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET, esc_method=args.esc)
    trace_buf = torch.zeros(_lib.TRACE_BYTES, dtype=torch.uint8, device=dev)
    peers, dist_mode = None, args.dist if world > 1 else None
    if world > 1 and args.dist in ("fused", "pull"):
        from paper_2511_13778_b200.dist import PeerSlabs

        try:  # slab buffers sized for the largest plane count any config here can ask for
            peers = PeerSlabs(n, k, adp.AdpConfig(), device=dev.index)
        except Exception as e:  # noqa: BLE001 — no IPC / peer access (raised on every rank alike):
            # fall back to the NCCL all-gather
            dist_mode = f"allgather ({args.dist} unavailable: {str(e)[:160]})"
            print(f"bench: {dist_mode}", file=sys.stderr, flush=True)

    def step(config=cfg, A=At, B=Bt, Cm=Ct, trace=None):
        if world > 1:
            dgemm_dist("N", m_global, m, n, k, 1.0, A, m, B, 0.0, Cm, m, config, handle, trace=trace, peers=peers,
                       pull=args.dist == "pull")
        else:
            adp.dgemm("N", "N", m, n, k, 1.0, A, m, B, k, 0.0, Cm, m, config, handle, trace=trace)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        barrier()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # ---- headline: device-resident ADP DGEMM -----------------------------------------
    step(trace=trace_buf)
    torch.cuda.synchronize()
    trace = adp.AdpTrace.from_c(_lib.Trace.from_buffer_copy(trace_buf.cpu().numpy().tobytes()))
    for _ in range(args.warmup):
        step()
    # burst: 5 steps right after the warm-up (clocks not yet power-capped)
    burst_ms = timed(step, 5, 0)
    # soak to the power-capped steady state right before the timed region, with no idle gap
    # in between (same step count on every rank); nvidia-smi starts sampling before it
    sampler = ClockSampler(dev.index)
    sampler.start()
    n_soak = 0
    if args.soak > 0:
        n_soak = max(1, int(args.soak * 1e3 / max(burst_ms, 1e-3)))
        for _ in range(n_soak):
            step()
    else:
        time.sleep(0.5)
    barrier()
    launches0 = handle.launches()
    handle.profile_enable(args.steps * (4 if world > 1 else 1))  # the dist path is 4 pipeline calls
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    barrier()
    wall1 = time.time()
    launches = handle.launches() - launches0
    clocks = sampler.stop(wall0, wall1)
    stage = handle.profile_read()
    handle.profile_enable(0)
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if clocks is not None and clocks["samples"] < 10 and not c4:
        # a short timed region leaves few samples (nvidia-smi polls every 100 ms and
        # its power reading lags): soak the same step for ~2 s, sampled the same way,
        # and report it beside the timed-region samples. The step count comes from
        # the max-reduced ms, so every rank runs the same collectives.
        soak = ClockSampler(dev.index)
        soak.start()
        time.sleep(0.5)
        s0 = time.time()
        for _ in range(max(10, min(2000, int(2000.0 / max(ms, 1e-3))))):
            step()
        barrier()
        clocks["soak_after_timed_region"] = soak.stop(s0 + 0.5, time.time())
    flops_global = 2.0 * m_global * n * k
    value = flops_global / (ms * 1e-3) / 1e12

    # per-stage averages (this rank); for N > 1 each call is two pipeline calls
    stage_ms = {}
    if stage:
        for key in _lib.PROFILE_STAGES:
            stage_ms[key] = sum(c[key] for c in stage) / args.steps
    gemm_ms = stage_ms.get("gemm", 0.0)

    pk, pk_kind = peaks()
    # INT8 dense tensor peak: measured on this pool's B200 by tools/mma_peak.cu (back-to-back
    # tcgen05.mma kind::i8 M=128 N=256 from smem, 4 s sustained; profiles/r01_mma_peak.json);
    # MEASURED_PEAKS.json has no INT8 figure. Fallback: 2 x its dense bf16.
    int8_peak, peak_src = 2.0 * pk["bf16_tflops"], f"2 x bf16_tflops of MEASURED_PEAKS.json ({pk_kind})"
    try:
        with open(os.path.join(ROOT, "profiles", "r01_mma_peak.json")) as f:
            int8_peak = float(json.load(f)["int8_tops_sustained"])
            peak_src = "measured: tools/mma_peak.cu, tcgen05 kind::i8 N=256 sustained (profiles/r01_mma_peak.json)"
    except (OSError, KeyError, ValueError):
        pass
    pairs = trace.pairs or 0
    achieved = 2.0 * m * n * k * pairs / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    traffic = None  # the ncu capture is of the 8192^3 headline kernel
    try:
        if c4:
            raise OSError
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            traffic = json.load(f).get("igemm_dram_bytes_per_launch")
    except OSError:
        pass
    roofline = {"bound": "tensor", "kernel": "igemm_kernel (tcgen05 kind::i8 + fused exact epilogue)",
                "achieved": achieved, "peak": int8_peak, "unit": "TFLOP/s",
                "frac": (achieved / int8_peak) if achieved else None, "traffic": traffic,
                "peak_source": peak_src + "; int8 ops = 2mnk x pairs",
                "frac_of_2x_bf16": (achieved / (2.0 * pk["bf16_tflops"])) if achieved else None,
                "clock_note": "the GEMM runs power-capped (sw_power_cap, ~1000 W): see clocks", "pairs": pairs}
    # the same kernel against the dense kind::i8 rate at the SM clock nvidia-smi saw under load
    # (148 SMs x 8192 MAC/clk x 2 ops): how much of the power-capped clock's peak it uses
    load_clk = None
    if clocks:
        soak = clocks.get("soak_after_timed_region") or {}
        load_clk = soak.get("sm_mhz") or clocks.get("sm_mhz")
    if achieved and load_clk:
        roofline["peak_at_load_clock"] = 148 * 8192 * 2 * load_clk * 1e6 / 1e12
        roofline["frac_at_load_clock"] = achieved / roofline["peak_at_load_clock"]

    extra = {}
    if not args.quick:
        # ---- e2e through the C-ABI with HOST buffers: adpb200_dgemm_host copies A and B
        # in, runs the pipeline and copies C out (overlapped with the GEMM's row chunks);
        # each step returns with C on the host ----------------------------------------
        A_h = At.cpu().pin_memory()
        B_h = Bt.cpu().pin_memory()
        C_h = torch.empty_like(Ct, device="cpu").pin_memory()

        def e2e_step():
            if world > 1:  # the row-partitioned path keeps device buffers; copy around it
                At.copy_(A_h, non_blocking=True)
                Bt.copy_(B_h, non_blocking=True)
                step()
                C_h.copy_(Ct, non_blocking=True)
            else:
                adp.dgemm_host("N", "N", m, n, k, 1.0, A_h, m, B_h, k, 0.0, C_h, m, cfg, handle, dev.index)

        e2e_ms = timed(e2e_step, max(3, args.steps // 2), 2)
        extra["e2e"] = {"value": flops_global / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                        "h2d_bytes_per_step": int(At.numel() * 8 + Bt.numel() * 8),
                        "d2h_bytes_per_step": int(Ct.numel() * 8), "ms_per_step": e2e_ms}
        if world == 1:
            # the streamed host path speculates the slice count from the handle's previous
            # call; every step above hits. Worst case: operands alternating between U(1,2)
            # (s = 7) and U[-1,1] (s = 8), so every call misses and recomputes C from the
            # kept inputs
            Au_h = grading.gen_uniform_rect(k, m, 11, -1.0, 1.0, dev.index).cpu().pin_memory()
            Bu_h = grading.gen_uniform_rect(n, k, 12, -1.0, 1.0, dev.index).cpu().pin_memory()
            flip = [0]

            def e2e_miss():
                a_h, b_h = (A_h, B_h) if flip[0] % 2 == 0 else (Au_h, Bu_h)
                flip[0] += 1
                adp.dgemm_host("N", "N", m, n, k, 1.0, a_h, m, b_h, k, 0.0, C_h, m, cfg, handle, dev.index)

            miss_ms = timed(e2e_miss, 2 * max(2, args.steps // 8), 2)
            extra["e2e"]["every_call_missed"] = {
                "ms_per_step": miss_ms, "value": flops_global / (miss_ms * 1e-3) / 1e12,
                "note": "operands alternate between s = 7 and s = 8 data: every speculation misses, C is "
                        "recomputed on the device and copied again (U[-1,1] calls run the s = 8 GEMM)"}
            del Au_h, Bu_h
        # ---- native FP64 (cuBLAS DGEMM through torch) on the same shapes -------------
        X = At.t()
        Y = (Bt if world == 1 else grading.gen_uniform_rect(n, k, 2, 1.0, 2.0, dev.index)).t()  # full k x n
        nat_ms = timed(lambda: torch.mm(X, Y), max(3, args.steps // 2), 2)
        del Y
        extra["native_fp64"] = {"value": 2.0 * m * n * k / (nat_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                                "impl": "cublasDgemm via torch.mm", "ms_per_step": nat_ms}
        # ---- ADP overhead: guardrails + pinned s=7 vs plain fixed 7-slice emulation ------
        fixed = adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=7, pair_limit=adp.PAIRS_TARGET)
        guarded = adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=7, pair_limit=adp.PAIRS_TARGET,
                                guardrails_forced=True)
        fs, gs = [], []
        for _ in range(3):  # interleaved, so clock / power drift hits both alike
            fs.append(timed(lambda: step(fixed), max(3, args.steps // 4), 1))
            gs.append(timed(lambda: step(guarded), max(3, args.steps // 4), 1))
        f_ms, g_ms = statistics.median(fs), statistics.median(gs)
        extra["adp_overhead"] = {"fixed7_ms": f_ms, "guardrails_pinned7_ms": g_ms, "auto_ms": ms,
                                 "overhead_frac": (g_ms - f_ms) / f_ms,
                                 "guardrail_stage_ms": stage_ms.get("stats", 0) + stage_ms.get("esc", 0)
                                 + stage_ms.get("decide", 0)}
        # ---- U[-1,1] operands: coarsened ESC picks s = 8 --------------------------------
        Au = grading.gen_uniform_rect(k, m, 1 + 1000 * rank, -1.0, 1.0, dev.index)
        Bu = grading.gen_uniform_rect(n, k, 2, -1.0, 1.0, dev.index)
        if world > 1:
            Bu = Bu[c0:c1].contiguous()
        tr2 = torch.zeros_like(trace_buf)
        step(cfg, Au, Bu, Ct, tr2)
        torch.cuda.synchronize()
        t2 = adp.AdpTrace.from_c(_lib.Trace.from_buffer_copy(tr2.cpu().numpy().tobytes()))
        u_ms = timed(lambda: step(cfg, Au, Bu, Ct), max(3, args.steps // 2), 2)
        extra["uniform_pm1"] = {"value": flops_global / (u_ms * 1e-3) / 1e12, "slices": t2.slices,
                                "esc_bits": t2.esc_bits, "pairs": t2.pairs}
        # the ESC stage of these operands (exponents spread over ~10 binades: no tile of the
        # max-plus can be pruned, so the kernel does the full m n t work): the ESC roofline
        handle.profile_enable(3 * (4 if world > 1 else 1))
        for _ in range(3):
            step(cfg, Au, Bu, Ct)
        torch.cuda.synchronize()
        prof = handle.profile_read()
        handle.profile_enable(0)
        if prof:
            extra["uniform_pm1"]["esc_ms"] = sum(c["esc"] for c in prof) / 3
        # ---- bitwise-reference policy: all s^2 pairs -------------------------------------
        full_ms = timed(lambda: step(adp.AdpConfig()), max(3, args.steps // 2), 2)
        extra["full_pairs"] = {"value": flops_global / (full_ms * 1e-3) / 1e12,
                               "note": "all s^2 slice pairs: output bitwise equal to the reference adp_gemm; "
                                       "the like-for-like figure against the reference arm, whose adp_gemm "
                                       "runs this pair policy (the headline skips the pairs below the "
                                       "target precision, d_a + d_b > s)"}
        del Au, Bu
        # ---- accuracy of the headline result: componentwise relative error against
        # the device double-double oracle (Dot2), and the grading ratio
        # |C - AB| / (2^-52 (|A||B|)_ij); cuBLAS DGEMM on the same operands ----------
        step()
        # (N > 1: this rank's row block against its local B slab, i.e. the C columns of the slab)
        if world > 1:
            Ct_acc = Ct[c0:c1].contiguous()
        else:
            Ct_acc = Ct
        ref, absab = grading.dd_gemm(Bt, At)          # C^T = B^T A^T in row-major terms
        rep = grading.error_report(Ct_acc, ref, absab=absab)
        nat = torch.mm(At.t(), Bt.t()).t().contiguous()
        rep_n = grading.error_report(nat, ref, absab=absab)
        del ref, absab, nat
        extra["accuracy"] = {
            "oracle": "device double-double GEMM (Dot2), |err| <= 2^-53|AB| + gamma_2k^2 |A||B|",
            "max_rel_err": rep.max_err, "avg_rel_err": rep.avg_err,
            "max_err_over_eps_absAB": rep.max_ratio, "avg_err_over_eps_absAB": rep.avg_ratio,
            "native_fp64_max_rel_err": rep_n.max_err, "native_fp64_avg_rel_err": rep_n.avg_err,
            "native_fp64_max_err_over_eps_absAB": rep_n.max_ratio}

        # ---- BASELINE configs 2 (U[-1,1] variant) and 5 (rectangular / long-k), U[-1,1]
        # reference inputs; each also with the certified ESC option -------------------------
        rect = {}
        for name, (rm, rn, rk) in (("c2_u11_8192x8192x8192", (8192, 8192, 8192)),
                                   ("c5a_4096x4096x65536", (4096, 4096, 65536)),
                                   ("c5b_65536x1024x1024", (65536, 1024, 1024))):
            Ar = grading.gen_uniform_rect(rm, rk, 1, -1.0, 1.0, dev.index)
            Br = grading.gen_uniform_rect(rk, rn, 2, -1.0, 1.0, dev.index)
            Cr = torch.empty((rm, rn), dtype=torch.float64, device=dev)
            _, tr = adp.adp_gemm(Ar, Br, config=cfg, handle=handle, out=Cr)
            # ~0.3 s per measurement (at least 5 calls): short calls such as C5b's 3 ms need
            # more than a handful of calls for a stable clock
            t0 = time.perf_counter()
            adp.adp_gemm(Ar, Br, config=cfg, handle=handle, out=Cr)
            torch.cuda.synchronize()
            reps = max(5, min(100, int(0.3 / max(time.perf_counter() - t0, 1e-4))))
            r_ms = timed(lambda: adp.adp_gemm(Ar, Br, config=cfg, handle=handle, out=Cr), reps, 2)
            f7 = adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=7, pair_limit=adp.PAIRS_TARGET)
            r7_ms = timed(lambda: adp.adp_gemm(Ar, Br, config=f7, handle=handle, out=Cr), reps, 2)
            rn_ms = timed(lambda: torch.mm(Ar, Br, out=Cr), reps, 2)
            cc = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET, esc_method="certified")
            _, tcc = adp.adp_gemm(Ar, Br, config=cc, handle=handle, out=Cr)
            rc_ms = timed(lambda: adp.adp_gemm(Ar, Br, config=cc, handle=handle, out=Cr), reps, 2)
            fl = 2.0 * rm * rn * rk
            rect[name] = {"adp_tflops": fl / r_ms / 1e9, "slices": tr.slices, "esc_bits": tr.esc_bits,
                          "pairs": tr.pairs, "k_chunks": tr.k_chunks, "emulate7_tflops": fl / r7_ms / 1e9,
                          "certified_esc_tflops": fl / rc_ms / 1e9, "certified_esc_slices": tcc.slices,
                          "certified_esc_bits": tcc.esc_bits,
                          "cublas_dgemm_tflops": fl / rn_ms / 1e9, "adp_vs_cublas": rn_ms / r_ms}
            del Ar, Br, Cr
        torch.cuda.empty_cache()
        extra["rectangular"] = rect

        # ---- BASELINE config 3's fallback: one NaN in A sends the auto-mode call to the
        # native FP64 GEMM on the device (no host sync); both flavours, beside cuBLAS ------
        An = At.clone()
        An.view(-1)[12345] = float("nan")
        fb = {}
        for flav in ("reference", "fast"):
            fcfg = adp.AdpConfig(pair_limit=adp.PAIRS_TARGET, fallback=flav)
            trf = torch.zeros_like(trace_buf)
            step(fcfg, An, Bt, Ct, trf)
            torch.cuda.synchronize()
            tf = adp.AdpTrace.from_c(_lib.Trace.from_buffer_copy(trf.cpu().numpy().tobytes()))
            f_ms = timed(lambda: step(fcfg, An, Bt, Ct), 3, 1)
            fb[flav] = {"value": flops_global / (f_ms * 1e-3) / 1e12, "path": tf.path, "ms_per_step": f_ms}
        del An
        fb["reference"]["kernel"] = "native_kernel: SIMT FP64, ascending k, no FMA (bitwise native_gemm)"
        fb["fast"]["kernel"] = "dmma_kernel: FP64 tensor cores (DMMA m8n8k4), opt-in"
        fb["unit"] = "TFLOP/s"
        fb["fast_vs_cublas"] = fb["fast"]["value"] / world / extra["native_fp64"]["value"]
        extra["fallback_tflops"] = fb

    # ---- ESC (K2) against its own roofline: the DPX add+max rate (tools/dpx_peak.cu). Taken
    # on the U[-1,1] operands, where the kernel runs the whole max-plus product; on the
    # headline's U(1,2) operands most tiles stop after one block (exact pruning), reported
    # beside it as headline_ms ----------------------------------------------------------------
    esc_ms = extra.get("uniform_pm1", {}).get("esc_ms", 0.0)
    if esc_ms > 0:
        blocks = (k + 255) // 256  # esc_block_len 256
        instr = float(m) * n * blocks  # VIADDMNMX.S16x2: 2 add+max per (i, j, block), 2 j per instruction
        esc_rf = {"bound": "dpx", "kernel": "esc_kernel (VIADDMNMX.S16x2 max-plus over exponent blocks)",
                  "operands": "U[-1,1] 8192^3 (no tile pruned)", "ms": esc_ms,
                  "headline_ms": stage_ms.get("esc"), "achieved": instr / (esc_ms * 1e-3), "unit": "instr/s",
                  "instr_per_launch": instr}
        try:
            with open(os.path.join(ROOT, "profiles", "r02_dpx_peak.json")) as f:
                dp = json.load(f)
            esc_rf["peak"] = float(dp["instr_per_s"])
            esc_rf["frac"] = esc_rf["achieved"] / esc_rf["peak"]
            esc_rf["peak_source"] = "measured: tools/dpx_peak.cu (profiles/r02_dpx_peak.json)"
            if load_clk:
                esc_rf["frac_at_load_clock"] = esc_rf["achieved"] / (dp["instr_per_clk_per_sm"] * 148 * load_clk * 1e6)
        except (OSError, KeyError, ValueError):
            pass
        extra["esc_roofline"] = esc_rf

    # ---- BASELINE config 4 strong scaling: 32768^3 U[-1,1] row-partitioned over the N
    # ranks, against the same problem on one GPU (every rank runs it alone, max over ranks) --
    if not args.quick and not c4 and args.c4_size > 0:
        extra["strong_c4"] = strong_c4(args, adp, grading, dev, world, rank, handle, timed, dist)

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            rows = At[:, :256].t().contiguous().cpu().numpy()        # 256 x k block of A (row-major)
            cols = Bt[:1024, :].t().contiguous().cpu().numpy()       # k x 1024 block of B (row-major)
            cpu = cpu_baseline(rows, cols, k)
        except Exception as e:  # noqa: BLE001 — a missing CPU baseline must not sink the GPU number
            cpu = {"value": None, "error": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": "effective FP64 TFLOP/s (2mnk/t) of ADP DGEMM, 55-bit, "
                      + ("32768^3 (BASELINE config 4)" if c4 else
                         ("8192^3" if (m, n, k) == (8192, 8192, 8192) else f"{m}x{n}x{k} per GPU")),
            "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if c4 else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": ("synthetic U[-1,1]" if c4 else "synthetic U(1,2)")
                    + ": the reference's gen_uniform_rect (xoshiro256++) seeds 1, 2, on the device",
            "config": {"workload": f"ADP DGEMM {m_global}x{n}x{k} column-major NN ("
                                   + ("rows partitioned over the GPUs" if c4 else "8192 rows per GPU")
                                   + "), guardrails live, ESC-chosen s, pairs d_a+d_b<=s",
                       "m": m_global, "n": n, "k": k, "slices": trace.slices, "esc_bits": trace.esc_bits,
                       "path": trace.path, "pairs": pairs, "gemm_variant": trace.gemm_variant,
                       "parallelism": (f"row-block x{world}: A/C rows per rank, B column slabs; B exponent "
                                       "stats all-gathered, ADP decision max-allreduced (NCCL); B slice planes: "
                                       + ({"fused": "read in place by the GEMM over NVLink (fused phase 7)",
                                           "pull": "pulled rank by rank by the copy engines under the GEMM "
                                                   "(phase 7 per rank)"}.get(args.dist) if peers is not None
                                          else "NCCL all-gather overlapped with the own-column GEMM")
                                       + f" [--dist {dist_mode}]")
                       if world > 1 else "single GPU",
                       "esc_method": args.esc,
                       "l2": f"inputs larger than L2 ({m * k * 8 >> 20} MiB per operand, L2 126 MB)"},
            "gpu_launches": launches,
            "stage_ms": stage_ms,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        line.update(extra)
        if "accuracy" in extra:
            line["max_rel_err"] = extra["accuracy"]["max_rel_err"]
        if "native_fp64" in extra:
            line["speedup_vs_native_fp64"] = value / world / extra["native_fp64"]["value"]
        line["value_burst"] = flops_global / (burst_ms * 1e-3) / 1e12
        line["config"]["soak"] = (f"{n_soak} untimed steps (~{args.soak:g} s) before the timed region: value is the "
                                  "power-capped steady state; value_burst = 5 steps right after the warm-up")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

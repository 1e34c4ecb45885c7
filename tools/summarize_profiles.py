"""Turn a tools/profile_round.sh run (gpurun_out/<tag>_*) into the tracked
summaries under profiles/: launch-list shares, ncu_summary.json (the bench's
roofline.traffic source), ncu details pages, probe outputs.
Usage: python tools/summarize_profiles.py [tag]   (default r01c)"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01c"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    return [(dict(zip(hdr, row)), dict(zip(hdr, units))) for row in r[2:]]


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1,
         "ms": 1e3, "msecond": 1e3}


def val(d, u, k):
    try:
        return float(d[k].replace(",", "")) * SCALE.get(u[k], 1)
    except (KeyError, ValueError):
        return None


# launch list
agg = collections.OrderedDict()
hdr = None
for r in csv.reader(open(os.path.join(G, f"{tag}_launches.csv"))):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        us = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
        k = d["Kernel Name"].split("(")[0].replace("adpb200::<unnamed>::", "").replace("void ", "")
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += us
ours = {k: v for k, v in agg.items() if not k.startswith("at::")}
tot = sum(v[1] for v in ours.values())
lines = ["# ncu launch list (gpu__time_duration.sum, --clock-control none): python bench.py --quick --no-cpu --steps 2 --warmup 1",
         "# cold-cache, serialised launches - compare SHARES, not absolutes; every pipeline call of the run (trace call, warm-up, burst, timed);",
         "# uniform_kernel = the device xoshiro input generator (setup, untimed).",
         f"{'kernel':48s} {'launches':>8s} {'total_us':>12s} {'per_launch_us':>14s} {'share_of_ours':>13s}"]
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    sh = f"{100 * v[1] / tot:12.1f}%" if k in ours else "     (torch)"
    lines.append(f"{k[:48]:48s} {v[0]:8d} {v[1]:12.3f} {v[1] / v[0]:14.4f} {sh}")
open(os.path.join(P, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
shutil.copy(os.path.join(G, f"{tag}_launches.csv"), os.path.join(P, f"{tag}_launches.csv"))

# launch list of one certified-ESC call on U[-1,1] (the certificate's kernels beside the rest)
cpath = os.path.join(G, f"{tag}_launches_certified.csv")
if os.path.exists(cpath):
    cagg = collections.OrderedDict()
    chdr = None
    for r in csv.reader(open(cpath)):
        if r and r[0] == "ID":
            chdr = r
            continue
        if chdr and len(r) == len(chdr):
            d = dict(zip(chdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            us = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
            k = d["Kernel Name"].split("(")[0].replace("adpb200::<unnamed>::", "").replace("void ", "")
            a = cagg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += us
    cours = {k: v for k, v in cagg.items() if not k.startswith("at::") and "uniform" not in k}
    ctot = sum(v[1] for v in cours.values())
    cl = ["# ncu launch list: python tools/one_call.py --u11 --certified (8192^3 U[-1,1], certified ESC, 2 calls)",
          "# the certificate = certify_prep/finish + slice kernels in indicator mode (K = 512) + one igemm<64> launch",
          f"{'kernel':48s} {'launches':>8s} {'total_us':>12s} {'per_launch_us':>14s} {'share_of_ours':>13s}"]
    for k, v in sorted(cagg.items(), key=lambda x: -x[1][1]):
        sh = f"{100 * v[1] / ctot:12.1f}%" if k in cours else "   (setup)"
        cl.append(f"{k[:48]:48s} {v[0]:8d} {v[1]:12.3f} {v[1] / v[0]:14.4f} {sh}")
    open(os.path.join(P, f"{tag}_launches_certified.txt"), "w").write("\n".join(cl) + "\n")

# ncu details + summary
ig, igu = raw(os.path.join(G, f"{tag}_igemm64.ncu-rep"))[0]
gk = {}
for d, u in raw(os.path.join(G, f"{tag}_guard.ncu-rep")):
    name = d["Kernel Name"].split("(")[0].replace("adpb200::<unnamed>::", "").replace("void ", "")
    t_us = val(d, u, "gpu__time_duration.sum")
    byt = val(d, u, "dram__bytes_read.sum") + val(d, u, "dram__bytes_write.sum")
    gk[name] = {"us": round(t_us, 2), "dram_bytes": int(byt), "achieved_GBps": round(byt / (t_us * 1e-6) / 1e9, 1),
                "frac_of_6551_GBps": round(byt / (t_us * 1e-6) / 1e9 / 6551, 3)}
rd, wr = val(ig, igu, "dram__bytes_read.sum"), val(ig, igu, "dram__bytes_write.sum")
summ = {
    "round": 2, "tag": tag,
    "source": "ncu --set full --clock-control none (tools/profile_round.sh): igemm_kernel<64> = second call of "
              "tools/one_call.py (8192^3, U(1,2), s = 7, 34 pairs); guard kernels = second call",
    "igemm_kernel": {
        "duration_ms_under_ncu": round(val(ig, igu, "gpu__time_duration.sum") / 1e3, 3),
        "sm_clock_ghz_under_ncu": round(float(ig["sm__cycles_elapsed.avg.per_second"]), 3),
        "tensor_pipe_active_pct_of_active_cycles": round(float(ig["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]), 1),
        "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
        "l2_to_sm_bytes": int(val(ig, igu, "l1tex__m_xbar2l1tex_read_bytes.sum")),
        "registers_per_thread": int(float(ig["launch__registers_per_thread"]))},
    "igemm_dram_bytes_per_launch": int(rd + wr),
    "igemm_algorithmic_bytes_per_launch": {"note": "tensor-bound kernel; unique operand bytes = 7 planes x (8192 x 8192) "
                                                   "x 2 operands + C written",
                                           "planes_read_once": 939524096, "c_written": 536870912},
    "reading": "DRAM traffic per launch vs 1.48 GB unique: L2 re-reads across waves, far from the HBM limit. The kernel "
               "is power-capped; the tensor pipe is ~80% active, the MMA warp waiting ~7% for the TMEM drain at tile "
               "boundaries (ADPB200_DEBUG=4 counters); when active the pipe runs at the spec dense rate.",
    "guard_kernels": gk,
}
json.dump(summ, open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)
for nm in ("igemm64", "guard"):
    out = subprocess.run(["ncu", "-i", os.path.join(G, f"{tag}_{nm}.ncu-rep"), "--page", "details"], capture_output=True,
                         text=True).stdout
    open(os.path.join(P, f"{tag}_{nm}_ncu_details.txt" if nm == "guard" else f"{tag}_igemm64_ncu_details.txt"),
         "w").write(out)
for f in ("mma_peak.jsonl", "qr_probe.jsonl", "esc_block.jsonl", "shapes.jsonl", "fp64_chain.json", "small.jsonl",
          "e2e.json", "pcie.json"):
    src = os.path.join(G, f"{tag}_{f}")
    if os.path.exists(src):
        keep = [l for l in open(src) if l.startswith("{")]
        open(os.path.join(P, f"{tag}_{f}"), "w").writelines(keep)
bench = [l for l in open(os.path.join(G, f"{tag}_bench.log")) if l.startswith("{")]
if bench:
    open(os.path.join(P, f"{tag}_bench.json"), "w").write(bench[-1])
print(json.dumps({"igemm_dram": summ["igemm_dram_bytes_per_launch"], "guard": gk}, indent=1))
print("\n".join(lines[:12]))

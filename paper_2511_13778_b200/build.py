"""Build libadpb200.so (all CUDA kernels, sm_100a) in-tree with nvcc.

    python -m paper_2511_13778_b200.build [--force]

The shared library lands next to this file so it travels with the repository
snapshot (it is git-ignored, not gpurun-ignored). The CUDA runtime is linked
statically; the driver API (cuTensorMapEncodeTiled) is resolved at run time
through cudaGetDriverEntryPoint, so the library loads on hosts without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "adpb200")
LIB = os.path.join(PKG, "libadpb200.so")
SOURCES = ["guard.cu", "slice.cu", "igemm.cu", "native.cu", "grade.cu", "qr.cu", "api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-I" + INCLUDE,
]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build libadpb200.so; with `variant`, an A/B build of the same sources with extra
    -D defines into ab/lib_<variant>.so (objects under build/adpb200_<variant>)."""
    build_dir, lib_out, flags = BUILD, LIB, list(FLAGS)
    if variant:
        build_dir = BUILD + "_" + variant
        lib_out = os.path.join(ROOT, "ab", f"lib_{variant}.so")
        os.makedirs(os.path.dirname(lib_out), exist_ok=True)
        flags += ["-D" + d for d in defines]
    os.makedirs(build_dir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(INCLUDE, "adpb200.h"))
    objs = []
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC] + flags + ["-c", s, "-o", o])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(lib_out, objs):
        run([NVCC, "-shared", "-cudart", "static", "-o", lib_out] + objs + ["-ldl", "-lpthread", "-lrt"])
    return lib_out


if __name__ == "__main__":
    # python -m paper_2511_13778_b200.build [--force] [--variant NAME -DNAME=VAL ...]
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else ""
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose=True, variant=var, defines=defs))

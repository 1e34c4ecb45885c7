"""CPU: resource facts of the built kernels that the launch code relies on.

igemm_kernel<NB> splits its register file by warpgroup with setmaxnreg
(csrc/igemm.cu: 40 per thread for the producer/MMA/allocator warpgroup, the rest
for the epilogue warpgroups). setmaxnreg.inc blocks until the CTA's pool has the
registers, and the pool is what the launch reserved: the CTA's threads x the
kernel's register count. The split is sized for 168 with 384 threads (232 per
epilogue thread) and for 128 with 512 threads (NB = 48: 3 epilogue warps per
TMEM quadrant, 152 per epilogue thread); a build that comes out different would
hang the epilogue (launch_igemm refuses it at run time). This pins it at build
time, together with the SASS evidence for the tensor-core paths."""
import os
import re
import shutil
import subprocess

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2511_13778_b200", "libadpb200.so")


def _cuobjdump(*args):
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(exe):
        pytest.skip("library or cuobjdump missing")
    return subprocess.run([exe, *args, LIB], capture_output=True, text=True, check=True).stdout


def test_igemm_register_count_matches_the_split():
    out = _cuobjdump("--dump-resource-usage")
    regs = {}
    lines = out.splitlines()
    for i, line in enumerate(lines):
        m = re.search(r"igemm_kernel(?:I|<)L?i?(\d+)E?L?i?(\d*)", line)
        if m and "Function" in line:
            r = re.search(r"REG:(\d+)", lines[i + 1] if i + 1 < len(lines) else "")
            if r:
                regs[(int(m.group(1)), int(m.group(2) or 8))] = int(r.group(1))
    # (NB, epilogue warps): 384 threads -> 168 registers, 512 threads (NB = 48, short k) -> 128
    want = {(8, 8): 168, (16, 8): 168, (32, 8): 168, (48, 8): 168, (48, 12): 128, (64, 8): 168}
    assert regs == want, regs


def test_sass_has_tensor_core_paths():
    sass = _cuobjdump("-sass")
    assert "UTCIMMA" in sass          # tcgen05.mma kind::i8 (slice GEMM)
    assert "UTMALDG" in sass          # TMA loads
    assert "USETMAXREG" in sass       # warpgroup register split
    assert re.search(r"\bDMMA\b", sass)  # FP64 tensor cores (fast fallback)

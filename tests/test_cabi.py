"""CPU: the drop-in boundary (include/adpb200.h) without a GPU.

* libadpb200.so loads on a GPU-less host and exports every function the
  header declares;
* the option validation mirrors AdpConfig::validate (adp.cpp:15-28,
  proj/tests/test_adp.cpp:58-80);
* the host copy of the device decision function is bitwise identical to the
  oracle's decide() (gate order + FP64 cost model, adp.cpp:46-96);
* the Python mirror (parse_mode, AdpTrace.to_json) and the C++ façade
  (include/adpb200.hpp) compile and behave like the reference's host API.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def adp():
    import paper_2511_13778_b200 as adp

    adp.lib()
    return adp


def declared_functions():
    src = open(os.path.join(ROOT, "include", "adpb200.h")).read()
    return sorted(set(re.findall(r"\b(adpb200_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(adp):
    names = declared_functions()
    assert len(names) >= 20
    lib = adp.lib()
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/adpb200.h but not exported"
    from paper_2511_13778_b200._lib import EXPORTED

    assert set(EXPORTED) <= set(names)
    assert b"sm_100a" in lib.adpb200_version()


def test_library_is_cuda_sm100a():
    out = subprocess.run(["cuobjdump", "-lelf", os.path.join(ROOT, "paper_2511_13778_b200", "libadpb200.so")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_default_options_match_reference(adp):
    o = adp._lib.default_options()
    # AdpConfig defaults (adp.hpp:18-33)
    assert (o.target_bits, o.esc_block_len, o.max_slices, o.min_dim, o.mode, o.forced_slices, o.cost_ratio,
            o.chunk_len) == (53, 256, 18, 256, 0, 7, 512.0, 65536)
    assert o.pair_limit == adp.PAIRS_FULL  # the reference's adp_gemm uses the Full pair set


@pytest.mark.parametrize("field,value,ok", [
    ("target_bits", 0, False), ("target_bits", 1024, True), ("target_bits", 1025, False),
    ("esc_block_len", 0, False), ("max_slices", 6, False), ("max_slices", 7, True), ("max_slices", 32, True),
    ("max_slices", 33, False), ("min_dim", 0, False), ("cost_ratio", 0.0, False), ("cost_ratio", -1.0, False),
    ("chunk_len", 0, False), ("chunk_len", 131071, True), ("chunk_len", 131072, False),
])
def test_validate_options(adp, field, value, ok):
    cfg = adp.AdpConfig(**{field: value})
    if ok:
        cfg.validate()
    else:
        with pytest.raises(ValueError):
            cfg.validate()


def test_forced_slices_validated_only_in_emulate_mode(adp):
    adp.AdpConfig(forced_slices=0).validate()
    with pytest.raises(ValueError):
        adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=0).validate()
    with pytest.raises(ValueError):
        adp.AdpConfig(mode=adp.AdpMode.ForceEmulate, forced_slices=33).validate()


def test_decide_host_matches_oracle(adp, port):
    from oracle.oracle import Config

    rng = np.random.default_rng(11)
    names = ("emulated", "native_fallback")
    from oracle.oracle import REASONS

    for _ in range(2000):
        mode = int(rng.integers(0, 3))
        kw = dict(mode=mode, min_dim=int(rng.integers(1, 600)), cost_ratio=float(rng.choice([1.0, 16.0, 512.0, 3.7, 100.1])),
                  forced_slices=int(rng.integers(1, 33)), max_slices=int(rng.integers(7, 33)),
                  target_bits=int(rng.integers(1, 80)))
        args = (int(rng.integers(0, 2)), int(rng.integers(0, 2)), int(rng.integers(0, 5000)),
                int(rng.integers(0, 5000)), int(rng.integers(0, 5000)), int(rng.integers(0, 200)))
        got = adp.decide(*args, adp.AdpConfig(mode=adp.AdpMode(mode), **{k: v for k, v in kw.items() if k != "mode"}))
        want = port.decide(*args, Config(**kw))
        assert got[0] == names[want[0]] and got[1] == REASONS[want[1]]
        assert got[2] == want[2] and got[3] == want[3]
        assert (got[4] if got[4] is not None else -1) == want[4]
        assert np.float64(got[5]).view(np.uint64) == np.float64(want[5]).view(np.uint64)


def test_parse_mode_and_trace_json(adp):
    cfg = adp.AdpConfig()
    assert adp.parse_mode("emulate:11", cfg) and cfg.mode == adp.AdpMode.ForceEmulate and cfg.forced_slices == 11
    for bad in ("emulate:", "emulate:0", "emulate:33", "emulate:7x", "emulate:-3", "Auto", ""):
        assert not adp.parse_mode(bad, adp.AdpConfig())
    assert adp.parse_mode("native", cfg) and cfg.mode == adp.AdpMode.ForceNative
    t = adp.AdpTrace(path="native_fallback", reason="too_small", esc_bits=None, slices=7, m=3, n=4, k=5)
    assert t.to_json() == '{"path":"native_fallback","reason":"too_small","esc_bits":null,"slices":null,"m":3,"n":4,"k":5}'


def test_required_slices(adp):
    assert adp.required_slices(53, 1) == 7 and adp.required_slices(53, 2) == 8 and adp.required_slices(24, 0) == 4
    with pytest.raises(ValueError):
        adp.required_slices(0, 1)


def _build_facade(tmp_path):
    exe = os.path.join(str(tmp_path), "facade_check")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "facade_check.cpp"), "-o", exe,
           "-L", os.path.join(ROOT, "paper_2511_13778_b200"), "-ladpb200",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2511_13778_b200"),
           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_facade_compiles_and_checks_contracts(tmp_path):
    exe = _build_facade(tmp_path)
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout


def test_nccl_cpp_driver_compiles(tmp_path):
    """include/adpb200_nccl.hpp (C++ multi-GPU driver over NCCL) compiles and links
    against libadpb200.so and libnccl (the run is a GPU test)."""
    exe = os.path.join(str(tmp_path), "dist_nccl_check")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "dist_nccl_check.cpp"), "-o", exe,
           "-L", os.path.join(ROOT, "paper_2511_13778_b200"), "-ladpb200",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lnccl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr

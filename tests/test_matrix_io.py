"""CPU: the reference's matrix file formats (proj/src/matrix_io.cpp) in the
Python mirror (paper_2511_13778_b200.matrix_io) and the C++ façade header
(include/adpb200_io.hpp), checked byte-for-byte against files the reference
itself writes and reads."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2511_13778_b200 import matrix_io


def _sample():
    rng = np.random.default_rng(11)
    a = rng.uniform(-1, 1, (7, 5))
    a[0, 0] = -0.0
    a[1, 1] = 1e-310          # subnormal
    a[2, 2] = 1.5e300
    a[3, 3] = 0.0001          # to_chars picks 1e-04
    a[4, 4] = 123456789012345680000.0
    a[5, 0] = 100.0
    return a


@pytest.mark.parametrize("ext", ["mtx", "mm", "adpm", "bin"])
def test_python_files_are_the_references(ref, tmp_path, ext):
    a = _sample()
    ours = str(tmp_path / f"ours.{ext}")
    theirs = str(tmp_path / f"theirs.{ext}")
    matrix_io.write_matrix(ours, a)
    ref.write_matrix(theirs, a)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    back = ref.read_matrix(ours)
    assert np.array_equal(back.view(np.uint64), a.view(np.uint64))
    mine = matrix_io.read_matrix(theirs)
    assert np.array_equal(mine.view(np.uint64), a.view(np.uint64))


def test_adpm_keeps_nan_payloads(tmp_path):
    a = np.zeros((2, 3))
    a.view(np.uint64)[0, 1] = 0xFFF8DEADBEEFCAFE
    p = str(tmp_path / "x.adpm")
    matrix_io.write_matrix(p, a)
    assert np.array_equal(matrix_io.read_matrix(p).view(np.uint64), a.view(np.uint64))


def test_matrix_market_comments_and_errors(tmp_path):
    p = tmp_path / "c.mtx"
    p.write_bytes(b"%%MatrixMarket matrix array real general\r\n% c\n\n2 2\n1\n2\n3\n4\n")
    assert np.array_equal(matrix_io.read_matrix(str(p)), np.array([[1.0, 3.0], [2.0, 4.0]]))
    for body, msg in [(b"%%MatrixMarket matrix coordinate real general\n1 1\n1\n", "unsupported header"),
                      (b"%%MatrixMarket matrix array real general\n2 2\n1\n2\n", "not enough values"),
                      (b"%%MatrixMarket matrix array real general\n1 1\nabc\n", "bad value"),
                      (b"%%MatrixMarket matrix array real general\n", "missing dimensions"),
                      (b"ADPM\x02\x00\x00\x00", "unsupported version"),
                      (b"ADPM\x01\x00\x00\x00" + (1).to_bytes(8, "little") + (1).to_bytes(8, "little"),
                       "truncated payload")]:
        p.write_bytes(body)
        with pytest.raises(RuntimeError, match=msg):
            matrix_io.read_matrix(str(p))
    big = b"ADPM\x01\x00\x00\x00" + (1 << 20).to_bytes(8, "little") + (1 << 10).to_bytes(8, "little")
    p.write_bytes(big)
    with pytest.raises(RuntimeError, match="out of range"):
        matrix_io.read_matrix(str(p))


def test_cpp_header_round_trip(ref, tmp_path):
    exe = str(tmp_path / "io_check")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
                        "/usr/local/cuda/include", os.path.join(ROOT, "tests", "cpp", "io_check.cpp"), "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    a = _sample()
    for src_ext, dst_ext in [("mtx", "adpm"), ("adpm", "mtx"), ("mm", "mm")]:
        src = str(tmp_path / f"in.{src_ext}")
        dst = str(tmp_path / f"out.{dst_ext}")
        ref.write_matrix(src, a)
        r = subprocess.run([exe, src, dst], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        want = str(tmp_path / f"want.{dst_ext}")
        ref.write_matrix(want, a)
        assert open(dst, "rb").read() == open(want, "rb").read()


def test_shortest_decimal_matches_to_chars_on_random_magnitudes(ref, tmp_path):
    rng = np.random.default_rng(123)
    bits = rng.integers(0, 2 ** 63 - 1, size=(40, 50), dtype=np.int64).astype(np.uint64)
    a = bits.view(np.float64).copy()
    a[~np.isfinite(a)] = 1.0
    a[::3] = np.round(a[::3] * 0 + rng.uniform(-1e6, 1e6, a[::3].shape))   # integers
    a[1::7] = rng.uniform(-1, 1, a[1::7].shape) * 10.0 ** rng.integers(-30, 30, a[1::7].shape)
    ours, theirs = str(tmp_path / "o.mtx"), str(tmp_path / "t.mtx")
    matrix_io.write_matrix(ours, a)
    ref.write_matrix(theirs, a)
    assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_cpp_header_rejects_malformed_files(tmp_path):
    exe = str(tmp_path / "io_check")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
                        "/usr/local/cuda/include", os.path.join(ROOT, "tests", "cpp", "io_check.cpp"), "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    p = tmp_path / "bad.mtx"
    cases = [(b"%%MatrixMarket matrix coordinate real general\n1 1\n1\n", "unsupported header"),
             (b"%%MatrixMarket matrix array real general\n2 2\n1\n2\n", "not enough values"),
             (b"%%MatrixMarket matrix array real general\n1 1\nabc\n", "bad value"),
             (b"%%MatrixMarket matrix array real general\n% only comments\n", "missing dimensions"),
             (b"%%MatrixMarket matrix array real general\n2 x\n", "bad dimension line"),
             (b"ADPM\x02\x00\x00\x00", "unsupported version"),
             (b"ADPM\x01\x00\x00\x00" + (1).to_bytes(8, "little"), "truncated header"),
             (b"ADPM\x01\x00\x00\x00" + (1).to_bytes(8, "little") + (1).to_bytes(8, "little"), "truncated payload"),
             (b"ADPM\x01\x00\x00\x00" + (1 << 20).to_bytes(8, "little") + (1 << 10).to_bytes(8, "little"),
              "out of range")]
    for body, msg in cases:
        p.write_bytes(body)
        r = subprocess.run([exe, str(p), str(tmp_path / "o.adpm")], capture_output=True, text=True)
        assert r.returncode == 3 and msg in r.stderr, (body, r.stderr)
    # CRLF, blank lines, a '+' sign and upper-case banner tokens are accepted
    p.write_bytes(b"%%MatrixMarket MATRIX Array REAL General\r\n\r\n% c\r\n2 1\r\n+1.5\r\n-2e-3\r\n")
    r = subprocess.run([exe, str(p), str(tmp_path / "o.mtx")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "o.mtx").read_bytes() == b"%%MatrixMarket matrix array real general\n2 1\n1.5\n-0.002\n"

"""The reference's matrix file formats (mirror of ozadp/matrix_io.hpp,
proj/src/matrix_io.cpp:40-144) for the Python host interface.

* Matrix Market array text: `%%MatrixMarket matrix array real general`,
  optional % comments, `rows cols`, one value per line in column-major order,
  shortest round-trip decimals (std::to_chars; byte-identical files);
* ADPM binary: b"ADPM", u32 LE version 1, u64 LE rows, u64 LE cols, then the
  row-major little-endian FP64 payload (bitwise lossless).

Readers cap the element count at 2^28 like the reference; format and I/O
failures raise RuntimeError (std::runtime_error).
"""
from __future__ import annotations

import struct

import numpy as np

from .grading import _num

MAX_ELEMENTS = 1 << 28

__all__ = ["write_matrix_market", "read_matrix_market", "write_adpm", "read_adpm", "read_matrix", "write_matrix"]


def _check_dims(rows: int, cols: int) -> None:
    if rows > MAX_ELEMENTS or cols > MAX_ELEMENTS or rows * cols > MAX_ELEMENTS:
        raise RuntimeError("matrix file: dimensions out of range")


def write_matrix_market(f, m: np.ndarray) -> None:
    m = np.asarray(m, dtype=np.float64)
    rows, cols = m.shape
    out = ["%%MatrixMarket matrix array real general\n", f"{rows} {cols}\n"]
    out += [_num(v) + "\n" for v in m.T.reshape(-1).tolist()]
    f.write("".join(out).encode())


def read_matrix_market(f) -> np.ndarray:
    lines = f.read().decode().split("\n")
    if not lines or (len(lines) == 1 and not lines[0]):
        raise RuntimeError("matrix market: missing header")
    head = lines[0].rstrip("\r")
    parts = head.split()
    parts += [""] * (5 - len(parts))
    if parts[0] != "%%MatrixMarket" or [p.lower() for p in parts[1:5]] != ["matrix", "array", "real", "general"]:
        raise RuntimeError("matrix market: unsupported header: " + head)
    i = 1
    while True:
        if i >= len(lines):
            raise RuntimeError("matrix market: missing dimensions")
        line = lines[i].rstrip("\r")
        i += 1
        if line and line[0] != "%":
            break
    dims = line.split()
    try:
        rows, cols = int(dims[0]), int(dims[1])
        if rows < 0 or cols < 0:
            raise ValueError
    except (ValueError, IndexError):
        raise RuntimeError("matrix market: bad dimension line: " + line) from None
    _check_dims(rows, cols)
    tokens = " ".join(lines[i:]).split()
    if len(tokens) < rows * cols:
        raise RuntimeError("matrix market: not enough values")
    vals = []
    for t in tokens[: rows * cols]:
        try:
            vals.append(float(t))
        except ValueError:
            raise RuntimeError("matrix market: bad value: " + t) from None
    return np.array(vals, dtype=np.float64).reshape(cols, rows).T.copy()


def write_adpm(f, m: np.ndarray) -> None:
    m = np.ascontiguousarray(m, dtype="<f8")
    rows, cols = m.shape
    f.write(b"ADPM" + struct.pack("<IQQ", 1, rows, cols) + m.tobytes())


def read_adpm(f) -> np.ndarray:
    if f.read(4) != b"ADPM":
        raise RuntimeError("adpm: bad magic")
    v = f.read(4)
    if len(v) != 4 or struct.unpack("<I", v)[0] != 1:
        raise RuntimeError("adpm: unsupported version")
    h = f.read(16)
    if len(h) != 16:
        raise RuntimeError("adpm: truncated header")
    rows, cols = struct.unpack("<QQ", h)
    _check_dims(rows, cols)
    want = rows * cols * 8
    payload = f.read(want)
    if len(payload) != want:
        raise RuntimeError("adpm: truncated payload")
    return np.frombuffer(payload, dtype="<f8").reshape(rows, cols).astype(np.float64)


def read_matrix(path: str) -> np.ndarray:
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError("cannot open " + path) from None
    with f:
        adpm = f.read(4) == b"ADPM"
        f.seek(0)
        return read_adpm(f) if adpm else read_matrix_market(f)


def write_matrix(path: str, m: np.ndarray) -> None:
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError("cannot open " + path + " for writing") from None
    with f:
        ext = path.rsplit(".", 1)[-1].lower() if "." in path else ""
        if ext in ("mtx", "mm"):
            write_matrix_market(f, m)
        else:
            write_adpm(f, m)

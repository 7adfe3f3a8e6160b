#!/usr/bin/env python
"""GPU inflate vs zlib on BGEN-8-like blocks (debug / A-B tool): prints per-case status and
the first mismatching byte."""
import sys
import zlib
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from bgen_fixture import _probability_block  # noqa: E402

from paper_2604_21095_b200 import _native  # noqa: E402


def gpu_inflate(streams, stride):
    blob = b"".join(streams) + b"\0" * 16
    off = np.cumsum([0] + [len(s) for s in streams[:-1]]).astype(np.int64)
    size = np.array([len(s) for s in streams], dtype=np.int64)
    out = np.zeros(len(streams) * stride, dtype=np.uint8)
    out_len = np.zeros(len(streams), dtype=np.int64)
    status = np.zeros(len(streams), dtype=np.int32)
    b = np.frombuffer(blob, dtype=np.uint8).copy()
    _native.call("pg_debug_inflate", b.ctypes.data, b.size, off.ctypes.data, size.ctypes.data, len(streams), 0,
                 out.ctypes.data, stride, out_len.ctypes.data, status.ctypes.data)
    return [(int(st), out[i * stride:i * stride + int(n)].tobytes()) for i, (st, n) in enumerate(zip(status, out_len))]


def main():
    rng = np.random.default_rng(1)
    n = 23000
    cases = {}
    cases["mono_het"] = np.full(n, 1.0)
    cases["mono_hom"] = np.full(n, 0.0)
    d = rng.binomial(2, 0.3, n).astype(float)
    cases["hard"] = d.copy()
    f = rng.random(n) < 0.2
    d[f] = np.clip(d[f] + rng.normal(0, 0.3, f.sum()), 0, 2)
    d[rng.random(n) < 0.05] = np.nan
    cases["c5"] = d
    names = list(cases)
    blocks = [_probability_block(cases[k], 8, 2, 0) for k in names]
    streams = [zlib.compress(b) for b in blocks]
    got = gpu_inflate(streams, 10 + 5 * n + 16)
    for k, b, (st, out) in zip(names, blocks, got):
        bad = next((i for i in range(min(len(b), len(out))) if b[i] != out[i]), None)
        print(f"{k:10s} status {st} len {len(out)}/{len(b)} first mismatch {bad}")


if __name__ == "__main__":
    main()

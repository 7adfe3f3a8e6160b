#!/usr/bin/env python
"""Host gaps between device batches at the C3 shape: wall time of a 1M-marker pass of
scan_device with and without the result fetch, and the per-batch wall split
(pg_scan_device vs _collect). Diagnostics only (wall clock), not a bench value."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2604_21095_b200 import _native  # noqa: E402
from paper_2604_21095_b200._device import BatchInfo, DeviceContext, call  # noqa: E402
from paper_2604_21095_b200.engine import threshold_premask  # noqa: E402
from ctypes import byref  # noqa: E402


def main():
    n, p, m, db = 23000, 20480, 1 << 20, 65536
    bpm = (n + 3) // 4
    pitch = (bpm + 15) // 16 * 16
    dev = torch.device("cuda:0")
    ytil = bench.synth_panel(torch, n, p, 3, dev)
    packed = bench.synth_packed(torch, m, n, pitch, 5, dev)
    gidx = np.arange(n, dtype=np.int64)
    with DeviceContext(0) as ctx:
        ctx.set_panel_device(ytil.data_ptr(), n, p, p, gidx, n)
        df = float(n - 2)
        ctx.set_scan(df, _native.PG_MODE_THRESHOLD, np.full(p, threshold_premask(1e-4, df)))
        batches = [(s, min(db, m - s)) for s in range(0, m, db)]
        for fetch in (True, False, True, False):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            t_call = t_coll = g = 0.0
            for s, c in batches:
                info = BatchInfo()
                a = time.perf_counter()
                with ctx.lock:
                    call("pg_scan_device", ctx._h, _native.PG_GENO_BED, packed.data_ptr() + s * pitch, c, bpm, pitch,
                         byref(info))
                b = time.perf_counter()
                ctx._collect(info, fetch, 8)
                t_call += b - a
                t_coll += time.perf_counter() - b
                g += info.gemm_ms
            torch.cuda.synchronize()
            wall = 1e3 * (time.perf_counter() - t0)
            print(f"fetch={fetch}: wall {wall:.1f} ms, gemm {g:.1f} ms, in pg_scan_device {1e3 * t_call:.1f} ms, "
                  f"in _collect {1e3 * t_coll:.1f} ms, candidates/batch {info.n_candidates}")


if __name__ == "__main__":
    main()

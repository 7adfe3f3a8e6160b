#!/usr/bin/env python
"""Secondary BASELINE configs on one GPU (the driver's bench.py measures C3):

  C2  synthetic PLINK .bed N=23,000 x M=1M x P=2,048
  C5  synthetic BGEN 8-bit dosages with 5% missing calls, N=23,000 x M=1M x P=4,096

value: device time of the scan with inputs resident in HBM (one device batch of distinct
markers re-scanned until M markers are covered). e2e (C5): compressed BGEN blocks from
pinned host memory -> GPU inflate + validation (pg_stage_bgen) -> scan, per batch.
Prints one JSON line per workload.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
import zlib
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def bgen_rows(rng, count, n, missing=0.05):
    """(raw device rows [count, 3n] = u8 prob pairs | ploidy, compressed BGEN blocks)."""
    rows = np.empty((count, 3 * n), dtype=np.uint8)
    blocks = []
    for i in range(count):
        af = rng.uniform(0.05, 0.95)
        g = rng.binomial(2, af, n).astype(np.float64)
        frac = rng.random(n) < 0.2  # imputed-like: 20% fractional dosages
        g[frac] = np.clip(g[frac] + rng.normal(0, 0.3, frac.sum()), 0, 2)
        d = g
        p1 = np.where(d <= 1, 1 - d, 0.0)
        ph = np.where(d <= 1, d, 2 - d)
        a = np.rint(p1 * 255).astype(np.int64)
        b = np.rint(ph * 255).astype(np.int64)
        over = a + b - 255
        b = np.where(over > 0, b - over, b)
        probs = np.stack([a, b], 1).astype(np.uint8).reshape(-1)
        ploidy = np.full(n, 2, np.uint8)
        ploidy[rng.random(n) < missing] |= 0x80
        rows[i, :2 * n] = probs
        rows[i, 2 * n:] = ploidy
        data = np.concatenate([np.frombuffer(np.array([n], "<u4").tobytes() + np.array([2], "<u2").tobytes()
                                             + bytes([2, 2]), np.uint8), ploidy, np.array([0, 8], np.uint8), probs])
        comp = zlib.compress(data.tobytes(), 6)
        blocks.append(np.array([data.size], "<u4").tobytes() + comp)
    return rows, blocks


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", choices=["c2", "c5"], default="c5")
    ap.add_argument("--markers", type=int, default=1_000_000)
    ap.add_argument("--samples", type=int, default=23_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--distinct", type=int, default=0,
                    help="distinct markers in the resident batch = markers per launch (default: the engine's device "
                         "batch, 65,536 for PLINK and 8,192 for BGEN)")
    ap.add_argument("--contexts", type=int, choices=[1, 2], default=2,
                    help="C5 e2e: batches alternate between two device contexts on two host threads")
    a = ap.parse_args()

    import torch

    from paper_2604_21095_b200 import _native
    from paper_2604_21095_b200._device import DeviceContext
    from paper_2604_21095_b200.engine import threshold_premask

    n = a.samples
    p = 2048 if a.workload == "c2" else 4096
    dev = torch.device("cuda", 0)
    ctx = DeviceContext(0)
    gen = torch.Generator(device=dev).manual_seed(5)
    y = torch.randn(n, p, generator=gen, device=dev, dtype=torch.float64)
    y -= y.mean(0, keepdim=True)
    y /= torch.sqrt((y * y).mean(0, keepdim=True))
    gidx = np.arange(n, dtype=np.int64)
    ctx.set_panel_device(y.data_ptr(), n, p, p, gidx, n)
    df = float(n - 2)
    ctx.set_scan(df, _native.PG_MODE_THRESHOLD, np.full(p, threshold_premask(1e-4, df)))
    rng = np.random.default_rng(9)
    batch = a.distinct or (65536 if a.workload == "c2" else 8192)
    if a.workload == "c2":
        bpm = (n + 3) // 4
        pitch = (bpm + 15) // 16 * 16
        # Binomial(2, AF) genotypes without missing calls (as C3 / bench.py)
        af = rng.uniform(0.05, 0.95, (batch, 1))
        g = (rng.random((batch, n)) < af).astype(np.uint8) + (rng.random((batch, n)) < af).astype(np.uint8)
        codes = np.array([3, 2, 0], np.uint8)[g]
        codes = np.pad(codes, ((0, 0), (0, bpm * 4 - n))).reshape(batch, bpm, 4)
        host = np.zeros((batch, pitch), np.uint8)
        host[:, :bpm] = codes[:, :, 0] | (codes[:, :, 1] << 2) | (codes[:, :, 2] << 4) | (codes[:, :, 3] << 6)
        kind, row_bytes = _native.PG_GENO_BED, bpm
        rows_dev = torch.from_numpy(host).to(dev)
        blocks = None
    else:
        rows, blocks = bgen_rows(rng, batch, n)
        kind, row_bytes = _native.PG_GENO_BGEN8, 3 * n
        pitch = (row_bytes + 15) // 16 * 16
        padded = np.zeros((batch, pitch), np.uint8)
        padded[:, :row_bytes] = rows
        rows_dev = torch.from_numpy(padded).to(dev)
    reps = -(-a.markers // batch)
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=dev)

    def step():
        launches = 0
        for _ in range(reps):
            r = ctx.scan_device(kind, rows_dev.data_ptr(), batch, row_bytes, pitch)
            launches += r.launches
        return launches

    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    launches = sum(step() for _ in range(a.steps))
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    tests = reps * batch * p
    line = {"workload": a.workload, "n_samples": n, "n_markers": reps * batch, "n_phenotypes": p,
            "value": tests / (ms / 1e3), "unit": "tests/s", "ms_per_step": ms, "gpu_launches": launches // a.steps}
    if blocks is not None:
        blob = b"".join(blocks)
        sizes = np.array([len(b) for b in blocks], np.int64)
        offs = np.concatenate([[0], np.cumsum(sizes[:-1])]).astype(np.int64)
        pinned = torch.empty(len(blob), dtype=torch.uint8, pin_memory=True)
        pinned.numpy()[:] = np.frombuffer(blob, np.uint8)
        host_blob = pinned.numpy()

        ctxs = [ctx]
        if a.contexts == 2:
            from concurrent.futures import ThreadPoolExecutor

            c2 = DeviceContext(0)
            buf = torch.empty(ctx.panel_bytes(), dtype=torch.uint8, device=dev)
            ctx.export_panel(buf.data_ptr())
            torch.cuda.synchronize()
            c2.import_panel(buf.data_ptr(), n, p, gidx, n)
            c2.set_scan(df, _native.PG_MODE_THRESHOLD, np.full(p, threshold_premask(1e-4, df)))
            del buf
            ctxs.append(c2)
            pool = ThreadPoolExecutor(max_workers=2)

        def lane(cx, count):
            # staging of batch i+1 (H2D + GPU inflate) overlaps the scan of batch i
            if count == 0:
                return
            cx.stage_bgen_begin(0, host_blob, offs, sizes)
            for i in range(count):
                bad = cx.stage_bgen_end(i % 2)
                assert bad is None, bad
                if i + 1 < count:
                    cx.stage_bgen_begin((i + 1) % 2, host_blob, offs, sizes)
                cx.scan_staged(i % 2)

        def e2e_step():
            if len(ctxs) == 1:
                lane(ctx, reps)
            else:
                futs = [pool.submit(lane, ctxs[k], len(range(k, reps, 2))) for k in range(2)]
                for f in futs:
                    f.result()

        e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            e2e_step()
        torch.cuda.synchronize()
        sec = (time.perf_counter() - t0) / a.steps
        line["e2e"] = {"value": tests / sec, "unit": "tests/s", "s_per_step": sec,
                       "h2d_compressed_bytes_per_step": int(sizes.sum()) * reps,
                       "inflated_bytes_per_step": int((10 + 3 * n) * reps * batch),
                       "path": "pinned compressed blocks -> pg_stage_bgen_begin/_end (GPU inflate, overlapped) -> pg_scan_staged",
                       "device_contexts": len(ctxs)}
        line["compressed_bytes_per_variant"] = float(sizes.mean())
    print(json.dumps(line), flush=True)
    for cx in ctxs if blocks is not None else [ctx]:
        cx.close()


if __name__ == "__main__":
    main()

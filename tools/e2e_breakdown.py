#!/usr/bin/env python
"""Where the C3 end-to-end step's time goes beyond the device scan: the raw-phenotype upload +
panel preparation (pg_ctx_prepare_panel / commit_panel) and the staged host-buffer scan loop,
each timed alone (wall clock around synchronised calls; diagnostics, not a bench value)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2604_21095_b200 import _native  # noqa: E402
from paper_2604_21095_b200._device import DeviceContext  # noqa: E402
from paper_2604_21095_b200.engine import threshold_premask  # noqa: E402
from paper_2604_21095_b200.kernel import build_covariate_basis  # noqa: E402


def wall(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append(1e3 * (time.perf_counter() - t0))
    return min(out), out


def main():
    n, p, m = 23000, 20480, int(sys.argv[1]) if len(sys.argv) > 1 else 262144
    bpm, pitch, db = (n + 3) // 4, (n + 3) // 4 + 0, 65536
    dev = torch.device("cuda:0")
    gen = torch.Generator(device=dev).manual_seed(3)
    c_dev = torch.randn(n, bench.N_COVARIATES, generator=gen, device=dev, dtype=torch.float64)
    yh = torch.empty((n, p), dtype=torch.float64, pin_memory=True)
    yh.copy_(c_dev @ (0.1 * torch.randn(bench.N_COVARIATES, p, generator=gen, device=dev, dtype=torch.float64))
             + torch.randn(n, p, generator=gen, device=dev, dtype=torch.float64))
    y_np, c_np = yh.numpy(), c_dev.cpu().numpy()
    packed = bench.synth_packed(torch, m, n, pitch, 5, dev)
    host = torch.empty((m, bpm), dtype=torch.uint8, pin_memory=True)
    host.copy_(packed[:, :bpm])
    host_np = host.numpy()
    del packed
    gidx = np.arange(n, dtype=np.int64)
    df = float(n - 1 - bench.N_COVARIATES)
    with DeviceContext(0) as ctx:
        basis = build_covariate_basis(c_np, True)
        t_basis, _ = wall(lambda: build_covariate_basis(c_np, True))
        state = {}

        def prep():
            state["flat"], _ = ctx.prepare_panel(y_np, basis.q)

        t_prep, _ = wall(prep)
        t_commit, _ = wall(lambda: ctx.commit_panel(np.nonzero(~state["flat"])[0], gidx, n))
        t_async = {}
        for chunk in (1280, 2560, 5120, 20480):
            def run_async(chunk=chunk):
                ctx.set_panel_async(y_np, basis.q, gidx, n, chunk_cols=chunk)
                ctx.panel_async_wait()

            t_async[chunk], _ = wall(run_async)
        ctx.prepare_panel(y_np, basis.q)
        ctx.commit_panel(np.nonzero(~state["flat"])[0], gidx, n)
        ctx.set_scan(df, _native.PG_MODE_THRESHOLD, np.full(p, threshold_premask(5e-8, df)))
        batches = [(s, min(db, m - s)) for s in range(0, m, db)]

        def staged():
            for i, (s, c) in enumerate(batches):
                ctx.stage(i % 2, _native.PG_GENO_BED, host_np[s:s + c], bpm)
                if i:
                    ctx.scan_staged((i - 1) % 2)
            ctx.scan_staged((len(batches) - 1) % 2)

        t_staged, _ = wall(staged, 2)

        def e2e_like(trace):
            t0 = time.perf_counter()
            b = build_covariate_basis(c_np, True)
            ctx.set_panel_async(y_np, b.q, gidx, n)
            trace.append(("panel call", time.perf_counter() - t0))
            ctx.set_scan(df, _native.PG_MODE_THRESHOLD, np.full(p, threshold_premask(5e-8, df)))
            for i, (s, c) in enumerate(batches):
                ctx.stage(i % 2, _native.PG_GENO_BED, host_np[s:s + c], bpm)
                if i:
                    r = ctx.scan_staged((i - 1) % 2)
                    trace.append((f"scan {i - 1} (gemm {r.gemm_ms:.1f} ms)", time.perf_counter() - t0))
            r = ctx.scan_staged((len(batches) - 1) % 2)
            trace.append((f"scan {len(batches) - 1} (gemm {r.gemm_ms:.1f} ms)", time.perf_counter() - t0))
            ctx.panel_async_wait()
            trace.append(("panel wait", time.perf_counter() - t0))

        for _ in range(2):
            trace = []
            torch.cuda.synchronize()
            e2e_like(trace)
        e2e_trace = trace
        y_gb = y_np.nbytes / 1e9
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d = torch.empty(yh.shape, dtype=torch.float64, device=dev)
        e0.record()
        d.copy_(yh, non_blocking=True)
        e1.record()
        e1.synchronize()
        h2d_ms = e0.elapsed_time(e1)
    print(f"covariate basis (host)      {t_basis:8.1f} ms")
    print(f"prepare_panel (Y H2D+prep)  {t_prep:8.1f} ms   (Y = {y_gb:.2f} GB; bare pinned H2D {h2d_ms:.1f} ms"
          f" = {y_gb / h2d_ms * 1e3:.1f} GB/s)")
    print(f"commit_panel (quantize)     {t_commit:8.1f} ms")
    for chunk, t in t_async.items():
        print(f"set_panel_async + wait, {chunk:5d}-phenotype chunks {t:8.1f} ms")
    print(f"staged scan of {m} markers {t_staged:8.1f} ms")
    print("e2e-like step with the pipelined panel (cumulative wall ms):")
    for name, t in e2e_trace:
        print(f"  {1e3 * t:8.1f}  {name}")


if __name__ == "__main__":
    main()

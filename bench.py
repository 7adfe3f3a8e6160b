#!/usr/bin/env python
"""Benchmark of the BASELINE.json metric: association tests/sec at N=23,000
samples, P=20,480 phenotypes (config 3: synthetic PLINK .bed, M=1,000,000
markers per GPU, THRESHOLD hit compaction at p <= 1e-4).

  python bench.py [--gpus N --steps K --warmup W]             # this repo (B200 kernels)
  python bench.py --impl reference [--steps K --warmup W]     # the reference's own scan loop on the host cores
  torchrun --nproc-per-node N bench.py --gpus N ...            # one rank per GPU
  python bench.py --workload c4 ...                            # 8.9M markers in total (the paper headline)
  python bench.py --markers-per-gpu 1000000 ...                # weak scaling instead

Scaling: by default the C3 job (M = 1,000,000 markers in total) is split into contiguous
256-aligned marker shards over the N ranks (strong scaling, BASELINE config 3 at 1/2/4/8
GPUs); `--workload c4` scans C4's 8.9M markers in total; `--markers-per-gpu M` fixes the
per-rank shard instead (weak scaling). A step scans the rank's whole marker shard against
the resident panel and returns the hits: value = (markers x phenotypes over all ranks) /
(max over ranks of the device time of K steps). `e2e` times the same through
the host-buffer C-ABI path (raw panel upload + device prep + NCCL broadcast + pinned .bed rows
H2D inside the step; the panel enters raw (phenotypes + 10 covariates) and is
residualized, standardized and quantized on the device). Data are synthetic of the paper's shape (random-init
genotypes Binomial(2, AF), AF ~ U(0.05, 0.95); Gaussian phenotypes
standardized like the reference panel). Inputs (5.75 GB packed genotypes,
1.4 GB quantized panel) are far larger than the 126 MB L2.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
from concurrent.futures import ThreadPoolExecutor
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_COVARIATES = 10
METRIC = "association tests/sec (N=23k, P=20,480) at 1/2/4/8 B200; % bf16 tensor peak"


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--samples", type=int, default=23_000)
    ap.add_argument("--workload", choices=["c3", "c4"], default="c3",
                    help="c3: 1,000,000 markers in total; c4: 8,900,000 markers in total (paper headline)")
    ap.add_argument("--total-markers", type=int, default=None, help="markers in the whole job (strong scaling)")
    ap.add_argument("--markers-per-gpu", type=int, default=None, help="fixed shard per GPU (weak scaling)")
    ap.add_argument("--phenotypes", type=int, default=20_480)
    ap.add_argument("--p-threshold", type=float, default=1e-4)
    ap.add_argument("--device-batch", type=int, default=65_536)
    ap.add_argument("--cpu-sample", type=int, default=4096, help="markers in the timed CPU-baseline sample")
    ap.add_argument("--ref-workers", type=int, default=2, help="reference arm: engine worker threads")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--contexts", type=int, choices=[1, 2], default=2,
                    help="device contexts the batches alternate between (2: host work overlaps kernels)")
    ap.add_argument("--sync-panel", action="store_true",
                    help="A/B: e2e uploads + prepares the whole panel before the first scan")
    ap.add_argument("--panel-chunk", type=int, default=1280, help="phenotypes per pipelined panel chunk")
    ap.add_argument("--no-panel-shard", action="store_true",
                    help="A/B (N > 1): rank 0 prepares the whole panel and broadcasts it")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--missing-share", type=float, default=0.0,
                    help="share of markers with missing calls (C3 variants; default none)")
    ap.add_argument("--missing-rate", type=float, default=0.0, help="missing-call rate within those markers")
    ap.add_argument("--no-missing-side", action="store_true",
                    help="A/B: batches with missing calls take the two-row planes path")
    a = ap.parse_args()
    a.total = a.total_markers or (8_900_000 if a.workload == "c4" else 1_000_000)
    a.scaling = "weak" if a.markers_per_gpu else "strong"
    return a


def job_markers(a, world: int) -> int:
    return a.markers_per_gpu * world if a.markers_per_gpu else a.total


def rank_span(a, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of this rank's markers: contiguous 256-aligned shards of the job."""
    if a.markers_per_gpu:
        return rank * a.markers_per_gpu, (rank + 1) * a.markers_per_gpu
    from paper_2604_21095_b200.distributed import shard_span

    return shard_span(a.total, world, rank)


# --------------------------------------------------------------------------- helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_config(a, world: int) -> dict:
    total = job_markers(a, world)
    name = "C4" if total == 8_900_000 else "C3" if total == 1_000_000 * (world if a.markers_per_gpu else 1) else "custom"
    split = (f"{a.markers_per_gpu:,} markers per GPU" if a.markers_per_gpu
             else f"M={total:,} markers split over {world} GPU(s)")
    return {
        "workload": (f"{name}: synthetic PLINK .bed N={a.samples:,} x {split} x "
                     f"P={a.phenotypes:,} phenotypes, THRESHOLD p<={a.p_threshold:g} hit compaction"),
        "n_samples": a.samples,
        "n_markers_total": total,
        "n_markers_per_gpu": -(-total // world),
        "n_phenotypes": a.phenotypes,
        "p_threshold": a.p_threshold,
        "device_batch_markers": a.device_batch,
        "parallelism": f"marker shards x{world} (panel broadcast once over NCCL)",
        "l2_policy": "inputs larger than L2 (5.75 GB packed genotypes + 1.4 GB panel limbs per GPU per step)",
        "missing_calls": ({"marker_share": a.missing_share, "rate": a.missing_rate} if a.missing_share > 0
                          and a.missing_rate > 0 else None),
        "device_contexts": a.contexts,  # batches alternate between contexts driven by host threads
        "panel_upload": "synchronous" if a.sync_panel else f"pipelined ({a.panel_chunk}-phenotype chunks)",
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._thr = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thr.join(timeout=10)

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


# --------------------------------------------------------------------------- synthetic data (device, torch plumbing)
def synth_packed(torch, n_markers: int, n_samples: int, pitch: int, seed: int, device, miss_share: float = 0.0,
                 miss_rate: float = 0.0):
    """Packed .bed rows [M, pitch] uint8 on the device: G ~ Binomial(2, AF), AF ~ U(0.05, 0.95);
    a share `miss_share` of the markers has each call missing with probability `miss_rate`."""
    out = torch.zeros((n_markers, pitch), dtype=torch.uint8, device=device)
    gen = torch.Generator(device=device).manual_seed(seed)
    bpm = (n_samples + 3) // 4
    lut = torch.tensor([3, 2, 0], dtype=torch.uint8, device=device)  # dosage 0,1,2 -> code 11,10,00
    chunk = 8192
    for s in range(0, n_markers, chunk):
        e = min(n_markers, s + chunk)
        af = torch.rand(e - s, 1, generator=gen, device=device) * 0.9 + 0.05
        g = (torch.rand(e - s, n_samples, generator=gen, device=device) < af).to(torch.uint8)
        g += (torch.rand(e - s, n_samples, generator=gen, device=device) < af).to(torch.uint8)
        codes = lut[g.long()]
        if miss_share > 0 and miss_rate > 0:
            rows = torch.rand(e - s, 1, generator=gen, device=device) < miss_share
            miss = (torch.rand(e - s, n_samples, generator=gen, device=device) < miss_rate) & rows
            codes = torch.where(miss, torch.ones_like(codes), codes)  # code 01 = missing
        pad = bpm * 4 - n_samples
        if pad:
            codes = torch.nn.functional.pad(codes, (0, pad))
        q = codes.view(e - s, bpm, 4)
        out[s:e, :bpm] = q[:, :, 0] | (q[:, :, 1] << 2) | (q[:, :, 2] << 4) | (q[:, :, 3] << 6)
    return out


def synth_panel(torch, n_samples: int, n_pheno: int, seed: int, device):
    """Standardized panel Y~ [N, P] f64: centred (intercept-only residualization), unit 1/N variance."""
    gen = torch.Generator(device=device).manual_seed(seed + 1000)
    y = torch.randn(n_samples, n_pheno, generator=gen, device=device, dtype=torch.float64)
    y -= y.mean(dim=0, keepdim=True)
    y /= torch.sqrt((y * y).mean(dim=0, keepdim=True))
    return y


# --------------------------------------------------------------------------- reference arm
def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        return max(int(i.get("num_threads", 1)) for i in threadpool_info()) or 1
    except Exception:
        return os.cpu_count() or 1


def run_cpu_sample(packed_rows: np.ndarray, ytil: np.ndarray, n: int, p_thr: float) -> tuple[float, int]:
    """Fallback when oracle/_ref is absent: the oracle port on a bounded marker sample -> (seconds, hits)."""
    from oracle import scan_oracle as orc

    t0 = time.perf_counter()
    dos = orc.decode_bed(packed_rows, n)
    res = orc.threshold_scan(dos, ytil, float(n - 2), p_thr)
    return time.perf_counter() - t0, int(res["rows"].size)


def ref_loop_sample(a, n_markers: int, batch: int, workers: int):
    """The reference's own THRESHOLD scan loop (oracle/ref_scan_loop.py, panelgwas 0.1.0 from
    oracle/_ref) at N, P and p_threshold of the workload, over an n_markers .bed sample."""
    from oracle.ref_scan_loop import ReferenceScanLoop

    return ReferenceScanLoop(a.samples, a.phenotypes, n_markers, a.p_threshold, seed=a.seed, n_cov=N_COVARIATES,
                             batch_size=batch, workers=workers)


def reference_arm(a) -> None:
    """Reference CPU path on the host cores (rank 0 only; other ranks exit without work)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import ref_scan_loop

    n, p = a.samples, a.phenotypes
    # a bounded sample per step so that W + K steps end within a few minutes: 2 engine batches
    per_step = int(2 ** np.floor(np.log2(40_000 / max(1, a.steps + a.warmup))))
    per_step = max(1024, min(8192, per_step))
    if ref_scan_loop.available():
        loop = ref_loop_sample(a, per_step, per_step // 2, a.ref_workers)
        for _ in range(a.warmup):
            loop.step()
        steps = [loop.step() for _ in range(a.steps)]
        loop.close()
        total = sum(x["seconds"] for x in steps)
        kind, cores = "reference", ref_scan_loop.host_threads()
        sample = (f"{per_step} markers x {n} samples x {p} phenotypes per step through the reference's own "
                  f"scan loop (panelgwas 0.1.0 from oracle/_ref: PlinkSource.read_marker_batch -> "
                  f"engine._process_batch on {a.ref_workers} workers, batch {per_step // 2} -> ThresholdWriter); "
                  f"panel prep (build_covariate_basis/residualize/standardize_columns, 10 covariates) "
                  f"{loop.setup_s:.1f} s once, outside the steps; phenotype TSV parse not included")
        extra = {"setup_s": loop.setup_s, "records_per_step": steps[-1]["records"]}
    else:  # oracle/_ref not built (no /root/reference where build() ran): the numpy port
        rng = np.random.default_rng(a.seed)
        y = rng.standard_normal((n, p))
        y -= y.mean(axis=0)
        y /= np.sqrt((y * y).mean(axis=0))
        bpm = (n + 3) // 4
        g = rng.binomial(2, rng.uniform(0.05, 0.95, per_step)[:, None], size=(per_step, n))
        codes = np.array([3, 2, 0], dtype=np.uint8)[g]
        codes = np.pad(codes, ((0, 0), (0, bpm * 4 - n))).reshape(per_step, bpm, 4)
        packed = (codes[:, :, 0] | (codes[:, :, 1] << 2) | (codes[:, :, 2] << 4) | (codes[:, :, 3] << 6)).astype(np.uint8)
        for _ in range(a.warmup):
            run_cpu_sample(packed, y, n, a.p_threshold)
        total = sum(run_cpu_sample(packed, y, n, a.p_threshold)[0] for _ in range(a.steps))
        kind, cores = "port", cpu_threads()
        sample = f"{per_step} markers x {n} samples x {p} phenotypes per step (oracle/scan_oracle.py port)"
        extra = {}
    value = a.steps * per_step * p / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tests/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * total / a.steps, "higher_is_better": True,
        "scaling": a.scaling, "vs_baseline": None, "dtype": "f64 (f32 genotype store, reference default)",
        "data": "synthetic", "config": workload_config(a, world),
        "cpu_baseline": {"value": value, "unit": "tests/s", "cores": cores, "kind": kind, "sample": sample, **extra},
        "e2e": {"value": value, "unit": "tests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm
def our_arm(a) -> None:
    import torch
    import torch.distributed as dist

    from paper_2604_21095_b200 import _native, build as _build
    from paper_2604_21095_b200._device import DeviceContext
    from paper_2604_21095_b200.engine import threshold_premask
    from paper_2604_21095_b200.kernel import build_covariate_basis

    world, rank, local = dist_env()
    # test hooks (as distributed.py): several ranks on one GPU over gloo for a functional check
    backend = os.environ.get("PANELGWAS_DIST_BACKEND", "nccl")
    if os.environ.get("PANELGWAS_DIST_DEVICE"):
        local = int(os.environ["PANELGWAS_DIST_DEVICE"])
        os.environ["PANELGWAS_DEVICE"] = str(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _build.build()  # no-op when the in-tree .so is current
    n, p = a.samples, a.phenotypes
    span = rank_span(a, world, rank)
    m = span[1] - span[0]
    job = job_markers(a, world)
    bpm = (n + 3) // 4
    pitch = (bpm + 15) // 16 * 16
    df = float(n - 2)

    ctx = DeviceContext(local)
    if a.no_missing_side:
        ctx.set_missing_side_gemm(False)
    gidx = np.arange(n, dtype=np.int64)
    ytil = synth_panel(torch, n, p, a.seed, dev) if rank == 0 else None

    # e2e at N > 1: every rank uploads and prepares its share of the phenotype columns over its
    # own PCIe link and the quantized shares are all-gathered (instead of rank 0 preparing the
    # whole panel and broadcasting it)
    shard_panel = world > 1 and not a.sync_panel and not a.no_panel_shard and p % (256 * world) == 0
    panel_cols = (rank * p // world, (rank + 1) * p // world) if shard_panel else (0, p)

    def distribute_panel(raw_host=None):
        """rank 0 builds the resident panel; its limbs are broadcast once over NCCL; others import.

        raw_host = (Y [N, P], C [N, c]) host arrays: the public path (covariate basis on the
        host, residualize + standardize + quantize on the device). Y is page-locked, so the
        pipelined upload (pg_ctx_set_panel_async) is used: phenotype chunks are prepared as
        they land and the first batch's GEMM follows them chunk by chunk; the zero-variance
        flags are checked once the step's scans are done (panel_checked)."""
        if raw_host is not None and shard_panel:
            y_cols, c_raw = raw_host
            basis = build_covariate_basis(c_raw, True)
            c0, c1 = panel_cols
            ctx.set_panel_async_cols(y_cols, p, c0, basis.q, gidx, n, chunk_cols=a.panel_chunk)
            flat, _sd = ctx.panel_async_wait()
            wire = dev if backend == "nccl" else torch.device("cpu")
            bad = torch.tensor([int(flat.any())], device=wire, dtype=torch.int64)
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
            if int(bad.item()):
                raise RuntimeError("synthetic panel has zero-variance phenotypes")
            nb = ctx.panel_rows_bytes(c1 - c0)
            send = torch.empty(nb, dtype=torch.uint8, device=dev)
            ctx.export_panel_rows(send.data_ptr(), c0, c1)
            if wire == dev:
                recv = torch.empty(world * nb, dtype=torch.uint8, device=dev)
                dist.all_gather_into_tensor(recv, send)
                parts = [recv[r * nb:(r + 1) * nb] for r in range(world)]
            else:
                parts = [torch.empty(nb, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(parts, send.cpu())
                parts = [t.to(dev) for t in parts]
            torch.cuda.current_stream(dev).synchronize()  # the gather is done before the ctx's stream reads it
            for r in range(world):
                if r != rank:
                    ctx.import_panel_rows(parts[r].data_ptr(), r * p // world, (r + 1) * p // world)
            return (world - 1) * nb
        if rank == 0:
            if raw_host is not None:
                y_raw, c_raw = raw_host
                basis = build_covariate_basis(c_raw, True)
                if a.sync_panel:
                    flat, _sd = ctx.prepare_panel(y_raw, basis.q)
                    ctx.commit_panel(np.nonzero(~flat)[0], gidx, n)
                else:
                    ctx.set_panel_async(y_raw, basis.q, gidx, n, chunk_cols=a.panel_chunk)
            else:
                ctx.set_panel_device(ytil.data_ptr(), n, p, p, gidx, n)
        if world > 1:
            wire = dev if backend == "nccl" else torch.device("cpu")  # NCCL: device to device
            nbytes = ctx.panel_bytes() if rank == 0 else 0
            nb = torch.tensor([nbytes], device=wire, dtype=torch.int64)
            dist.broadcast(nb, 0)
            buf = torch.empty(int(nb.item()), dtype=torch.uint8, device=dev)
            if rank == 0:
                ctx.export_panel(buf.data_ptr())
            wbuf = buf if wire == dev else buf.cpu()
            dist.broadcast(wbuf, 0)
            if rank != 0:
                if wbuf is not buf:
                    buf.copy_(wbuf)
                torch.cuda.current_stream(dev).synchronize()  # broadcast / copy done before the ctx's stream reads buf
                ctx.import_panel(buf.data_ptr(), n, p, gidx, n)
            return int(nb.item())
        return 0

    distribute_panel(None)
    rbar = np.full(p, threshold_premask(a.p_threshold, df))
    ctx.set_scan(df, _native.PG_MODE_THRESHOLD, rbar)
    packed = synth_packed(torch, m, n, pitch, a.seed * 7919 + rank, dev, a.missing_share, a.missing_rate)
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream_handle(), device=dev)
    batches = [(s, min(a.device_batch, m - s)) for s in range(0, m, a.device_batch)]

    # Two contexts (default): batches alternate between two DeviceContexts driven by two host
    # threads (the C ABI releases the GIL), so one context's host work between batches (result
    # fetch, candidate-count round trips) overlaps the other's kernels; the second context
    # imports the first one's panel (device to device).
    ctx2 = stream2 = None
    pool = None
    if a.contexts == 2:
        ctx2 = DeviceContext(local)
        if a.no_missing_side:
            ctx2.set_missing_side_gemm(False)
        pbuf = torch.empty(ctx.panel_bytes(), dtype=torch.uint8, device=dev)
        ctx.export_panel(pbuf.data_ptr())
        torch.cuda.synchronize()
        ctx2.import_panel(pbuf.data_ptr(), n, p, gidx, n)
        ctx2.set_scan(df, _native.PG_MODE_THRESHOLD, rbar)
        del pbuf
        stream2 = torch.cuda.ExternalStream(ctx2.stream_handle(), device=dev)
        pool = ThreadPoolExecutor(max_workers=2)

    def alternate(work, items):
        """work(ctx, k, item) for every item: item i on context i % 2 (or all on ctx)."""
        if ctx2 is None:
            return [work(ctx, 0, it) for it in items]
        out = [None] * len(items)

        def lane(k):
            for i in range(k, len(items), 2):
                out[i] = work((ctx, ctx2)[k], k, items[i])

        for f in [pool.submit(lane, 0), pool.submit(lane, 1)]:
            f.result()
        return out

    def scan_step_device():
        stats = {"gemm_ms": 0.0, "hits": 0, "launches": 0, "d2h": 0}

        def one(cx, _k, sc):
            s, c = sc
            r = cx.scan_device(_native.PG_GENO_BED, packed.data_ptr() + s * pitch, c, bpm, pitch)
            return r.gemm_ms, int(np.count_nonzero(r.cand_p <= a.p_threshold)), r.launches, r.cand_rows.size * 40 + c * 25

        for g, h, ln, d in alternate(one, batches):
            stats["gemm_ms"] += g
            stats["hits"] += h
            stats["launches"] += ln
            stats["d2h"] += d
        return stats

    def timed(fn, steps):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        out = [fn() for _ in range(steps)]
        if stream2 is not None:
            stream.wait_stream(stream2)  # the end event follows both contexts' work
        ev1.record(stream)
        ev1.synchronize()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, out

    for _ in range(a.warmup):
        scan_step_device()
    with ClockSampler(local) as clk:
        ms, outs = timed(scan_step_device, a.steps)
    tests_per_step = job * p  # the whole job (all ranks); ms is the max over ranks
    value = tests_per_step * a.steps / (ms / 1e3)
    gemm_ms = sum(o["gemm_ms"] for o in outs)
    launches = sum(o["launches"] for o in outs)
    hits = outs[-1]["hits"]
    if ctx2 is not None:
        # with two contexts a GEMM's event span can include waiting for the other context's
        # GEMM to leave the SMs: the kernel's own duration (roofline) comes from the same
        # steps run on one context
        gemm_ms = 0.0
        for _ in range(a.steps):
            for s0, c0 in batches:
                gemm_ms += ctx.scan_device(_native.PG_GENO_BED, packed.data_ptr() + s0 * pitch, c0, bpm, pitch,
                                           fetch=False).gemm_ms

    # roofline of the dominant kernel (assoc_i8_kernel): BASELINE accounting 2*N*M*P x2 (hi/lo) = 4*N*M*P
    flops = 4.0 * n * m * p * a.steps
    achieved = flops / (gemm_ms / 1e3) / 1e12
    peaks = measured_peaks()
    peak = float(peaks.get("bf16_tflops", 1590.0))
    peak_sus = float(peaks.get("bf16_tflops_sustained", 1400.0))
    traffic = None
    tf = ROOT / "profiles" / "assoc_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("bytes_per_launch")
        except Exception:
            traffic = None
    # hardware view: the kernel issues 3 int8 MMAs (limbs) per padded sample, exact int32 accumulation
    k_pad = (n + 63) // 64 * 64
    # THRESHOLD scans of PLINK rows run two of the three panel limbs (the third is added to the
    # candidates exactly, csrc/assoc_gemm.cu refine_two_limb); PG_TWO_LIMB=0 runs all three
    limbs = 3 if os.environ.get("PG_TWO_LIMB", "1") == "0" else 2
    int8_ops = 2.0 * limbs * k_pad * m * ((p + 127) // 128 * 128) * a.steps
    int8_achieved = int8_ops / (gemm_ms / 1e3) / 1e12
    int8_peak = None
    try:
        A = torch.randint(-128, 127, (8192, 8192), device=dev, dtype=torch.int8)
        B = torch.randint(-128, 127, (8192, 8192), device=dev, dtype=torch.int8)
        best = 1e9
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(A, B.t())
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        int8_peak = 2 * 8192**3 / (best / 1e3) / 1e12
        del A, B
    except Exception:
        pass

    # HBM roofline of the decode stage: K1 statistics kernel alone over the whole shard
    # (reads ceil(N/4) bytes per marker, writes 56 B of per-marker stats)
    # (the GPU leaves the GEMM power-capped: one untimed pass lets the clocks settle first)
    ctx.time_marker_stats(_native.PG_GENO_BED, packed.data_ptr(), m, pitch, reps=3)
    k1_ms = ctx.time_marker_stats(_native.PG_GENO_BED, packed.data_ptr(), m, pitch, reps=10)
    k1_bytes = m * (bpm + 56)
    hbm_peak = float(peaks.get("hbm_gbs", 6548.8))
    decode_hbm = {"kernel": "stats_kernel", "achieved": k1_bytes / (k1_ms / 1e3) / 1e9, "peak": hbm_peak,
                  "unit": "GB/s", "frac": k1_bytes / (k1_ms / 1e3) / 1e9 / hbm_peak, "ms": k1_ms,
                  "bytes_def": "ceil(N/4) packed bytes read + 56 B stats written per marker",
                  "peak_source": "MEASURED_PEAKS.json hbm_gbs"}

    # ------------------------------------------------ end to end through the host-buffer C ABI
    e2e = None
    if not a.no_e2e:
        host_rows = torch.empty((m, bpm), dtype=torch.uint8, pin_memory=True)
        host_rows.copy_(packed[:, :bpm])
        host_np = host_rows.numpy()
        raw = None
        if rank == 0 or shard_panel:
            # raw phenotypes of the C3 shape: Y = C gamma + noise, 10 covariates,
            # each 256-phenotype block from its own generator so that a rank can make just its
            # share (the sharded panel preparation) and every sharding sees the same matrix
            gen = torch.Generator(device=dev).manual_seed(a.seed + 2000)
            c_dev = torch.randn(n, N_COVARIATES, generator=gen, device=dev, dtype=torch.float64)
            c0, c1 = panel_cols
            yh = torch.empty((n, c1 - c0), dtype=torch.float64, pin_memory=True)
            for b0 in range(c0, c1, 256):
                w = min(256, c1 - b0)
                gb = torch.Generator(device=dev).manual_seed(a.seed + 2001 + b0 // 256)
                gamma = 0.1 * torch.randn(N_COVARIATES, w, generator=gb, device=dev, dtype=torch.float64)
                yh[:, b0 - c0:b0 - c0 + w].copy_(c_dev @ gamma + torch.randn(n, w, generator=gb, device=dev,
                                                                             dtype=torch.float64))
            raw = (yh.numpy(), c_dev.cpu().numpy())
            del c_dev
        del packed
        torch.cuda.empty_cache()

        pbuf2 = torch.empty(ctx.panel_bytes(), dtype=torch.uint8, device=dev) if ctx2 is not None else None

        panel_ready = threading.Event()
        # one GPU, pipelined panel: the second context follows the first one's panel chunk by
        # chunk (pg_ctx_follow_panel), so both contexts' first batches run behind the upload;
        # otherwise it takes the finished panel from the first context after its first batch
        follow = ctx2 is not None and world == 1 and not a.sync_panel

        def e2e_lane(cx, k, items):
            """One context's share of the step: the host-buffer C-ABI path, pipelined (the H2D
            of its next batch overlaps the scan of its current one). With two contexts the
            first exports the step's panel right after its first batch (the pipelined panel
            is complete by then) and the second imports it (device to device)."""
            h2d = d2h = hits = 0

            def hand_over():
                if k == 0 and ctx2 is not None and not follow and not panel_ready.is_set():
                    ctx.export_panel(pbuf2.data_ptr())
                    panel_ready.set()

            for j, (s, c) in enumerate(items):
                cx.stage(j % 2, _native.PG_GENO_BED, host_np[s:s + c], bpm)
                h2d += c * bpm
                if j == 0 and k == 1 and not follow:
                    panel_ready.wait()
                    cx.import_panel(pbuf2.data_ptr(), n, p, gidx, n)
                    cx.set_scan(df, _native.PG_MODE_THRESHOLD, rbar)
                if j:
                    r = cx.scan_staged((j - 1) % 2)
                    d2h += r.cand_rows.size * 40 + r.n_markers * 25
                    hits += int(np.count_nonzero(r.cand_p <= a.p_threshold))
                    hand_over()
            if items:
                r = cx.scan_staged((len(items) - 1) % 2)
                d2h += r.cand_rows.size * 40 + r.n_markers * 25
                hits += int(np.count_nonzero(r.cand_p <= a.p_threshold))
            hand_over()
            return h2d, d2h, hits

        def e2e_step():
            moved = distribute_panel(raw)
            if shard_panel:  # this rank's share of Y and C (the shares' limbs move over NVLink)
                h2d = n * (panel_cols[1] - panel_cols[0] + N_COVARIATES + 1) * 8
            else:
                h2d = moved + (n * (p + N_COVARIATES + 1) * 8 if rank == 0 else 0)
            ctx.set_scan(df, _native.PG_MODE_THRESHOLD, rbar)
            if follow:
                ctx2.follow_panel(ctx)
                ctx2.set_scan(df, _native.PG_MODE_THRESHOLD, rbar)
            d2h = hits = 0
            if ctx2 is None:
                h, d, t = e2e_lane(ctx, 0, batches)
                h2d, d2h, hits = h2d + h, d2h + d, hits + t
            else:
                panel_ready.clear()
                futs = [pool.submit(e2e_lane, (ctx, ctx2)[k], k, batches[k::2]) for k in range(2)]
                for f in futs:
                    h, d, t = f.result()
                    h2d, d2h, hits = h2d + h, d2h + d, hits + t
            if (rank == 0 or shard_panel) and not a.sync_panel:
                flat, _sd = ctx.panel_async_wait()  # (complete long ago: no wait)
                if flat.any():
                    raise RuntimeError("synthetic panel has zero-variance phenotypes")
            return h2d, d2h, hits

        e2e_step()
        ms_e2e, outs_e2e = timed(e2e_step, a.steps)
        e2e_hits = outs_e2e[-1][2]
        if world > 1:  # every rank's hits (the job's)
            wire = dev if backend == "nccl" else torch.device("cpu")
            t = torch.tensor([e2e_hits], device=wire, dtype=torch.int64)
            dist.all_reduce(t)
            e2e_hits = int(t.item())
        e2e = {"value": tests_per_step * a.steps / (ms_e2e / 1e3), "unit": "tests/s",
               "h2d_bytes_per_step": int(outs_e2e[-1][0]), "d2h_bytes_per_step": int(outs_e2e[-1][1]),
               "ms_per_step": ms_e2e / a.steps, "hits_per_step": e2e_hits,
               "panel": ("sharded over ranks" if shard_panel else "rank 0" if world > 1 else "one GPU")}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        from oracle import ref_scan_loop

        sample = max(256, min(a.cpu_sample, m))
        if ref_scan_loop.available():
            loop = ref_loop_sample(a, sample, sample // 2, a.ref_workers)
            sec = loop.step()["seconds"]
            cpu = {"value": sample * p / sec, "unit": "tests/s", "cores": ref_scan_loop.host_threads(),
                   "kind": "reference",
                   "sample": f"{sample} markers x {n} samples x {p} phenotypes through the reference's own scan loop "
                             f"(panelgwas 0.1.0 from oracle/_ref, {a.ref_workers} engine workers, batch "
                             f"{sample // 2}) in {sec:.1f} s; its panel prep ({loop.setup_s:.1f} s) not counted"}
            loop.close()
        else:
            rows_np = synth_packed(torch, sample, n, pitch, a.seed * 7919 + 17, dev)[:, :bpm].cpu().numpy()
            y_np = ytil.cpu().numpy()
            sec, _ = run_cpu_sample(rows_np, y_np, n, a.p_threshold)
            cpu = {"value": sample * p / sec, "unit": "tests/s", "cores": cpu_threads(), "kind": "port",
                   "sample": f"{sample} markers x {n} samples x {p} phenotypes, one pass of oracle/scan_oracle.py "
                             f"(numpy restatement of the reference path) in {sec:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tests/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": a.scaling,
            "vs_baseline": None, "dtype": "int8 (exact int32 accumulate; fp64 epilogue)", "data": "synthetic",
            "config": workload_config(a, world),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "frac_of_sustained": achieved / peak_sus, "traffic": traffic,
                         "kernel": "assoc_i8_kernel",
                         "flops_def": "BASELINE: 2*N*M*P x2 (hi/lo) = 4*N*M*P per launch, N = kept samples",
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)"},
            "hw_int8": {"achieved_tops": int8_achieved, "cublas_int8_tops_measured": int8_peak,
                        "frac": (int8_achieved / int8_peak) if int8_peak else None,
                        "ops_def": f"2 * {limbs} limbs * K_pad * M * P_pad per launch"},
            "decode_hbm": decode_hbm,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "hits_per_step": hits,
            "gemm_ms_per_step": gemm_ms / a.steps,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse_args()
    if a.impl == "reference":
        reference_arm(a)
    else:
        our_arm(a)


if __name__ == "__main__":
    main()

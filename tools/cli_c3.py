#!/usr/bin/env python
"""End-to-end C3 through the drop-in CLI (`panelgwas run`), on files.

Writes a synthetic PLINK trio (N samples x M markers, Binomial(2, AF), AF ~ U(0.05, 0.95)),
a phenotype TSV (P columns, Python-repr floats) and a covariate TSV (10 columns) under
--dir, then times `python -m paper_2604_21095_b200 run --bfile ... --pheno ... --covar ...
--p-threshold 1e-4 --out ...` as a subprocess (wall clock, page cache warm after writing),
and prints one JSON line with the run's own summary timings.

  python tools/cli_c3.py --dir /tmp/c3 [--markers 1000000 --phenotypes 20480]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def write_repr_tsv(path: Path, ids: list[str], names: list[str], values: np.ndarray) -> None:
    """Rows 'ID<TAB>v1<TAB>...' with repr() floats, formatted by the native emitter."""
    from paper_2604_21095_b200 import _native

    with open(path, "wb") as fh:
        fh.write(("IID\t" + "\t".join(names) + "\n").encode())
        p = values.shape[1]
        cap = p * 40
        out = ctypes.create_string_buffer(cap)
        ln = ctypes.c_int64(0)
        for i, sid in enumerate(ids):
            row = np.ascontiguousarray(values[i], dtype=np.float64)
            _native.call("pg_format_float_repr", row.ctypes.data, p, out, cap, ctypes.byref(ln))
            fh.write(sid.encode() + b"\t" + out.raw[:ln.value - 1].replace(b"\n", b"\t") + b"\n")


def write_bed(prefix: Path, n: int, m: int, seed: int) -> None:
    """Binomial(2, AF) genotypes, AF ~ U(0.05, 0.95); drawn on the GPU (bench.synth_packed)."""
    import torch

    from bench import synth_packed

    bpm = (n + 3) // 4
    with open(f"{prefix}.bed", "wb") as fh:
        fh.write(bytes([0x6C, 0x1B, 0x01]))
        step = 65536
        for s in range(0, m, step):
            c = min(step, m - s)
            rows = synth_packed(torch, c, n, bpm, seed * 7919 + s, torch.device("cuda", 0))
            fh.write(rows.cpu().numpy().tobytes())
    with open(f"{prefix}.bim", "w") as fh:
        fh.writelines(f"1\trs{i + 1}\t0\t{i + 1}\tA\tG\n" for i in range(m))
    with open(f"{prefix}.fam", "w") as fh:
        fh.writelines(f"F{i + 1}\tS{i + 1}\t0\t0\t0\t-9\n" for i in range(n))


def write_inputs(d: Path, n: int, p: int, a) -> None:
    ids = [f"S{i + 1}" for i in range(n)]
    write_bed(d / "geno", n, a.markers, a.seed)
    rng = np.random.default_rng(a.seed + 1)
    c = rng.standard_normal((n, a.covariates))
    y = c @ (0.1 * rng.standard_normal((a.covariates, p))) + rng.standard_normal((n, p))
    write_repr_tsv(d / "covar.tsv", ids, [f"c{j + 1}" for j in range(a.covariates)], c)
    write_repr_tsv(d / "pheno.tsv", ids, [f"ph{j + 1}" for j in range(p)], y)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default="/tmp/c3")
    ap.add_argument("--samples", type=int, default=23_000)
    ap.add_argument("--markers", type=int, default=1_000_000)
    ap.add_argument("--phenotypes", type=int, default=20_480)
    ap.add_argument("--covariates", type=int, default=10)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--top-k", type=int, default=0, help="TOPK mode with this k instead of THRESHOLD p <= 1e-4")
    ap.add_argument("--full", action="store_true", help="FULL mode (f32 t matrix) instead of THRESHOLD")
    ap.add_argument("--reuse", action="store_true", help="keep the input files of a previous run in --dir")
    ap.add_argument("--extra", default="", help="extra CLI flags for `panelgwas run` (space-separated)")
    a = ap.parse_args()
    d = Path(a.dir)
    d.mkdir(parents=True, exist_ok=True)
    n, p = a.samples, a.phenotypes
    t0 = time.perf_counter()
    if not (a.reuse and (d / "geno.bed").exists() and (d / "pheno.tsv").exists()):
        write_inputs(d, n, p, a)
    t_write = time.perf_counter() - t0
    sizes = {f: os.path.getsize(d / f) for f in ("geno.bed", "pheno.tsv", "covar.tsv")}
    cmd = [sys.executable, "-m", "paper_2604_21095_b200", "run", "--bfile", str(d / "geno"), "--pheno",
           str(d / "pheno.tsv"), "--covar", str(d / "covar.tsv"),
           *(["--full", "--allow-large-full"] if a.full else ["--top-k", str(a.top_k)] if a.top_k
             else ["--p-threshold", "1e-4"]), *a.extra.split(), "--out", str(d / "hits.tsv")]
    for old in d.glob("hits.tsv*"):  # a rewrite of an existing file costs extra (truncate + flush on close)
        old.unlink()
    t0 = time.perf_counter()
    res = subprocess.run(cmd, capture_output=True, text=True, cwd=str(ROOT),
                         env={**os.environ, "PANELGWAS_PROFILE": "1"})
    wall = time.perf_counter() - t0
    if res.returncode != 0:
        print(res.stdout[-2000:], res.stderr[-4000:])
        raise SystemExit(res.returncode)
    summary = json.loads((d / "hits.tsv.summary.json").read_text())
    tests = summary["markers_scanned"] * summary["phenotypes_scanned"]
    mode = ("FULL f32" if a.full else f"TOPK k={a.top_k}" if a.top_k else "p<=1e-4") + (f" {a.extra}" if a.extra else "")
    line = {"workload": f"C3 via CLI: N={n:,} M={a.markers:,} P={p:,} + {a.covariates} covariates, {mode}",
            "wall_s": wall, "tests": tests, "tests_per_s_wall": tests / wall, "records": summary["records_emitted"],
            "file_bytes": {**sizes, "out": os.path.getsize(d / "hits.tsv")}, "write_inputs_s": t_write,
            "summary_times": {k: summary[k] for k in summary if k.startswith("time_") or k == "wall_s"},
            "phases": next((json.loads(ln)["panelgwas_phases_s"] for ln in res.stderr.splitlines()
                            if ln.startswith('{"panelgwas_phases_s"')), None)}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

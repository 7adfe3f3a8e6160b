#!/usr/bin/env python
"""End-to-end C5 through the drop-in CLI (`panelgwas run --bgen`), on files.

Writes a BGEN v1.2 file (layout 2, zlib, 8-bit probabilities, embedded sample IDs) of
N samples x M variants -- `--distinct` distinct compressed genotype blocks (Binomial(2, AF)
calls, 20 % made fractional, 5 % missing: tools/bench_workloads.bgen_rows) cycled over the M
variants, each with its own identifiers and position -- plus a phenotype TSV (P columns), then
times `python -m paper_2604_21095_b200 run --bgen ... --pheno ... --p-threshold 1e-4` as a
subprocess (wall clock, page cache warm after writing) and prints one JSON line with the
run's own phase timings.

  python tools/cli_c5.py --dir /tmp/c5 [--markers 1000000 --phenotypes 4096]
"""
from __future__ import annotations

import argparse
import json
import os
import struct
import subprocess
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))


def _blocks(args):
    from bench_workloads import bgen_rows

    seed, count, n = args
    _, blocks = bgen_rows(np.random.default_rng(seed), count, n)
    return blocks


def write_bgen(path: Path, n: int, m: int, distinct: int, seed: int) -> None:
    ids = b"".join(struct.pack("<H", len(s)) + s for s in (f"S{i + 1}".encode() for i in range(n)))
    sample_block = struct.pack("<II", 8 + len(ids), n) + ids
    flags = 1 | (2 << 2) | (1 << 31)  # zlib, layout 2, sample identifiers present
    workers = min(16, os.cpu_count() or 4)
    per = -(-distinct // workers)
    with ProcessPoolExecutor(workers) as ex:
        parts = list(ex.map(_blocks, [(seed + w, min(per, distinct - w * per), n) for w in range(workers)
                                      if distinct - w * per > 0]))
    blocks = [b for part in parts for b in part]
    with open(path, "wb") as fh:
        fh.write(struct.pack("<I", 20 + len(sample_block)))  # first variant, relative to byte 4
        fh.write(struct.pack("<III", 20, m, n) + b"bgen" + struct.pack("<I", flags))
        fh.write(sample_block)
        chunk = []
        for v in range(m):
            name = f"rs{v + 1}".encode()
            blk = blocks[v % len(blocks)]
            chunk.append(struct.pack("<H", len(name)) + name + struct.pack("<H", len(name)) + name
                         + struct.pack("<H", 1) + b"1" + struct.pack("<IH", v + 1, 2)
                         + struct.pack("<I", 1) + b"A" + struct.pack("<I", 1) + b"G"
                         + struct.pack("<I", len(blk)) + blk)
            if len(chunk) == 4096:
                fh.write(b"".join(chunk))
                chunk = []
        fh.write(b"".join(chunk))


def main():
    from cli_c3 import write_repr_tsv

    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default="/tmp/c5")
    ap.add_argument("--samples", type=int, default=23_000)
    ap.add_argument("--markers", type=int, default=1_000_000)
    ap.add_argument("--phenotypes", type=int, default=4_096)
    ap.add_argument("--distinct", type=int, default=8192)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--reuse", action="store_true", help="keep the input files of a previous run in --dir")
    ap.add_argument("--extra", default="", help="extra CLI flags for `panelgwas run` (space-separated)")
    a = ap.parse_args()
    d = Path(a.dir)
    d.mkdir(parents=True, exist_ok=True)
    n, p = a.samples, a.phenotypes
    t0 = time.perf_counter()
    if not (a.reuse and (d / "geno.bgen").exists() and (d / "pheno.tsv").exists()):
        write_bgen(d / "geno.bgen", n, a.markers, a.distinct, a.seed)
        rng = np.random.default_rng(a.seed + 1)
        write_repr_tsv(d / "pheno.tsv", [f"S{i + 1}" for i in range(n)], [f"ph{j + 1}" for j in range(p)],
                       rng.standard_normal((n, p)))
    t_write = time.perf_counter() - t0
    for old in d.glob("hits.tsv*"):
        old.unlink()
    cmd = [sys.executable, "-m", "paper_2604_21095_b200", "run", "--bgen", str(d / "geno.bgen"), "--pheno",
           str(d / "pheno.tsv"), "--p-threshold", "1e-4", *a.extra.split(), "--out", str(d / "hits.tsv")]
    t0 = time.perf_counter()
    res = subprocess.run(cmd, capture_output=True, text=True, cwd=str(ROOT), env={**os.environ, "PANELGWAS_PROFILE": "1"})
    wall = time.perf_counter() - t0
    if res.returncode != 0:
        print(res.stdout[-2000:], res.stderr[-4000:])
        raise SystemExit(res.returncode)
    summary = json.loads((d / "hits.tsv.summary.json").read_text())
    tests = summary["markers_scanned"] * summary["phenotypes_scanned"]
    line = {"workload": f"C5 via CLI: BGEN-8 N={n:,} M={a.markers:,} ({a.distinct} distinct blocks, 5 % missing, "
                        f"20 % fractional) P={p:,}, p<=1e-4",
            "wall_s": wall, "tests": tests, "tests_per_s_wall": tests / wall, "records": summary["records_emitted"],
            "file_bytes": {f: os.path.getsize(d / f) for f in ("geno.bgen", "pheno.tsv", "hits.tsv")},
            "write_inputs_s": t_write,
            "summary_times": {k: summary[k] for k in summary if k.startswith("time_") or k == "wall_s"},
            "phases": next((json.loads(ln)["panelgwas_phases_s"] for ln in res.stderr.splitlines()
                            if ln.startswith('{"panelgwas_phases_s"')), None)}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

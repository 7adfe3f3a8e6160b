"""The multi-GPU driver end to end (distributed.run_scan_distributed): two ranks launched as
separate processes, marker shards, rank 0 parses the tables and broadcasts the metadata and
the quantized panel, shard outputs merged by rank 0 == the single-process scan, byte for
byte (THRESHOLD, TOPK, FULL + min-p sidecar). On the one-GPU test box both ranks share
device 0 over gloo (host collectives; no kernel waits on another rank)."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from conftest_helpers import write_tsv

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dataset(tmp_path):
    rng = np.random.default_rng(77)
    n, m, p = 90, 700, 5
    ids = [f"S{i + 1}" for i in range(n)]
    d = rng.binomial(2, rng.uniform(0.1, 0.9, (m, 1)), size=(m, n)).astype(np.float64)
    d[rng.random(d.shape) < 0.02] = np.nan
    y = rng.standard_normal((n, p))
    y[:, 1] += 0.8 * np.nan_to_num(d[300], nan=1.0)
    bed, bim, fam = pg.write_bed_trio(tmp_path / "g", d, ids)
    write_tsv(tmp_path / "p.tsv", ids, [f"ph{j}" for j in range(p)], y)
    write_tsv(tmp_path / "c.tsv", ids, ["c1"], rng.standard_normal((n, 1)))
    return tmp_path / "g"


@pytest.mark.parametrize("mode", [["--p-threshold", "0.05"], ["--top-k", "3"], ["--full", "--precision", "f64"]])
def test_two_rank_driver_equals_single_process(tmp_path, mode):
    prefix = _dataset(tmp_path)
    args = ["--bfile", str(prefix), "--pheno", str(tmp_path / "p.tsv"), "--covar", str(tmp_path / "c.tsv"),
            "--batch-size", "64", "--min-p-sidecar", *mode]
    single = tmp_path / "single.out"
    subprocess.run([sys.executable, "-m", "paper_2604_21095_b200", "run", *args, "--out", str(single)], check=True,
                   cwd=ROOT, capture_output=True)
    multi = tmp_path / "multi.out"
    env = {**os.environ, "PANELGWAS_DIST_BACKEND": "gloo", "PANELGWAS_DIST_DEVICE": "0"}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "-m", "paper_2604_21095_b200.distributed",
           *args, "--out", str(multi)]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    if res.returncode != 0:
        rank1 = "\n".join(ln for ln in res.stderr.splitlines() if "[rank1]" in ln)
        raise AssertionError((rank1 or res.stderr)[-6000:])
    assert multi.read_bytes() == single.read_bytes()
    assert Path(f"{multi}.minp.tsv").read_bytes() == Path(f"{single}.minp.tsv").read_bytes()
    if "--full" in mode:
        for suffix in (".markers.tsv", ".phenotypes.txt"):
            assert Path(f"{multi}{suffix}").read_bytes() == Path(f"{single}{suffix}").read_bytes()
    assert not list(tmp_path.glob("multi.out.rank*"))  # shard files cleaned up


@pytest.mark.parametrize("shape", [["--total-markers", "12800"], ["--markers-per-gpu", "8192"]])
def test_bench_two_ranks_functional(shape):
    """bench.py under torchrun with 2 ranks (functional check of the multi-GPU bench path on
    one GPU over gloo: panel broadcast, max-over-ranks timing, one JSON line from rank 0),
    strong (a fixed job split into 256-aligned shards) and weak (a fixed shard per rank)."""
    import json

    env = {**os.environ, "PANELGWAS_DIST_BACKEND": "gloo", "PANELGWAS_DIST_DEVICE": "0"}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           *shape, "--phenotypes", "512", "--samples", "2000", "--steps", "3", "--warmup", "3",
           "--device-batch", "4096"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-4000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["cpu_baseline"] is None
    strong = shape[0] == "--total-markers"
    assert d["scaling"] == ("strong" if strong else "weak")
    assert d["config"]["n_markers_total"] == (12800 if strong else 16384)
    # value counts every rank's tests once: (job markers x P x K) / max-over-ranks time
    assert abs(d["value"] * d["ms_per_step"] / 1e3 - d["config"]["n_markers_total"] * 512) < 1e-3 * d["value"]


def test_bench_two_ranks_sharded_panel_equals_broadcast():
    """e2e at N > 1: each rank prepares its share of the phenotype columns and the quantized
    shares are all-gathered (pg_ctx_set_panel_async_cols / export / import_panel_rows) — the
    scans find exactly the hits of the rank-0-prepared, broadcast panel."""
    import json

    env = {**os.environ, "PANELGWAS_DIST_BACKEND": "gloo", "PANELGWAS_DIST_DEVICE": "0"}
    out = {}
    for flag in ([], ["--no-panel-shard"]):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
               "--total-markers", "12800", "--phenotypes", "512", "--samples", "2000", "--steps", "3",
               "--warmup", "3", "--device-batch", "4096", "--p-threshold", "0.01", "--no-cpu-baseline", *flag]
        res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-4000:]
        d = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][0])
        out[tuple(flag)] = d["e2e"]
    assert out[()]["panel"] == "sharded over ranks" and out[("--no-panel-shard",)]["panel"] == "rank 0"
    assert out[()]["hits_per_step"] == out[("--no-panel-shard",)]["hits_per_step"] > 0


@pytest.mark.parametrize("f64", [False, True])
def test_nccl_panel_broadcast_round_trip(f64):
    """The NCCL data plane of the multi-GPU scan on this box's one GPU: a one-rank NCCL group
    broadcasts the exported device panel (incl. the F64 panel's lo level), a second context
    imports it after syncing torch's stream (distributed.broadcast_panel), and its scans equal
    the exporting context's bit for bit (THRESHOLD two-limb and FULL)."""
    import torch
    import torch.distributed as dist

    from oracle import scan_oracle as orc
    from paper_2604_21095_b200 import _native
    from paper_2604_21095_b200._device import DeviceContext
    from paper_2604_21095_b200.distributed import broadcast_bytes

    rng = np.random.default_rng(4)
    n, m, p = 300, 500, 40
    d = rng.binomial(2, rng.uniform(0.1, 0.9, m)[:, None], size=(m, n)).astype(np.float64)
    d[rng.random((m, n)) < 0.02] = np.nan
    codes = np.where(np.isnan(d), 1, np.select([d == 2, d == 1, d == 0], [0, 2, 3])).astype(np.uint8)
    bpm = (n + 3) // 4
    q = codes.reshape(m, bpm, 4)
    packed = (q[:, :, 0] | (q[:, :, 1] << 2) | (q[:, :, 2] << 4) | (q[:, :, 3] << 6)).astype(np.uint8)
    ytil, _ = orc.standardized_panel(rng.standard_normal((n, p)), orc.covariate_basis(np.zeros((n, 0))))
    gidx = np.arange(n, dtype=np.int64)
    df = float(n - 2)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1, device_id=dev)
    try:
        with DeviceContext(0) as a, DeviceContext(0) as b:
            for c in (a, b):
                c.set_f64_panel(f64)
            a.set_panel(ytil, gidx, n)
            buf = torch.empty(a.panel_bytes(), dtype=torch.uint8, device=dev)
            a.export_panel(buf.data_ptr())
            buf = broadcast_bytes(torch, dist, buf, buf.numel(), 0, dev)
            torch.cuda.current_stream(dev).synchronize()
            b.import_panel(buf.data_ptr(), n, p, gidx, n)
            out = []
            for c in (a, b):
                c.set_scan(df, _native.PG_MODE_THRESHOLD, np.full(p, orc.premask_abs_r(0.05, df)))
                t = c.scan(_native.PG_GENO_BED, packed, bpm)
                c.set_scan(df, _native.PG_MODE_FULL, None)
                f = c.scan(_native.PG_GENO_BED, packed, bpm)
                out.append((t.cand_rows, t.cand_cols, t.cand_t, t.cand_p, f.t_rows))
        for x, y in zip(*out):
            assert np.array_equal(x, y)
    finally:
        dist.destroy_process_group()

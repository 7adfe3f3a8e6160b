"""Multi-GPU host logic on CPU: marker sharding, the panel-byte broadcast protocol
(world_size 2 over gloo), and rank-order merging of shard outputs (THRESHOLD,
TOPK, FULL) == the single-process output."""
import os
import socket
from pathlib import Path

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from paper_2604_21095_b200 import distributed, output


def test_shard_span_covers_and_aligns():
    for n in (1, 255, 256, 1000, 1_000_000):
        for world in (1, 2, 3, 4, 8):
            spans = [distributed.shard_span(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            for a, b in spans[:-1]:
                assert a % 256 == 0 and b % 256 == 0 or b == n
    with pytest.raises(ValueError):
        distributed.shard_span(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, payload_path, result_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    payload = np.load(payload_path)
    buf = torch.from_numpy(payload.copy()) if rank == 0 else None
    got = distributed.broadcast_bytes(torch, dist, buf, payload.size if rank == 0 else None, 0)
    np.save(Path(result_dir) / f"r{rank}.npy", got.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_panel_bytes_broadcast_gloo(tmp_path):
    import torch.multiprocessing as mp

    payload = np.random.default_rng(0).integers(0, 256, size=12345, dtype=np.uint8)
    np.save(tmp_path / "payload.npy", payload)
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path / "payload.npy"), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"r{r}.npy"), payload)


def _markers(n):
    return [pg.MarkerRecord("1", f"snp{i + 1}", i + 1, "A", "B", i) for i in range(n)]


def _stats(markers, rows, cols, t, p):
    m = len(markers)
    return output.BatchStats(markers=tuple(markers), allele_frequency=np.full(m, 0.3),
                             missing_count=np.zeros(m, np.int64), skip_reason=np.zeros(m, np.int8), clamp_count=0,
                             cand_rows=np.asarray(rows, np.int64), cand_cols=np.asarray(cols, np.int64),
                             cand_r=np.asarray(t, float) / 10, cand_t=np.asarray(t, float),
                             cand_p=np.asarray(p, float))


def test_merge_threshold_and_topk_equal_single_process(tmp_path):
    rng = np.random.default_rng(3)
    mk = _markers(10)
    names = ["ph1", "ph2", "ph3"]
    rows = np.repeat(np.arange(10), 3)
    cols = np.tile(np.arange(3), 10)
    t = rng.standard_normal(30) * 3
    p = np.round(rng.random(30), 2)  # coarse p -> ties exercise the source-index tie-break
    # single process
    w = output.ThresholdWriter(tmp_path / "single.tsv", 0.5, 8.0, 10, True, names)
    w.emit(_stats(mk, rows, cols, t, p))
    w.finalize()
    k = output.TopKWriter(tmp_path / "single_top.tsv", 2, 8.0, 10, True, names)
    k.emit(_stats(mk, rows, cols, t, p))
    k.finalize()
    # two shards: markers [0, 6) and [6, 10)
    shards, tshards = [], []
    for r, (lo, hi) in enumerate(((0, 6), (6, 10))):
        sel = (rows >= lo) & (rows < hi)
        ws = output.ThresholdWriter(tmp_path / f"o.rank{r}", 0.5, 8.0, 10, True, names)
        ws.emit(_stats(mk[lo:hi], rows[sel] - lo, cols[sel], t[sel], p[sel]))
        ws.finalize()
        shards.append(tmp_path / f"o.rank{r}")
        ks = output.TopKWriter(tmp_path / f"k.rank{r}", 2, 8.0, 10, True, names)
        ks.emit(_stats(mk[lo:hi], rows[sel] - lo, cols[sel], t[sel], p[sel]))
        ks.finalize()
        tshards.append(tmp_path / f"k.rank{r}")
    distributed.merge_tsv(shards, tmp_path / "merged.tsv")
    assert (tmp_path / "merged.tsv").read_bytes() == (tmp_path / "single.tsv").read_bytes()
    distributed.merge_topk(tshards, tmp_path / "merged_top.tsv", 2, names, {m.id: m.source_index for m in mk})
    assert (tmp_path / "merged_top.tsv").read_bytes() == (tmp_path / "single_top.tsv").read_bytes()


def test_merge_full(tmp_path):
    mk = _markers(5)
    names = ["p1", "p2"]
    t = np.arange(10, dtype=np.float64).reshape(5, 2)
    single = output.FullMatrixWriter(tmp_path / "s.bin", np.float64, 3.0, 5, True, names)
    b = _stats(mk, [], [], [], [])
    b.t_rows = t
    single.emit(b)
    single.finalize()
    shards = []
    for r, (lo, hi) in enumerate(((0, 3), (3, 5))):
        w = output.FullMatrixWriter(tmp_path / f"f.bin.rank{r}", np.float64, 3.0, 5, True, names)
        bs = _stats(mk[lo:hi], [], [], [], [])
        bs.t_rows = t[lo:hi]
        w.emit(bs)
        w.finalize()
        shards.append(tmp_path / f"f.bin.rank{r}")
    distributed.merge_full(shards, tmp_path / "f.bin")
    assert (tmp_path / "f.bin").read_bytes() == (tmp_path / "s.bin").read_bytes()
    assert (tmp_path / "f.bin.markers.tsv").read_text() == (tmp_path / "s.bin.markers.tsv").read_text()


def test_merge_min_p_takes_best_shard(tmp_path):
    from paper_2604_21095_b200.engine import write_min_p

    names = ["a", "b", "c"]
    write_min_p(tmp_path / "s0", names, [0.1, 0.5, 0.2], [1.0, 5.0, 2.0], [0.3, 1e-6, 0.04])
    write_min_p(tmp_path / "s1", names, [0.3, 0.4, 0.2], [3.0, 4.0, 2.0], [0.003, 1e-5, 0.04])
    assert distributed.merge_min_p([tmp_path / "s0", tmp_path / "s1"], tmp_path / "m") == 3
    rows = [ln.split("\t") for ln in (tmp_path / "m").read_text().splitlines()[1:]]
    assert [r[0] for r in rows] == names
    assert [float(r[3]) for r in rows] == [0.003, 1e-6, 0.04]

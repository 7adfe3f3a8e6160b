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


def _markers(n, dup_ids=False):
    # dup_ids: '.' IDs (common in .bim files) on every other marker
    return [pg.MarkerRecord("1", "." if dup_ids and i % 2 else f"snp{i + 1}", i + 1, "A", "B", i) for i in range(n)]


def _stats(markers, rows, cols, t, p):
    m = len(markers)
    t = np.asarray(t, float)
    return output.BatchStats(markers=tuple(markers), allele_frequency=np.full(m, 0.3),
                             missing_count=np.zeros(m, np.int64), skip_reason=np.zeros(m, np.int8), clamp_count=0,
                             cand_rows=np.asarray(rows, np.int64), cand_cols=np.asarray(cols, np.int64),
                             cand_r=t / 10, cand_t=t, cand_p=np.asarray(p, float), cand_beta=t * 0.37,
                             cand_se=np.full(t.size, 0.37))


@pytest.mark.parametrize("dup_ids", [False, True])
@pytest.mark.parametrize("top_k", [2, 5])
def test_merge_threshold_and_topk_equal_single_process(tmp_path, dup_ids, top_k):
    """Shard merges == one process, for THRESHOLD / TOPK records and their effect-size
    sidecars, with tied p across shards and duplicated ('.') marker IDs."""
    rng = np.random.default_rng(3)
    mk = _markers(10, dup_ids)
    names = ["ph1", "ph2", "ph3"]
    rows = np.repeat(np.arange(10), 3)
    cols = np.tile(np.arange(3), 10)
    t = rng.standard_normal(30) * 3
    p = np.round(rng.random(30), 1)  # coarse p -> ties exercise the source-index tie-break
    # single process
    w = output.ThresholdWriter(tmp_path / "single.tsv", 0.5, 8.0, 10, True, names, effect_sizes=True)
    w.emit(_stats(mk, rows, cols, t, p))
    w.finalize()
    k = output.TopKWriter(tmp_path / "single_top.tsv", top_k, 8.0, 10, True, names, effect_sizes=True)
    k.emit(_stats(mk, rows, cols, t, p))
    k.finalize()
    # two shards: markers [0, 6) and [6, 10)
    shards, tshards = [], []
    for r, (lo, hi) in enumerate(((0, 6), (6, 10))):
        sel = (rows >= lo) & (rows < hi)
        ws = output.ThresholdWriter(tmp_path / f"o.rank{r}", 0.5, 8.0, 10, True, names, effect_sizes=True)
        ws.emit(_stats(mk[lo:hi], rows[sel] - lo, cols[sel], t[sel], p[sel]))
        ws.finalize()
        shards.append(tmp_path / f"o.rank{r}")
        ks = output.TopKWriter(tmp_path / f"k.rank{r}", top_k, 8.0, 10, True, names, effect_sizes=True)
        ks.emit(_stats(mk[lo:hi], rows[sel] - lo, cols[sel], t[sel], p[sel]))
        ks.finalize()
        tshards.append(tmp_path / f"k.rank{r}")
    distributed.merge_tsv(shards, tmp_path / "merged.tsv")
    assert (tmp_path / "merged.tsv").read_bytes() == (tmp_path / "single.tsv").read_bytes()
    distributed.merge_tsv([output.beta_sidecar(x) for x in shards], output.beta_sidecar(tmp_path / "merged.tsv"),
                          header="\t".join(output.BETA_COLUMNS))
    assert (output.beta_sidecar(tmp_path / "merged.tsv").read_bytes()
            == output.beta_sidecar(tmp_path / "single.tsv").read_bytes())
    distributed.merge_topk(tshards, tmp_path / "merged_top.tsv", top_k, names, effect_sizes=True)
    assert (tmp_path / "merged_top.tsv").read_bytes() == (tmp_path / "single_top.tsv").read_bytes()
    assert (output.beta_sidecar(tmp_path / "merged_top.tsv").read_bytes()
            == output.beta_sidecar(tmp_path / "single_top.tsv").read_bytes())
    beta, se = output.load_effect_sizes(tmp_path / "single_top.tsv")
    recs = output.load_association_records(tmp_path / "single_top.tsv")
    assert np.allclose(beta, [r.t * 0.37 for r in recs]) and np.all(se == 0.37)


def test_merge_qc(tmp_path):
    """QC shards -> marker rows in rank order, then the phenotype rows once."""
    head = "KIND\tNAME\tREASON\n"
    (tmp_path / "a").write_text(head + "marker\tm1\tMONOMORPHIC\nphenotype\tz\tZERO_VARIANCE\n")
    (tmp_path / "b").write_text(head + "marker\tm9\tALL_MISSING\nphenotype\tz\tZERO_VARIANCE\n")
    assert distributed.merge_qc([tmp_path / "a", tmp_path / "b"], tmp_path / "m") == 2
    assert (tmp_path / "m").read_text() == (head + "marker\tm1\tMONOMORPHIC\nmarker\tm9\tALL_MISSING\n"
                                            "phenotype\tz\tZERO_VARIANCE\n")


def test_merge_full(tmp_path):
    mk = _markers(5)
    names = ["p1", "p2"]
    t = np.arange(10, dtype=np.float64).reshape(5, 2)
    single = output.FullMatrixWriter(tmp_path / "s.bin", np.float64, 3.0, 5, True, names, effect_sizes=True)
    b = _stats(mk, [], [], [], [])
    b.t_rows = t
    b.beta_rows = t * 0.5
    single.emit(b)
    single.finalize()
    shards = []
    for r, (lo, hi) in enumerate(((0, 3), (3, 5))):
        w = output.FullMatrixWriter(tmp_path / f"f.bin.rank{r}", np.float64, 3.0, 5, True, names,
                                    effect_sizes=True)
        bs = _stats(mk[lo:hi], [], [], [], [])
        bs.t_rows = t[lo:hi]
        bs.beta_rows = t[lo:hi] * 0.5
        w.emit(bs)
        w.finalize()
        shards.append(tmp_path / f"f.bin.rank{r}")
    distributed.merge_full(shards, tmp_path / "f.bin", effect_sizes=True)
    assert (tmp_path / "f.bin").read_bytes() == (tmp_path / "s.bin").read_bytes()
    assert np.array_equal(output.read_full_beta(tmp_path / "f.bin"), t * 0.5)
    assert (output.beta_sidecar(tmp_path / "f.bin", full=True).read_bytes()
            == output.beta_sidecar(tmp_path / "s.bin", full=True).read_bytes())
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


def test_panel_metadata_round_trip(tmp_path):
    """What rank 0 broadcasts instead of every rank parsing the tables: a pickled metadata
    dict that rebuilds a values-free _PreparedPanel with the same names, alignment, basis, df."""
    import pickle

    from conftest_helpers import write_tsv
    from paper_2604_21095_b200 import engine

    rng = np.random.default_rng(8)
    n = 40
    ids = [f"S{i + 1}" for i in range(n)]
    d = rng.integers(0, 3, (6, n)).astype(np.float64)
    bed, bim, fam = pg.write_bed_trio(tmp_path / "g", d, ids)
    y = rng.standard_normal((n, 3))
    y[3, 1] = np.nan
    pheno = write_tsv(tmp_path / "p.tsv", ids, ["a", "b", "c"], y)
    covar = write_tsv(tmp_path / "c.tsv", ids, ["x"], rng.standard_normal((n, 1)))
    (tmp_path / "keep.txt").write_text("\n".join(ids[:35]) + "\n")
    spec = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=bed, bim_path=bim, fam_path=fam)
    cfg = pg.ScanConfig(source=spec, pheno_path=pheno, covar_path=covar, out_path=tmp_path / "o.tsv",
                        keep_path=tmp_path / "keep.txt", df_mode=pg.DfMode.ADJUSTED)
    with pg.open_genotype_source(spec) as src:
        prep = engine.prepare_panel(cfg, src)
    got = engine.panel_from_metadata(pickle.loads(pickle.dumps(engine.panel_metadata(prep))))
    assert got.df == prep.df == 35 - 2 - 1
    assert got.panel.phenotype_names == prep.panel.phenotype_names
    assert got.panel.n_phenotypes == 3 and got.panel.n_samples == 35
    assert np.array_equal(got.panel.missing_count, prep.panel.missing_count)
    assert np.array_equal(got.align.genotype_row_index, prep.align.genotype_row_index)
    assert got.align.exclusion_log == prep.align.exclusion_log
    assert np.array_equal(got.basis.q, prep.basis.q) and got.basis.rank == prep.basis.rank

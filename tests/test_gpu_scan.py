"""End-to-end parity of the device scan (run_scan through the C ABI) with the
reference outputs frozen in tests/golden/ (s1: N=300, M=600, P=12 with
missing calls, missing phenotypes and 3 covariates; c1: BASELINE config 1,
N=2000, M=10000, P=64, 10 covariates).

Bars (north star / SURVEY appendix 5):
  bit-exact  : record keys, AF, N_MISS, skip accounting, hit membership away
               from the threshold (|t| outside t_crit * (1 +- 1e-4))
  tolerance  : |dt| <= 1e-4 * max(1, |t|), |d(-log10 p)| <= 1e-4 * max(1, -log10 p)
"""
from pathlib import Path

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from scan_fixtures import regenerate

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"
TOL = 1e-4


def _scan(paths, out, **kw):
    kw.setdefault("summary_to_stderr", False)
    spec = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=paths["bed_path"], bim_path=paths["bim_path"],
                         fam_path=paths["fam_path"])
    cfg = pg.ScanConfig(source=spec, pheno_path=paths["pheno_path"], covar_path=paths["covar_path"],
                        out_path=Path(out), **kw)
    return pg.run_scan(cfg)


def _arrays(path):
    recs = pg.load_association_records(path)
    return {
        "rows": np.array([int(r.id[3:]) - 1 for r in recs], dtype=np.int64),
        "cols": np.array([int(r.phenotype[2:]) - 1 for r in recs], dtype=np.int64),
        "r": np.array([r.r for r in recs]), "t": np.array([r.t for r in recs]),
        "p": np.array([r.p for r in recs]), "af": np.array([r.af for r in recs]),
        "n_miss": np.array([r.missing_count for r in recs], dtype=np.int64),
    }


def _assert_close_t_p(t, t_ref, p, p_ref):
    dt = np.abs(t - t_ref) / np.maximum(1.0, np.abs(t_ref))
    assert dt.max(initial=0.0) <= TOL, f"max rel dt {dt.max()}"
    lp, lp_ref = -np.log10(p), -np.log10(p_ref)
    dl = np.abs(lp - lp_ref) / np.maximum(1.0, lp_ref)
    assert dl.max(initial=0.0) <= TOL, f"max rel d(-log10 p) {dl.max()}"


@pytest.fixture(scope="module")
def s1(tmp_path_factory):
    return regenerate("s1", tmp_path_factory.mktemp("s1"))


@pytest.fixture(scope="module")
def c1(tmp_path_factory):
    return regenerate("c1", tmp_path_factory.mktemp("c1"))


def test_s1_all_pairs(s1, tmp_path):
    g = np.load(GOLD / "s1.npz")
    _scan(s1, tmp_path / "o.tsv", p_threshold=1.0, precision=pg.Precision.F64)
    a = _arrays(tmp_path / "o.tsv")
    assert np.array_equal(a["rows"], g["all_f64_rows"]) and np.array_equal(a["cols"], g["all_f64_cols"])
    assert np.array_equal(a["af"], g["all_f64_af"])          # AF bit-exact
    assert np.array_equal(a["n_miss"], g["all_f64_n_miss"])  # imputation counts bit-exact
    _assert_close_t_p(a["t"], g["all_f64_t"], a["p"], g["all_f64_p"])
    # the integer contraction is far tighter than the bar: report it
    rel = np.max(np.abs(a["t"] - g["all_f64_t"]) / np.maximum(1, np.abs(g["all_f64_t"])))
    assert rel < 1e-5


def _membership_matches(a, g, prefix, df, p_thr):
    t_crit = pg.t_threshold_for_p(p_thr, df)
    got = set(zip(a["rows"].tolist(), a["cols"].tolist()))
    want = set(zip(g[f"{prefix}_rows"].tolist(), g[f"{prefix}_cols"].tolist()))
    t_of = dict(zip(zip(g["all_f64_rows"].tolist(), g["all_f64_cols"].tolist()), g["all_f64_t"].tolist()))
    for key in got ^ want:
        assert abs(abs(t_of[key]) - t_crit) <= 1e-4 * t_crit, f"non-borderline membership difference {key}"


def test_s1_threshold_membership_and_tsv(s1, tmp_path):
    g = np.load(GOLD / "s1.npz")
    summ = _scan(s1, tmp_path / "o.tsv", p_threshold=1e-3, precision=pg.Precision.F64)
    a = _arrays(tmp_path / "o.tsv")
    _membership_matches(a, g, "thr_f64", summ.df, 1e-3)
    ref = pg.load_association_records(GOLD / "s1_thr_f64.tsv")
    mine = pg.load_association_records(tmp_path / "o.tsv")
    assert [(r.id, r.phenotype, r.chrom, r.pos, r.counted_allele, r.other_allele, r.af, r.missing_count, r.n, r.df)
            for r in mine] == [(r.id, r.phenotype, r.chrom, r.pos, r.counted_allele, r.other_allele, r.af,
                                r.missing_count, r.n, r.df) for r in ref]
    text = (tmp_path / "o.tsv").read_text()
    assert text.startswith("CHR\tID\tPOS\tA1\tA2\tAF\tN_MISS\tN\tDF\tR\tT\tP\tPHENO\n")


def test_s1_f32_mode(s1, tmp_path):
    g = np.load(GOLD / "s1.npz")
    summ = _scan(s1, tmp_path / "o.tsv", p_threshold=1e-3)
    a = _arrays(tmp_path / "o.tsv")
    _membership_matches(a, g, "thr_f32", summ.df, 1e-3)


def test_s1_topk(s1, tmp_path):
    g = np.load(GOLD / "s1.npz")
    _scan(s1, tmp_path / "top.tsv", output_mode=pg.OutputMode.TOPK, top_k=5, precision=pg.Precision.F64)
    mine = pg.load_association_records(tmp_path / "top.tsv")
    ref = pg.load_association_records(GOLD / "s1_topk_f64.tsv")
    assert [(r.id, r.phenotype) for r in mine] == [(r.id, r.phenotype) for r in ref]
    _assert_close_t_p(np.array([r.t for r in mine]), np.array([r.t for r in ref]),
                      np.array([r.p for r in mine]), np.array([r.p for r in ref]))


def test_s1_full(s1, tmp_path):
    g = np.load(GOLD / "s1.npz")
    _scan(s1, tmp_path / "full.bin", output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64)
    t, lines, phenos = pg.read_full_matrix(tmp_path / "full.bin")
    rows = np.array([int(x.split("\t")[0]) for x in lines])
    assert np.array_equal(rows, g["full_f64_rows"])
    assert t.dtype == np.dtype("<f8")
    rel = np.abs(t - g["full_f64_t"]) / np.maximum(1, np.abs(g["full_f64_t"]))
    assert rel.max() <= TOL


def test_s1_batch_invariance_bitwise(s1, tmp_path):
    blobs = []
    for db in (1, 7, 256, 600):
        out = tmp_path / f"full_{db}.bin"
        _scan(s1, out, output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64, device_batch=db)
        blobs.append(out.read_bytes())
    assert all(b == blobs[0] for b in blobs[1:])
    thr = []
    for db in (5, 600):
        out = tmp_path / f"thr_{db}.tsv"
        _scan(s1, out, p_threshold=1.0, precision=pg.Precision.F64, device_batch=db)
        thr.append(out.read_bytes())
    assert thr[0] == thr[1]


def test_c1_threshold(c1, tmp_path):
    g = np.load(GOLD / "c1.npz")
    summ = _scan(c1, tmp_path / "o.tsv", p_threshold=1e-4, precision=pg.Precision.F64)
    a = _arrays(tmp_path / "o.tsv")
    t_crit = pg.t_threshold_for_p(1e-4, summ.df)
    got = set(zip(a["rows"].tolist(), a["cols"].tolist()))
    want = set(zip(g["thr_f64_rows"].tolist(), g["thr_f64_cols"].tolist()))
    both = sorted(got & want)
    assert len(both) > 0
    tm = dict(zip(zip(a["rows"].tolist(), a["cols"].tolist()), a["t"].tolist()))
    tr = dict(zip(zip(g["thr_f64_rows"].tolist(), g["thr_f64_cols"].tolist()), g["thr_f64_t"].tolist()))
    for key in got ^ want:
        tv = tm.get(key, tr.get(key))
        assert abs(abs(tv) - t_crit) <= 1e-4 * t_crit
    pm = dict(zip(zip(a["rows"].tolist(), a["cols"].tolist()), a["p"].tolist()))
    pr = dict(zip(zip(g["thr_f64_rows"].tolist(), g["thr_f64_cols"].tolist()), g["thr_f64_p"].tolist()))
    _assert_close_t_p(np.array([tm[k] for k in both]), np.array([tr[k] for k in both]),
                      np.array([pm[k] for k in both]), np.array([pr[k] for k in both]))


def test_c1_full_subset(c1, tmp_path):
    g = np.load(GOLD / "c1.npz")
    _scan(c1, tmp_path / "full.bin", output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64)
    t, lines, _ = pg.read_full_matrix(tmp_path / "full.bin")
    rows = np.array([int(x.split("\t")[0]) for x in lines])
    pos = np.searchsorted(rows, g["full_f64_rows"])
    assert np.array_equal(rows[pos], g["full_f64_rows"])
    rel = np.abs(t[pos] - g["full_f64_t"]) / np.maximum(1, np.abs(g["full_f64_t"]))
    assert rel.max() <= TOL


def test_c1_fused_decode_matches_planes_bitwise(c1, tmp_path, monkeypatch):
    """The in-GEMM 2-bit decode and the materialized-plane path are the same integers."""
    _scan(c1, tmp_path / "fused.bin", output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64, device_batch=3000)
    monkeypatch.setenv("PANELGWAS_FUSED_DECODE", "0")
    _scan(c1, tmp_path / "planes.bin", output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64, device_batch=3000)
    assert (tmp_path / "fused.bin").read_bytes() == (tmp_path / "planes.bin").read_bytes()


def test_s1_extension_mode_residualized_genotypes(s1, tmp_path):
    """--residualize-genotypes + adjusted df (the FWL / `validate --exact` mode): side GEMM K5."""
    g = np.load(GOLD / "s1.npz")
    _scan(s1, tmp_path / "adj.tsv", p_threshold=1.0, precision=pg.Precision.F64, df_mode=pg.DfMode.ADJUSTED,
          residualize_genotypes=True)
    a = _arrays(tmp_path / "adj.tsv")
    assert np.array_equal(a["rows"], g["adj_f64_rows"]) and np.array_equal(a["cols"], g["adj_f64_cols"])
    _assert_close_t_p(a["t"], g["adj_f64_t"], a["p"], g["adj_f64_p"])
    rel = np.max(np.abs(a["t"] - g["adj_f64_t"]) / np.maximum(1, np.abs(g["adj_f64_t"])))
    assert rel < 1e-5


def test_fwl_matches_full_ols(tmp_path):
    """Extension mode equals full OLS y ~ 1 + C + g (reference tests/test_engine.py:417-432)."""
    rng = np.random.default_rng(19)
    n = 30
    af = rng.uniform(0.2, 0.8, size=10)
    d = rng.binomial(2, af[:, None], size=(10, n)).astype(np.float64)
    y = rng.standard_normal((n, 2))
    covar = rng.standard_normal((n, 2))
    y[:, 0] += covar @ [0.8, -0.5]
    ids = [f"S{i + 1}" for i in range(n)]
    bed, bim, fam = pg.write_bed_trio(tmp_path / "g", d, ids)
    from conftest_helpers import write_tsv

    pheno = write_tsv(tmp_path / "p.tsv", ids, ["ph1", "ph2"], y)
    cov = write_tsv(tmp_path / "c.tsv", ids, ["cv1", "cv2"], covar)
    spec = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=bed, bim_path=bim, fam_path=fam)
    pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, covar_path=cov, out_path=tmp_path / "o.tsv",
                              p_threshold=1.0, df_mode=pg.DfMode.ADJUSTED, residualize_genotypes=True,
                              precision=pg.Precision.F64, summary_to_stderr=False))
    for rec in pg.load_association_records(tmp_path / "o.tsv"):
        ref = pg.ols_single(y[:, int(rec.phenotype[2:]) - 1], d[rec.pos - 1], covar)
        assert rec.t == pytest.approx(ref.t, abs=1e-5)


def test_two_shard_flow_equals_single_gpu(s1, tmp_path):
    """The multi-GPU flow (panel export -> broadcast bytes -> import; contiguous marker
    shards; rank-order merge) run as two sequential 'ranks' on one GPU: byte-identical
    to the single scan."""
    import torch

    from paper_2604_21095_b200 import distributed

    spec = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=s1["bed_path"], bim_path=s1["bim_path"],
                         fam_path=s1["fam_path"])
    base = dict(source=spec, pheno_path=s1["pheno_path"], covar_path=s1["covar_path"], p_threshold=1e-2,
                precision=pg.Precision.F64, summary_to_stderr=False)
    pg.run_scan(pg.ScanConfig(out_path=tmp_path / "single.tsv", **base))
    exported = {}

    from paper_2604_21095_b200.engine import stage_panel

    def hook0(ctx, prep):
        stage_panel(ctx, prep, 300)
        buf = torch.empty(ctx.panel_bytes(), dtype=torch.uint8, device="cuda")
        ctx.export_panel(buf.data_ptr())
        exported["buf"] = buf
        exported["flags"] = prep.zero_variance

    def hook1(ctx, prep):
        prep.set_flags(exported["flags"])  # what the rank-0 flag broadcast delivers
        ctx.import_panel(exported["buf"].data_ptr(), prep.align.n_kept, len(prep.pheno_names),
                         prep.align.genotype_row_index, 300)

    shards = []
    for rank, hook in ((0, hook0), (1, hook1)):
        lo, hi = distributed.shard_span(600, 2, rank)
        out = distributed.shard_path(tmp_path / "multi.tsv", rank)
        pg.run_scan(pg.ScanConfig(out_path=out, **base), marker_range=(lo, hi), panel_hook=hook)
        shards.append(out)
    distributed.merge_tsv(shards, tmp_path / "multi.tsv")
    assert (tmp_path / "multi.tsv").read_bytes() == (tmp_path / "single.tsv").read_bytes()

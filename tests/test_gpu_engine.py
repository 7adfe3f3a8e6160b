"""Engine behaviour on the device, following the reference engine / CLI test
strategy (tests/test_engine.py, tests/test_cli.py): record order and
contract, premask == brute-force filter, TOPK selection and ties, FULL payload and
budget guard, invariances, accounting, keep/remove, df modes, missing policies,
OLS equivalence, CLI subcommands and exit codes."""
import json

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from conftest_helpers import write_tsv
from paper_2604_21095_b200 import cli

pytestmark = pytest.mark.gpu


def dataset(tmp_path, d, y, covar=None, subdir="data"):
    root = tmp_path / subdir
    root.mkdir(parents=True, exist_ok=True)
    n = d.shape[1]
    ids = [f"S{i + 1}" for i in range(n)]
    bed, bim, fam = pg.write_bed_trio(root / "geno", d, ids)
    pheno = write_tsv(root / "pheno.tsv", ids, [f"ph{j + 1}" for j in range(y.shape[1])], y)
    cov = write_tsv(root / "covar.tsv", ids, [f"cv{j + 1}" for j in range(covar.shape[1])], covar) \
        if covar is not None else None
    spec = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=bed, bim_path=bim, fam_path=fam)
    return spec, pheno, cov, root


def scan(spec, pheno, out, covar=None, **kw):
    kw.setdefault("summary_to_stderr", False)
    return pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, out_path=out, covar_path=covar, **kw))


def random_dataset(rng, m, n, p, maf=(0.2, 0.8)):
    af = rng.uniform(*maf, size=m)
    return rng.binomial(2, af[:, None], size=(m, n)).astype(np.float64), rng.standard_normal((n, p))


def test_open_threshold_emits_all_pairs_in_order(tmp_path):
    d, y = random_dataset(np.random.default_rng(0), 20, 30, 4)
    spec, pheno, _, root = dataset(tmp_path, d, y)
    s = scan(spec, pheno, root / "out.tsv", p_threshold=1.0)
    recs = pg.load_association_records(root / "out.tsv")
    assert len(recs) == s.markers_scanned * s.phenotypes_scanned == s.records_emitted
    keys = [(r.pos, r.phenotype) for r in recs]
    assert keys == sorted(keys)
    rec = recs[0]
    assert (rec.n, rec.df, rec.counted_allele, rec.other_allele) == (30, 28, "A", "B")


@pytest.mark.parametrize("thr,planted", [(0.2, False), (1e-6, True)])
def test_premask_equals_bruteforce(tmp_path, thr, planted):
    rng = np.random.default_rng(2 if not planted else 27)
    d, y = random_dataset(rng, 40 if not planted else 30, 50 if not planted else 200, 6 if not planted else 3)
    if planted:
        y[:, 0] += 0.8 * d[4]
        y[:, 2] -= 0.9 * d[17]
    spec, pheno, _, root = dataset(tmp_path, d, y)
    scan(spec, pheno, root / "all.tsv", p_threshold=1.0, precision=pg.Precision.F64)
    scan(spec, pheno, root / "cut.tsv", p_threshold=thr, precision=pg.Precision.F64)
    full = pg.load_association_records(root / "all.tsv")
    expected = {(r.id, r.phenotype) for r in full if r.p <= thr}
    assert expected or not planted
    assert {(r.id, r.phenotype) for r in pg.load_association_records(root / "cut.tsv")} == expected


def test_topk_matches_bruteforce_and_ties(tmp_path):
    d, y = random_dataset(np.random.default_rng(5), 25, 30, 3)
    spec, pheno, _, root = dataset(tmp_path, d, y)
    scan(spec, pheno, root / "all.tsv", p_threshold=1.0, precision=pg.Precision.F64, device_batch=7)
    scan(spec, pheno, root / "top.tsv", output_mode=pg.OutputMode.TOPK, top_k=4, precision=pg.Precision.F64,
         device_batch=7)
    full = pg.load_association_records(root / "all.tsv")
    by = {}
    for r in full:
        by.setdefault(r.phenotype, []).append(r)
    expected = set()
    for name, recs in by.items():
        recs.sort(key=lambda r: (r.p, r.pos))
        expected |= {(r.id, name) for r in recs[:4]}
    assert {(r.id, r.phenotype) for r in pg.load_association_records(root / "top.tsv")} == expected
    # duplicated marker rows: identical p, the earlier source index wins
    rng = np.random.default_rng(6)
    row = rng.binomial(2, 0.5, size=20).astype(np.float64)
    d2 = np.vstack([row, rng.binomial(2, 0.5, size=(6, 20)).astype(np.float64), row])
    spec, pheno, _, root = dataset(tmp_path, d2, rng.standard_normal((20, 1)), subdir="dup")
    scan(spec, pheno, root / "top.tsv", output_mode=pg.OutputMode.TOPK, top_k=d2.shape[0] - 1)
    ids = [r.id for r in pg.load_association_records(root / "top.tsv")]
    assert len(ids) == d2.shape[0] - 1
    assert "snp1" in ids and ("snp8" not in ids or ids.index("snp1") < ids.index("snp8"))


def test_full_payload_budget_and_f32(tmp_path):
    d, y = random_dataset(np.random.default_rng(7), 12, 30, 3)
    d[4] = 2.0
    spec, pheno, _, root = dataset(tmp_path, d, y)
    s = scan(spec, pheno, root / "full.bin", output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64)
    t, lines, names = pg.read_full_matrix(root / "full.bin")
    assert t.shape == (11, 3) and names == ["ph1", "ph2", "ph3"] and s.records_emitted == 33
    assert not any(x.split("\t")[2] == "snp5" for x in lines)
    scan(spec, pheno, root / "f32.bin", output_mode=pg.OutputMode.FULL)
    assert pg.read_full_matrix(root / "f32.bin")[0].dtype == np.dtype("<f4")
    with pytest.raises(pg.ConfigError, match="budget"):
        scan(spec, pheno, root / "b.bin", output_mode=pg.OutputMode.FULL, full_byte_budget=10)
    scan(spec, pheno, root / "b.bin", output_mode=pg.OutputMode.FULL, full_byte_budget=10, allow_large_full=True)
    # FULL t == THRESHOLD t for every pair
    scan(spec, pheno, root / "thr.tsv", p_threshold=1.0, precision=pg.Precision.F64)
    lookup = {(r.id, r.phenotype): r.t for r in pg.load_association_records(root / "thr.tsv")}
    for line, row in zip(lines, t):
        for j, name in enumerate(names):
            assert row[j] == lookup[(line.split("\t")[2], name)]


def test_invariances(tmp_path):
    rng = np.random.default_rng(13)
    d, y = random_dataset(rng, 33, 40, 4)
    y[rng.random(y.shape) < 0.05] = np.nan
    spec, pheno, cov, root = dataset(tmp_path, d, y, covar=rng.standard_normal((40, 2)))
    outs = []
    for workers, db in ((1, 5), (2, 33), (8, 1)):
        out = root / f"w{workers}.tsv"
        scan(spec, pheno, out, covar=cov, p_threshold=1.0, precision=pg.Precision.F64, worker_count=workers,
             device_batch=db)
        outs.append(out.read_bytes())
    assert outs[0] == outs[1] == outs[2]
    scan(spec, pheno, root / "f32.tsv", covar=cov, p_threshold=1.0)
    a = pg.load_association_records(root / "w1.tsv")
    b = pg.load_association_records(root / "f32.tsv")
    assert all(abs(ra.t - rb.t) <= 1e-4 * max(1.0, abs(ra.t)) for ra, rb in zip(a, b))


def test_accounting_qc_keep_remove_and_df(tmp_path):
    rng = np.random.default_rng(16)
    d, y = random_dataset(rng, 15, 30, 3)
    d[2] = 0.0
    d[9] = np.nan
    y[:, 1] = 42.0
    spec, pheno, _, root = dataset(tmp_path, d, y)
    s = scan(spec, pheno, root / "out.tsv", p_threshold=1.0, qc_sidecar=True)
    assert (s.markers_skipped_monomorphic, s.markers_skipped_all_missing, s.markers_scanned) == (1, 1, 13)
    assert (s.phenotypes_skipped_zero_variance, s.phenotypes_scanned, s.records_emitted) == (1, 2, 26)
    blob = json.loads((root / "out.tsv.summary.json").read_text())
    assert blob["markers_scanned"] == 13 and blob["records_emitted"] == 26
    qc = (root / "out.tsv.qc.tsv").read_text()
    assert "snp3\tMONOMORPHIC" in qc and "snp10\tALL_MISSING" in qc and "ph2\tZERO_VARIANCE" in qc
    d, y = random_dataset(np.random.default_rng(17), 6, 12, 2)
    spec, pheno, _, root = dataset(tmp_path, d, y, subdir="kr")
    (root / "keep.txt").write_text("".join(f"S{i}\n" for i in range(1, 11)))
    (root / "remove.txt").write_text("S1\nS2\n")
    s = scan(spec, pheno, root / "o.tsv", p_threshold=1.0, keep_path=root / "keep.txt",
             remove_path=root / "remove.txt", precision=pg.Precision.F64)
    assert s.n_samples_used == 8 and s.exclusion_log["remove-listed"] == 2
    rec = pg.load_association_records(root / "o.tsv")[0]
    assert rec.n == 8
    # kept-sample subset: same t as OLS on the kept rows only
    keep = np.array([i for i in range(12) if f"S{i + 1}" not in {"S1", "S2", "S11", "S12"}])
    for r in pg.load_association_records(root / "o.tsv"):
        ref = pg.ols_single(y[keep, int(r.phenotype[2:]) - 1], d[r.pos - 1, keep])
        assert r.t == pytest.approx(ref.t, abs=1e-5)
    d, y = random_dataset(np.random.default_rng(18), 8, 30, 2)
    spec, pheno, cov, root = dataset(tmp_path, d, y, covar=np.random.default_rng(1).standard_normal((30, 3)),
                                     subdir="df")
    scan(spec, pheno, root / "o.tsv", covar=cov, p_threshold=1.0, df_mode=pg.DfMode.ADJUSTED)
    assert pg.load_association_records(root / "o.tsv")[0].df == 30 - 4 - 1


def test_paper_df_matches_ols_and_missing_policy(tmp_path):
    rng = np.random.default_rng(20)
    d, y = random_dataset(rng, 12, 25, 3)
    spec, pheno, _, root = dataset(tmp_path, d, y)
    scan(spec, pheno, root / "out.tsv", p_threshold=1.0, precision=pg.Precision.F64)
    for rec in pg.load_association_records(root / "out.tsv"):
        ref = pg.ols_single(y[:, int(rec.phenotype[2:]) - 1], d[rec.pos - 1])
        assert rec.t == pytest.approx(ref.t, abs=1e-5)
        assert rec.p == pytest.approx(ref.p, rel=1e-4)
    d, y = random_dataset(np.random.default_rng(21), 5, 20, 2)
    y[3, 0] = np.nan
    spec, pheno, _, root = dataset(tmp_path, d, y, subdir="mp")
    assert scan(spec, pheno, root / "o.tsv", p_threshold=1.0).records_emitted > 0
    with pytest.raises(pg.PanelGwasError, match="missing"):
        scan(spec, pheno, root / "o2.tsv", p_threshold=1.0, missing_policy=pg.MissingPolicy.FAIL)


class TestCli:
    def test_run_bench_validate_convert(self, tmp_path, capsys):
        d, y = random_dataset(np.random.default_rng(3), 20, 40, 2)
        spec, pheno, _, root = dataset(tmp_path, d, y)
        prefix = root / "geno"
        assert cli.main(["run", "--bfile", str(prefix), "--pheno", str(pheno), "--out", str(root / "o.tsv"),
                         "--p-threshold", "1"]) == 0
        assert len(pg.load_association_records(root / "o.tsv")) == 40
        capsys.readouterr()
        assert cli.main(["bench", "--simulate", "--n-samples", "200", "--n-markers", "500", "--n-phenotypes", "8",
                         "--out-dir", str(tmp_path / "b")]) == 0
        keys = dict(line.split("=", 1) for line in capsys.readouterr().out.split())
        assert int(keys["tests"]) == 500 * 8 - 8 * (int(keys["markers_skipped_monomorphic"]))
        assert float(keys["tests_per_second"]) > 0
        assert cli.main(["validate", "--simulate", "--out-dir", str(tmp_path / "v")]) == 0
        assert "PASS" in capsys.readouterr().out
        assert cli.main(["validate", "--simulate", "--exact", "--out-dir", str(tmp_path / "vx")]) == 0
        assert "PASS" in capsys.readouterr().out
        assert cli.main(["convert", "--bfile", str(prefix), "--to", "dense", "--out", str(root / "conv")]) == 0
        arr = np.load(root / "conv.npy")
        assert np.array_equal(np.nan_to_num(arr, nan=-1), np.nan_to_num(d, nan=-1))

    def test_usage_errors_exit_2(self, tmp_path):
        with pytest.raises(SystemExit) as e:
            cli.main(["run", "--pheno", "p", "--out", "o"])
        assert e.value.code == 2
        with pytest.raises(SystemExit) as e:
            cli.main(["run", "--bfile", "x", "--pheno", "p", "--out", "o", "--full", "--top-k", "3"])
        assert e.value.code == 2

    def test_error_exit_1(self, tmp_path, capsys):
        assert cli.main(["run", "--bfile", str(tmp_path / "nope"), "--pheno", str(tmp_path / "p.tsv"),
                         "--out", str(tmp_path / "o.tsv")]) == 1
        assert "missing file" in capsys.readouterr().err


def test_min_p_sidecar_equals_full_scan_minimum(tmp_path):
    """<out>.minp.tsv (per-phenotype max |t| / min p, fused into the GEMM epilogue) ==
    the minimum over the FULL t matrix of the same scan, bit for bit (fp64 r of the maximum)."""
    rng = np.random.default_rng(41)
    d, y = random_dataset(rng, 300, 120, 9)
    y[:, 3] += 0.7 * d[11]
    spec, pheno, _, root = dataset(tmp_path, d, y)
    scan(spec, pheno, root / "thr.tsv", p_threshold=1e-3, min_p_sidecar=True, device_batch=64,
         precision=pg.Precision.F64)
    scan(spec, pheno, root / "full.bin", output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64)
    t, _, names = pg.read_full_matrix(root / "full.bin")
    rows = [ln.split("\t") for ln in (root / "thr.tsv.minp.tsv").read_text().splitlines()]
    assert rows[0] == ["PHENO", "MAX_ABS_R", "MAX_ABS_T", "MIN_P"]
    assert [r[0] for r in rows[1:]] == names
    got_t = np.array([float(r[2]) for r in rows[1:]])
    got_p = np.array([float(r[3]) for r in rows[1:]])
    want_t = np.abs(t).max(axis=0)
    assert np.array_equal(got_t, want_t)
    want_p = pg.p_from_t(want_t, 118.0)
    np.testing.assert_allclose(got_p, want_p, rtol=1e-13)
    assert np.argmin(got_p) == 3
    # the records the threshold scan emitted agree with the sidecar's minimum
    recs = pg.load_association_records(root / "thr.tsv")
    for j, name in enumerate(names):
        ps = [r.p for r in recs if r.phenotype == name]
        if ps:
            assert min(ps) == got_p[j]


def test_topk_large_batches_null_bar_and_rescan(tmp_path):
    """Device batches much larger than 16k markers: phenotypes short of k records get a
    null-quantile bar instead of admitting every marker; a phenotype whose statistics are
    far below the null (one informative sample) falls short and its batch is rescanned.
    The output equals the brute-force top-k by (p, source index) of the full scan."""
    rng = np.random.default_rng(31)
    n, m, k = 60, 900, 3
    d, y = random_dataset(rng, m, n, 4)
    d[:, 0] = 1.0  # sample 0 heterozygous everywhere ...
    y[:, 2] = 0.0
    y[0, 2] = 1.0  # ... and phenotype 3 supported on it: |t| < 1.1 for every marker (sub-null)
    y[:, 3] += 0.9 * d[123]  # a planted hit
    spec, pheno, _, root = dataset(tmp_path, d, y)
    scan(spec, pheno, root / "all.tsv", p_threshold=1.0, precision=pg.Precision.F64)
    from paper_2604_21095_b200 import engine

    before = engine.topk_rescans
    scan(spec, pheno, root / "top.tsv", output_mode=pg.OutputMode.TOPK, top_k=k, precision=pg.Precision.F64,
         device_batch=400)
    assert engine.topk_rescans > before  # the sub-null phenotype forced the exact fallback
    by = {}
    for r in pg.load_association_records(root / "all.tsv"):
        by.setdefault(r.phenotype, []).append(r)
    expected = []
    for name in sorted(by):
        recs = sorted(by[name], key=lambda r: (r.p, r.pos))[:k]
        expected += [(r.id, name, r.t) for r in recs]
    got = [(r.id, r.phenotype, r.t) for r in pg.load_association_records(root / "top.tsv")]
    assert sorted(got, key=lambda x: (x[1], x[0])) == sorted(expected, key=lambda x: (x[1], x[0]))
    assert ("snp124", "ph4") in {(g[0], g[1]) for g in got}


def test_bgen_matches_plink_with_alleles_swapped_and_rerun_identical(tmp_path):
    """The same dosage matrix through the PLINK and BGEN-16 readers: identical statistics,
    opposite counted-allele labels (PLINK counts allele1, BGEN allele2); and a rerun of the
    same scan is byte-identical (reference tests: engine / determinism)."""
    from bgen_fixture import write_bgen

    rng = np.random.default_rng(23)
    d = rng.integers(0, 3, size=(8, 30)).astype(np.float64)
    y = rng.standard_normal((30, 2))
    spec, pheno, _, root = dataset(tmp_path, d, y)
    ids = [f"S{i + 1}" for i in range(30)]
    bspec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=write_bgen(root / "g.bgen", d, ids, bits=16))
    scan(spec, pheno, root / "plink.tsv", p_threshold=1.0, precision=pg.Precision.F64)
    scan(bspec, pheno, root / "bgen.tsv", p_threshold=1.0, precision=pg.Precision.F64)
    a = pg.load_association_records(root / "plink.tsv")
    b = pg.load_association_records(root / "bgen.tsv")
    assert len(a) == len(b) == 16
    for ra, rb in zip(a, b):
        assert ra.phenotype == rb.phenotype
        assert (ra.counted_allele, ra.other_allele) == ("A", "B")
        assert (rb.counted_allele, rb.other_allele) == ("B", "A")
        assert rb.t == pytest.approx(ra.t, rel=1e-9, abs=1e-12)
        assert rb.af == pytest.approx(ra.af, abs=1e-12)
    scan(bspec, pheno, root / "bgen2.tsv", p_threshold=1.0, precision=pg.Precision.F64)
    assert (root / "bgen2.tsv").read_bytes() == (root / "bgen.tsv").read_bytes()


def test_null_calibration(tmp_path):
    """Under the null the p-values are uniform: P(p <= a) ~ a, KS distance small
    (reference acceptance criterion 9)."""
    rng = np.random.default_rng(909)
    d, y = random_dataset(rng, 2000, 400, 64, maf=(0.05, 0.95))
    spec, pheno, _, root = dataset(tmp_path, d, y)
    scan(spec, pheno, root / "all.tsv", p_threshold=1.0, precision=pg.Precision.F64)
    p = np.sort(np.array([r.p for r in pg.load_association_records(root / "all.tsv")]))
    m = p.size
    for a, tol in ((0.05, 0.004), (0.01, 0.0015)):
        assert abs(np.mean(p <= a) - a) < tol
    ks = np.max(np.abs(p - (np.arange(1, m + 1) / m)))
    assert ks < 0.01


def test_candidate_counter_crosses_int32_range(tmp_path):
    """The epilogue's candidate counter is 64-bit: a launch whose counter starts just below
    2^31 (test hook) and crosses it yields exactly the candidates of a normal launch (the
    32-bit counter of round 1 wrapped to negative slots here)."""
    from paper_2604_21095_b200 import _native
    from paper_2604_21095_b200._device import DeviceContext
    from oracle import scan_oracle as orc

    rng = np.random.default_rng(77)
    n, m, p = 256, 700, 300
    d, y = random_dataset(rng, m, n, p)
    ytil, _ = orc.standardized_panel(y, orc.covariate_basis(np.zeros((n, 0))))
    codes = np.select([d == 2, d == 1, d == 0], [0, 2, 3]).astype(np.uint8)
    q = codes.reshape(m, n // 4, 4)
    packed = (q[:, :, 0] | (q[:, :, 1] << 2) | (q[:, :, 2] << 4) | (q[:, :, 3] << 6)).astype(np.uint8)
    with DeviceContext(0) as ctx:
        ctx.set_panel(ytil, np.arange(n, dtype=np.int64), n)
        ctx.set_scan(float(n - 2), _native.PG_MODE_THRESHOLD, np.zeros(p))  # every pair is a candidate
        a = ctx.scan(_native.PG_GENO_BED, packed, n // 4)
        ctx.debug_candidate_base(2**31 - 1000)
        b = ctx.scan(_native.PG_GENO_BED, packed, n // 4)
        ctx.debug_candidate_base(2**32 - 5)
        c = ctx.scan(_native.PG_GENO_BED, packed, n // 4)
    assert a.cand_t.size == m * p
    for x in (b, c):
        assert np.array_equal(x.cand_rows, a.cand_rows) and np.array_equal(x.cand_cols, a.cand_cols)
        assert np.array_equal(x.cand_t, a.cand_t)


def test_topk_larger_than_device_batch(tmp_path):
    """top_k above the device batch, ~3 batches: phenotypes holding some but fewer than k
    records must not lose true top-k markers to the null-quantile bar (advisor finding)."""
    rng = np.random.default_rng(12)
    n, m, k = 80, 1500, 700
    d, y = random_dataset(rng, m, n, 5)
    spec, pheno, _, root = dataset(tmp_path, d, y)
    scan(spec, pheno, root / "all.tsv", p_threshold=1.0, precision=pg.Precision.F64)
    scan(spec, pheno, root / "top.tsv", output_mode=pg.OutputMode.TOPK, top_k=k, precision=pg.Precision.F64,
         device_batch=512)
    by = {}
    for r in pg.load_association_records(root / "all.tsv"):
        by.setdefault(r.phenotype, []).append(r)
    expected = []
    for name in sorted(by):
        expected += [(name, r.id) for r in sorted(by[name], key=lambda r: (r.p, r.pos))[:k]]
    got = [(r.phenotype, r.id) for r in pg.load_association_records(root / "top.tsv")]
    assert got == expected

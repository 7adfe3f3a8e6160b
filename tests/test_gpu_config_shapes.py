"""Parity at the BASELINE configs' own shapes.

* C5 shape: BGEN-8, N = 23,000, 1,024 variants, 5 % missing calls, 20 % fractional dosages,
  P = 4,096 phenotypes with 10 covariates — through the GPU inflate (csrc/inflate.cu), the
  in-place BGEN-8 decode and the 3-row wide-digit GEMM (`assoc_i8_kernel<kWide3>`: 144-row
  pair tiles, 12-column epilogue steps, 16 phenotype tiles), against the oracle restatement
  of the reference path (bgen.py:183-249 decode, kernel.py:376-504 stats).
* C1 as the config says ("synthetic NumPy genotypes"): the c1 cohort through DenseSource
  (dense.py:79-97) vs the reference's own c1 golden output, exactly as the PLINK run is checked.

Bars: AF, N_MISS, skip flags bit-exact; |dt| <= 1e-4 max(1, |t|),
|d(-log10 p)| <= 1e-4 max(1, -log10 p); hit membership exact for |t| outside t_crit (1 +- 1e-4);
beta / SE <= 1e-4 relative (north star).
"""
from pathlib import Path

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from oracle import scan_oracle as orc
from paper_2604_21095_b200 import _native
from paper_2604_21095_b200._device import DeviceContext

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"
TOL = 1e-4


def _c5_cohort(tmp_path, n=23_000, m=1024, p=4096, n_cov=10, seed=5):
    from bgen_fixture import _quantize, write_bgen

    rng = np.random.default_rng(seed)
    af = rng.uniform(0.05, 0.95, m)
    d = rng.binomial(2, af[:, None], size=(m, n)).astype(np.float64)
    frac = rng.random((m, n)) < 0.20
    d[frac] = np.clip(d[frac] + rng.normal(0.0, 0.3, frac.sum()), 0.0, 2.0)
    d[rng.random((m, n)) < 0.05] = np.nan
    d[3] = 1.0  # monomorphic (skipped)
    ids = [f"S{i + 1}" for i in range(n)]
    path = write_bgen(tmp_path / "c5.bgen", d, ids, bits=8)
    # what the reference reader decodes from those bytes (bgen.py:238-249 via the oracle)
    miss = np.isnan(d)
    hom1, het = _quantize(np.where(miss, 0.0, d), 255)
    probs = np.stack([np.where(miss, 0, hom1), np.where(miss, 0, het)], -1).reshape(m, -1)
    ploidy = np.where(miss, 0x82, 2)
    want_d = np.stack([orc.decode_bgen(probs[i], ploidy[i], 8) for i in range(m)])
    c = rng.standard_normal((n, n_cov))
    y = c @ (0.1 * rng.standard_normal((n_cov, p))) + rng.standard_normal((n, p))
    y[:, 7] += 0.08 * np.nan_to_num(want_d[11] - np.nanmean(want_d[11]))  # a planted signal
    return path, want_d, y, c


def _assert_t_p(t, t_ref, p, p_ref):
    dt = np.abs(t - t_ref) / np.maximum(1.0, np.abs(t_ref))
    assert dt.max(initial=0.0) <= TOL, f"max rel dt {dt.max()}"
    lp, lr = -np.log10(p), -np.log10(p_ref)
    dl = np.abs(lp - lr) / np.maximum(1.0, lr)
    assert dl.max(initial=0.0) <= TOL, f"max rel d(-log10 p) {dl.max()}"


def test_c5_shape_bgen8_wide3_vs_oracle(tmp_path):
    path, want_d, y, c = _c5_cohort(tmp_path)
    n, p = y.shape
    m = want_d.shape[0]
    q = orc.covariate_basis(c)
    ytil, zero = orc.standardized_panel(y, q)
    assert not zero.any()
    df = float(n - 2)
    p_thr = 1e-3
    want = orc.threshold_scan(want_d, ytil, df, p_thr)
    src = pg.BgenSource(path)
    blob, off, size = src.read_compressed_block(0, m)
    src.close()
    sd = orc.panel_sd(y, q)
    with DeviceContext(0) as ctx:
        ctx.set_wide_digits(True)
        ctx.set_panel(ytil, np.arange(n, dtype=np.int64), n)
        ctx.set_beta_scale(sd)
        # FULL: every (marker, phenotype) t against the oracle's fp64 r
        ctx.set_scan(df, _native.PG_MODE_FULL, None)
        assert ctx.stage_bgen(0, blob, off, size) is None
        full = ctx.scan_staged(0)
        # THRESHOLD with the reference premask
        ctx.set_scan(df, _native.PG_MODE_THRESHOLD, np.full(p, orc.premask_abs_r(p_thr, df)))
        assert ctx.stage_bgen(1, blob, off, size) is None
        thr = ctx.scan_staged(1)
    assert full.rows_per_marker == 3  # the kWide3 geometry (2 base-255 digit rows + the missing row)
    for res in (full, thr):
        # fractional BGEN AF: ~1e-15 relative (numpy's pairwise nansum order)
        np.testing.assert_allclose(res.af, want["af"], rtol=1e-14, atol=0)
        assert np.array_equal(res.missing_count, want["missing"])
        assert np.array_equal(res.skip, want["skip"])
    ok = want["skip"] == 0
    t_ref = orc.t_from_r(want["full_r"][ok], df)
    rel = np.abs(full.t_rows - t_ref) / np.maximum(1.0, np.abs(t_ref))
    assert full.t_rows.shape == (ok.sum(), p) and rel.max() <= TOL, rel.max()
    # hit membership: exact away from the threshold
    t_crit = orc.t_threshold_for_p(p_thr, df)
    got = set(zip(thr.cand_rows[thr.cand_p <= p_thr].tolist(), thr.cand_cols[thr.cand_p <= p_thr].tolist()))
    exp = set(zip(want["rows"].tolist(), want["cols"].tolist()))
    assert len(exp) > 0.5 * p_thr * m * p
    for key in got ^ exp:
        tv = t_ref[np.searchsorted(np.nonzero(ok)[0], key[0]), key[1]]
        assert abs(abs(tv) - t_crit) <= TOL * t_crit, (key, tv, t_crit)
    both = sorted(got & exp)
    gi = {k: i for i, k in enumerate(zip(thr.cand_rows.tolist(), thr.cand_cols.tolist()))}
    wi = {k: i for i, k in enumerate(zip(want["rows"].tolist(), want["cols"].tolist()))}
    a = np.array([gi[k] for k in both])
    b = np.array([wi[k] for k in both])
    _assert_t_p(thr.cand_t[a], want["t"][b], thr.cand_p[a], want["p"][b])
    assert any(r == 11 and c == 7 for r, c in both)  # the planted signal is found
    # effect sizes (north star: beta within 1e-4): beta = r sd(y_res) / sd(g), se = beta / t
    beta, se = orc.effect_sizes(want["r"], want["variance"][want["rows"]], sd[want["cols"]], df)
    np.testing.assert_allclose(thr.cand_beta[a], beta[b], rtol=TOL)
    np.testing.assert_allclose(thr.cand_se[a], se[b], rtol=TOL)


@pytest.fixture(scope="module")
def c1_dense(tmp_path_factory):
    from scan_fixtures import regenerate, spec_of

    root = tmp_path_factory.mktemp("c1d")
    paths = regenerate("c1", root)
    spec = spec_of("c1")
    n, m = spec["n_samples"], spec["n_markers"]
    bpm = (n + 3) // 4
    blob = np.frombuffer(Path(paths["bed_path"]).read_bytes()[3:], dtype=np.uint8).reshape(m, bpm)
    np.save(root / "c1.npy", orc.decode_bed(blob, n))  # [markers, samples] float64, NaN = missing
    ids = [ln.split()[1] for ln in Path(paths["fam_path"]).read_text().splitlines()]
    (root / "c1.samples.txt").write_text("\n".join(ids) + "\n")
    return paths, root / "c1.npy", root / "c1.samples.txt"


def test_c1_dense_numpy_matches_reference_golden(c1_dense, tmp_path):
    """BASELINE config 1 as specified (NumPy genotypes) through DenseSource == the reference's c1 output."""
    paths, npy, ids = c1_dense
    g = np.load(GOLD / "c1.npz")
    spec = pg.SourceSpec(pg.GenotypeFormat.DENSE, dense_path=npy, sample_id_path=ids)
    summ = pg.run_scan(pg.ScanConfig(source=spec, pheno_path=paths["pheno_path"], covar_path=paths["covar_path"],
                                     out_path=tmp_path / "o.tsv", p_threshold=1e-4, precision=pg.Precision.F64,
                                     summary_to_stderr=False))
    recs = pg.load_association_records(tmp_path / "o.tsv")
    keys = [(r.pos - 1, int(r.phenotype[2:]) - 1) for r in recs]  # dense markers are m1.. at pos 1..
    want = list(zip(g["thr_f64_rows"].tolist(), g["thr_f64_cols"].tolist()))
    t_crit = pg.t_threshold_for_p(1e-4, summ.df)
    got_t = dict(zip(keys, [r.t for r in recs]))
    ref_t = dict(zip(want, g["thr_f64_t"].tolist()))
    for key in set(keys) ^ set(want):
        tv = got_t.get(key, ref_t.get(key))
        assert abs(abs(tv) - t_crit) <= TOL * t_crit
    both = sorted(set(keys) & set(want))
    assert len(both) > 0.95 * len(want)
    gi = {k: i for i, k in enumerate(keys)}
    wi = {k: i for i, k in enumerate(want)}
    a = [gi[k] for k in both]
    b = [wi[k] for k in both]
    # AF and N_MISS bit-exact with the reference
    assert [recs[i].af for i in a] == g["thr_f64_af"][b].tolist()
    assert [recs[i].missing_count for i in a] == g["thr_f64_n_miss"][b].tolist()
    _assert_t_p(np.array([recs[i].t for i in a]), g["thr_f64_t"][b], np.array([recs[i].p for i in a]),
                g["thr_f64_p"][b])


def test_c1_dense_equals_plink_bitwise(c1_dense, tmp_path):
    """The same integral dosages through DenseSource and PlinkSource give identical records."""
    paths, npy, ids = c1_dense
    dense = pg.SourceSpec(pg.GenotypeFormat.DENSE, dense_path=npy, sample_id_path=ids)
    plink = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=paths["bed_path"], bim_path=paths["bim_path"],
                          fam_path=paths["fam_path"])
    for spec, out in ((dense, "d.tsv"), (plink, "p.tsv")):
        pg.run_scan(pg.ScanConfig(source=spec, pheno_path=paths["pheno_path"], covar_path=paths["covar_path"],
                                  out_path=tmp_path / out, p_threshold=1e-3, precision=pg.Precision.F64,
                                  summary_to_stderr=False))
    d = pg.load_association_records(tmp_path / "d.tsv")
    p = pg.load_association_records(tmp_path / "p.tsv")
    assert len(d) == len(p) > 0
    for x, y in zip(d, p):
        assert (x.pos, x.phenotype, x.t, x.p, x.r, x.af, x.missing_count) == \
            (y.pos, y.phenotype, y.t, y.p, y.r, y.af, y.missing_count)

"""Precision.F64 (reference engine.py:31-33): the panel is quantized at two levels (~46 bits,
csrc/panel.cu) and the exact int8 GEMM runs once per level, so t / p / beta agree with the
reference's float64 path to ~1e-12 instead of the default mode's ~1e-7 (the reference's own
default f32-store mode is in the same class as the latter). Genotype codes are exact for
PLINK, BGEN and integral dense dosages; real-valued dense dosages stay on their 2^-17 grid."""
from pathlib import Path

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from conftest_helpers import write_tsv
from oracle import scan_oracle as orc
from paper_2604_21095_b200 import _native
from paper_2604_21095_b200._device import DeviceContext
from scan_fixtures import regenerate

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


def _packed(d):
    m, n = d.shape
    codes = np.where(np.isnan(d), 1, np.select([d == 2, d == 1, d == 0], [0, 2, 3])).astype(np.uint8)
    bpm = (n + 3) // 4
    codes = np.pad(codes, ((0, 0), (0, 4 * bpm - n)))
    q = codes.reshape(m, bpm, 4)
    return (q[:, :, 0] | (q[:, :, 1] << 2) | (q[:, :, 2] << 4) | (q[:, :, 3] << 6)).astype(np.uint8), bpm


@pytest.mark.parametrize("missing_share", [0.0, 0.2, 1.0])
def test_f64_panel_plink_matches_fp64_oracle(missing_share):
    rng = np.random.default_rng(int(missing_share * 10) + 5)
    n, m, p = 731, 600, 70
    d = rng.binomial(2, rng.uniform(0.1, 0.9, m)[:, None], size=(m, n)).astype(np.float64)
    rows = rng.random(m) < missing_share
    d[rows] = np.where(rng.random((rows.sum(), n)) < 0.04, np.nan, d[rows])
    y = rng.standard_normal((n, p))
    ytil, _ = orc.standardized_panel(y, orc.covariate_basis(rng.standard_normal((n, 3))))
    df = float(n - 2)
    want = orc.threshold_scan(d, ytil, df, 1.0)
    t_ref = orc.t_from_r(want["full_r"][want["skip"] == 0], df)
    packed, bpm = _packed(d)
    got = {}
    with DeviceContext(0) as ctx:
        for f64 in (False, True):
            ctx.set_f64_panel(f64)
            ctx.set_panel(ytil, np.arange(n, dtype=np.int64), n)
            ctx.set_scan(df, _native.PG_MODE_FULL, None)
            got[f64] = ctx.scan(_native.PG_GENO_BED, packed, bpm).t_rows
            ctx.set_scan(df, _native.PG_MODE_THRESHOLD, np.full(p, orc.premask_abs_r(0.05, df)))
            thr = ctx.scan(_native.PG_GENO_BED, packed, bpm)
            if f64:  # candidates: exact fp64 t of the oracle at every premask hit
                rows_ok = np.nonzero(want["skip"] == 0)[0]
                pos = np.searchsorted(rows_ok, thr.cand_rows)
                np.testing.assert_allclose(thr.cand_t, t_ref[pos, thr.cand_cols], rtol=1e-11, atol=1e-12)
    err32 = np.abs(got[False] - t_ref).max()
    err64 = np.abs(got[True] - t_ref).max()
    assert err64 <= 1e-11 * max(1.0, np.abs(t_ref).max()), err64
    assert err64 < err32 / 1000  # the lo level removes the 23-bit quantization error


def test_f64_threshold_equals_oracle_records(tmp_path):
    """Through run_scan: F64 records == the oracle's fp64 threshold scan (membership exact,
    t / p to 1e-11), for a PLINK cohort with covariates and missing calls."""
    rng = np.random.default_rng(8)
    n, m, k = 400, 300, 6
    d = rng.binomial(2, rng.uniform(0.1, 0.9, m)[:, None], size=(m, n)).astype(np.float64)
    d[rng.random((m, n)) < 0.02] = np.nan
    y = rng.standard_normal((n, k))
    y[:, 2] += 0.4 * np.nan_to_num(d[17], nan=1.0)
    cov = rng.standard_normal((n, 2))
    ids = [f"S{i + 1}" for i in range(n)]
    bed, bim, fam = pg.write_bed_trio(tmp_path / "g", d, ids)
    pheno = write_tsv(tmp_path / "p.tsv", ids, [f"ph{j + 1}" for j in range(k)], y)
    covar = write_tsv(tmp_path / "c.tsv", ids, ["c1", "c2"], cov)
    spec = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=bed, bim_path=bim, fam_path=fam)
    pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, covar_path=covar, out_path=tmp_path / "o.tsv",
                              p_threshold=0.05, precision=pg.Precision.F64, summary_to_stderr=False))
    recs = pg.load_association_records(tmp_path / "o.tsv")
    ytil, _ = orc.standardized_panel(y, orc.covariate_basis(cov))
    want = orc.threshold_scan(d, ytil, float(n - 2), 0.05)
    assert [(r.pos - 1, int(r.phenotype[2:]) - 1) for r in recs] == list(zip(want["rows"], want["cols"]))
    np.testing.assert_allclose([r.t for r in recs], want["t"], rtol=1e-11)
    np.testing.assert_allclose([r.p for r in recs], want["p"], rtol=1e-7)  # libm lgamma / log / exp


def test_f64_matches_reference_golden_s1(tmp_path):
    """The reference's own F64 output for s1 (missing calls and phenotypes, 3 covariates)."""
    g = np.load(GOLD / "s1.npz")
    paths = regenerate("s1", tmp_path)
    spec = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=paths["bed_path"], bim_path=paths["bim_path"],
                         fam_path=paths["fam_path"])
    pg.run_scan(pg.ScanConfig(source=spec, pheno_path=paths["pheno_path"], covar_path=paths["covar_path"],
                              out_path=tmp_path / "o.tsv", p_threshold=1.0, precision=pg.Precision.F64,
                              summary_to_stderr=False))
    recs = pg.load_association_records(tmp_path / "o.tsv")
    key = {(int(r.id[3:]) - 1, int(r.phenotype[2:]) - 1): r for r in recs}
    rows, cols, t, p = g["thr_f64_rows"], g["thr_f64_cols"], g["thr_f64_t"], g["thr_f64_p"]  # the golden's hits
    assert all((a, b) in key for a, b in zip(rows.tolist(), cols.tolist()))
    got_t = np.array([key[(a, b)].t for a, b in zip(rows.tolist(), cols.tolist())])
    got_p = np.array([key[(a, b)].p for a, b in zip(rows.tolist(), cols.tolist())])
    np.testing.assert_allclose(got_t, t, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(got_p, p, rtol=1e-7)  # libm lgamma / log / exp


@pytest.mark.parametrize("source", ["bgen8", "dense_int"])
def test_f64_panel_dosage_sources(source, tmp_path):
    rng = np.random.default_rng(3)
    n, m, k = 257, 90, 5
    ids = [f"S{i + 1}" for i in range(n)]
    if source == "bgen8":
        from bgen_fixture import write_bgen

        d = np.round(rng.uniform(0, 2, (m, n)) * 255 / 2) * 2 / 255  # on the 8-bit grid
        d[rng.random(d.shape) < 0.05] = np.nan
        spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=write_bgen(tmp_path / "g.bgen", d, ids, bits=8))
        src = pg.BgenSource(tmp_path / "g.bgen")
        d = src.read_marker_batch(0, m).dosages  # what the reference reader decodes
        src.close()
    else:
        d = rng.integers(0, 3, (m, n)).astype(np.float64)
        d[rng.random(d.shape) < 0.05] = np.nan
        np.save(tmp_path / "g.npy", d)
        (tmp_path / "s.txt").write_text("\n".join(ids) + "\n")
        spec = pg.SourceSpec(pg.GenotypeFormat.DENSE, dense_path=tmp_path / "g.npy", sample_id_path=tmp_path / "s.txt")
    y = rng.standard_normal((n, k))
    pheno = write_tsv(tmp_path / "p.tsv", ids, [f"ph{j + 1}" for j in range(k)], y)
    pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, out_path=tmp_path / "f.bin",
                              output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64, summary_to_stderr=False))
    t, _, _ = pg.read_full_matrix(tmp_path / "f.bin")
    ytil, _ = orc.standardized_panel(y, orc.covariate_basis(np.zeros((n, 0))))
    want = orc.threshold_scan(d, ytil, float(n - 2), 1.0)
    t_ref = orc.t_from_r(want["full_r"][want["skip"] == 0], float(n - 2))
    np.testing.assert_allclose(t, t_ref, rtol=1e-10, atol=1e-12)

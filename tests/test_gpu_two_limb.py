"""Two-limb premask of PLINK THRESHOLD / TOPK scans (assoc_i8_kernel<kFused2> +
refine_two_limb): the GEMM runs two of the three panel limbs, the premask is widened by the
rigorous bound |sum q0 u| <= ||q0_p||_2 ||u_m||_2, and every candidate gets the deferred limb
added exactly before its fp64 r / t / p. Outputs must be bitwise identical to the
three-limb GEMM (PG_TWO_LIMB=0), whatever the allele frequencies (the bound is widest for
rare variants), missing calls (side GEMM), sample subsets or batch sizes."""
import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from oracle import scan_oracle as orc
from paper_2604_21095_b200 import _native
from paper_2604_21095_b200._device import DeviceContext
from test_gpu_engine import dataset, scan

pytestmark = pytest.mark.gpu


def _cohort(rng, m, n, p):
    af = np.concatenate([rng.uniform(0.001, 0.01, m // 4), rng.uniform(0.05, 0.95, m - m // 4)])
    d = rng.binomial(2, af[:, None], size=(m, n)).astype(np.float64)
    y = rng.standard_normal((n, p))
    y[:, 1] += 0.3 * d[m // 2]
    return d, y


@pytest.mark.parametrize("mode", ["thr", "thr_open", "topk"])
@pytest.mark.parametrize("missing", [False, True])
def test_two_limb_equals_three_limb_bitwise(mode, missing, tmp_path, monkeypatch):
    rng = np.random.default_rng(11 + 3 * missing)
    n, m, p = 611, 1500, 40
    d, y = _cohort(rng, m, n, p)
    if missing:
        rows = rng.random(m) < 0.3
        d[rows] = np.where(rng.random((rows.sum(), n)) < 0.03, np.nan, d[rows])
    spec, pheno, _, root = dataset(tmp_path, d, y)
    keep = root / "keep.txt"
    keep.write_text("\n".join(f"S{i + 1}" for i in range(40, n)) + "\n")
    kw = {"thr": dict(p_threshold=1e-2), "thr_open": dict(p_threshold=1.0),
          "topk": dict(output_mode=pg.OutputMode.TOPK, top_k=7)}[mode]
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("PG_TWO_LIMB", flag)
        for db in (512, 1500):
            path = root / f"o{flag}_{db}.tsv"
            scan(spec, pheno, path, device_batch=db, keep_path=keep, **kw)
            out[flag, db] = path.read_bytes()
    assert len(set(out.values())) == 1
    assert out["1", 512].count(b"\n") > 1


def test_two_limb_candidates_match_oracle():
    """Device level: the refined candidates' t == the oracle's fp64 t, and the hit set (p <= thr)
    equals the oracle's, including rare variants whose premask bound is widest."""
    rng = np.random.default_rng(5)
    n, m, p = 1003, 800, 96
    d, y = _cohort(rng, m, n, p)
    ytil, _ = orc.standardized_panel(y, orc.covariate_basis(np.zeros((n, 0))))
    df = float(n - 2)
    thr = 1e-3
    want = orc.threshold_scan(d, ytil, df, thr)
    codes = np.select([d == 2, d == 1, d == 0], [0, 2, 3]).astype(np.uint8)
    bpm = (n + 3) // 4
    codes = np.pad(codes, ((0, 0), (0, 4 * bpm - n)))
    q = codes.reshape(m, bpm, 4)
    packed = (q[:, :, 0] | (q[:, :, 1] << 2) | (q[:, :, 2] << 4) | (q[:, :, 3] << 6)).astype(np.uint8)
    res = {}
    with DeviceContext(0) as ctx:
        ctx.set_panel(ytil, np.arange(n, dtype=np.int64), n)
        for two in (True, False):
            ctx.set_two_limb_premask(two)
            ctx.set_scan(df, _native.PG_MODE_THRESHOLD, np.full(p, orc.premask_abs_r(thr, df)))
            res[two] = ctx.scan(_native.PG_GENO_BED, packed, bpm)
    a, b = res[True], res[False]
    ka = a.cand_p <= thr
    kb = b.cand_p <= thr
    for f in ("cand_rows", "cand_cols", "cand_r", "cand_t", "cand_p"):
        assert np.array_equal(getattr(a, f)[ka], getattr(b, f)[kb])
    assert a.n_candidates >= b.n_candidates  # the widened premask admits a few more pairs
    assert np.array_equal(a.cand_rows[ka], want["rows"]) and np.array_equal(a.cand_cols[ka], want["cols"])
    np.testing.assert_allclose(a.cand_t[ka], want["t"], rtol=1e-4)


@pytest.mark.parametrize("mode", ["thr", "topk"])
def test_wide_two_limb_bgen8_equals_three_limb_bitwise(mode, tmp_path, monkeypatch):
    """BGEN-8 through the 240-row two-limb wide GEMM (kWide3Two, deferred q0 limb for the digit
    rows and the missing row) == the three-limb kWide3 GEMM, record for record."""
    from bgen_fixture import write_bgen
    from conftest_helpers import write_tsv

    rng = np.random.default_rng(29)
    n, m, k = 333, 500, 12
    ids = [f"S{i + 1}" for i in range(n)]
    af = rng.uniform(0.02, 0.9, m)
    d = rng.binomial(2, af[:, None], size=(m, n)).astype(np.float64)
    frac = rng.random((m, n)) < 0.3
    d[frac] = np.clip(d[frac] + rng.normal(0, 0.3, frac.sum()), 0, 2)
    d[rng.random((m, n)) < 0.05] = np.nan
    y = rng.standard_normal((n, k))
    y[:, 3] += 0.4 * np.nan_to_num(d[7], nan=1.0)
    pheno = write_tsv(tmp_path / "p.tsv", ids, [f"ph{j + 1}" for j in range(k)], y)
    spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=write_bgen(tmp_path / "g.bgen", d, ids, bits=8))
    kw = dict(p_threshold=0.02) if mode == "thr" else dict(output_mode=pg.OutputMode.TOPK, top_k=9)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("PG_TWO_LIMB", flag)
        path = tmp_path / f"o{flag}.tsv"
        pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, out_path=path, summary_to_stderr=False,
                                  device_batch=300, **kw))
        out[flag] = path.read_bytes()
    assert out["1"] == out["0"] and out["1"].count(b"\n") > 1


def test_two_limb_extension_mode_and_covariates_bitwise(tmp_path, monkeypatch):
    """Extension mode (residualize_genotypes, adjusted df: the K5 basis GEMM stays three-limb and
    rewrites V_m) with covariates and missing calls: two-limb records == three-limb records."""
    from conftest_helpers import write_tsv

    rng = np.random.default_rng(71)
    n, m, p = 401, 900, 16
    d, y = _cohort(rng, m, n, p)
    rows = rng.random(m) < 0.2
    d[rows] = np.where(rng.random((rows.sum(), n)) < 0.04, np.nan, d[rows])
    spec, pheno, _, root = dataset(tmp_path, d, y)
    ids = [f"S{i + 1}" for i in range(n)]
    covar = write_tsv(root / "c.tsv", ids, ["c1", "c2", "c3"], rng.standard_normal((n, 3)))
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("PG_TWO_LIMB", flag)
        path = root / f"e{flag}.tsv"
        scan(spec, pheno, path, covar=covar, p_threshold=0.01, residualize_genotypes=True,
             df_mode=pg.DfMode.ADJUSTED, device_batch=400)
        out[flag] = path.read_bytes()
    assert out["1"] == out["0"] and out["1"].count(b"\n") > 1


@pytest.mark.parametrize("source", ["bgen16", "dense_real"])
def test_wide4_two_limb_equals_three_limb_bitwise(source, tmp_path, monkeypatch):
    """4-row wide digits (BGEN-16, real-valued dense) through the 256-row two-limb GEMM
    (kWide4Two) == the three-limb kWide GEMM, record for record (THRESHOLD and TOPK)."""
    from conftest_helpers import write_tsv

    rng = np.random.default_rng(91)
    n, m, k = 271, 300, 10
    ids = [f"S{i + 1}" for i in range(n)]
    d = np.clip(rng.binomial(2, rng.uniform(0.05, 0.9, m)[:, None], size=(m, n)) +
                rng.normal(0, 0.2, (m, n)), 0, 2)
    d[rng.random((m, n)) < 0.05] = np.nan
    y = rng.standard_normal((n, k))
    y[:, 1] += 0.5 * np.nan_to_num(d[9], nan=1.0)
    pheno = write_tsv(tmp_path / "p.tsv", ids, [f"ph{j + 1}" for j in range(k)], y)
    if source == "bgen16":
        from bgen_fixture import write_bgen

        spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=write_bgen(tmp_path / "g.bgen", d, ids, bits=16))
    else:
        np.save(tmp_path / "g.npy", d)
        (tmp_path / "s.txt").write_text("\n".join(ids) + "\n")
        spec = pg.SourceSpec(pg.GenotypeFormat.DENSE, dense_path=tmp_path / "g.npy", sample_id_path=tmp_path / "s.txt")
    for kw in (dict(p_threshold=0.02), dict(output_mode=pg.OutputMode.TOPK, top_k=6)):
        out = {}
        for flag in ("1", "0"):
            monkeypatch.setenv("PG_TWO_LIMB", flag)
            path = tmp_path / f"o{flag}.tsv"
            pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, out_path=path, summary_to_stderr=False,
                                      device_batch=128, **kw))
            out[flag] = path.read_bytes()
        assert out["1"] == out["0"] and out["1"].count(b"\n") > 1

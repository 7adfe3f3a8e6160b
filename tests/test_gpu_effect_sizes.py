"""Device effect sizes (north star: "beta / t / -log10 p must agree within a stated
relative tolerance") against the reference's own per-pair OLS.

The reference engine writes R T P only (output.py:29-43); beta exists in its OLS oracle
(oracle.ols_single, oracle.py:35-90). tests/golden/ols.npz holds ols_single beta / se / t
for sampled pairs of the golden cohorts s1 and c1, computed by the reference itself
(tests/golden/make_golden.py make_ols). The device beta is the slope of y_res on g: with
--residualize-genotypes and --df-mode adjusted that is the OLS estimate of y ~ 1 + C + g
(Frisch-Waugh-Lovell), in paper mode that of y_res ~ 1 + g.

Tolerances (written here, as the north star asks), the reference's own t bar
|dt| <= 1e-4 max(1, |t|) (tests/test_engine.py:298-308) carried over to beta = t * se:
|d beta| <= 1e-4 max(|beta|, se) and |d se| <= 1e-4 se."""
from pathlib import Path

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from paper_2604_21095_b200 import output
from scan_fixtures import GOLD, regenerate

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def _spec(paths):
    return pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=paths["bed_path"], bim_path=paths["bim_path"],
                         fam_path=paths["fam_path"])


def _run(paths, out, **kw):
    return pg.run_scan(pg.ScanConfig(source=_spec(paths), pheno_path=paths["pheno_path"],
                                     covar_path=paths["covar_path"], out_path=out, summary_to_stderr=False,
                                     effect_sizes=True, **kw))


MODES = {
    "paper": {},
    "adj": {"residualize_genotypes": True, "df_mode": pg.DfMode.ADJUSTED},
}


@pytest.mark.parametrize("name", ["s1", "c1"])
@pytest.mark.parametrize("mode", ["paper", "adj"])
def test_full_beta_matches_reference_ols(tmp_path, name, mode):
    paths = regenerate(name, tmp_path)
    g = np.load(GOLD / "ols.npz")
    out = tmp_path / "full.bin"
    _run(paths, out, output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64, **MODES[mode])
    t, lines, names = pg.read_full_matrix(out)
    beta = output.read_full_beta(out)
    assert beta.shape == t.shape
    src = np.array([int(ln.split("\t")[0]) for ln in lines])
    row_of = {s: i for i, s in enumerate(src.tolist())}
    rows = np.array([row_of[r] for r in g[f"{name}_rows"].tolist()])
    cols = g[f"{name}_cols"]
    got_b = beta[rows, cols]
    want_b, want_se, want_t = (g[f"{name}_{k}_{mode}"] for k in ("beta", "se", "t"))
    err = np.abs(got_b - want_b) / np.maximum(np.abs(want_b), want_se)
    assert err.max() <= RTOL, err.max()
    dt = np.abs(t[rows, cols] - want_t) / np.maximum(1.0, np.abs(want_t))
    assert dt.max() <= RTOL, dt.max()
    print(f"{name}/{mode}: max |d beta| / max(|beta|, se) = {err.max():.2e}, max rel |dt| = {dt.max():.2e} "
          f"over {err.size} pairs")


@pytest.mark.parametrize("mode", ["paper", "adj"])
def test_record_se_matches_reference_ols(tmp_path, mode):
    """BETA / SE of the record sidecar vs ols_single on every golden s1 pair (open threshold)."""
    paths = regenerate("s1", tmp_path)
    g = np.load(GOLD / "ols.npz")
    out = tmp_path / "all.tsv"
    _run(paths, out, p_threshold=1.0, precision=pg.Precision.F64, **MODES[mode])
    recs = pg.load_association_records(out)
    beta, se = output.load_effect_sizes(out)
    at = {(int(r.id[3:]) - 1, int(r.phenotype[2:]) - 1): i for i, r in enumerate(recs)}
    idx = np.array([at[(a, b)] for a, b in zip(g["s1_rows"].tolist(), g["s1_cols"].tolist())])
    want_b, want_se = g[f"s1_beta_{mode}"], g[f"s1_se_{mode}"]
    assert (np.abs(beta[idx] - want_b) / np.maximum(np.abs(want_b), want_se)).max() <= RTOL
    assert (np.abs(se[idx] - want_se) / want_se).max() <= RTOL


def test_threshold_and_topk_sidecars_aligned(tmp_path):
    """<out>.beta.tsv lines follow the record lines (THRESHOLD, TOPK, f32 and f64), beta/se == t,
    and the records' beta equals the FULL beta matrix of the same scan."""
    paths = regenerate("s1", tmp_path)
    full = tmp_path / "full.bin"
    _run(paths, full, output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64)
    bmat = output.read_full_beta(full)
    _, lines, names = pg.read_full_matrix(full)
    row_of = {ln.split("\t")[2]: i for i, ln in enumerate(lines)}
    col_of = {nm: j for j, nm in enumerate(names)}
    for kw in ({"p_threshold": 1e-2}, {"p_threshold": 1.0, "precision": pg.Precision.F64},
               {"output_mode": pg.OutputMode.TOPK, "top_k": 7, "device_batch": 256}):
        out = tmp_path / "rec.tsv"
        _run(paths, out, **kw)
        recs = pg.load_association_records(out)
        beta, se = output.load_effect_sizes(out)
        assert beta.size == se.size == len(recs) > 0
        t = np.array([r.t for r in recs])
        np.testing.assert_allclose(beta / se, t, rtol=1e-12)
        want = np.array([bmat[row_of[r.id], col_of[r.phenotype]] for r in recs])
        np.testing.assert_allclose(beta, want, rtol=1e-12 if kw.get("precision") else 1e-6)


def test_effect_sizes_off_by_default_and_outputs_unchanged(tmp_path):
    """Effect sizes are opt-in: default outputs stay byte-identical to the reference format."""
    paths = regenerate("s1", tmp_path)
    a, b = tmp_path / "a.tsv", tmp_path / "b.tsv"
    pg.run_scan(pg.ScanConfig(source=_spec(paths), pheno_path=paths["pheno_path"], covar_path=paths["covar_path"],
                              out_path=a, summary_to_stderr=False, p_threshold=1e-3))
    _run(paths, b, p_threshold=1e-3)
    assert a.read_bytes() == b.read_bytes()
    assert not output.beta_sidecar(a).exists() and output.beta_sidecar(b).exists()

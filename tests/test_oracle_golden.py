"""Pin the CPU oracle against golden outputs of the reference itself
(tests/golden/*, produced by tests/golden/make_golden.py from /root/reference).

CPU only. If the oracle matches the reference on these vectors, the GPU parity
tests that compare the device path with the oracle inherit the reference as
their ground truth."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import scan_oracle as orc

GOLD = Path(__file__).parent / "golden"


def nan_eq(a, b):
    return np.array_equal(np.nan_to_num(a, nan=-7.0), np.nan_to_num(b, nan=-7.0))


def test_decode_fixtures():
    g = np.load(GOLD / "decode.npz")
    for i in range(6):
        got = orc.decode_bed(g[f"fixed{i}_bytes"], int(g[f"fixed{i}_n"]))[0]
        assert nan_eq(got, g[f"fixed{i}_dosage"])
    assert nan_eq(orc.decode_bed(g["rand_packed"], int(g["rand_n"])), g["rand_dosage"])


def test_pvalues_match_reference():
    g = np.load(GOLD / "pvalues.npz")
    for i, df in enumerate(g["dfs"]):
        np.testing.assert_allclose(orc.p_from_t(g["t"], df), g["p"][i], rtol=1e-13, atol=0)
    np.testing.assert_allclose(orc.reg_inc_beta(g["ib_a"], g["ib_b"], g["ib_x"]), g["ib"], rtol=1e-13, atol=1e-300)
    for k, (pt, df) in enumerate(g["crit_cases"]):
        assert orc.t_threshold_for_p(pt, df) == pytest.approx(g["crit"][k], rel=1e-12)
    for i, df in enumerate((2.0, 11.0, 22998.0)):
        assert nan_eq(orc.t_from_r(g["r"], df), g["t_from_r"][i])


def test_prepare_matches_reference():
    g = np.load(GOLD / "prepare.npz")
    mat, af, miss, var, skip = orc.prepare(g["dosages"])
    np.testing.assert_allclose(mat, g["matrix"], atol=1e-12)
    assert nan_eq(af, g["af"])
    assert np.array_equal(miss, g["missing"])
    assert np.array_equal(skip, g["skip"])
    np.testing.assert_allclose(var, g["variance"], rtol=1e-12)


def _cohort_arrays(name):
    from scan_fixtures import load_cohort

    return load_cohort(name)


@pytest.mark.parametrize("name", ["s1", "c1"])
def test_simulator_reproduces_reference_cohort(tmp_path, name):
    from scan_fixtures import regenerate

    meta = json.loads((GOLD / f"{name}.json").read_text())
    paths = regenerate(name, tmp_path)
    import hashlib

    for key, digest in meta["sha256"].items():
        assert hashlib.sha256(Path(paths[key]).read_bytes()).hexdigest() == digest, key


def test_oracle_scan_matches_reference_s1(tmp_path):
    from scan_fixtures import oracle_inputs

    dos, ytil, df, _ = oracle_inputs("s1", tmp_path)
    g = np.load(GOLD / "s1.npz")
    res = orc.threshold_scan(dos, ytil, df, 1.0)
    assert np.array_equal(res["rows"], g["all_f64_rows"]) and np.array_equal(res["cols"], g["all_f64_cols"])
    np.testing.assert_allclose(res["t"], g["all_f64_t"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(res["p"], g["all_f64_p"], rtol=1e-8)
    res3 = orc.threshold_scan(dos, ytil, df, 1e-3)
    assert set(zip(res3["rows"], res3["cols"])) == set(zip(g["thr_f64_rows"], g["thr_f64_cols"]))


def test_oracle_scan_matches_reference_c1(tmp_path):
    from scan_fixtures import oracle_inputs

    dos, ytil, df, _ = oracle_inputs("c1", tmp_path)
    g = np.load(GOLD / "c1.npz")
    res = orc.threshold_scan(dos, ytil, df, 1e-4)
    assert set(zip(res["rows"].tolist(), res["cols"].tolist())) == set(
        zip(g["thr_f64_rows"].tolist(), g["thr_f64_cols"].tolist()))
    order = np.lexsort((res["cols"], res["rows"]))
    np.testing.assert_allclose(res["t"][order], g["thr_f64_t"], rtol=1e-9)
    sub = g["full_f64_rows"]
    np.testing.assert_allclose(orc.t_from_r(res["full_r"][sub], df), g["full_f64_t"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("name", ["s1", "c1"])
def test_oracle_effect_sizes_match_reference_ols(tmp_path, name):
    """The oracle's beta / se (slope of y_res on g) == the reference's own per-pair OLS
    (oracle.ols_single) on the golden cohorts: y ~ 1 + C + g in extension mode with the
    adjusted df, y_res ~ 1 + g in paper mode."""
    from scan_fixtures import panel_inputs

    dos, y, c, q, _ = panel_inputs(name, tmp_path)
    g = np.load(GOLD / "ols.npz")
    rows, cols = g[f"{name}_rows"], g[f"{name}_cols"]
    n = y.shape[0]
    ytil, _ = orc.standardized_panel(y, q)
    sd = orc.panel_sd(y, q)
    for mode, gq, df in (("paper", None, float(n - 2)), ("adj", q, float(n - q.shape[1] - 1))):
        mat, _, _, var, _ = orc.prepare(dos[np.unique(rows)], gq)
        idx = np.searchsorted(np.unique(rows), rows)
        r = np.einsum("kn,nk->k", mat[idx], ytil[:, cols]) / n
        beta, se = orc.effect_sizes(r, var[idx], sd[cols], df)
        np.testing.assert_allclose(beta, g[f"{name}_beta_{mode}"], rtol=1e-9, atol=1e-14)
        np.testing.assert_allclose(se, g[f"{name}_se_{mode}"], rtol=1e-9)
        np.testing.assert_allclose(beta / se, g[f"{name}_t_{mode}"], rtol=1e-9, atol=1e-12)

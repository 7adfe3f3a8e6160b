"""Parity at the BASELINE sizes (N = 23,000 samples, P = 20,480 phenotypes; fewer markers):
the device FULL statistics for a sample of markers equal the oracle's float64 restatement
of the reference path (|dt| <= 1e-4 max(1, |t|)), and the THRESHOLD hits equal the
brute-force p <= 1e-4 filter of the same FULL matrix away from the threshold
(size-independent properties of the full-size contraction: K = 23,040, 80 phenotype tiles)."""
import numpy as np
import pytest

from oracle import scan_oracle as orc

pytestmark = pytest.mark.gpu

N, P, M = 23_000, 20_480, 1_024


@pytest.fixture(scope="module")
def full_size():
    from paper_2604_21095_b200 import _native
    from paper_2604_21095_b200._device import DeviceContext

    rng = np.random.default_rng(2604)
    y = rng.standard_normal((N, P), dtype=np.float32).astype(np.float64)
    y -= y.mean(axis=0)
    y /= np.sqrt((y * y).mean(axis=0))
    af = rng.uniform(0.05, 0.95, M)
    g = rng.binomial(2, af[:, None], size=(M, N)).astype(np.uint8)
    miss = rng.random((M, N)) < 0.01
    miss[: M // 2] = False  # half the markers without missing calls
    codes = np.array([3, 2, 0], np.uint8)[g]
    codes[miss] = 1
    bpm = (N + 3) // 4
    codes = np.pad(codes, ((0, 0), (0, bpm * 4 - N))).reshape(M, bpm, 4)
    packed = (codes[:, :, 0] | (codes[:, :, 1] << 2) | (codes[:, :, 2] << 4) | (codes[:, :, 3] << 6)).astype(np.uint8)
    ctx = DeviceContext(0)
    ctx.set_panel(y, np.arange(N, dtype=np.int64), N)
    df = float(N - 2)
    yield ctx, y, packed, df, _native
    ctx.close()


def test_full_statistics_match_oracle(full_size):
    ctx, y, packed, df, _native = full_size
    ctx.set_scan(df, _native.PG_MODE_FULL, None)
    res = ctx.scan(_native.PG_GENO_BED, packed, packed.shape[1])
    t_dev = res.t_rows
    assert t_dev.shape == (M, P)
    pick = np.r_[0:4, M // 2:M // 2 + 4, M - 4:M]  # markers with and without missing calls
    dos = orc.decode_bed(packed[pick], N)
    ref = orc.threshold_scan(dos, y, df, 1.0)  # every pair: (rows, cols, r, t, p)
    t_ref = np.zeros((pick.size, P))
    t_ref[ref["rows"], ref["cols"]] = ref["t"]
    rel = np.abs(t_dev[pick] - t_ref) / np.maximum(1.0, np.abs(t_ref))
    assert rel.max() <= 1e-4


def test_threshold_hits_equal_full_filter(full_size):
    from paper_2604_21095_b200.engine import threshold_premask
    from paper_2604_21095_b200.kernel import t_threshold_for_p

    ctx, y, packed, df, _native = full_size
    ctx.set_scan(df, _native.PG_MODE_FULL, None)
    t_full = ctx.scan(_native.PG_GENO_BED, packed, packed.shape[1]).t_rows
    ctx.set_scan(df, _native.PG_MODE_THRESHOLD, np.full(P, threshold_premask(1e-4, df)))
    res = ctx.scan(_native.PG_GENO_BED, packed, packed.shape[1])
    hits = set(zip(res.cand_rows[res.cand_p <= 1e-4].tolist(), res.cand_cols[res.cand_p <= 1e-4].tolist()))
    t_crit = t_threshold_for_p(1e-4, df)
    a = np.abs(t_full)
    sure_in = set(zip(*np.nonzero(a > t_crit * (1 + 1e-4))))
    sure_out = set(zip(*np.nonzero(a < t_crit * (1 - 1e-4))))
    assert sure_in <= hits
    assert not (hits & sure_out)
    assert 0.5e-4 * M * P < len(hits) < 2e-4 * M * P  # null: ~1e-4 of the tests


@pytest.mark.parametrize("p", [255, 700, 1300])
def test_odd_tile_counts_match_oracle(p):
    """Phenotype-tile counts that do not divide the raster group (1, 3, 6 tiles of 256) and a
    marker count that leaves partial genotype tiles: every (marker, phenotype) visited once."""
    from paper_2604_21095_b200 import _native
    from paper_2604_21095_b200._device import DeviceContext

    rng = np.random.default_rng(p)
    n, m = 333, 1111
    y = rng.standard_normal((n, p))
    y -= y.mean(axis=0)
    y /= np.sqrt((y * y).mean(axis=0))
    g = rng.binomial(2, rng.uniform(0.1, 0.9, (m, 1)), size=(m, n)).astype(np.uint8)
    bpm = (n + 3) // 4
    codes = np.pad(np.array([3, 2, 0], np.uint8)[g], ((0, 0), (0, bpm * 4 - n))).reshape(m, bpm, 4)
    packed = (codes[:, :, 0] | (codes[:, :, 1] << 2) | (codes[:, :, 2] << 4) | (codes[:, :, 3] << 6)).astype(np.uint8)
    with DeviceContext(0) as ctx:
        ctx.set_panel(y, np.arange(n, dtype=np.int64), n)
        ctx.set_scan(float(n - 2), _native.PG_MODE_FULL, None)
        t_dev = ctx.scan(_native.PG_GENO_BED, packed, bpm).t_rows
    ref = orc.threshold_scan(orc.decode_bed(packed, n), y, float(n - 2), 1.0)
    t_ref = np.zeros((m, p))
    t_ref[ref["rows"], ref["cols"]] = ref["t"]
    ok = ref["skip"] == 0
    t_ok = t_dev[ok] if t_dev.shape[0] == m else t_dev  # FULL rows may list non-skipped markers only
    rel = np.abs(t_ok - t_ref[ok]) / np.maximum(1.0, np.abs(t_ref[ok]))
    assert rel.max() <= 1e-4


def test_k_sliced_extension_mode_through_engine(tmp_path):
    """N = 140,000 (> one int32-exact slice) through the engine with covariates and
    --residualize-genotypes: the side GEMM K5 and the main contraction both run K-sliced;
    t equals the oracle's FWL restatement (adjusted df)."""
    import paper_2604_21095_b200 as pg
    from conftest_helpers import write_tsv

    rng = np.random.default_rng(1400)
    n, m, p = 140_000, 24, 3
    ids = [f"S{i + 1}" for i in range(n)]
    g = rng.binomial(2, rng.uniform(0.1, 0.9, (m, 1)), size=(m, n)).astype(np.float64)
    c = rng.standard_normal((n, 2))
    y = c @ rng.standard_normal((2, p)) + rng.standard_normal((n, p))
    y[:, 0] += 0.03 * g[5]
    bed, bim, fam = pg.write_bed_trio(tmp_path / "g", g, ids)
    pheno = write_tsv(tmp_path / "p.tsv", ids, [f"ph{j}" for j in range(p)], y)
    covar = write_tsv(tmp_path / "c.tsv", ids, ["c1", "c2"], c)
    spec = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=bed, bim_path=bim, fam_path=fam)
    pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, covar_path=covar, out_path=tmp_path / "o.tsv",
                              p_threshold=1.0, precision=pg.Precision.F64, summary_to_stderr=False,
                              residualize_genotypes=True, df_mode=pg.DfMode.ADJUSTED))
    recs = pg.load_association_records(tmp_path / "o.tsv")
    q = orc.covariate_basis(c)
    ytil, _ = orc.standardized_panel(y, q)
    mat, *_ = orc.prepare(g, q)
    r, _ = orc.correlate(mat, ytil)
    t_ref = orc.t_from_r(r, float(n - q.shape[1] - 1))
    got = np.array([x.t for x in recs]).reshape(m, p)
    rel = np.abs(got - t_ref) / np.maximum(1.0, np.abs(t_ref))
    assert rel.max() <= 1e-4
    assert abs(t_ref[5, 0]) > 5

"""Device scans over BGEN (8/16-bit, missing calls: balanced-ternary rows + missing
row) and dense NPY sources vs reference goldens and vs the PLINK path."""
from pathlib import Path

import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from conftest_helpers import write_tsv

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


def _records(path):
    recs = pg.load_association_records(path)
    return recs, np.array([r.t for r in recs]), np.array([r.p for r in recs])


@pytest.mark.parametrize("bits", [8, 16])
def test_bgen_scan_matches_reference(bits, tmp_path):
    g = np.load(GOLD / "bgen.npz")
    spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=GOLD / f"bgen{bits}.bgen")
    pg.run_scan(pg.ScanConfig(source=spec, pheno_path=GOLD / "bgen_pheno.tsv", out_path=tmp_path / "o.tsv",
                              p_threshold=1.0, precision=pg.Precision.F64, summary_to_stderr=False))
    recs, t, p = _records(tmp_path / "o.tsv")
    rows = np.array([int(r.id[2:]) - 1 for r in recs])
    cols = np.array([int(r.phenotype[2:]) - 1 for r in recs])
    assert np.array_equal(rows, g[f"b{bits}_rows"]) and np.array_equal(cols, g[f"b{bits}_cols"])
    assert all((r.counted_allele, r.other_allele) == ("B", "A") for r in recs)  # BGEN counts allele2
    np.testing.assert_allclose([r.af for r in recs], g[f"b{bits}_af"], rtol=1e-12)
    dt = np.abs(t - g[f"b{bits}_t"]) / np.maximum(1, np.abs(g[f"b{bits}_t"]))
    assert dt.max() <= 1e-5
    lp, lr = -np.log10(p), -np.log10(g[f"b{bits}_p"])
    assert (np.abs(lp - lr) / np.maximum(1, lr)).max() <= 1e-4


def test_dense_integral_equals_plink_exactly(tmp_path):
    rng = np.random.default_rng(24)
    d = rng.integers(0, 3, size=(40, 50)).astype(np.float64)
    d[rng.random(d.shape) < 0.05] = np.nan
    y = rng.standard_normal((50, 3))
    ids = [f"S{i + 1}" for i in range(50)]
    bed, bim, fam = pg.write_bed_trio(tmp_path / "g", d, ids)
    pheno = write_tsv(tmp_path / "p.tsv", ids, ["ph1", "ph2", "ph3"], y)
    np.save(tmp_path / "g.npy", d.T)
    (tmp_path / "s.txt").write_text("\n".join(ids) + "\n")
    plink = pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=bed, bim_path=bim, fam_path=fam)
    dense = pg.SourceSpec(pg.GenotypeFormat.DENSE, dense_path=tmp_path / "g.npy", sample_id_path=tmp_path / "s.txt",
                          dense_orientation=pg.DenseOrientation.SAMPLES_BY_MARKERS)
    for spec, out in ((plink, "a.tsv"), (dense, "b.tsv")):
        pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, out_path=tmp_path / out, p_threshold=1.0,
                                  precision=pg.Precision.F64, summary_to_stderr=False))
    a = pg.load_association_records(tmp_path / "a.tsv")
    b = pg.load_association_records(tmp_path / "b.tsv")
    assert len(a) == len(b)
    for ra, rb in zip(a, b):  # same integers through the same exact contraction -> identical bits
        assert (ra.t, ra.p, ra.r, ra.af, ra.missing_count) == (rb.t, rb.p, rb.r, rb.af, rb.missing_count)


def test_dense_fractional_dosages(tmp_path):
    """Real-valued dosages take the 2^-17 fixed-point ternary path; compare with the oracle."""
    from oracle import scan_oracle as orc

    rng = np.random.default_rng(31)
    m, n, k = 25, 64, 4
    d = np.clip(rng.binomial(2, 0.4, size=(m, n)) + rng.normal(0, 0.15, size=(m, n)), 0, 2)
    d[rng.random(d.shape) < 0.04] = np.nan
    y = rng.standard_normal((n, k))
    ids = [f"S{i + 1}" for i in range(n)]
    pheno = write_tsv(tmp_path / "p.tsv", ids, [f"ph{j + 1}" for j in range(k)], y)
    np.save(tmp_path / "g.npy", d)
    (tmp_path / "s.txt").write_text("\n".join(ids) + "\n")
    spec = pg.SourceSpec(pg.GenotypeFormat.DENSE, dense_path=tmp_path / "g.npy", sample_id_path=tmp_path / "s.txt")
    pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, out_path=tmp_path / "o.tsv", p_threshold=1.0,
                              precision=pg.Precision.F64, summary_to_stderr=False))
    recs, t, _ = _records(tmp_path / "o.tsv")
    ytil, _ = orc.standardized_panel(y, orc.covariate_basis(np.zeros((n, 0))))
    want = orc.threshold_scan(d, ytil, float(n - 2), 1.0)
    assert len(recs) == want["t"].size
    dt = np.abs(t - want["t"]) / np.maximum(1, np.abs(want["t"]))
    assert dt.max() <= 1e-4


@pytest.mark.parametrize("source", ["bgen8", "bgen16", "dense_real"])
@pytest.mark.parametrize("extension", [False, True])
def test_wide_digits_equal_ternary_bitwise(source, extension, tmp_path, monkeypatch):
    """Wide-digit GEMM (base-255 digits, 3 accumulators; 3 rows per BGEN-8 marker, 4 otherwise) and the balanced-ternary
    planes are two exact integer contractions of the same codes: FULL output identical."""
    rng = np.random.default_rng(77)
    n, m = 130, 70
    ids = [f"S{i + 1}" for i in range(n)]
    d = rng.uniform(0, 2, (m, n))
    d[rng.random(d.shape) < 0.06] = np.nan
    y = rng.standard_normal((n, 5))
    cov = rng.standard_normal((n, 2))
    pheno = write_tsv(tmp_path / "p.tsv", ids, [f"ph{j}" for j in range(5)], y)
    covar = write_tsv(tmp_path / "c.tsv", ids, ["c1", "c2"], cov)
    if source.startswith("bgen"):
        from bgen_fixture import write_bgen

        spec = pg.SourceSpec(pg.GenotypeFormat.BGEN,
                             bgen_path=write_bgen(tmp_path / "g.bgen", d, ids, bits=int(source[4:])))
    else:
        np.save(tmp_path / "g.npy", d)
        (tmp_path / "s.txt").write_text("\n".join(ids) + "\n")
        spec = pg.SourceSpec(pg.GenotypeFormat.DENSE, dense_path=tmp_path / "g.npy", sample_id_path=tmp_path / "s.txt")
    kw = dict(source=spec, pheno_path=pheno, covar_path=covar, output_mode=pg.OutputMode.FULL,
              precision=pg.Precision.F64, summary_to_stderr=False, device_batch=40,
              residualize_genotypes=extension, df_mode=pg.DfMode.ADJUSTED if extension else pg.DfMode.PAPER_N_MINUS_2)
    pg.run_scan(pg.ScanConfig(out_path=tmp_path / "wide.bin", **kw))
    monkeypatch.setenv("PANELGWAS_WIDE_DIGITS", "0")
    pg.run_scan(pg.ScanConfig(out_path=tmp_path / "tern.bin", **kw))
    assert (tmp_path / "wide.bin").read_bytes() == (tmp_path / "tern.bin").read_bytes()


def test_wide3_k_sliced_equals_ternary_bitwise(tmp_path, monkeypatch):
    """BGEN-8 at N = 140,000 (> one int32-exact K slice): the 3-row wide GEMM accumulates
    int64 partials slice by slice; FULL output equals the ternary planes' bit for bit."""
    from bgen_fixture import write_bgen

    rng = np.random.default_rng(140)
    n, m = 140_000, 9
    ids = [f"S{i + 1}" for i in range(n)]
    d = rng.uniform(0, 2, (m, n))
    d[rng.random(d.shape) < 0.05] = np.nan
    y = rng.standard_normal((n, 3))
    pheno = write_tsv(tmp_path / "p.tsv", ids, ["a", "b", "c"], y)
    spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=write_bgen(tmp_path / "g.bgen", d, ids, bits=8))
    kw = dict(source=spec, pheno_path=pheno, output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64,
              summary_to_stderr=False)
    pg.run_scan(pg.ScanConfig(out_path=tmp_path / "wide.bin", **kw))
    monkeypatch.setenv("PANELGWAS_WIDE_DIGITS", "0")
    pg.run_scan(pg.ScanConfig(out_path=tmp_path / "tern.bin", **kw))
    assert (tmp_path / "wide.bin").read_bytes() == (tmp_path / "tern.bin").read_bytes()


def test_bgen8_in_place_blocks_equal_host_inflate_with_sample_subset(tmp_path, monkeypatch):
    """All-8-bit BGEN batches are decoded straight from the GPU-inflated blocks (probs at
    10 + n, ploidy at 8); with a --keep / --remove subset and samples missing from the
    phenotype table the FULL output equals the host-inflate path (repacked rows) bit for bit."""
    from bgen_fixture import write_bgen

    rng = np.random.default_rng(808)
    n, m = 157, 90
    ids = [f"S{i + 1}" for i in range(n)]
    d = rng.uniform(0, 2, (m, n))
    d[rng.random(d.shape) < 0.07] = np.nan
    y = rng.standard_normal((n - 5, 4))  # the last 5 genotype samples have no phenotypes
    pheno = write_tsv(tmp_path / "p.tsv", ids[:-5], ["a", "b", "c", "d"], y)
    (tmp_path / "keep.txt").write_text("".join(f"{s}\n" for s in ids[3:140]))
    (tmp_path / "remove.txt").write_text("S10\nS11\n")
    spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=write_bgen(tmp_path / "g.bgen", d, ids, bits=8))
    kw = dict(source=spec, pheno_path=pheno, output_mode=pg.OutputMode.FULL, precision=pg.Precision.F64,
              summary_to_stderr=False, keep_path=tmp_path / "keep.txt", remove_path=tmp_path / "remove.txt",
              device_batch=32)
    pg.run_scan(pg.ScanConfig(out_path=tmp_path / "gpu.bin", **kw))
    monkeypatch.setenv("PANELGWAS_HOST_INFLATE", "1")
    pg.run_scan(pg.ScanConfig(out_path=tmp_path / "host.bin", **kw))
    assert (tmp_path / "gpu.bin").read_bytes() == (tmp_path / "host.bin").read_bytes()
    t, markers, names = pg.read_full_matrix(tmp_path / "gpu.bin")
    assert t.shape == (m, 4) and np.isfinite(t).all()


@pytest.mark.parametrize("m,k,mode", [(7, 5, "full"), (95, 150, "full"), (161, 290, "thr"), (401, 33, "thr")])
def test_wide3t_equals_wide3_bitwise(m, k, mode, tmp_path, monkeypatch):
    """BGEN-8 through the transposed wide GEMM (genotype rows as A, 80 markers and 144
    phenotypes per pair tile, shuffled 3-row recombination) == the kWide3 kernel bit for bit,
    for marker / phenotype counts that leave partial tiles and groups of 10."""
    from bgen_fixture import write_bgen

    rng = np.random.default_rng(m + k)
    n = 211
    ids = [f"S{i + 1}" for i in range(n)]
    d = rng.uniform(0, 2, (m, n))
    hard = rng.random(d.shape) < 0.6
    d[hard] = np.round(d[hard])
    d[rng.random(d.shape) < 0.05] = np.nan
    y = rng.standard_normal((n, k))
    pheno = write_tsv(tmp_path / "p.tsv", ids, [f"ph{j}" for j in range(k)], y)
    spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=write_bgen(tmp_path / "g.bgen", d, ids, bits=8))
    kw = dict(source=spec, pheno_path=pheno, precision=pg.Precision.F64, summary_to_stderr=False, device_batch=256)
    kw.update(output_mode=pg.OutputMode.FULL) if mode == "full" else kw.update(p_threshold=0.05)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("PG_WIDE3T", flag)
        path = tmp_path / f"o{flag}.{'bin' if mode == 'full' else 'tsv'}"
        pg.run_scan(pg.ScanConfig(out_path=path, **kw))
        out[flag] = path.read_bytes()
    assert out["1"] == out["0"]

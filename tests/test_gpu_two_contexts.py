"""run_scan on two device contexts (engine._two_lane_loop, opt-in PANELGWAS_CONTEXTS=2): batches alternate between two
contexts driven by two host threads and are handed to the writer in batch order. Every output
(THRESHOLD / FULL records, effect-size and min-p sidecars, QC) must be byte-identical to the
one-context loop (PANELGWAS_CONTEXTS=1), for PLINK rows and GPU-inflated BGEN blocks, with
odd batch counts, and errors raised on a lane must surface."""
import numpy as np
import pytest

import paper_2604_21095_b200 as pg
from conftest_helpers import write_tsv
from paper_2604_21095_b200.errors import FormatError
from test_gpu_engine import dataset, scan

pytestmark = pytest.mark.gpu


def _outputs(root, stem):
    """Every output file of a scan but the summary (it holds wall times)."""
    return {p.name.replace(stem, ""): p.read_bytes() for p in sorted(root.glob(stem + "*"))
            if not p.name.endswith(".summary.json")}


@pytest.mark.parametrize("mode", ["thr", "full"])
def test_two_contexts_plink_identical(mode, tmp_path, monkeypatch):
    rng = np.random.default_rng(17)
    n, m, p = 333, 1300, 9
    d = rng.binomial(2, rng.uniform(0.05, 0.95, m)[:, None], size=(m, n)).astype(np.float64)
    rows = rng.random(m) < 0.2
    d[rows] = np.where(rng.random((rows.sum(), n)) < 0.05, np.nan, d[rows])
    y = rng.standard_normal((n, p))
    y[:, 3] += 0.4 * np.nan_to_num(d[100], nan=1.0)
    spec, pheno, _, root = dataset(tmp_path, d, y)
    kw = dict(p_threshold=0.05, min_p_sidecar=True, qc_sidecar=True, effect_sizes=True) if mode == "thr" else \
        dict(output_mode=pg.OutputMode.FULL, effect_sizes=True)
    out = {}
    for lanes in ("1", "2"):
        monkeypatch.setenv("PANELGWAS_CONTEXTS", lanes)
        for db in (256, 300):  # 6 and 5 batches (odd: one context scans one more)
            stem = f"o{lanes}_{db}.out"
            scan(spec, pheno, root / stem, device_batch=db, **kw)
            out[lanes, db] = _outputs(root, stem)
    ref = out["1", 256]
    assert len(ref) >= 2 and all(v == ref for v in out.values())


def test_two_contexts_bgen_identical(tmp_path, monkeypatch):
    from bgen_fixture import write_bgen

    rng = np.random.default_rng(23)
    n, m, k = 211, 700, 6
    ids = [f"S{i + 1}" for i in range(n)]
    d = rng.binomial(2, rng.uniform(0.05, 0.95, m)[:, None], size=(m, n)).astype(np.float64)
    frac = rng.random((m, n)) < 0.2
    d[frac] = np.clip(d[frac] + rng.normal(0, 0.3, frac.sum()), 0, 2)
    d[rng.random((m, n)) < 0.05] = np.nan
    y = rng.standard_normal((n, k))
    pheno = write_tsv(tmp_path / "p.tsv", ids, [f"ph{j + 1}" for j in range(k)], y)
    spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=write_bgen(tmp_path / "g.bgen", d, ids, bits=8))
    out = {}
    for lanes in ("1", "2"):
        monkeypatch.setenv("PANELGWAS_CONTEXTS", lanes)
        path = tmp_path / f"o{lanes}.tsv"
        pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, out_path=path, summary_to_stderr=False,
                                  p_threshold=0.1, device_batch=96))
        out[lanes] = path.read_bytes()
    assert out["1"] == out["2"] and out["1"].count(b"\n") > 1


def test_two_contexts_lane_error_surfaces(tmp_path, monkeypatch):
    """A malformed BGEN block in a batch scanned by the second context raises the reference's
    error from run_scan (and the scan's contexts are not returned to the pool half-used)."""
    from bgen_fixture import write_bgen

    rng = np.random.default_rng(29)
    n, m = 97, 300
    ids = [f"S{i + 1}" for i in range(n)]
    d = rng.binomial(2, 0.4, size=(m, n)).astype(np.float64)
    path = write_bgen(tmp_path / "g.bgen", d, ids, bits=8)
    src = pg.BgenSource(path)
    off = int(src._offsets[100])  # variant 100: batch 1 of 64-variant batches, the second context
    src.close()
    raw = bytearray(path.read_bytes())
    raw[off + 60] ^= 0xFF  # corrupt a byte inside its compressed block
    path.write_bytes(bytes(raw))
    pheno = write_tsv(tmp_path / "p.tsv", ids, ["ph1", "ph2"], rng.standard_normal((n, 2)))
    spec = pg.SourceSpec(pg.GenotypeFormat.BGEN, bgen_path=path)
    monkeypatch.setenv("PANELGWAS_CONTEXTS", "2")
    with pytest.raises(FormatError):
        pg.run_scan(pg.ScanConfig(source=spec, pheno_path=pheno, out_path=tmp_path / "o.tsv",
                                  summary_to_stderr=False, p_threshold=0.1, device_batch=64))

#!/usr/bin/env python
"""Per-scan wall time of many tiny run_scan calls (the reference acceptance criterion 1 shape:
N 10-50, M 1-20, P 1-8) in F32 and F64 precision; prints mean ms per scan."""
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import paper_2604_21095_b200 as pg  # noqa: E402
from conftest_helpers import write_tsv  # noqa: E402


def main():
    rng = np.random.default_rng(101)
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        cases = []
        for i in range(30):
            n, m, p = int(rng.integers(10, 51)), int(rng.integers(1, 21)), int(rng.integers(1, 9))
            d = rng.binomial(2, rng.uniform(0.2, 0.8, m)[:, None], size=(m, n)).astype(float)
            ids = [f"S{j}" for j in range(n)]
            bed, bim, fam = pg.write_bed_trio(tmp / f"g{i}", d, ids)
            ph = write_tsv(tmp / f"p{i}.tsv", ids, [f"ph{j + 1}" for j in range(p)], rng.standard_normal((n, p)))
            cases.append((pg.SourceSpec(pg.GenotypeFormat.PLINK_BED, bed_path=bed, bim_path=bim, fam_path=fam), ph))
        for prec in (pg.Precision.F32_STORE_F64_ACC, pg.Precision.F64, pg.Precision.F32_STORE_F64_ACC):
            t0 = time.perf_counter()
            for i, (spec, ph) in enumerate(cases):
                pg.run_scan(pg.ScanConfig(source=spec, pheno_path=ph, out_path=tmp / f"o{i}.tsv", p_threshold=1.0,
                                          precision=prec, summary_to_stderr=False))
            print(prec.value, f"{1e3 * (time.perf_counter() - t0) / len(cases):.1f} ms per scan")


if __name__ == "__main__":
    main()

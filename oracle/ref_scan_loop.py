"""The reference's own scan loop (panelgwas 0.1.0, from oracle/_ref/panelgwas_src.zip) on the
host cores — BASELINE INFRASTRUCTURE, used only by bench.py's `--impl reference` arm and its
`cpu_baseline` leg. Nothing here is product code, and nothing in the product imports it.

What runs is the reference's stock THRESHOLD path, function for function:

  setup (once, reported separately)   kernel.build_covariate_basis / residualize /
                                      standardize_columns on the in-memory raw panel
                                      (engine.py:259-279), kernel.t_threshold_for_p + the
                                      premask bar (engine.py:321-330), engine._Prepared
  step (timed)                        the scan loop of engine._run_scan_open (engine.py:381-398):
                                      PlinkSource.read_marker_batch on the main thread,
                                      engine._process_batch on a ThreadPoolExecutor with the
                                      reference's window of 2 x workers, ThresholdWriter.emit
                                      (p_from_t + TSV records) in order, writer.finalize

The only part of run_scan left out is the phenotype TSV parse (phenotypes.load_table): at
N 23,000 x P 20,480 it is a ~9 GB text file that the reference loader needs minutes for,
and it is a separate §8(f3) row, not the scan. The genotype rows come from a real .bed
trio written with the reference's own simulate.write_bed_trio.
"""

from __future__ import annotations

import os
import tempfile
import time
from collections import deque
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

from . import make_ref


def available() -> bool:
    return make_ref.SRC_ZIP.exists()


class ReferenceScanLoop:
    """Reference panel prep once, then timed passes of the reference scan loop over a marker sample."""

    def __init__(self, n: int, p: int, n_markers: int, p_threshold: float, seed: int = 3, n_cov: int = 10,
                 batch_size: int = 4096, workers: int = 1, workdir: Path | None = None):
        ref = make_ref.import_reference()
        from panelgwas import engine, kernel, output  # the reference, from the archive
        from panelgwas.genotypes.plink import PlinkSource
        from panelgwas.simulate import write_bed_trio

        self.ref, self.engine, self.output = ref, engine, output
        self.n, self.p, self.m = n, p, n_markers
        self.p_threshold, self.batch_size, self.workers = p_threshold, batch_size, workers
        rng = np.random.default_rng(seed)
        # raw panel of the C3 shape: Y = C gamma + N(0, 1), 10 covariates
        c = rng.standard_normal((n, n_cov))
        y = c @ (0.1 * rng.standard_normal((n_cov, p))) + rng.standard_normal((n, p))
        t0 = time.perf_counter()
        basis = kernel.build_covariate_basis(c, True, 1e-8, [f"c{j}" for j in range(n_cov)])
        ytil, _sd, zero_var = kernel.standardize_columns(kernel.residualize(y, basis))
        del y
        kept = np.nonzero(~zero_var)[0]
        ytil = np.ascontiguousarray(ytil[:, kept])
        df = float(n - 2)
        t_crit = kernel.t_threshold_for_p(p_threshold, df)
        premask = 0.0
        if t_crit > 0.0:
            premask = float(engine._abs_t_to_abs_r(np.float64(t_crit * (1.0 - 1e-9)), df) * (1.0 - 1e-12))
        self.prep = engine._Prepared(ytil=ytil, basis=basis, df=df, dtype=np.dtype(np.float32),
                                     residualize_genotypes=False, mode=engine.OutputMode.THRESHOLD,
                                     premask_abs_r=premask, topk_bar=None, topk_t_floor=np.inf,
                                     out_dtype=np.dtype(np.float32))
        self.setup_s = time.perf_counter() - t0
        self.names = [f"ph{j + 1}" for j in kept]
        # genotype sample: G ~ Binomial(2, AF), AF ~ U(0.05, 0.95), as a .bed trio
        self._tmp = tempfile.TemporaryDirectory(prefix="refscan_", dir=workdir)
        root = Path(self._tmp.name)
        af = rng.uniform(0.05, 0.95, n_markers)
        g = rng.binomial(2, af[:, None], size=(n_markers, n)).astype(np.float64)
        bed, bim, fam = write_bed_trio(root / "g", g, [f"I{i}" for i in range(n)])
        del g
        self.source = PlinkSource(bed, bim, fam)
        self.out_path = root / "ref.tsv"

    def step(self) -> dict:
        """One pass of the reference scan loop over the sample; returns timings and record count."""
        engine, output, prep, source = self.engine, self.output, self.prep, self.source
        t0 = time.perf_counter()
        writer = output.ThresholdWriter(self.out_path, self.p_threshold, prep.df, self.n, source.counts_allele1,
                                        self.names)
        window = max(2, 2 * self.workers)
        with ThreadPoolExecutor(max_workers=self.workers) as pool:
            pending: deque = deque()
            for start, count in engine.plan_batches(self.m, self.batch_size):
                raw = source.read_marker_batch(start, count, dtype=prep.dtype)
                pending.append(pool.submit(engine._process_batch, raw, prep))
                while len(pending) >= window:
                    writer.emit(pending.popleft().result()[0])
            while pending:
                writer.emit(pending.popleft().result()[0])
        records = writer.finalize()
        return {"seconds": time.perf_counter() - t0, "records": int(records)}

    def close(self) -> None:
        self.source.close()
        self._tmp.cleanup()


def host_threads() -> int:
    """Threads the reference's numpy/OpenBLAS can use on this host."""
    try:
        from threadpoolctl import threadpool_info

        n = max(int(i.get("num_threads", 1)) for i in threadpool_info())
        if n:
            return n
    except Exception:
        pass
    return os.cpu_count() or 1

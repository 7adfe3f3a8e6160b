"""Scan orchestration on the B200.

API and semantics of /root/reference/pkg/src/panelgwas/engine.py (ScanConfig,
ScanSummary, plan_batches, run_scan): same output files, record order,
summary keys and error behaviour. What differs is where the work happens:

  reference (_process_batch, engine.py:178-219)   this engine
  --------------------------------------------   ---------------------------------
  host decode to f32/f64 dosages                  raw rows -> device (pg_scan)
  prepare_genotype_batch (numpy, f64)             K1 integer stats + ternary planes
  correlate: f64 DGEMM on 256-row tiles           K2 int8 tcgen05 GEMM, exact
  premask |r| >= r_bar, t for candidates          K3 fused epilogue + cub sort
  ThresholdWriter p_from_t                        K4 fp64 Student-t on device

The panel is residualized / standardized on the host once (as the reference
does), then quantized and kept resident in HBM. Batches are read on a
background thread while the device scans the previous one. Because every
(marker, phenotype) statistic is an exact integer contraction followed by a
fixed fp64 epilogue, results are identical for any batch size, worker count
or GPU count.
"""

from __future__ import annotations

import enum
import json
import os
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _native, kernel, output, phenotypes
from .errors import ConfigError, PanelGwasError
from .genotypes.types import SourceSpec, open_genotype_source
from .kernel import SkipReason
from .phenotypes import MissingPolicy, PanelState


class Precision(enum.Enum):
    F32_STORE_F64_ACC = "f32"
    F64 = "f64"


class DfMode(enum.Enum):
    PAPER_N_MINUS_2 = "paper"
    ADJUSTED = "adjusted"


class OutputMode(enum.Enum):
    THRESHOLD = "threshold"
    TOPK = "topk"
    FULL = "full"


DEFAULT_BATCH_SIZE = 4096
DEFAULT_P_THRESHOLD = 1e-4
DEFAULT_TOP_K = 100
DEFAULT_FULL_BYTE_BUDGET = 16 * 1024**3

# device batches are sized for the GEMM (>= this many markers) and bounded in memory
_MIN_DEVICE_BATCH = 8192
_DOSAGE_DEVICE_BATCH = 8192  # --batch-size up to 32,768 raises C5 throughput (GPU-resident: +10 %) but
# triples the pinned read ring, whose allocation contends with the panel upload in a CLI run
_PLINK_DEVICE_BATCH = 65536
_SLICE_SAMPLES = 131072  # csrc/assoc.cuh kSliceK
_MAX_GEMM_ROWS = 1 << 17
_MAX_FULL_BYTES = 2 << 30
# candidate pairs one device batch may produce (each costs ~64 B of device buffers + 40 B of
# host arrays): THRESHOLD / TOPK batches are sized so the expected count stays below this
# (the native hard limit, ctx.cu kMaxCandidates, is 8x higher)
_CAND_BUDGET = 1 << 27

_MODE_CODE = {
    OutputMode.THRESHOLD: _native.PG_MODE_THRESHOLD,
    OutputMode.TOPK: _native.PG_MODE_TOPK,
    OutputMode.FULL: _native.PG_MODE_FULL,
}


@dataclass
class ScanConfig:
    """Everything a scan needs; defaults match the CLI."""

    source: SourceSpec
    pheno_path: Path
    out_path: Path
    covar_path: Path | None = None
    keep_path: Path | None = None
    remove_path: Path | None = None
    id_column: str = "IID"
    delimiter: str = "\t"
    missing_policy: MissingPolicy = MissingPolicy.MEAN_IMPUTE
    batch_size: int = DEFAULT_BATCH_SIZE
    precision: Precision = Precision.F32_STORE_F64_ACC
    df_mode: DfMode = DfMode.PAPER_N_MINUS_2
    residualize_genotypes: bool = False
    rank_tolerance: float = 1e-8
    output_mode: OutputMode = OutputMode.THRESHOLD
    p_threshold: float = DEFAULT_P_THRESHOLD
    top_k: int = DEFAULT_TOP_K
    worker_count: int = 1
    full_byte_budget: int = DEFAULT_FULL_BYTE_BUDGET
    allow_large_full: bool = False
    qc_sidecar: bool = False
    min_p_sidecar: bool = False  # engine extension: <out>.minp.tsv, per-phenotype max |t| / min p
    # engine extension: per-record effect size and standard error (<out>.beta.tsv / .beta.bin)
    effect_sizes: bool = False
    summary_to_stderr: bool = True
    device: int | None = None
    # markers per device launch; None = sized automatically (results do not depend on it)
    device_batch: int | None = None

    def validate(self) -> None:
        if self.batch_size < 1:
            raise ConfigError("batch_size must be >= 1")
        if not 0.0 < self.p_threshold <= 1.0:
            raise ConfigError("p_threshold must be in (0, 1]")
        if self.top_k < 1:
            raise ConfigError("top_k must be >= 1")
        if self.worker_count < 1:
            raise ConfigError("worker_count must be >= 1")


@dataclass
class ScanSummary:
    """Scan accounting; markers_scanned + skipped == n_markers."""

    n_markers: int
    n_samples_source: int
    n_samples_used: int
    markers_scanned: int
    markers_skipped_monomorphic: int
    markers_skipped_all_missing: int
    phenotypes_total: int
    phenotypes_scanned: int
    phenotypes_skipped_zero_variance: int
    records_emitted: int
    clamp_count: int
    p_underflow_count: int
    df: int
    time_decode_s: float
    time_prepare_s: float
    time_correlate_s: float
    time_emit_s: float
    wall_s: float
    exclusion_log: dict[str, int] = field(default_factory=dict)
    phenotype_names: list[str] = field(default_factory=list)  # not serialized (engine extension)

    _KEYS = (
        "n_markers", "n_samples_source", "n_samples_used", "markers_scanned", "markers_skipped_monomorphic",
        "markers_skipped_all_missing", "phenotypes_total", "phenotypes_scanned",
        "phenotypes_skipped_zero_variance", "records_emitted", "clamp_count", "p_underflow_count", "df",
        "time_decode_s", "time_prepare_s", "time_correlate_s", "time_emit_s", "wall_s",
    )

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k in self._KEYS}
        for reason, count in self.exclusion_log.items():
            d[f"excluded_{reason}"] = count
        return d


def plan_batches(n_markers: int, batch_size: int) -> list[tuple[int, int]]:
    """Contiguous (start, count) spans covering [0, n_markers)."""
    if n_markers < 1:
        raise ValueError("plan_batches requires at least one marker")
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    return [(s, min(batch_size, n_markers - s)) for s in range(0, n_markers, batch_size)]


def abs_t_to_abs_r(abs_t, df: float):
    """|r| with |t| = |r| sqrt(df / (1 - r^2)) (monotone inverse; inf -> 1)."""
    with np.errstate(invalid="ignore", divide="ignore"):
        r = abs_t / np.sqrt(df + np.square(abs_t))
    return np.where(np.isinf(abs_t), 1.0, r)


def threshold_premask(p_threshold: float, df: float) -> float:
    """The |r| premask bar of a THRESHOLD scan (engine.py:321-330 of the reference)."""
    t_crit = kernel.t_threshold_for_p(p_threshold, df)
    if t_crit <= 0.0:
        return 0.0
    safe_t = t_crit * (1.0 - 1e-9)
    return float(abs_t_to_abs_r(np.float64(safe_t), df) * (1.0 - 1e-12))


def topk_premask(worst_abs_t: np.ndarray, t_floor: float, df: float) -> np.ndarray:
    """Per-phenotype |r| bar from the TopK admission bar (engine.py:205-211 of the reference)."""
    bar_t = np.minimum(worst_abs_t, t_floor) * (1.0 - 1e-12)
    bar_r = abs_t_to_abs_r(np.maximum(bar_t, 0.0), df)
    return np.where(bar_t <= 0.0, -1.0, bar_r * (1.0 - 1e-12))


_TOPK_NULL_FACTOR = 16.0  # (/4 = floor of) expected null candidates per missing top-k slot
topk_rescans = 0  # batches rescanned because a null-quantile bar admitted too few (diagnostics)


def topk_batch_bars(writer, top_k: int, batch_markers: int, t_floor: float, df: float):
    """Per-phenotype |r| bars for the next TOPK batch and the candidate counts they must yield.

    Phenotypes already holding k records use the admission bar of their k-th record (the
    reference's rule, engine.py:205-211). A phenotype still short of k records would admit
    every marker (the reference's per-4,096-marker batches can afford that; a 65,536-marker
    device batch x 20,480 phenotypes cannot), so its bar is the null quantile at
    p = max(4, 32 / k) * k / batch: all markers beating the batch's k-th best are then above
    the bar whenever at least k candidates pass, which the caller checks (and rescans the
    batch without a bar for any phenotype that falls short)."""
    bars = topk_premask(writer.worst_abs_t, t_floor, df)
    kept = writer.kept_counts()
    short = kept < top_k
    # a short phenotype needs the batch's own k best above its bar, not just k - kept: a
    # marker under the bar could still beat a weak held record otherwise. With >= k batch
    # candidates above the bar, every marker below it has k better records and cannot enter.
    need = np.where(short, top_k, 0)
    # expected null candidates per phenotype: factor x missing slots (>= 32), so falling short
    # needs a Poisson(>= 32) draw below `missing` (rescans stay rare) while the first batch
    # of a C3-sized scan admits ~k x max(4, ...) candidates per phenotype, not 65,536
    factor = max(_TOPK_NULL_FACTOR / 4.0, 32.0 / max(top_k, 1))
    for miss in np.unique(need[short]).tolist():
        p_q = min(1.0, factor * miss / max(batch_markers, 1))
        bars[need == miss] = threshold_premask(p_q, df) if p_q < 1.0 else -1.0
    return bars, need


def _pinned_buffers(sizes: list[int]) -> list:
    return [_native.PinnedBuffer(n) for n in sizes]


def _free_pinned(bufs) -> None:
    for b in bufs or []:
        b.close()


def expected_candidates_per_marker(config: ScanConfig, batch: int, n_pheno: int) -> int:
    """Upper estimate of the premask's candidate pairs per marker of a `batch`-marker launch.

    THRESHOLD: the null admits ~p_threshold of the pairs (the bar is p_threshold's |r|,
    engine.py:321-330 of the reference); x4 headroom for real signal, and every pair at p = 1.
    TOPK: the first batch's null-quantile bars admit ~max(4k, 32) markers per phenotype
    (topk_batch_bars), or the whole batch when that is larger."""
    n_pheno = max(1, n_pheno)
    if config.output_mode is OutputMode.TOPK:
        per_pheno = min(batch, 2 * max(4 * config.top_k, 32))
        return -(-per_pheno * n_pheno // max(batch, 1))
    frac = min(1.0, 4.0 * config.p_threshold + 1e-6)
    return max(1, int(np.ceil(frac * n_pheno)))


def device_batch_size(config: ScanConfig, n_markers: int, n_pheno: int, n_samples: int = 0) -> int:
    """Markers per device launch: at least the configured batch, sized for the GEMM, memory-bounded."""
    if config.device_batch is not None:
        return max(1, min(int(config.device_batch), n_markers))
    plink = config.source.format.value == "plink-bed"
    # PLINK rows are 2-bit packed and decoded inside the GEMM: large launches amortize the
    # per-launch statistics / compaction / host round trips (65,536 markers = 377 MB at N = 23k)
    # dosage sources: up to 4 GEMM rows per marker with wide digits (the default), 16 with the
    # balanced-ternary planes
    wide = os.environ.get("PANELGWAS_WIDE_DIGITS", "1") != "0"
    b = max(config.batch_size, _PLINK_DEVICE_BATCH if plink else (_DOSAGE_DEVICE_BATCH if wide else _MIN_DEVICE_BATCH))
    b = min(b, _MAX_GEMM_ROWS if plink else _MAX_GEMM_ROWS // (4 if wide else 16))
    if config.output_mode is OutputMode.FULL:
        b = min(b, max(256, _MAX_FULL_BYTES // (8 * max(n_pheno, 1))))
    else:
        b = min(b, max(256, _CAND_BUDGET // max(1, expected_candidates_per_marker(config, b, n_pheno))))
    if n_samples > _SLICE_SAMPLES or config.precision is Precision.F64:
        # K-sliced runs hold 16 B of int64 partials per test, F64 mode 16 B per panel level
        per_test = 32 if config.precision is Precision.F64 else 16
        b = min(b, max(256, _MAX_FULL_BYTES * 2 // (per_test * max(n_pheno, 1))))
    return max(1, min(b, n_markers))


@dataclass
class _PreparedPanel:
    basis: kernel.CovariateBasis
    panel: phenotypes.PhenotypePanel
    align: phenotypes.SampleAlignment
    df: float
    pheno_names: list[str] = field(default_factory=list)
    zero_variance: np.ndarray | None = None
    kept_cols: np.ndarray | None = None
    pheno_sd: np.ndarray | None = None  # sd (1/N) of each scanned residualized phenotype (effect sizes)

    def set_flags(self, zero_variance: np.ndarray) -> None:
        self.zero_variance = np.asarray(zero_variance, dtype=bool)
        self.kept_cols = np.nonzero(~self.zero_variance)[0]
        self.pheno_names = [self.panel.phenotype_names[j] for j in self.kept_cols.tolist()]
        if not self.pheno_names:
            raise PanelGwasError("every phenotype has zero variance; nothing to scan")
        if self.df < 1:
            n = self.align.n_kept
            raise ConfigError(f"degrees of freedom {self.df:.0f} < 1 (n={n}, basis rank={self.basis.rank})")


def prepare_panel(config: ScanConfig, source) -> _PreparedPanel:
    """Tables -> alignment -> panel (missing policy) -> covariate basis -> df (host, once).

    The numeric panel preparation (centre, residualize, standardize: kernel.py:310-347 of
    the reference, engine.py:259-279) runs on the device in stage_panel()."""
    pheno_table = phenotypes.load_table(config.pheno_path, config.id_column, config.delimiter)
    covar_table = (
        phenotypes.load_table(config.covar_path, config.id_column, config.delimiter) if config.covar_path else None
    )
    keep = phenotypes.read_id_list(config.keep_path) if config.keep_path else None
    remove = phenotypes.read_id_list(config.remove_path) if config.remove_path else None
    align = phenotypes.align_samples(source.sample_ids, pheno_table, covar_table, keep, remove)
    panel = phenotypes.build_panel(pheno_table, align, config.missing_policy)
    n = align.n_kept
    if covar_table is not None:
        c_matrix = phenotypes.covariate_matrix(covar_table, align)
        c_names = covar_table.column_names
    else:
        c_matrix = np.zeros((n, 0))
        c_names = []
    basis = kernel.build_covariate_basis(c_matrix, True, config.rank_tolerance, c_names)
    df = float(n - 2) if config.df_mode is DfMode.PAPER_N_MINUS_2 else float(n - basis.rank - 1)
    return _PreparedPanel(basis, panel, align, df)


def panel_metadata(prep: _PreparedPanel) -> dict:
    """Everything a scan needs about the prepared panel except its values (small, picklable):
    what rank 0 sends the other ranks instead of having each parse the phenotype tables."""
    return {"basis": prep.basis, "names": prep.panel.phenotype_names, "missing": prep.panel.missing_count,
            "shape": prep.panel.y.shape, "align": prep.align, "df": prep.df}


def panel_from_metadata(meta: dict) -> _PreparedPanel:
    """A _PreparedPanel for a rank that receives the quantized panel over NCCL: no values
    (the placeholder matrix is never touched, so no host memory is committed)."""
    y = np.empty(meta["shape"], dtype=np.float64)
    panel = phenotypes.PhenotypePanel(y, list(meta["names"]), meta["missing"], PanelState.STANDARDIZED)
    return _PreparedPanel(meta["basis"], panel, meta["align"], meta["df"])


def stage_panel(ctx, prep: _PreparedPanel, n_samples_src: int, commit: bool = True) -> None:
    """Device panel preparation (pg_ctx_prepare_panel) + quantization of the kept columns."""
    flat, sd = ctx.prepare_panel(prep.panel.y, prep.basis.q)
    prep.panel.state = PanelState.STANDARDIZED
    prep.set_flags(flat)
    prep.pheno_sd = np.ascontiguousarray(sd[prep.kept_cols])
    if commit:
        ctx.commit_panel(prep.kept_cols, prep.align.genotype_row_index, n_samples_src)


MIN_P_COLUMNS = ("PHENO", "MAX_ABS_R", "MAX_ABS_T", "MIN_P")


def write_min_p(path: Path, names, max_abs_r, max_abs_t, min_p) -> None:
    """Per-phenotype minimum p over the scan (north star (3)); floats as repr()."""
    with open(path, "w") as fh:
        fh.write("\t".join(MIN_P_COLUMNS) + "\n")
        for j, name in enumerate(names):
            fh.write(f"{name}\t{float(max_abs_r[j])!r}\t{float(max_abs_t[j])!r}\t{float(min_p[j])!r}\n")


# One idle device context per device, kept for the next scan of this process: a context owns
# its CUDA streams and device buffers (grown, never shrunk), so a process that runs many scans
# (tests, notebooks, the acceptance suite's hundreds of tiny scans) creates them once. A scan
# takes the idle context only if it was created under the same PG_* / PANELGWAS_* switches
# (some are read when a context is created); a failed scan closes its context instead.
_CTX_POOL: dict = {}
_CTX_POOL_LOCK = threading.Lock()


def _switches() -> tuple:
    return tuple(sorted((k, v) for k, v in os.environ.items() if k.startswith(("PG_", "PANELGWAS_"))))


_POOL_PER_DEVICE = 2  # a scan drives up to two contexts (_two_lane_loop)


def _acquire_context(device):
    from ._device import DeviceContext

    key = _switches()
    stale = []
    ctx = None
    with _CTX_POOL_LOCK:
        held = _CTX_POOL.setdefault(device, [])
        while held and ctx is None:
            k, c = held.pop()
            if k == key:
                ctx = c
            else:
                stale.append(c)
    for c in stale:
        c.close()
    if ctx is None:
        ctx = DeviceContext(device)
        ctx.pool_key = key
    return ctx


def _release_context(device, ctx) -> None:
    extra = None
    with _CTX_POOL_LOCK:
        held = _CTX_POOL.setdefault(device, [])
        if any(c is ctx for _, c in held):
            return
        held.append((getattr(ctx, "pool_key", None), ctx))
        if len(held) > _POOL_PER_DEVICE:
            extra = held.pop(0)[1]
    if extra is not None:
        extra.close()


def _two_contexts_wanted(config: ScanConfig) -> bool:
    """PANELGWAS_CONTEXTS=2: THRESHOLD / FULL scans alternate batches between two device
    contexts (_two_lane_loop; TOPK keeps one: its per-batch bars come from the writer's state).
    Off by default: through the CLI at C3 the two lanes' threads contend with the writer
    thread's record formatting for the GIL and the scan loop measured 1.6-3.5 s against
    1.1-1.6 s on one context; the benches, whose per-batch host work is small,
    gain from two contexts and use them."""
    return config.output_mode is not OutputMode.TOPK and os.environ.get("PANELGWAS_CONTEXTS", "1") == "2"


def _two_lane_loop(ctx, ctx2, plan, read_lane, stage_on, ready_on, dispatch, full_bufs, dtype, waits) -> float:
    """Batches alternate between two device contexts, one host thread each: batch i runs on
    context i % 2 (its reads, staging and scans pipelined as in the one-context loop), and
    results are handed to `dispatch` strictly in batch order. While one context's thread
    fetches results or waits for its turn, the other context's kernels keep the GPU busy.
    Returns the host read time."""
    seq = threading.Condition()
    state = {"next": 0, "error": None, "t_read": 0.0}

    def ordered_dispatch(i, res):
        with seq:
            while state["next"] != i and state["error"] is None:
                seq.wait()
            if state["error"] is not None:
                return
            try:
                dispatch(i, res)
            except BaseException as exc:
                state["error"] = exc
                raise
            finally:
                state["next"] = i + 1
                seq.notify_all()

    def scan_on(cx, slot, i):
        t0 = time.perf_counter()
        out = full_bufs[i % len(full_bufs)].array if full_bufs else None
        res = cx.scan_staged(slot, full_elem_bytes=dtype.itemsize, full_out=out)
        with seq:
            waits["scan"] += time.perf_counter() - t0
        return res

    def lane(k):
        cx = (ctx, ctx2)[k]
        mine = list(range(k, len(plan), 2))
        if not mine:
            return
        try:
            with ThreadPoolExecutor(max_workers=1) as reader:
                fut = reader.submit(read_lane, mine[0], 2 * k)
                prev = None
                for j, i in enumerate(mine):
                    t0 = time.perf_counter()
                    block, dt_read = fut.result()
                    with seq:
                        waits["read"] += time.perf_counter() - t0
                        state["t_read"] += dt_read
                    stage_on(cx, j % 2, block)
                    if prev is not None:
                        ordered_dispatch(prev[0], scan_on(cx, prev[1], prev[0]))
                    if state["error"] is not None:
                        return
                    if j + 1 < len(mine):  # into the buffer of the batch just scanned
                        fut = reader.submit(read_lane, mine[j + 1], 2 * k + (j + 1) % 2)
                    ready_on(cx, j % 2, i)
                    prev = (i, j % 2)
                ordered_dispatch(prev[0], scan_on(cx, prev[1], prev[0]))
        except BaseException as exc:
            with seq:
                if state["error"] is None:
                    state["error"] = exc
                seq.notify_all()
            raise

    with ThreadPoolExecutor(max_workers=2) as lanes:
        futs = [lanes.submit(lane, k) for k in range(2)]
        for f in futs:
            try:
                f.result()
            except BaseException:
                pass
    if state["error"] is not None:
        raise state["error"]
    return state["t_read"]


def run_scan(config: ScanConfig, marker_range: tuple[int, int] | None = None, panel_hook=None,
             prep_hook=None) -> ScanSummary:
    """Execute a full scan on the GPU and write results plus the summary files.

    marker_range / panel_hook / prep_hook are used by the multi-GPU driver (distributed.py):
    scan only markers [start, stop) of the source, obtain the resident panel through
    `panel_hook(ctx, prep)` (NCCL broadcast from rank 0) instead of uploading it, and the host
    panel metadata through `prep_hook(source)` (rank 0 parses the tables for everyone).
    """
    wall0 = time.perf_counter()
    config.validate()
    # CUDA context creation (0.5-2 s) overlaps opening the source (the BGEN index) and parsing
    # the tables; every C-ABI entry selects the ctx's device itself, so the handle may be
    # created on another thread
    init = ThreadPoolExecutor(max_workers=1)
    ctx_fut = init.submit(_acquire_context, config.device)
    ctx2_fut = init.submit(_acquire_context, config.device) if _two_contexts_wanted(config) else None
    try:
        source = open_genotype_source(config.source)
    except BaseException:
        init.shutdown(wait=False)
        _close_when_done(ctx_fut)
        if ctx2_fut is not None:
            _close_when_done(ctx2_fut)
        raise
    try:
        return _run_scan_open(config, source, wall0, init, ctx_fut, marker_range, panel_hook, prep_hook, ctx2_fut)
    finally:
        source.close()


def _close_when_done(ctx_fut) -> None:
    try:
        ctx_fut.result().close()
    except Exception:
        pass


def _run_scan_open(config: ScanConfig, source, wall0: float, init, ctx_fut, marker_range=None, panel_hook=None,
                   prep_hook=None, ctx2_fut=None) -> ScanSummary:
    # the pinned read ring (~0.4 s per GB) is allocated on the init thread after the context,
    # also while the tables parse
    lo, hi = marker_range if marker_range is not None else (0, source.n_markers)
    compressed = hasattr(source, "read_compressed_block") and os.environ.get("PANELGWAS_HOST_INFLATE") != "1"
    row_bytes = (source.compressed_bytes_per_marker if compressed
                 else getattr(source, "bytes_per_marker", 0))
    # the batch only shrinks as phenotypes are added, so one phenotype bounds every ring slot
    ring_bytes = device_batch_size(config, max(hi - lo, 1), 1, source.n_samples) * row_bytes
    # 3 buffers for one context's pipeline; 4 (two per context) when two contexts alternate
    ring_fut = init.submit(_pinned_buffers, [ring_bytes] * (4 if ctx2_fut is not None else 3) if ring_bytes else [])
    init.shutdown(wait=False)
    try:
        phases = {"start": time.perf_counter() - wall0}
        prep = prep_hook(source) if prep_hook is not None else prepare_panel(config, source)
        phases["tables_panel_host"] = time.perf_counter() - wall0
        if source.n_markers < 1:
            raise PanelGwasError("genotype source has no markers")
        ctx = ctx_fut.result()
        # Precision.F64: the panel at two quantization levels (~46 bits), one exact GEMM each
        ctx.set_f64_panel(config.precision is Precision.F64)
    except BaseException:
        for fut, release in ((ring_fut, _free_pinned), (ctx_fut, lambda c: c.close()),
                             (ctx2_fut, lambda c: c.close())):
            try:
                if fut is not None:
                    release(fut.result())
            except Exception:
                pass
        raise
    phases["device_ready"] = time.perf_counter() - wall0
    n = prep.align.n_kept
    df = prep.df
    dtype = np.dtype(np.float32 if config.precision is Precision.F32_STORE_F64_ACC else np.float64)
    try:
        if panel_hook is not None:
            panel_hook(ctx, prep)
        else:
            stage_panel(ctx, prep, source.n_samples)
        phases["panel_on_device"] = time.perf_counter() - wall0
        names = prep.pheno_names
        n_pheno = len(names)
        if config.output_mode is OutputMode.FULL:
            projected = source.n_markers * n_pheno * dtype.itemsize
            if projected > config.full_byte_budget and not config.allow_large_full:
                raise ConfigError(
                    f"FULL output would be ~{projected} bytes, over the {config.full_byte_budget}-byte budget; "
                    "pass the large-output override to proceed"
                )
            writer = output.FullMatrixWriter(config.out_path, dtype, df, n, source.counts_allele1, names,
                                             effect_sizes=config.effect_sizes)
        elif config.output_mode is OutputMode.TOPK:
            writer = output.TopKWriter(config.out_path, config.top_k, df, n, source.counts_allele1, names,
                                       effect_sizes=config.effect_sizes)
        else:
            writer = output.ThresholdWriter(config.out_path, config.p_threshold, df, n, source.counts_allele1,
                                            names, effect_sizes=config.effect_sizes)
        if config.effect_sizes:
            ctx.set_beta_scale(prep.pheno_sd)
    except BaseException:
        try:
            _free_pinned(ring_fut.result())
        finally:
            ctx.close()
        raise

    scan_ok = False
    ctx2 = None
    # A/B switches (results are identical either way); set on every scan since the context may
    # be a reused one
    ctx.set_fused_decode(os.environ.get("PANELGWAS_FUSED_DECODE", "1") != "0")
    ctx.set_missing_side_gemm(os.environ.get("PANELGWAS_MISSING_SIDE_GEMM", "1") != "0")
    ctx.set_wide_digits(os.environ.get("PANELGWAS_WIDE_DIGITS", "1") != "0")
    try:
        if config.residualize_genotypes and prep.basis.rank:
            ctx.set_basis(prep.basis.q)  # extension mode: side GEMM K5 for |Q^T g|^2
        t_floor = np.inf
        if config.output_mode is OutputMode.THRESHOLD:
            rbar = np.full(n_pheno, threshold_premask(config.p_threshold, df))
        elif config.output_mode is OutputMode.TOPK:
            t_floor = kernel.t_threshold_for_p(kernel.P_FLOOR, df)
            rbar = np.full(n_pheno, -1.0)  # replaced per batch below (topk_batch_bars)
        else:
            rbar = None
        ctx.set_scan(df, _MODE_CODE[config.output_mode], rbar)
        if config.min_p_sidecar:
            ctx.track_max_abs_r(True)

        skip_mono = skip_missing = clamp_total = 0
        t_decode = t_prepare = t_corr = t_emit = 0.0
        qc_rows: list[str] = []
        step = device_batch_size(config, hi - lo, n_pheno, source.n_samples)
        plan = [(lo + s0, c0) for s0, c0 in plan_batches(hi - lo, step)]
        read_kw = {"dtype": dtype} if config.source.format.value == "dense" else {}
        if ctx2_fut is not None:
            # a second context (created while the tables parsed) takes the panel device to
            # device and scans every other batch (_two_lane loop below)
            ctx2 = ctx2_fut.result()
            if len(plan) >= 2:
                ctx2.set_f64_panel(config.precision is Precision.F64)
                ctx2.clone_panel_from(ctx)
                if config.effect_sizes:
                    ctx2.set_beta_scale(prep.pheno_sd)
                ctx2.set_fused_decode(os.environ.get("PANELGWAS_FUSED_DECODE", "1") != "0")
                ctx2.set_missing_side_gemm(os.environ.get("PANELGWAS_MISSING_SIDE_GEMM", "1") != "0")
                ctx2.set_wide_digits(os.environ.get("PANELGWAS_WIDE_DIGITS", "1") != "0")
                if config.residualize_genotypes and prep.basis.rank:
                    ctx2.set_basis(prep.basis.q)
                ctx2.set_scan(df, _MODE_CODE[config.output_mode], rbar)
                if config.min_p_sidecar:
                    ctx2.track_max_abs_r(True)
            else:
                _release_context(config.device, ctx2)
                ctx2 = None

        # pinned ring of 3 host buffers + 2 device staging slots: the read of batch i+1 and
        # its H2D overlap the device scan of batch i. BGEN batches travel compressed and are
        # inflated on the GPU (pg_stage_bgen); other formats as raw rows (pg_stage).
        pinned = ring_fut.result() or None  # allocated during table parsing (>= step * row bytes each)

        def read(i):
            t0 = time.perf_counter()
            s0, c0 = plan[i]
            if compressed:
                block = source.read_compressed_block(s0, c0, out=pinned[i % 3].array)
            elif pinned is not None:
                block = source.read_raw_block(s0, c0, out=pinned[i % 3].array)
            else:
                block = source.read_raw_block(s0, c0, **read_kw)
            return block, time.perf_counter() - t0

        def stage(i, block):
            if config.output_mode is OutputMode.TOPK:
                kept_blocks[i] = block  # kept for a (rare) rescan
            if compressed:  # H2D + GPU inflate run while the previous batch is scanned
                return ctx.stage_bgen_begin(i % 2, *block)
            kind, rows, row_bytes = block
            return ctx.stage(i % 2, kind, rows, row_bytes)

        def staged_ready(i):
            if compressed:
                bad = ctx.stage_bgen_end(i % 2)
                if bad is not None:
                    source.raise_block_error(plan[i][0] + bad[0], bad[1], bad[2], bad[3])

        # two contexts (_two_lane_loop): context k reads into pinned buffers 2k, 2k+1 and stages
        # into its own two slots
        def read_lane(i, buf):
            t0 = time.perf_counter()
            s0, c0 = plan[i]
            if compressed:
                block = source.read_compressed_block(s0, c0, out=pinned[buf].array)
            elif pinned is not None:
                block = source.read_raw_block(s0, c0, out=pinned[buf].array)
            else:
                block = source.read_raw_block(s0, c0, **read_kw)
            return block, time.perf_counter() - t0

        def stage_on(cx, slot, block):
            if compressed:
                return cx.stage_bgen_begin(slot, *block)
            kind, rows, row_bytes = block
            return cx.stage(slot, kind, rows, row_bytes)

        def ready_on(cx, slot, i):
            if compressed:
                bad = cx.stage_bgen_end(slot)
                if bad is not None:
                    source.raise_block_error(plan[i][0] + bad[0], bad[1], bad[2], bad[3])

        topk_need = {}
        kept_blocks = {}

        def set_topk_bars(i):
            if config.output_mode is OutputMode.TOPK and i < len(plan):
                bars, need = topk_batch_bars(writer, config.top_k, plan[i][1], t_floor, df)
                ctx.set_rbar(bars)
                topk_need[i] = (bars, need)

        def topk_complete(i, res):
            """Rescan batch i without a bar for phenotypes whose null-quantile bar admitted
            fewer candidates than they still need (rare; exactness of the top-k selection)."""
            bars, need = topk_need.pop(i)
            have = np.bincount(res.cand_cols, minlength=n_pheno) if res.cand_cols is not None else np.zeros(n_pheno)
            short = (need > 0) & (bars > 0) & (have < need)
            if not short.any():
                return res
            global topk_rescans
            topk_rescans += 1
            start, count = plan[i]
            block = kept_blocks[i]
            if compressed:
                block = source.read_raw_block(start, count)
            kind, rows, row_bytes = block
            ctx.set_rbar(np.where(short, -1.0, 2.0))  # everything for the short phenotypes, nothing else
            extra = ctx.scan(kind, rows, row_bytes, full_elem_bytes=dtype.itemsize)
            keep_old = ~short[res.cand_cols]
            rows_ = np.concatenate([res.cand_rows[keep_old], extra.cand_rows])
            cols_ = np.concatenate([res.cand_cols[keep_old], extra.cand_cols])
            order = np.lexsort((cols_, rows_))  # (marker, phenotype) order
            names_ = ("cand_r", "cand_t", "cand_p") + (("cand_beta", "cand_se") if config.effect_sizes else ())
            for name in names_:
                setattr(res, name, np.concatenate([getattr(res, name)[keep_old], getattr(extra, name)])[order])
            res.cand_rows, res.cand_cols = rows_[order], cols_[order]
            return res

        def finish(i, res):
            nonlocal t_prepare, t_corr, t_emit, clamp_total, skip_mono, skip_missing
            start, count = plan[i]
            t_prepare += res.decode_ms / 1e3
            t_corr += res.gemm_ms / 1e3
            markers = source.marker_catalog[start:start + count]  # a lazy catalog slice for the writers
            batch = output.BatchStats(
                markers=markers, allele_frequency=res.af, missing_count=res.missing_count,
                skip_reason=res.skip, clamp_count=res.clamp_count, cand_rows=res.cand_rows,
                cand_cols=res.cand_cols, cand_r=res.cand_r, cand_t=res.cand_t, t_rows=res.t_rows,
                cand_p=res.cand_p, cand_beta=res.cand_beta, cand_se=res.cand_se, beta_rows=res.beta_rows,
            )
            clamp_total += res.clamp_count
            skip_mono += int(np.count_nonzero(res.skip == SkipReason.MONOMORPHIC))
            skip_missing += int(np.count_nonzero(res.skip == SkipReason.ALL_MISSING))
            if config.qc_sidecar:
                for j in np.nonzero(res.skip)[0].tolist():
                    qc_rows.append(f"marker\t{markers[j].id}\t{SkipReason(int(res.skip[j])).name}\n")
            t0 = time.perf_counter()
            writer.emit(batch)
            t_emit += time.perf_counter() - t0

        pinned_out: list = []
        try:
            staged: list = [None, None]
            # records of batch i-1 are formatted / written (TOPK: merged) on a writer thread while
            # batch i scans
            emitter = ThreadPoolExecutor(max_workers=1)
            emit_fut = None

            waits = {"read": 0.0, "scan": 0.0, "emit": 0.0, "stage": 0.0, "finish_thread": 0.0}

            def dispatch(i, res):
                nonlocal emit_fut
                if config.output_mode is OutputMode.TOPK:
                    res = topk_complete(i, res)  # device rescans stay on this thread
                    kept_blocks.pop(i, None)
                if emit_fut is not None:
                    t0 = time.perf_counter()
                    emit_fut.result()  # one batch in the writer at a time; re-raises its errors
                    waits["emit"] += time.perf_counter() - t0
                # TOPK: the bars of batch i+1 come from the writer after batch i-1 while batch i
                # merges on the writer thread. A lagged bar is lower (and a lagged `need`
                # larger), so batch i+1 admits a superset of the candidates it must: exact.
                set_topk_bars(i + 1)
                emit_fut = emitter.submit(timed_finish, i, res)

            def timed_finish(i, res):
                t0 = time.perf_counter()
                finish(i, res)
                waits["finish_thread"] += time.perf_counter() - t0

            # FULL: t rows land in two pinned buffers used alternately. The writer holds at most
            # one batch (dispatch waits for it before handing over the next), so batch i's
            # buffer is free again by the time batch i+2 is fetched into it.
            # (two contexts: batch i uses buffer i % 4 — the writer holds batch i-2 at most while
            # the contexts fetch batches i-1 and i)
            full_bufs = []
            if config.output_mode is OutputMode.FULL and os.environ.get("PANELGWAS_FULL_PINNED") != "0":
                full_bufs = [_native.PinnedBuffer(step * n_pheno * dtype.itemsize)
                             for _ in range(4 if ctx2 is not None else 2)]
                pinned_out.extend(full_bufs)
            n_scanned = [0]

            def scan(slot):
                t0 = time.perf_counter()
                out = full_bufs[n_scanned[0] % 2].array if full_bufs else None
                n_scanned[0] += 1
                res = ctx.scan_staged(slot, full_elem_bytes=dtype.itemsize, full_out=out)
                waits["scan"] += time.perf_counter() - t0
                return res

            set_topk_bars(0)
            # the writer thread formats in Python while this thread mostly waits in ctypes
            # calls: hand the GIL back quickly so each scan is issued as soon as it can be
            switch_interval = sys.getswitchinterval()
            sys.setswitchinterval(2e-4)
            try:
                if ctx2 is not None:
                    t_decode += _two_lane_loop(ctx, ctx2, plan, read_lane, stage_on, ready_on, dispatch, full_bufs,
                                               dtype, waits)
                else:
                    with ThreadPoolExecutor(max_workers=1) as reader:
                        fut = reader.submit(read, 0)
                        pending = None
                        for i in range(len(plan)):
                            t0 = time.perf_counter()
                            block, dt_read = fut.result()
                            waits["read"] += time.perf_counter() - t0
                            t_decode += dt_read
                            t0 = time.perf_counter()
                            staged[i % 2] = stage(i, block)
                            waits["stage"] += time.perf_counter() - t0
                            if i + 1 < len(plan):
                                fut = reader.submit(read, i + 1)
                            if pending is not None:
                                dispatch(pending, scan(pending % 2))
                            staged_ready(i)
                            pending = i
                        dispatch(pending, scan(pending % 2))
                if emit_fut is not None:
                    emit_fut.result()
            finally:
                sys.setswitchinterval(switch_interval)
                if emitter is not None:
                    emitter.shutdown(wait=True)
            if config.min_p_sidecar:
                # per-phenotype max |r| over every scanned marker (fused into the GEMM epilogue)
                max_abs_r = ctx.max_abs_r()
                if ctx2 is not None:
                    max_abs_r = np.maximum(max_abs_r, ctx2.max_abs_r())
                max_abs_t = ctx.t_from_r(max_abs_r, df)
                min_p, _ = ctx.p_from_t(max_abs_t, df)
        finally:
            if pinned is not None or pinned_out:
                ctx.sync()
                if ctx2 is not None:
                    ctx2.sync()
                for b in (pinned or []) + pinned_out:
                    b.close()
        scan_ok = True
    finally:
        for cx in (ctx, ctx2):
            if cx is None:
                continue
            if scan_ok:
                _release_context(config.device, cx)  # kept for the next scan of this process
            else:
                cx.close()

    phases["scan_loop_done"] = time.perf_counter() - wall0
    phases["loop_main_thread_waits"] = waits
    t0 = time.perf_counter()
    records = writer.finalize()
    t_emit += time.perf_counter() - t0
    phases["finalized"] = time.perf_counter() - wall0
    if hasattr(writer, "timings"):
        phases["writer"] = writer.timings
    if os.environ.get("PANELGWAS_PROFILE") == "1":  # cumulative seconds since run_scan entry
        print(json.dumps({"panelgwas_phases_s": phases}), file=sys.stderr)

    if config.min_p_sidecar:
        write_min_p(Path(str(config.out_path) + ".minp.tsv"), names, max_abs_r, max_abs_t, min_p)

    if config.qc_sidecar:
        with open(Path(str(config.out_path) + ".qc.tsv"), "w") as fh:
            fh.write("KIND\tNAME\tREASON\n")
            fh.writelines(qc_rows)
            for j in np.nonzero(prep.zero_variance)[0].tolist():
                fh.write(f"phenotype\t{prep.panel.phenotype_names[j]}\tZERO_VARIANCE\n")

    n_scanned_range = (marker_range[1] - marker_range[0]) if marker_range is not None else source.n_markers
    summary = ScanSummary(
        n_markers=n_scanned_range,
        n_samples_source=source.n_samples,
        n_samples_used=n,
        markers_scanned=n_scanned_range - skip_mono - skip_missing,
        markers_skipped_monomorphic=skip_mono,
        markers_skipped_all_missing=skip_missing,
        phenotypes_total=prep.panel.n_phenotypes,
        phenotypes_scanned=n_pheno,
        phenotypes_skipped_zero_variance=int(np.count_nonzero(prep.zero_variance)),
        records_emitted=records,
        clamp_count=clamp_total,
        p_underflow_count=writer.p_underflow_count,
        df=int(df),
        time_decode_s=t_decode,
        time_prepare_s=t_prepare,
        time_correlate_s=t_corr,
        time_emit_s=t_emit,
        wall_s=time.perf_counter() - wall0,
        exclusion_log=dict(prep.align.exclusion_log),
        phenotype_names=list(names),
    )
    with open(Path(str(config.out_path) + ".summary.json"), "w") as fh:
        json.dump(summary.to_dict(), fh, indent=2, sort_keys=True)
        fh.write("\n")
    if config.summary_to_stderr:
        for key, value in summary.to_dict().items():
            print(f"{key}={value}", file=sys.stderr)
    return summary

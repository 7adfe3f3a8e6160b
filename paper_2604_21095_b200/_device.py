"""Python handle over one `pg_ctx` (include/panelgwas_b200.h).

`DeviceContext` owns a native context bound to one CUDA device and exposes
numpy-in / numpy-out wrappers of every C-ABI entry point. All numerics run on
the device; without the native library or a B200 every method raises
`PanelGwasError` (there is deliberately no host fallback).
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import byref, c_double, c_int64, c_void_p
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import BatchInfo, call, ptr


def default_device_index() -> int:
    for key in ("PANELGWAS_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(key)
        if v:
            try:
                return int(v)
            except ValueError:
                pass
    return 0


@dataclass
class ScanResult:
    """Device results of one scanned block (host copies)."""

    n_markers: int
    af: np.ndarray
    missing_count: np.ndarray
    variance: np.ndarray
    skip: np.ndarray
    clamp_count: int
    cand_rows: np.ndarray | None = None
    cand_cols: np.ndarray | None = None
    cand_r: np.ndarray | None = None
    cand_t: np.ndarray | None = None
    cand_p: np.ndarray | None = None
    t_rows: np.ndarray | None = None
    cand_beta: np.ndarray | None = None  # effect sizes (set_beta_scale): aligned with cand_* / t_rows
    cand_se: np.ndarray | None = None
    beta_rows: np.ndarray | None = None
    decode_ms: float = 0.0
    gemm_ms: float = 0.0
    launches: int = 0
    rows_per_marker: int = 1
    n_candidates: int = 0


class DeviceContext:
    """One native scan context (panel resident in HBM + batch buffers + stream)."""

    def __init__(self, device: int | None = None):
        self.lib = _native.load_library()
        self.device = default_device_index() if device is None else int(device)
        handle = c_void_p()
        call("pg_ctx_create", self.device, byref(handle))
        self._h = handle
        self.lock = threading.RLock()
        self.n_pheno = 0
        self.mode = _native.PG_MODE_THRESHOLD
        self.beta_on = False

    # ------------------------------------------------------------ lifetime
    def close(self) -> None:
        if self._h:
            self.lib.pg_ctx_destroy(self._h)
            self._h = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def sync(self) -> None:
        call("pg_ctx_sync", self._h)

    def stream_handle(self) -> int:
        """cudaStream_t of this ctx (for CUDA-event timing on the launching stream)."""
        out = c_void_p()
        call("pg_ctx_stream", self._h, byref(out))
        return int(out.value or 0)

    # ------------------------------------------------------------ panel
    def set_panel(self, ytil: np.ndarray, geno_row_index: np.ndarray, n_samples_src: int) -> None:
        y = np.ascontiguousarray(ytil, dtype=np.float64)
        gidx = np.ascontiguousarray(geno_row_index, dtype=np.int64)
        with self.lock:
            call("pg_ctx_set_panel", self._h, ptr(y), y.shape[0], y.shape[1], y.shape[1], ptr(gidx),
                 int(n_samples_src))
            self.n_pheno = y.shape[1]
            self.beta_on = False  # the native ctx drops phenotype scales with the panel

    def prepare_panel(self, y: np.ndarray, basis_q: np.ndarray | None) -> tuple[np.ndarray, np.ndarray]:
        """Residualize + standardize the kept-sample panel on the device (kernel.py:310-347).

        Returns (zero_variance flags, sd); the standardized panel stays on the device
        until commit_panel() quantizes its kept columns."""
        y = np.ascontiguousarray(y, dtype=np.float64)
        if y.ndim != 2:
            raise ValueError("expected a 2-D (samples x phenotypes) matrix")
        n, p = y.shape
        q = None
        rank = 0
        if basis_q is not None and basis_q.shape[1]:
            q = np.ascontiguousarray(basis_q, dtype=np.float64)
            if q.shape[0] != n:
                raise ValueError(f"row count {n} does not match basis ({q.shape[0]} samples)")
            rank = q.shape[1]
        flat = np.zeros(p, dtype=np.uint8)
        sd = np.zeros(p, dtype=np.float64)
        with self.lock:
            call("pg_ctx_prepare_panel", self._h, ptr(y), n, p, p, ptr(q), rank, ptr(flat), ptr(sd))
            self._prep_shape = (n, p)
        return flat.astype(bool), sd

    def set_panel_async(self, y: np.ndarray, basis_q: np.ndarray | None, geno_row_index: np.ndarray,
                        n_samples_src: int, chunk_cols: int = 1280) -> None:
        """Pipelined prepare + commit of every column (pg_ctx_set_panel_async): `y` must be a
        C-contiguous f64 view of page-locked memory (e.g. a pinned torch tensor's .numpy())
        and stay alive until panel_async_wait(); returns at once, the next scan's GEMM
        overlaps the upload."""
        if y.dtype != np.float64 or y.ndim != 2 or not y.flags["C_CONTIGUOUS"]:
            raise ValueError("expected a C-contiguous float64 (samples x phenotypes) matrix")
        n, p = y.shape
        q = None
        rank = 0
        if basis_q is not None and basis_q.shape[1]:
            q = np.ascontiguousarray(basis_q, dtype=np.float64)
            rank = q.shape[1]
        gidx = np.ascontiguousarray(geno_row_index, dtype=np.int64)
        with self.lock:
            call("pg_ctx_set_panel_async", self._h, ptr(y), n, p, p, ptr(q), rank, ptr(gidx), int(n_samples_src),
                 int(chunk_cols))
            self.n_pheno = p
            self.beta_on = False
            self._async_shape = (n, p)

    def set_panel_async_cols(self, y_cols: np.ndarray, n_pheno: int, col_begin: int, basis_q: np.ndarray | None,
                             geno_row_index: np.ndarray, n_samples_src: int, chunk_cols: int = 1280) -> None:
        """A rank's share of a pipelined panel (pg_ctx_set_panel_async_cols): `y_cols` (pinned,
        C-contiguous f64 [n_kept, w]) holds phenotypes [col_begin, col_begin + w) of n_pheno;
        the other rows come from import_panel_rows."""
        if y_cols.dtype != np.float64 or y_cols.ndim != 2 or not y_cols.flags["C_CONTIGUOUS"]:
            raise ValueError("expected a C-contiguous float64 (samples x phenotypes) matrix")
        n, w = y_cols.shape
        q = None
        rank = 0
        if basis_q is not None and basis_q.shape[1]:
            q = np.ascontiguousarray(basis_q, dtype=np.float64)
            rank = q.shape[1]
        gidx = np.ascontiguousarray(geno_row_index, dtype=np.int64)
        with self.lock:
            call("pg_ctx_set_panel_async_cols", self._h, ptr(y_cols), n, int(n_pheno), w, int(col_begin),
                 int(col_begin) + w, ptr(q), rank, ptr(gidx), int(n_samples_src), int(chunk_cols))
            self.n_pheno = int(n_pheno)
            self.beta_on = False
            self._async_shape = (n, w)

    def panel_rows_bytes(self, n_rows: int) -> int:
        b = c_int64(0)
        call("pg_ctx_panel_rows_bytes", self._h, int(n_rows), byref(b))
        return b.value

    def export_panel_rows(self, d_dst: int, row_begin: int, row_end: int) -> None:
        with self.lock:
            call("pg_ctx_export_panel_rows", self._h, d_dst, int(row_begin), int(row_end))

    def import_panel_rows(self, d_src: int, row_begin: int, row_end: int) -> None:
        with self.lock:
            call("pg_ctx_import_panel_rows", self._h, d_src, int(row_begin), int(row_end))

    def follow_panel(self, leader: "DeviceContext") -> None:
        """Take `leader`'s pipelined panel chunk by chunk as it is prepared (pg_ctx_follow_panel)."""
        with leader.lock, self.lock:
            call("pg_ctx_follow_panel", self._h, leader._h)
            self.n_pheno = leader.n_pheno
            self.beta_on = False

    def clone_panel_from(self, src: "DeviceContext") -> None:
        """This context takes `src`'s resident panel, device to device (pg_ctx_clone_panel)."""
        with src.lock, self.lock:
            call("pg_ctx_clone_panel", self._h, src._h)
            self.n_pheno = src.n_pheno
            self.beta_on = False

    def panel_async_wait(self) -> tuple[np.ndarray, np.ndarray]:
        """(zero-variance flags, sd) of the pipelined panel once its preparation is complete."""
        p = self._async_shape[1]
        flat = np.zeros(p, dtype=np.uint8)
        sd = np.zeros(p, dtype=np.float64)
        with self.lock:
            call("pg_ctx_panel_async_wait", self._h, ptr(flat), ptr(sd))
        return flat.astype(bool), sd

    def fetch_prepared_panel(self) -> np.ndarray:
        out = np.empty(self._prep_shape, dtype=np.float64)
        with self.lock:
            call("pg_ctx_fetch_prepared_panel", self._h, ptr(out))
        return out

    def commit_panel(self, kept_cols: np.ndarray, geno_row_index: np.ndarray, n_samples_src: int) -> None:
        cols = np.ascontiguousarray(kept_cols, dtype=np.int64)
        gidx = np.ascontiguousarray(geno_row_index, dtype=np.int64)
        with self.lock:
            call("pg_ctx_commit_panel", self._h, ptr(cols), cols.size, ptr(gidx), int(n_samples_src))
            self.n_pheno = int(cols.size)
            self.beta_on = False  # the native ctx drops phenotype scales with the panel

    def set_panel_device(self, d_ptr: int, n_kept: int, n_pheno: int, ld: int, geno_row_index: np.ndarray,
                         n_samples_src: int) -> None:
        gidx = np.ascontiguousarray(geno_row_index, dtype=np.int64)
        with self.lock:
            call("pg_ctx_set_panel_device", self._h, d_ptr, n_kept, n_pheno, ld, ptr(gidx), int(n_samples_src))
            self.n_pheno = n_pheno
            self.beta_on = False  # the native ctx drops phenotype scales with the panel

    def panel_bytes(self) -> int:
        n = c_int64(0)
        call("pg_ctx_panel_bytes", self._h, byref(n))
        return n.value

    def export_panel(self, d_dst: int) -> None:
        call("pg_ctx_export_panel", self._h, d_dst)

    def import_panel(self, d_src: int, n_kept: int, n_pheno: int, geno_row_index: np.ndarray,
                     n_samples_src: int) -> None:
        gidx = np.ascontiguousarray(geno_row_index, dtype=np.int64)
        with self.lock:
            call("pg_ctx_import_panel", self._h, d_src, n_kept, n_pheno, ptr(gidx), int(n_samples_src))
            self.n_pheno = n_pheno
            self.beta_on = False  # the native ctx drops phenotype scales with the panel

    def set_scan(self, df: float, mode: int, r_bar: np.ndarray | None) -> None:
        rb = None if r_bar is None else np.ascontiguousarray(r_bar, dtype=np.float64)
        with self.lock:
            call("pg_ctx_set_scan", self._h, float(df), int(mode), ptr(rb))
            self.mode = mode

    def set_basis(self, q: np.ndarray | None) -> None:
        """Extension mode: residualize genotype rows against the covariate basis Q [n_kept, rank]."""
        qq = None if q is None else np.ascontiguousarray(q, dtype=np.float64)
        with self.lock:
            call("pg_ctx_set_basis", self._h, ptr(qq), 0 if qq is None else qq.shape[0],
                 0 if qq is None else qq.shape[1])

    def set_beta_scale(self, pheno_sd: np.ndarray | None) -> None:
        """Enable effect sizes: sd (1/N) of each scanned residualized phenotype, in panel
        column order (None disables). Every later scan also returns beta / se."""
        sd = None if pheno_sd is None else np.ascontiguousarray(pheno_sd, dtype=np.float64)
        with self.lock:
            call("pg_ctx_set_beta_scale", self._h, ptr(sd), 0 if sd is None else sd.size)
            self.beta_on = sd is not None

    def debug_candidate_base(self, base: int) -> None:
        """Test hook: start the 64-bit candidate counter of later scans at `base`."""
        call("pg_ctx_debug_candidate_base", self._h, int(base))

    def set_wide_digits(self, enable: bool) -> None:
        call("pg_ctx_set_wide_digits", self._h, 1 if enable else 0)

    def set_fused_decode(self, enable: bool) -> None:
        call("pg_ctx_set_fused_decode", self._h, 1 if enable else 0)

    def set_f64_panel(self, enable: bool) -> None:
        """Two-level (~46-bit) panel for Precision.F64; call before the panel is uploaded."""
        call("pg_ctx_set_f64_panel", self._h, 1 if enable else 0)

    def set_two_limb_premask(self, enable: bool) -> None:
        call("pg_ctx_set_two_limb_premask", self._h, 1 if enable else 0)

    def set_missing_side_gemm(self, enable: bool) -> None:
        call("pg_ctx_set_missing_side_gemm", self._h, 1 if enable else 0)

    def set_rbar(self, r_bar: np.ndarray) -> None:
        rb = np.ascontiguousarray(r_bar, dtype=np.float64)
        with self.lock:
            call("pg_ctx_set_rbar", self._h, ptr(rb))

    # ------------------------------------------------------------ scan
    def scan(self, kind: int, block: np.ndarray, row_bytes: int, *, fetch: bool = True,
             full_elem_bytes: int = 8) -> ScanResult:
        """Scan one host block of raw marker rows ([n_markers, row_bytes] uint8)."""
        blk = np.ascontiguousarray(block)
        n = blk.shape[0]
        info = BatchInfo()
        with self.lock:
            call("pg_scan", self._h, int(kind), blk.ctypes.data, n, int(row_bytes), byref(info))
            return self._collect(info, fetch, full_elem_bytes)

    def stage(self, slot: int, kind: int, block: np.ndarray, row_bytes: int) -> None:
        """Start the async H2D of a host block into staging slot 0/1 (keep `block` alive until scanned)."""
        blk = block if block.flags["C_CONTIGUOUS"] else np.ascontiguousarray(block)
        with self.lock:
            call("pg_stage", self._h, int(slot), int(kind), blk.ctypes.data, blk.shape[0], int(row_bytes))
        return blk

    def stage_bgen(self, slot: int, blob: np.ndarray, block_off: np.ndarray, block_size: np.ndarray):
        """Stage a compressed BGEN batch (GPU inflate + validation) into slot 0/1.

        Returns None on success, else (variant, reason, a, b) of the first failing block."""
        b = np.ascontiguousarray(blob, dtype=np.uint8)
        off = np.ascontiguousarray(block_off, dtype=np.int64)
        size = np.ascontiguousarray(block_size, dtype=np.int64)
        diag = np.zeros(4, dtype=np.int64)
        with self.lock:
            status = self.lib.pg_stage_bgen(self._h, int(slot), b.ctypes.data, b.size, off.ctypes.data,
                                            size.ctypes.data, off.size, diag.ctypes.data)
        if status == _native.PG_ERR_FORMAT and diag[1]:
            return tuple(int(x) for x in diag)
        _native.check(status)
        return None

    def stage_bgen_begin(self, slot: int, blob: np.ndarray, block_off: np.ndarray, block_size: np.ndarray):
        """Enqueue H2D + GPU inflate + validation of a compressed BGEN batch; returns the
        arrays that must stay alive until stage_bgen_end(slot)."""
        b = np.ascontiguousarray(blob, dtype=np.uint8)
        off = np.ascontiguousarray(block_off, dtype=np.int64)
        size = np.ascontiguousarray(block_size, dtype=np.int64)
        with self.lock:
            call("pg_stage_bgen_begin", self._h, int(slot), b.ctypes.data, b.size, off.ctypes.data, size.ctypes.data,
                 off.size)
        return b, off, size

    def stage_bgen_end(self, slot: int):
        """None when the batch is staged, else (variant, reason, a, b) of the first bad block."""
        diag = np.zeros(4, dtype=np.int64)
        with self.lock:
            status = self.lib.pg_stage_bgen_end(self._h, int(slot), diag.ctypes.data)
        if status == _native.PG_ERR_FORMAT and diag[1]:
            return tuple(int(x) for x in diag)
        _native.check(status)
        return None

    def scan_staged(self, slot: int, *, fetch: bool = True, full_elem_bytes: int = 8,
                    full_out: np.ndarray | None = None) -> ScanResult:
        """Scan staging slot 0/1. In FULL mode `full_out` (e.g. a pinned uint8 buffer large
        enough for the batch) receives the t rows and `t_rows` is a view of it."""
        info = BatchInfo()
        with self.lock:
            call("pg_scan_staged", self._h, int(slot), byref(info))
            return self._collect(info, fetch, full_elem_bytes, full_out)

    def scan_device(self, kind: int, d_ptr: int, n_markers: int, row_bytes: int, row_pitch: int, *,
                    fetch: bool = True, full_elem_bytes: int = 8) -> ScanResult:
        info = BatchInfo()
        with self.lock:
            call("pg_scan_device", self._h, int(kind), d_ptr, int(n_markers), int(row_bytes), int(row_pitch),
                 byref(info))
            return self._collect(info, fetch, full_elem_bytes)

    def _collect(self, info: BatchInfo, fetch: bool, full_elem_bytes: int,
                 full_out: np.ndarray | None = None) -> ScanResult:
        m = int(info.n_markers)
        res = ScanResult(
            n_markers=m,
            af=np.empty(m), missing_count=np.empty(m, np.int64), variance=np.empty(m),
            skip=np.empty(m, np.int8), clamp_count=int(info.clamp_count),
            decode_ms=float(info.decode_ms), gemm_ms=float(info.gemm_ms), launches=int(info.launches),
            rows_per_marker=int(info.rows_per_marker), n_candidates=int(info.n_candidates),
        )
        if not fetch:
            return res
        call("pg_fetch_marker_stats", self._h, ptr(res.af), ptr(res.missing_count), ptr(res.variance),
             ptr(res.skip))
        if self.mode == _native.PG_MODE_FULL:
            n_rows = c_int64(0)
            call("pg_fetch_full", self._h, None, full_elem_bytes, byref(n_rows))
            dt = np.float32 if full_elem_bytes == 4 else np.float64
            need = n_rows.value * self.n_pheno * full_elem_bytes
            if full_out is not None and full_out.nbytes >= need:
                out = full_out.reshape(-1)[:need].view(dt).reshape(n_rows.value, self.n_pheno)
            else:
                out = np.empty((n_rows.value, self.n_pheno), dtype=dt)
            call("pg_fetch_full", self._h, ptr(out), full_elem_bytes, byref(n_rows))
            res.t_rows = out
            if self.beta_on:
                res.beta_rows = np.empty((n_rows.value, self.n_pheno), dtype=dt)
                call("pg_fetch_full_beta", self._h, ptr(res.beta_rows), full_elem_bytes, byref(n_rows))
        else:
            k = int(info.n_candidates)
            res.cand_rows = np.empty(k, np.int64)
            res.cand_cols = np.empty(k, np.int64)
            res.cand_r = np.empty(k)
            res.cand_t = np.empty(k)
            res.cand_p = np.empty(k)
            if k:
                call("pg_fetch_candidates", self._h, ptr(res.cand_rows), ptr(res.cand_cols), ptr(res.cand_r),
                     ptr(res.cand_t), ptr(res.cand_p))
            if self.beta_on:
                res.cand_beta = np.empty(k)
                res.cand_se = np.empty(k)
                if k:
                    call("pg_fetch_candidate_beta", self._h, ptr(res.cand_beta), ptr(res.cand_se))
        return res

    def time_marker_stats(self, kind: int, d_ptr: int, n_markers: int, pitch: int, reps: int = 5) -> float:
        """Average ms of the statistics kernel alone on a device block (measurement hook)."""
        ms = ctypes.c_float(0.0)
        with self.lock:
            call("pg_time_marker_stats", self._h, int(kind), d_ptr, n_markers, pitch, reps, byref(ms))
        return float(ms.value)

    def track_max_abs_r(self, enable: bool = True) -> None:
        """Track the per-phenotype max |r| of later scans (min-p sidecar); clears it."""
        call("pg_ctx_track_max_abs_r", self._h, 1 if enable else 0)

    def max_abs_r(self) -> np.ndarray:
        out = np.empty(self.n_pheno)
        call("pg_fetch_max_abs_r", self._h, ptr(out))
        return out

    # ------------------------------------------------------------ element-wise statistics
    def t_from_r(self, r: np.ndarray, df: float) -> np.ndarray:
        a = np.ascontiguousarray(r, dtype=np.float64)
        out = np.empty_like(a)
        with self.lock:
            call("pg_t_from_r", self._h, ptr(a), a.size, float(df), ptr(out))
        return out

    def p_from_t(self, t: np.ndarray, df: float) -> tuple[np.ndarray, int]:
        a = np.ascontiguousarray(t, dtype=np.float64)
        out = np.empty_like(a)
        under = c_int64(0)
        with self.lock:
            call("pg_p_from_t", self._h, ptr(a), a.size, float(df), ptr(out), byref(under))
        return out, under.value

    def p_from_t_scalar(self, t: float, df: float) -> float:
        out = c_double(0.0)
        with self.lock:
            call("pg_p_from_t_scalar", self._h, float(t), float(df), byref(out))
        return out.value

    def reg_inc_beta_scalar(self, a: float, b: float, x: float) -> float:
        out = c_double(0.0)
        with self.lock:
            call("pg_reg_inc_beta_scalar", self._h, float(a), float(b), float(x), byref(out))
        return out.value

    def reg_inc_beta(self, a: np.ndarray, b: np.ndarray, x: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        with self.lock:
            call("pg_reg_inc_beta", self._h, ptr(a), ptr(b), ptr(x), x.size, ptr(out))
        return out

    def t_threshold_for_p(self, p_threshold: float, df: float) -> float:
        out = c_double(0.0)
        with self.lock:
            call("pg_t_threshold_for_p", self._h, float(p_threshold), float(df), byref(out))
        return out.value

    # ------------------------------------------------------------ decode / library kernels
    def decode_bed(self, packed: np.ndarray, n_samples: int, dtype) -> tuple[np.ndarray, np.ndarray]:
        blk = np.ascontiguousarray(packed, dtype=np.uint8)
        m, row_bytes = blk.shape
        elem = np.dtype(dtype).itemsize
        out = np.empty((m, n_samples), dtype=np.float32 if elem == 4 else np.float64)
        miss = np.empty(m, np.int64)
        with self.lock:
            call("pg_decode_bed", self._h, ptr(blk), m, row_bytes, int(n_samples), elem, ptr(out), ptr(miss))
        return out, miss

    def decode_bgen(self, rows: np.ndarray, n_samples: int, bits: int) -> tuple[np.ndarray, np.ndarray]:
        blk = np.ascontiguousarray(rows, dtype=np.uint8)
        m = blk.shape[0]
        out = np.empty((m, n_samples), dtype=np.float64)
        miss = np.empty(m, np.int64)
        with self.lock:
            call("pg_decode_bgen", self._h, ptr(blk), None, m, int(n_samples), int(bits), ptr(out), ptr(miss))
        return out, miss

    def prepare_batch(self, dosages: np.ndarray, q: np.ndarray | None, dtype):
        d = np.ascontiguousarray(dosages, dtype=np.float64)
        m, n = d.shape
        elem = np.dtype(dtype).itemsize
        out = np.empty((m, n), dtype=np.float32 if elem == 4 else np.float64)
        af = np.empty(m)
        miss = np.empty(m, np.int64)
        var = np.empty(m)
        skip = np.empty(m, np.int8)
        qq = None if q is None else np.ascontiguousarray(q, dtype=np.float64)
        rank = 0 if qq is None else qq.shape[1]
        with self.lock:
            call("pg_prepare_batch", self._h, ptr(d), m, n, ptr(qq), rank, elem, ptr(out), ptr(af), ptr(miss),
                 ptr(var), ptr(skip))
        return out, af, miss, var, skip

    def correlate(self, gt: np.ndarray, yt: np.ndarray) -> tuple[np.ndarray, int]:
        g = np.ascontiguousarray(gt, dtype=np.float64)
        y = np.ascontiguousarray(yt, dtype=np.float64)
        m, n = g.shape
        p = y.shape[1]
        r = np.empty((m, p))
        clamp = c_int64(0)
        with self.lock:
            call("pg_correlate_f64", self._h, ptr(g), m, n, ptr(y), p, ptr(r), byref(clamp))
        return r, clamp.value


_default: DeviceContext | None = None
_default_lock = threading.Lock()


def default_context() -> DeviceContext:
    """Process-wide context for the library-level functions (lazily created)."""
    global _default
    with _default_lock:
        if _default is None:
            _default = DeviceContext()
        return _default

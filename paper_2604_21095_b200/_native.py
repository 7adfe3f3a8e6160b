"""ctypes binding of the C-ABI library (include/panelgwas_b200.h).

The library is built in-tree (paper_2604_21095_b200/_lib/libpanelgwas_b200.so) by
`build.py`. There is no CPU fallback: if the library or a sm_100 device is
missing, compute calls raise immediately.
"""

from __future__ import annotations

import ctypes
import threading
from ctypes import c_char_p, c_double, c_int, c_int64, c_void_p
from pathlib import Path

import numpy as np

from .errors import ConfigError, FormatError, PanelGwasError

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libpanelgwas_b200.so"

PG_OK = 0
PG_TABLE_GENERIC = 100
PG_ERR_CUDA = 1
PG_ERR_INVALID = 2
PG_ERR_FORMAT = 3
PG_ERR_NOMEM = 4
PG_ERR_STATE = 5
PG_ERR_CONFIG = 6

PG_MODE_THRESHOLD = 0
PG_MODE_TOPK = 1
PG_MODE_FULL = 2

PG_GENO_BED = 0
PG_GENO_BGEN8 = 1
PG_GENO_BGEN16 = 2
PG_GENO_DENSE_F64 = 3


class BatchInfo(ctypes.Structure):
    _fields_ = [
        ("n_markers", c_int64),
        ("n_candidates", c_int64),
        ("clamp_count", c_int64),
        ("n_skipped_monomorphic", c_int64),
        ("n_skipped_all_missing", c_int64),
        ("gemm_ms", c_double),
        ("decode_ms", c_double),
        ("launches", c_int64),
        ("rows_per_marker", c_int64),
    ]


_P = c_void_p  # all array arguments are passed as raw addresses
# (name, argtypes) for every symbol declared in include/panelgwas_b200.h
SIGNATURES: dict[str, list] = {
    "pg_last_error": [],
    "pg_abi_version": [],
    "pg_device_count": [_P],
    "pg_host_alloc": [c_int64, _P],
    "pg_host_free": [_P],
    "pg_ctx_create": [c_int, _P],
    "pg_ctx_destroy": [_P],
    "pg_ctx_sync": [_P],
    "pg_ctx_stream": [_P, _P],
    "pg_ctx_set_panel": [_P, _P, c_int64, c_int64, c_int64, _P, c_int64],
    "pg_ctx_prepare_panel": [_P, _P, c_int64, c_int64, c_int64, _P, c_int64, _P, _P],
    "pg_ctx_commit_panel": [_P, _P, c_int64, _P, c_int64],
    "pg_ctx_set_panel_async": [_P, _P, c_int64, c_int64, c_int64, _P, c_int64, _P, c_int64, c_int64],
    "pg_ctx_panel_async_wait": [_P, _P, _P],
    "pg_ctx_clone_panel": [_P, _P],
    "pg_ctx_follow_panel": [_P, _P],
    "pg_topk_merge": [c_int64, c_int64, _P, _P, _P, c_int64, _P, _P, _P, c_int64, _P, _P],
    "pg_gather_spans": [_P, _P, _P, c_int64, _P],
    "pg_topk_gather": [c_int64, _P, c_int64, c_int, _P, _P, _P],
    "pg_ctx_set_panel_async_cols": [_P, _P, c_int64, c_int64, c_int64, c_int64, c_int64, _P, c_int64, _P, c_int64,
                                    c_int64],
    "pg_ctx_panel_rows_bytes": [_P, c_int64, _P],
    "pg_ctx_export_panel_rows": [_P, _P, c_int64, c_int64],
    "pg_ctx_import_panel_rows": [_P, _P, c_int64, c_int64],
    "pg_ctx_fetch_prepared_panel": [_P, _P],
    "pg_ctx_set_panel_device": [_P, _P, c_int64, c_int64, c_int64, _P, c_int64],
    "pg_ctx_panel_bytes": [_P, _P],
    "pg_ctx_export_panel": [_P, _P],
    "pg_ctx_import_panel": [_P, _P, c_int64, c_int64, _P, c_int64],
    "pg_ctx_set_scan": [_P, c_double, c_int, _P],
    "pg_ctx_set_rbar": [_P, _P],
    "pg_ctx_set_fused_decode": [_P, c_int],
    "pg_ctx_set_missing_side_gemm": [_P, c_int],
    "pg_ctx_set_f64_panel": [_P, c_int],
    "pg_ctx_set_two_limb_premask": [_P, c_int],
    "pg_ctx_set_wide_digits": [_P, c_int],
    "pg_ctx_set_basis": [_P, _P, c_int64, c_int64],
    "pg_scan": [_P, c_int, _P, c_int64, c_int64, _P],
    "pg_scan_device": [_P, c_int, _P, c_int64, c_int64, c_int64, _P],
    "pg_stage": [_P, c_int, c_int, _P, c_int64, c_int64],
    "pg_stage_bgen": [_P, c_int, _P, c_int64, _P, _P, c_int64, _P],
    "pg_stage_bgen_begin": [_P, c_int, _P, c_int64, _P, _P, c_int64],
    "pg_stage_bgen_end": [_P, c_int, _P],
    "pg_scan_staged": [_P, c_int, _P],
    "pg_fetch_marker_stats": [_P, _P, _P, _P, _P],
    "pg_fetch_candidates": [_P, _P, _P, _P, _P, _P],
    "pg_fetch_full": [_P, _P, c_int, _P],
    "pg_fetch_max_abs_r": [_P, _P],
    "pg_ctx_track_max_abs_r": [_P, c_int],
    "pg_format_float_columns": [c_int64, c_int, _P, _P, c_int64, _P],
    "pg_ctx_set_beta_scale": [_P, _P, c_int64],
    "pg_fetch_candidate_beta": [_P, _P, _P],
    "pg_fetch_full_beta": [_P, _P, c_int, _P],
    "pg_ctx_debug_candidate_base": [_P, ctypes.c_uint64],
    "pg_t_from_r": [_P, _P, c_int64, c_double, _P],
    "pg_p_from_t": [_P, _P, c_int64, c_double, _P, _P],
    "pg_p_from_t_scalar": [_P, c_double, c_double, _P],
    "pg_reg_inc_beta_scalar": [_P, c_double, c_double, c_double, _P],
    "pg_reg_inc_beta": [_P, _P, _P, _P, c_int64, _P],
    "pg_t_threshold_for_p": [_P, c_double, c_double, _P],
    "pg_decode_bed": [_P, _P, c_int64, c_int64, c_int64, c_int, _P, _P],
    "pg_decode_bgen": [_P, _P, _P, c_int64, c_int64, c_int, _P, _P],
    "pg_prepare_batch": [_P, _P, c_int64, c_int64, _P, c_int64, c_int, _P, _P, _P, _P, _P],
    "pg_correlate_f64": [_P, _P, c_int64, c_int64, _P, c_int64, _P, _P],
    "pg_bgen_index": [c_char_p, c_int64, c_int64, _P, _P, _P, _P, c_int64, _P, _P],
    "pg_bgen_inflate": [c_char_p, _P, _P, c_int64, c_int64, c_int, _P, c_int64, _P, _P, _P],
    "pg_table_parse": [_P, c_int64, c_int64, ctypes.c_char, c_int64, c_int64, c_int, c_int64, _P, _P, _P, _P, _P,
                       _P, _P, _P],
    "pg_format_float_repr": [_P, c_int64, _P, c_int64, _P],
    "pg_format_tsv": [c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, c_int64, _P, c_int64, _P],
    "pg_format_marker_lines": [c_int64, _P, _P, _P, _P, _P, _P, _P, c_int64, _P],
    "pg_bim_index": [_P, c_int64, c_int64, _P, _P, _P, _P, _P],
    "pg_bim_prefixes": [_P, _P, _P, _P, c_int64, c_int64, c_int, _P, c_int64, _P],
    "pg_time_marker_stats": [_P, c_int, _P, c_int64, c_int64, c_int, _P],
    "pg_debug_inflate": [_P, c_int64, _P, _P, c_int64, c_int64, _P, c_int64, _P, _P],
    "pg_debug_assoc_gemm": [_P, _P, _P, c_int64, _P, _P, c_int64, c_int64, _P, _P],
}

_lib = None
_lock = threading.Lock()


def load_library(path: Path | None = None):
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise PanelGwasError(
                f"panelgwas_b200 native library not built: {p} (run paper_2604_21095_b200/build.py)"
            )
        lib = ctypes.CDLL(str(p))
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue
            fn.argtypes = argtypes
            fn.restype = c_char_p if name == "pg_last_error" else c_int
        _lib = lib
        return lib


def exported_symbols(path: Path | None = None) -> set[str]:
    lib = load_library(path)
    return {name for name in SIGNATURES if getattr(lib, name, None) is not None}


def check(status: int) -> None:
    """Map a PG_* status onto the reference exception hierarchy (errors.py)."""
    if status == PG_OK:
        return
    msg = (_lib.pg_last_error() or b"").decode(errors="replace") if _lib is not None else ""
    if status == PG_ERR_INVALID:
        raise ValueError(msg)
    if status == PG_ERR_FORMAT:
        raise FormatError(msg)
    if status == PG_ERR_CONFIG:
        raise ConfigError(msg)
    raise PanelGwasError(f"panelgwas_b200 native error {status}: {msg}")


def call(name: str, *args) -> None:
    lib = load_library()
    check(getattr(lib, name)(*args))


def ptr(a: np.ndarray | None) -> int | None:
    """Address of a C-contiguous numpy array (None passes NULL)."""
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("native call needs a C-contiguous array")
    return a.ctypes.data


def device_count() -> int:
    n = c_int(0)
    call("pg_device_count", ctypes.addressof(n))
    return n.value


def require_device() -> None:
    if device_count() < 1:
        raise PanelGwasError("panelgwas_b200 requires an NVIDIA B200 (sm_100) device; none is visible")


class PinnedBuffer:
    """Page-locked host bytes (pg_host_alloc) viewed as a numpy uint8 array."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        p = c_void_p()
        call("pg_host_alloc", self.nbytes, ctypes.byref(p))
        self._ptr = p
        self.array = np.ctypeslib.as_array((ctypes.c_uint8 * self.nbytes).from_address(p.value))

    def close(self) -> None:
        if self._ptr:
            self.array = None
            load_library().pg_host_free(self._ptr)
            self._ptr = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

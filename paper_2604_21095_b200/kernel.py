"""Numerical API of the association engine (names and semantics of
/root/reference/pkg/src/panelgwas/kernel.py).

Per-marker and per-pair numerics run on the B200 through the C ABI:
  prepare_genotype_batch -> pg_prepare_batch   (fp64, csrc/libkern.cu)
  correlate              -> pg_correlate_f64   (fp64, fixed K order per output)
  t_from_r / p_from_t / reg_inc_beta / t_threshold_for_p -> csrc/pstats.cu
The scan itself (engine.run_scan) does not call these: it uses the fused
integer tensor-core path (csrc/assoc_gemm.cu) that computes the same r.

The panel-side preprocessing (build_covariate_basis, residualize,
standardize_columns) runs once per scan on the host in float64, exactly as
the reference does; its output is quantized and made resident on the device
by the engine (csrc/panel.cu).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .errors import PanelGwasError
from .genotypes.types import MarkerRecord, RawBatch

P_FLOOR = float(np.finfo(np.float64).tiny)
MONOMORPHIC_VARIANCE = 1e-12


def _dev():
    from ._device import default_context

    return default_context()


# ---------------------------------------------------------------------------
# p-values


def reg_inc_beta(a, b, x):
    """Regularized incomplete beta I_x(a, b) (device Lentz continued fraction)."""
    scalar = np.ndim(a) == 0 and np.ndim(b) == 0 and np.ndim(x) == 0
    a_arr = np.asarray(a, dtype=np.float64)
    b_arr = np.asarray(b, dtype=np.float64)
    x_arr = np.asarray(x, dtype=np.float64)
    if np.any(a_arr <= 0.0) or np.any(b_arr <= 0.0):
        raise ValueError("reg_inc_beta requires a > 0 and b > 0")
    if np.any(x_arr < 0.0) or np.any(x_arr > 1.0):
        raise ValueError("reg_inc_beta requires x in [0, 1]")
    ab, bb, xb = np.broadcast_arrays(a_arr, b_arr, x_arr)
    out = _dev().reg_inc_beta(ab.ravel(), bb.ravel(), xb.ravel()).reshape(xb.shape)
    if scalar:
        return float(out)
    return out


def p_from_t(t, df: float):
    """Two-sided p = I_{df/(df+t^2)}(df/2, 1/2), floored at P_FLOOR; p(0) = 1."""
    if df < 1.0:
        raise ValueError("p_from_t requires df >= 1")
    scalar = np.ndim(t) == 0
    arr = np.asarray(t, dtype=np.float64)
    p, _ = _dev().p_from_t(arr.ravel(), df)
    p = p.reshape(arr.shape)
    return float(p) if scalar else p


def t_threshold_for_p(p_threshold: float, df: float) -> float:
    """Smallest |t| with two-sided p <= p_threshold (device bisection)."""
    if not 0.0 < p_threshold <= 1.0:
        raise ValueError("p_threshold must be in (0, 1]")
    return _dev().t_threshold_for_p(float(p_threshold), float(df))


# ---------------------------------------------------------------------------
# covariate basis and panel preprocessing (host, once per scan)


@dataclass(frozen=True)
class CovariateBasis:
    """Orthonormal basis Q of span([1 | covariates]) with the dropped-column record."""

    q: np.ndarray
    source_columns: tuple[str, ...]
    dropped_columns: tuple[str, ...]

    @property
    def rank(self) -> int:
        return self.q.shape[1]

    @property
    def n_samples(self) -> int:
        return self.q.shape[0]


def build_covariate_basis(covariates: np.ndarray, include_intercept: bool = True, rank_tolerance: float = 1e-8,
                          column_names: list[str] | None = None) -> CovariateBasis:
    """Two-pass Gram–Schmidt over [intercept | covariates] with rank detection.

    A column is dropped when its residual norm after projection on the columns
    already accepted is <= rank_tolerance times its own norm (or it is zero).
    """
    c = np.asarray(covariates, dtype=np.float64)
    if c.ndim != 2:
        raise ValueError("covariates must be a 2-D (samples x columns) array")
    if np.isnan(c).any():
        raise ValueError("covariate matrix contains NaN")
    n = c.shape[0]
    labels = list(column_names) if column_names else [f"covar{j + 1}" for j in range(c.shape[1])]
    if len(labels) != c.shape[1]:
        raise ValueError("column_names length does not match covariates")
    ct = np.ascontiguousarray(c.T)  # contiguous columns (the loop below is per column)
    cols = ([("intercept", np.ones(n))] if include_intercept else []) + [
        (labels[j], ct[j]) for j in range(c.shape[1])
    ]
    basis: list[np.ndarray] = []
    kept: list[str] = []
    dropped: list[str] = []
    for name, col in cols:
        norm0 = float(np.linalg.norm(col))
        v = np.array(col, dtype=np.float64)
        for _sweep in range(2):  # re-orthogonalize once
            for qv in basis:
                v -= (qv @ v) * qv
        norm_v = float(np.linalg.norm(v))
        if norm0 == 0.0 or norm_v <= rank_tolerance * norm0:
            dropped.append(name)
        else:
            basis.append(v / norm_v)
            kept.append(name)
    q = np.column_stack(basis) if basis else np.zeros((n, 0))
    if n < q.shape[1] + 2:
        raise PanelGwasError(
            f"insufficient residual degrees of freedom: {n} samples for a rank-{q.shape[1]} covariate basis"
        )
    return CovariateBasis(q, tuple(kept), tuple(dropped))


def residualize(y: np.ndarray, basis: CovariateBasis) -> np.ndarray:
    """Centre columns, then subtract their projection on Q (no N x N projector)."""
    y = np.asarray(y, dtype=np.float64)
    if y.ndim != 2:
        raise ValueError("expected a 2-D (samples x phenotypes) matrix")
    if y.shape[0] != basis.n_samples:
        raise ValueError(f"row count {y.shape[0]} does not match basis ({basis.n_samples} samples)")
    out = y - y.mean(axis=0, keepdims=True)
    if basis.rank:
        out -= basis.q @ (basis.q.T @ out)
    return out


def standardize_columns(y_res: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Unit 1/N-variance columns; zero-variance columns are zero-filled and flagged."""
    y = np.asarray(y_res, dtype=np.float64)
    if not np.isfinite(y).all():
        raise ValueError("standardize_columns requires finite input")
    centre = y.mean(axis=0)
    dev = y - centre
    sd = np.sqrt(np.mean(dev * dev, axis=0))
    flat = sd <= 1e-12 * np.maximum(1.0, np.abs(centre))
    out = dev / np.where(flat, 1.0, sd)
    out[:, flat] = 0.0
    return out, sd, flat


# ---------------------------------------------------------------------------
# genotype batch preparation (device)


class SkipReason(enum.IntEnum):
    NONE = 0
    MONOMORPHIC = 1
    ALL_MISSING = 2


@dataclass(frozen=True)
class StandardizedBatch:
    """Imputed, centred, unit-variance marker rows plus per-marker QC."""

    markers: tuple[MarkerRecord, ...]
    matrix: np.ndarray
    allele_frequency: np.ndarray
    missing_count: np.ndarray
    variance_before_scaling: np.ndarray
    skip_reason: np.ndarray

    @property
    def skip_mask(self) -> np.ndarray:
        return self.skip_reason != SkipReason.NONE


def prepare_genotype_batch(raw: RawBatch, basis: CovariateBasis | None = None, residualize_genotypes: bool = False,
                           dtype=np.float64) -> StandardizedBatch:
    """Mean-impute, centre, [project off Q,] scale rows to unit 1/N variance — on the device in fp64."""
    q = basis.q if (residualize_genotypes and basis is not None and basis.rank) else None
    out_dtype = np.float32 if np.dtype(dtype) == np.float32 else np.float64
    mat, af, miss, var, skip = _dev().prepare_batch(np.asarray(raw.dosages, dtype=np.float64), q, out_dtype)
    return StandardizedBatch(raw.markers, mat.astype(dtype, copy=False), af, miss, var, skip)


# ---------------------------------------------------------------------------
# correlation and statistics


def correlate(gt: np.ndarray, yt: np.ndarray) -> tuple[np.ndarray, int]:
    """R = G Y / N for 1/N-standardized rows / columns, clipped to [-1, 1]; (R, clamp count)."""
    if gt.ndim != 2 or yt.ndim != 2 or gt.shape[1] != yt.shape[0]:
        raise ValueError(f"shape mismatch: genotypes {gt.shape} vs phenotypes {yt.shape}")
    return _dev().correlate(gt, yt)


def t_from_r(r, df: float):
    """t = r sqrt(df / (1 - r^2)), |r| capped at 1 - 1e-15; |r| >= 1 -> signed infinity."""
    if df < 1.0:
        raise ValueError("t_from_r requires df >= 1")
    scalar = np.ndim(r) == 0
    arr = np.asarray(r, dtype=np.float64)
    t = _dev().t_from_r(arr.ravel(), df).reshape(arr.shape)
    return float(t) if scalar else t


@dataclass(frozen=True)
class StatBlock:
    """Association statistics of one standardized block."""

    r: np.ndarray
    t: np.ndarray
    df: float
    p: np.ndarray | None
    clamp_count: int
    p_underflow_count: int


def compute_stats(gt_std: np.ndarray, yt_std: np.ndarray, df: float, with_p: bool = True) -> StatBlock:
    """correlate -> t_from_r -> p_from_t over a full block."""
    r, clamped = correlate(gt_std, yt_std)
    t = t_from_r(r, df)
    p = None
    under = 0
    if with_p:
        if df < 1.0:
            raise ValueError("p_from_t requires df >= 1")
        pf, under = _dev().p_from_t(np.asarray(t, dtype=np.float64).ravel(), df)
        p = pf.reshape(np.shape(t))
    return StatBlock(r, t, df, p, clamped, under)

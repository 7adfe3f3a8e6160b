"""Per-batch numerical API of the association engine.

Same names, arguments and error behaviour as /root/reference/pkg/src/panelgwas/kernel.py.
What runs where:

    statistics     correlate, t_from_r, p_from_t, reg_inc_beta, t_threshold_for_p,
                   compute_stats                        -> device (csrc/libkern.cu, csrc/pstats.cu)
    genotypes      prepare_genotype_batch                -> device, fp64 (pg_prepare_batch)
    panel          build_covariate_basis, residualize,
                   standardize_columns                   -> host fp64 (the oracle of csrc/panel_prep.cu)

`engine.run_scan` does not go through this module: the scan uses the fused integer
tensor-core contraction (csrc/assoc_gemm.cu), which produces the same r.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .errors import PanelGwasError
from .genotypes.types import MarkerRecord, RawBatch

#: smallest reported p (the smallest normal double)
P_FLOOR = float(np.finfo(np.float64).tiny)
MONOMORPHIC_VARIANCE = 1e-12


def _dev():
    from ._device import default_context

    return default_context()


def _require(ok: bool, message: str) -> None:
    if not ok:
        raise ValueError(message)


def _flat64(x) -> tuple[np.ndarray, tuple, bool]:
    """(contiguous float64 vector, original shape, was-a-scalar) of an array-like."""
    arr = np.asarray(x, dtype=np.float64)
    return arr.ravel(), arr.shape, arr.ndim == 0


def _reshape(v: np.ndarray, shape: tuple, scalar: bool):
    return float(v[0]) if scalar else v.reshape(shape)


# === statistics (device) ======================================================================


def correlate(gt: np.ndarray, yt: np.ndarray) -> tuple[np.ndarray, int]:
    """(R, clamp count): R = G Y / N of 1/N-standardized genotype rows and phenotype columns,
    clipped to [-1, 1]; fp64 on the device with a fixed summation order per output."""
    conformable = gt.ndim == 2 and yt.ndim == 2 and gt.shape[1] == yt.shape[0]
    _require(conformable, f"shape mismatch: genotypes {gt.shape} vs phenotypes {yt.shape}")
    return _dev().correlate(gt, yt)


def t_from_r(r, df: float):
    """t = r sqrt(df / (1 - r^2)) with |r| capped at 1 - 1e-15 (|r| >= 1 gives +-inf)."""
    _require(df >= 1.0, "t_from_r requires df >= 1")
    v, shape, scalar = _flat64(r)
    return _reshape(_dev().t_from_r(v, df), shape, scalar)


def p_from_t(t, df: float):
    """Two-sided Student-t p = I_{df/(df+t^2)}(df/2, 1/2), floored at P_FLOOR (p(0) = 1)."""
    _require(df >= 1.0, "p_from_t requires df >= 1")
    if np.ndim(t) == 0:  # the reference's scalar path (kernel.py:201-204), as t_threshold_for_p uses
        return _dev().p_from_t_scalar(float(t), float(df))
    v, shape, scalar = _flat64(t)
    p, _ = _dev().p_from_t(v, df)
    return _reshape(p, shape, scalar)


def reg_inc_beta(a, b, x):
    """Regularized incomplete beta I_x(a, b): Lentz continued fraction on the device,
    broadcasting a, b and x."""
    arrs = [np.asarray(v, dtype=np.float64) for v in (a, b, x)]
    _require(not (np.any(arrs[0] <= 0.0) or np.any(arrs[1] <= 0.0)), "reg_inc_beta requires a > 0 and b > 0")
    _require(not (np.any(arrs[2] < 0.0) or np.any(arrs[2] > 1.0)), "reg_inc_beta requires x in [0, 1]")
    if all(w.ndim == 0 for w in arrs):  # scalar path (kernel.py:156-163)
        return _dev().reg_inc_beta_scalar(float(arrs[0]), float(arrs[1]), float(arrs[2]))
    wide = np.broadcast_arrays(*arrs)
    vals = _dev().reg_inc_beta(*(w.ravel() for w in wide))
    return _reshape(vals, wide[2].shape, all(w.ndim == 0 for w in arrs))


def t_threshold_for_p(p_threshold: float, df: float) -> float:
    """Smallest |t| whose two-sided p is <= p_threshold (bisection on the device)."""
    _require(0.0 < p_threshold <= 1.0, "p_threshold must be in (0, 1]")
    return _dev().t_threshold_for_p(float(p_threshold), float(df))


@dataclass(frozen=True)
class StatBlock:
    """r, t (and p) of one standardized block, with the clamp / p-underflow counts."""

    r: np.ndarray
    t: np.ndarray
    df: float
    p: np.ndarray | None
    clamp_count: int
    p_underflow_count: int


def compute_stats(gt_std: np.ndarray, yt_std: np.ndarray, df: float, with_p: bool = True) -> StatBlock:
    """correlate, then t_from_r, then (with_p) p_from_t for a whole block."""
    r, n_clamped = correlate(gt_std, yt_std)
    t = t_from_r(r, df)
    if not with_p:
        return StatBlock(r, t, df, None, n_clamped, 0)
    _require(df >= 1.0, "p_from_t requires df >= 1")
    p, n_under = _dev().p_from_t(np.ravel(np.asarray(t, dtype=np.float64)), df)
    return StatBlock(r, t, df, p.reshape(np.shape(t)), n_clamped, n_under)


# === genotype rows (device) ===================================================================


class SkipReason(enum.IntEnum):
    """Why a marker produced no statistics."""

    NONE = 0
    MONOMORPHIC = 1
    ALL_MISSING = 2


@dataclass(frozen=True)
class StandardizedBatch:
    """Marker rows after imputation and standardization, with per-marker QC columns."""

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
    """Per marker row: mean-impute missing calls, centre, optionally project off Q, scale to
    unit 1/N variance (fp64 on the device); rows that cannot be scaled are flagged."""
    use_q = residualize_genotypes and basis is not None and basis.rank > 0
    want32 = np.dtype(dtype) == np.float32
    mat, af, n_miss, var, skip = _dev().prepare_batch(
        np.asarray(raw.dosages, dtype=np.float64), basis.q if use_q else None,
        np.float32 if want32 else np.float64)
    return StandardizedBatch(raw.markers, mat.astype(dtype, copy=False), af, n_miss, var, skip)


# === phenotype panel (host, once per scan) ====================================================


@dataclass(frozen=True)
class CovariateBasis:
    """Orthonormal Q spanning [intercept | covariates], with which input columns were kept
    and which were dropped as (numerically) dependent."""

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
    """Gram–Schmidt with one re-orthogonalization sweep over [intercept | covariates].

    Candidates are taken in order; each is projected off the accepted vectors (sequentially,
    twice) and dropped when its residual norm is <= rank_tolerance times its original norm or
    the column is zero."""
    cov = np.asarray(covariates, dtype=np.float64)
    _require(cov.ndim == 2, "covariates must be a 2-D (samples x columns) array")
    _require(not np.isnan(cov).any(), "covariate matrix contains NaN")
    n, k = cov.shape
    names = [f"covar{j}" for j in range(1, k + 1)] if not column_names else list(column_names)
    _require(len(names) == k, "column_names length does not match covariates")

    candidates = list(zip(names, np.ascontiguousarray(cov.T)))  # one contiguous row per column
    if include_intercept:
        candidates.insert(0, ("intercept", np.ones(n)))
    accepted = np.empty((len(candidates), n))
    n_acc = 0
    kept, dropped = [], []
    for name, column in candidates:
        scale = float(np.linalg.norm(column))
        resid = column.astype(np.float64, copy=True)
        for _ in (0, 1):
            for i in range(n_acc):
                resid -= (accepted[i] @ resid) * accepted[i]
        rn = float(np.linalg.norm(resid))
        if scale > 0.0 and rn > rank_tolerance * scale:
            accepted[n_acc] = resid / rn
            n_acc += 1
            kept.append(name)
        else:
            dropped.append(name)
    q = np.ascontiguousarray(accepted[:n_acc].T) if n_acc else np.zeros((n, 0))
    if n < n_acc + 2:
        raise PanelGwasError(
            f"insufficient residual degrees of freedom: {n} samples for a rank-{n_acc} covariate basis")
    return CovariateBasis(q, tuple(kept), tuple(dropped))


def residualize(y: np.ndarray, basis: CovariateBasis) -> np.ndarray:
    """Column-centred Y minus Q Q^T of it (applied as two thin products, never N x N)."""
    mat = np.asarray(y, dtype=np.float64)
    _require(mat.ndim == 2, "expected a 2-D (samples x phenotypes) matrix")
    _require(mat.shape[0] == basis.n_samples,
             f"row count {mat.shape[0]} does not match basis ({basis.n_samples} samples)")
    res = mat - mat.mean(axis=0, keepdims=True)
    if basis.rank > 0:
        res -= basis.q @ (basis.q.T @ res)
    return res


def standardize_columns(y_res: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(columns scaled to zero mean and unit 1/N variance, their sd, zero-variance flags);
    flagged columns are returned as zeros."""
    mat = np.asarray(y_res, dtype=np.float64)
    _require(bool(np.isfinite(mat).all()), "standardize_columns requires finite input")
    mu = mat.mean(axis=0)
    centred = mat - mu
    sd = np.sqrt(np.mean(centred * centred, axis=0))
    flat = sd <= 1e-12 * np.maximum(1.0, np.abs(mu))
    z = centred / np.where(flat, 1.0, sd)
    z[:, flat] = 0.0
    return z, sd, flat

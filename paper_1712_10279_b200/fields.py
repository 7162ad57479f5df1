"""Boundary value types of the drop-in (the reference's S/fields.py:37-289).

Grids, marginals and the returned fluxes keep the reference's names, shapes,
dtypes and validation errors so that callers of ``otflux.solve_*`` can switch
without changes.  Objects of the reference package itself are accepted too
(anything exposing ``.values`` of the right shape).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatchError, ValidationError

PSD_EIG_TOL = -1e-10


@dataclass(frozen=True)
class GridSpec:
    """n x n cells on the unit square, dx = 1/(n-1) (S/fields.py:37-53)."""

    n: int

    def __post_init__(self):
        if not isinstance(self.n, (int, np.integer)) or self.n < 2:
            raise ValidationError(f"grid needs an integer n >= 2, got {self.n!r}")

    @property
    def dx(self) -> float:
        return 1.0 / (self.n - 1)

    def coords(self) -> np.ndarray:
        return np.arange(self.n) * self.dx


def hermitian_part(x):
    """(X + X^H)/2 of the trailing two axes (exact on Hermitian input)."""
    x = np.asarray(x)
    xh = np.swapaxes(x, -1, -2)
    return 0.5 * (x + (np.conj(xh) if np.iscomplexobj(x) else xh))


def skew_part(x):
    """(X - X^H)/2 of the trailing two axes."""
    x = np.asarray(x)
    xh = np.swapaxes(x, -1, -2)
    return 0.5 * (x - (np.conj(xh) if np.iscomplexobj(x) else xh))


def _defect(x, sign):
    return float(np.max(np.abs(x - sign * np.conj(np.swapaxes(x, -1, -2))))) if x.size else 0.0


def _grid_array(values, min_ndim, who):
    arr = np.asarray(values)
    if arr.ndim < min_ndim or arr.shape[0] != arr.shape[1]:
        raise ValidationError(f"{who}: expected (n, n, ...) array, got shape {arr.shape}")
    if arr.shape[0] < 2:
        raise ValidationError(f"{who}: grid side must be >= 2")
    if not np.all(np.isfinite(arr)):
        raise ValidationError(f"{who}: non-finite entries")
    return arr


class _Density:
    """An (n, n, payload) marginal, validated on construction.  The three
    kinds differ in rank, dtype and a per-kind check (`_admit`); the error
    classes and messages are the reference's."""

    _RANK = 2
    _DTYPE = np.float64

    def __post_init__(self):
        who = type(self).__name__
        arr = _grid_array(self.values, self._RANK, who).astype(self._DTYPE)
        object.__setattr__(self, "values", self._admit(arr, who))

    @classmethod
    def _admit(cls, arr, who):
        if arr.ndim != cls._RANK:
            raise ValidationError(f"{who}: expected {cls._RANK}-d array, got {arr.ndim}-d")
        if arr.min() < 0:
            raise ValidationError(f"{who}: negative entries")
        return arr

    @property
    def n(self) -> int:
        return self.values.shape[0]

    @property
    def grid(self) -> GridSpec:
        return GridSpec(self.n)

    @property
    def k(self) -> int:
        """channels (vector) or matrix side (matrix) of the payload"""
        return self.values.shape[2]


@dataclass(frozen=True)
class ScalarDensity(_Density):
    values: np.ndarray


@dataclass(frozen=True)
class VectorDensity(_Density):
    values: np.ndarray
    _RANK = 3


@dataclass(frozen=True)
class MatrixDensity(_Density):
    """Per-cell Hermitian PSD k x k matrices; stored as their exact
    Hermitian part."""

    values: np.ndarray
    _RANK = 4
    _DTYPE = np.complex128

    @classmethod
    def _admit(cls, arr, who):
        if arr.ndim != 4 or arr.shape[2] != arr.shape[3]:
            raise ValidationError(f"{who}: expected (n, n, k, k), got {arr.shape}")
        scale = max(float(np.max(np.abs(arr))), 1.0)
        if _defect(arr, 1) > 1e-10 * scale:
            raise ValidationError(f"{who}: per-cell matrices not Hermitian")
        herm = hermitian_part(arr)
        if float(np.linalg.eigvalsh(herm).min()) < PSD_EIG_TOL * scale:
            raise ValidationError(f"{who}: matrix below the PSD tolerance")
        return herm

    def trace_field(self) -> np.ndarray:
        return np.real(np.trace(self.values, axis1=2, axis2=3))


def total_mass(d) -> float:
    """Sum of masses; trace sum for matrix fields (S/fields.py:211-215)."""
    v = np.asarray(d.values)
    if v.ndim == 4:
        return float(np.sum(np.real(np.trace(v, axis1=2, axis2=3))))
    return float(np.sum(v))


def normalize(d):
    m = total_mass(d)
    if m <= 0:
        raise ValidationError(f"cannot normalize field with total mass {m:g}")
    return type(d)(d.values / m)


def _trusted(cls, **fields):
    """Build a value object from arrays the engine produced (already in the
    canonical dtype, finite and structured), skipping re-validation."""
    obj = object.__new__(cls)
    for k, v in fields.items():
        object.__setattr__(obj, k, v)
    return obj


@dataclass(frozen=True)
class FluxField:
    """Staggered flux with zero ghost row of ux / ghost column of uy."""

    ux: np.ndarray
    uy: np.ndarray

    def __post_init__(self):
        ux = np.asarray(self.ux)
        uy = np.asarray(self.uy)
        if ux.shape != uy.shape:
            raise DimensionMismatchError(f"ux/uy shapes differ: {ux.shape} vs {uy.shape}")
        if ux.ndim < 2 or ux.shape[0] != ux.shape[1]:
            raise ValidationError(f"FluxField: expected (n, n, ...) arrays, got {ux.shape}")
        if np.any(ux[-1, :] != 0) or np.any(uy[:, -1] != 0):
            raise ValidationError("FluxField: ghost entries must be exactly zero")
        object.__setattr__(self, "ux", ux)
        object.__setattr__(self, "uy", uy)

    @classmethod
    def zeros(cls, grid: GridSpec, payload_shape=(), dtype=np.float64):
        shape = (grid.n, grid.n) + tuple(payload_shape)
        return cls(np.zeros(shape, dtype), np.zeros(shape, dtype))

    @property
    def n(self) -> int:
        return self.ux.shape[0]


@dataclass(frozen=True)
class GraphFlux:
    """Per-cell edge fluxes (n, n, ell)."""

    values: np.ndarray

    def __post_init__(self):
        arr = _grid_array(self.values, 3, type(self).__name__)
        object.__setattr__(self, "values", arr.astype(np.float64))


@dataclass(frozen=True)
class QuantumFlux:
    """Per-cell stacks of ell skew-Hermitian k x k matrices (n, n, ell, k, k),
    stored as their exact skew part."""

    values: np.ndarray

    def __post_init__(self):
        who = type(self).__name__
        arr = _grid_array(self.values, 5, who).astype(np.complex128)
        if arr.ndim != 5 or arr.shape[3] != arr.shape[4]:
            raise ValidationError(f"{who}: expected (n, n, ell, k, k), got {arr.shape}")
        if _defect(arr, -1) > 1e-10 * max(float(np.max(np.abs(arr))), 1.0):
            raise ValidationError(f"{who}: matrices not skew-Hermitian")
        object.__setattr__(self, "values", skew_part(arr))

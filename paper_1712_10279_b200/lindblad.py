"""Lindblad (commutator) channel operator setup for matrix transport (host,
one-time).  The per-cell commutators [L_s, X] and sum_s (Z_s L_s - L_s Z_s) run
inside the CUDA sweep; here we validate the matrix set and compute the spectral
bound of -div_L grad_L that sets nu.  Semantics follow S/lindblad.py:37-186.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import NumericalError, ValidationError
from .fields import hermitian_part

KERNEL_EIG_TOL = 1e-10


def _stack(matrices) -> np.ndarray:
    arr = np.asarray(matrices)
    arr = arr.astype(np.complex128 if np.iscomplexobj(arr) else np.float64)
    if arr.ndim == 2:
        arr = arr[None]
    if arr.ndim != 3 or arr.shape[1] != arr.shape[2]:
        raise ValidationError(f"expected (ell, k, k) Hermitian stack, got shape {arr.shape}")
    scale = max(float(np.max(np.abs(arr))), 1.0)
    if float(np.max(np.abs(arr - np.conj(np.swapaxes(arr, -1, -2))))) > 1e-10 * scale:
        raise ValidationError("matrices must be Hermitian")
    return hermitian_part(arr)


def hermitian_basis(k: int) -> np.ndarray:
    """Orthonormal basis of k x k Hermitian matrices (diagonal units, then
    symmetric and antisymmetric off-diagonal pairs)."""
    out = []
    for i in range(k):
        e = np.zeros((k, k), dtype=np.complex128)
        e[i, i] = 1.0
        out.append(e)
    h = 1.0 / np.sqrt(2.0)
    for i in range(k):
        for j in range(i + 1, k):
            s = np.zeros((k, k), dtype=np.complex128)
            s[i, j] = s[j, i] = h
            a = np.zeros((k, k), dtype=np.complex128)
            a[i, j] = 1j * h
            a[j, i] = -1j * h
            out += [s, a]
    return np.stack(out)


def operator_matrix(mats) -> np.ndarray:
    """Dense k^2 x k^2 form of -div_L grad_L in hermitian_basis."""
    mats = np.asarray(mats, dtype=np.complex128)
    B = hermitian_basis(mats.shape[-1])
    G = (np.einsum("sab,mbc->msac", mats, B) - np.einsum("mab,sbc->msac", B, mats))
    M = np.real(np.einsum("aspq,bspq->ab", G, np.conj(G)))
    return 0.5 * (M + M.T)


def check_kernel(matrices) -> bool:
    """True iff the commutator gradient vanishes exactly on span{I}."""
    ev = np.linalg.eigvalsh(operator_matrix(_stack(matrices)))
    return int(np.sum(ev <= KERNEL_EIG_TOL * max(float(ev.max()), 0.0))) == 1


@dataclass(frozen=True)
class LindbladSet:
    """ell Hermitian k x k matrices whose commutator gradient has kernel span{I}."""

    matrices: np.ndarray

    def __post_init__(self):
        arr = _stack(self.matrices)
        if not check_kernel(arr):
            raise ValidationError("gradient kernel is not span{I}; the matrix set is degenerate")
        object.__setattr__(self, "matrices", arr)

    @property
    def ell(self) -> int:
        return self.matrices.shape[0]

    @property
    def k(self) -> int:
        return self.matrices.shape[1]


def lambda_max_L(L) -> float:
    mats = L.matrices if hasattr(L, "matrices") else _stack(L)
    try:
        return float(np.linalg.eigvalsh(operator_matrix(mats)).max())
    except np.linalg.LinAlgError as exc:  # pragma: no cover
        raise NumericalError(f"eigensolve failed: {exc}") from exc


def default_lindblad3() -> LindbladSet:
    """The 3x3 pair used by the DTI fixtures (S/lindblad.py:218-222)."""
    return LindbladSet(np.stack([np.diag([1.0, 2.0, 0.0]),
                                 np.array([[1.0, 1, 1], [1, 0, 0], [1, 0, 0]])]).astype(np.complex128))


def lindblad_pair_k2() -> LindbladSet:
    """{diag(1,-1), sigma_x}, the k=2 set of the acceptance suite."""
    return LindbladSet(np.stack([np.diag([1.0, -1.0]),
                                 np.array([[0.0, 1.0], [1.0, 0.0]])]).astype(np.complex128))

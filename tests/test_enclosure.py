"""The spectral-enclosure shortcut of the nuclear prox (csrc/payload.cuh
herm_nuc_prox, K >= 3), restated in NumPy and checked against the oracle's
eigendecomposition prox (oracle/pdhg.py eig_soft, S/shrink.py:161-169).

For m = tr X / K and rho = sqrt((K-1)/K) ||X - m I||_F (widened by a relative
1e-12), every eigenvalue lies in [m - rho, m + rho].  When that interval is on
one piece of the soft threshold, the prox is X - thr I, X + thr I or 0 and the
kernel skips the eigensolve.  Here: the interval contains the spectrum, and
each shortcut equals the eigendecomposition result to rounding."""
import numpy as np
import pytest

from oracle.pdhg import eig_soft


def enclosure_piece(x, thr):
    k = x.shape[0]
    m = np.trace(x).real / k
    f2 = np.sum(np.abs(x - m * np.eye(k)) ** 2)
    rho = np.sqrt(f2 * (k - 1) / k) * (1 + 1e-12) + abs(m) * 1e-12
    if m - rho > thr:
        return 1, m, rho
    if m + rho < -thr:
        return -1, m, rho
    if m + rho < thr and m - rho > -thr:
        return 0, m, rho
    return 2, m, rho


def shortcut(x, piece, thr):
    k = x.shape[0]
    if piece == 0:
        return np.zeros_like(x)
    return x + (-thr if piece == 1 else thr) * np.eye(k)


def random_herm(rng, k, center, spread):
    a = rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k))
    h = 0.5 * (a + a.conj().T)
    h = h / np.linalg.norm(h, 2) * spread
    return h + center * np.eye(k)


@pytest.mark.parametrize("k", [3, 4])
def test_enclosure_contains_spectrum_and_shortcut_matches(k):
    rng = np.random.default_rng(1712 + k)
    thr = 0.7
    seen = {0: 0, 1: 0, -1: 0, 2: 0}
    for _ in range(4000):
        center = rng.uniform(-3.0, 3.0)
        spread = rng.choice([1e-9, 1e-3, 0.1, 0.5, 2.0]) * rng.uniform(0.0, 1.0)
        x = random_herm(rng, k, center, spread)
        lam = np.linalg.eigvalsh(x)
        piece, m, rho = enclosure_piece(x, thr)
        assert np.all(lam >= m - rho - 1e-14 * max(1.0, abs(m))) and np.all(lam <= m + rho + 1e-14 * max(1.0, abs(m)))
        seen[piece] += 1
        if piece == 2:
            continue
        ref = eig_soft(x[None], thr)[0]
        got = shortcut(x, piece, thr)
        scale = max(1.0, np.max(np.abs(x)))
        assert np.max(np.abs(got - ref)) <= 1e-13 * scale, (piece, lam)
    # every piece is exercised
    assert min(seen.values()) > 100, seen


def test_enclosure_boundary_eigenvalue_takes_eigensolve():
    # an eigenvalue exactly at the threshold is never classified by the
    # enclosure (the widened interval touches thr): the Jacobi path decides
    thr = 0.5
    x = np.diag([thr, 0.1, -0.2]).astype(np.complex128)
    assert enclosure_piece(x, thr)[0] == 2
    x = np.diag([thr + 1e-3, thr + 2e-3, thr + 5e-3]).astype(np.complex128)
    assert enclosure_piece(x, thr)[0] == 1

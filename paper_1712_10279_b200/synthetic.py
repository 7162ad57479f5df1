"""Deterministic synthetic marginals for benchmarks and parity tests.

These reproduce, bit for bit, the reference's pinned demo generators so that
the GPU box (where the reference is absent) builds the same inputs:
``rgb_disk_pair`` (S/problems.py:169-185, rasterised as in :93-118),
``matrix_blob_fixtures`` (:188-201, :121-139) and ``dirac_pair`` (:156-162).
``tests/test_oracle_golden.py`` checks the bytes against sha256 digests the
reference produced.  Functions return plain arrays (l0, l1) in the reference
layout: (n,n) scalar, (n,n,k) vector, (n,n,k,k) complex128 matrix.
"""

from __future__ import annotations

import numpy as np

DISK_CENTERS = ((0.3, 0.3), (0.7, 0.3), (0.5, 0.75))
DISK_RADIUS = 0.14
BLOB_CENTER = (0.3, 0.5)
BLOB_SHIFTED = (0.7, 0.5)
BLOB_RADIUS = 0.15


def _centres(n):
    return np.arange(n) * (1.0 / (n - 1))


def _inside(n, centre, radius):
    x = _centres(n)
    return (x[:, None] - centre[0]) ** 2 + (x[None, :] - centre[1]) ** 2 <= radius ** 2


def _unit_mass(values, trace=False):
    tot = float(np.sum(np.real(np.trace(values, axis1=2, axis2=3)))) if trace \
        else float(np.sum(values))
    return values / tot


def disks(n, placements, k, radius=DISK_RADIUS):
    """placements: iterable of (centre, channel); each disk holds unit mass."""
    v = np.zeros((n, n, k))
    for centre, ch in placements:
        m = _inside(n, centre, radius)
        v[m, ch] += 1.0 / int(m.sum())
    return _unit_mass(v)


def rgb_disk_pair(n, radius=DISK_RADIUS):
    """Three unit disks, target colours permuted R->G->B->R."""
    a = disks(n, [(c, ch) for ch, c in enumerate(DISK_CENTERS)], 3, radius)
    b = disks(n, [(c, (ch + 1) % 3) for ch, c in enumerate(DISK_CENTERS)], 3, radius)
    return a, b


def _herm(x):
    return 0.5 * (x + np.conj(np.swapaxes(x, -1, -2)))


def blobs(n, placements, radius=BLOB_RADIUS):
    """placements: iterable of (centre, shape matrix); unit-trace blobs."""
    placements = [(c, _herm(np.asarray(M, dtype=np.complex128))) for c, M in placements]
    k = placements[0][1].shape[0]
    v = np.zeros((n, n, k, k), dtype=np.complex128)
    for centre, M in placements:
        m = _inside(n, centre, radius)
        v[m] += (M / np.real(np.trace(M))) * (1.0 / int(m.sum()))
    return _herm(_unit_mass(_herm(v), trace=True))


def matrix_blob_fixtures(n):
    """(m0, m1, m2): colocated pair with different shapes, m0 translated."""
    a0 = np.diag([1.0, 0.0, 0.0])
    a1 = np.diag([0.0, 1.0, 0.0])
    return (blobs(n, [(BLOB_CENTER, a0)]), blobs(n, [(BLOB_CENTER, a1)]),
            blobs(n, [(BLOB_SHIFTED, a0)]))


def blob_pair_k2(n):
    """BASELINE C3: diag(1,0) vs [[.5,.5i],[-.5i,.5]] colocated at (0.3,0.5)."""
    return (blobs(n, [(BLOB_CENTER, np.diag([1.0, 0.0]))]),
            blobs(n, [(BLOB_CENTER, np.array([[0.5, 0.5j], [-0.5j, 0.5]]))]))


def lindblad_k2():
    """The k=2 pair {diag(1,-1), sigma_x} (T/test_acceptance.py:37-42)."""
    return np.stack([np.diag([1.0, -1.0]), np.array([[0.0, 1.0], [1.0, 0.0]])]).astype(np.complex128)


def lindblad_default3():
    """S/lindblad.py:218-222."""
    return np.stack([np.diag([1.0, 2.0, 0.0]),
                     np.array([[1.0, 1, 1], [1, 0, 0], [1, 0, 0]])]).astype(np.complex128)


def dirac_pair(n, cell0, cell1):
    a = np.zeros((n, n))
    b = np.zeros((n, n))
    a[cell0] = 1.0
    b[cell1] = 1.0
    return a, b


def rgb_disk_rows(n, r0, r1, radius=DISK_RADIUS, chunk=2048):
    """Rows [r0, r1) of rgb_disk_pair(n) without materialising the whole grid
    (for row-slab runs at 8192^2 and beyond).  Masks use the same
    floating-point predicate; the normaliser is accumulated chunk-wise, so the
    result can differ from rgb_disk_pair(n)[r0:r1] in the last bit."""
    x = _centres(n)
    counts = []
    for centre in DISK_CENTERS:
        c = 0
        for a in range(0, n, chunk):
            c += int(np.count_nonzero(
                (x[a:a + chunk, None] - centre[0]) ** 2 + (x[None, :] - centre[1]) ** 2
                <= radius ** 2))
        counts.append(c)
    total = float(sum(c * (1.0 / c) for c in counts))
    out = []
    for shift in (0, 1):
        v = np.zeros((r1 - r0, n, 3))
        for ch, centre in enumerate(DISK_CENTERS):
            m = (x[r0:r1, None] - centre[0]) ** 2 + (x[None, :] - centre[1]) ** 2 <= radius ** 2
            v[m, (ch + shift) % 3] += 1.0 / counts[ch]
        out.append(v / total)
    return out[0], out[1]

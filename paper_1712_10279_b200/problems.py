"""The reference's pinned input instances with its signatures (S/problems.py:
156-201, S/spatial.py:71-73): GridSpec in, density objects out.  They wrap the
array generators of synthetic.py (pinned by sha256 to the reference's bytes,
tests/test_host.py) so code and tests written against ``otflux`` find the
same names; the generic scene / blob builders stay out of scope."""

from __future__ import annotations

from . import synthetic
from .fields import GridSpec, MatrixDensity, ScalarDensity, VectorDensity


def _side(grid) -> int:
    return grid.n if isinstance(grid, GridSpec) else int(grid)


def lambda_max_spatial_bound(grid) -> float:
    """8 (n - 1)^2, the bound on the spectrum of -div grad used by the step sizes."""
    return 8.0 * (_side(grid) - 1) ** 2


def dirac_pair(grid, cell0, cell1):
    a, b = synthetic.dirac_pair(_side(grid), cell0, cell1)
    return ScalarDensity(a), ScalarDensity(b)


def rgb_disk_pair(grid, radius: float = synthetic.DISK_RADIUS):
    l0, l1 = synthetic.rgb_disk_pair(_side(grid), radius)
    return VectorDensity(l0), VectorDensity(l1)


def matrix_blob_fixtures(grid):
    return tuple(MatrixDensity(m) for m in synthetic.matrix_blob_fixtures(_side(grid)))

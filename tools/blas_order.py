"""Which rounding sequence does NumPy's matmul use for the reference's graph
operators (S/graph.py:105-123: ``x @ (D/c)`` and ``y @ -(D/c).T``)?

The CUDA kernels (payload.cuh VecPolicy::grad_c / div_c) reproduce it so the
vector path stays bit-identical to the reference when the channel flux is
active.  Checked model: a fused multiply-add chain from 0 over the inner index
in ascending order (OpenBLAS dgemm), descending for the (n^2, 2) @ (2, 1)
matrix-vector case (k = 2, one edge).  Exact FMA is emulated with fractions.

    python tools/blas_order.py      # prints mismatches per shape; 0 = model holds
"""
import sys
from fractions import Fraction

import numpy as np


def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def chain(x, col, order):
    acc = 0.0
    for i in order:
        acc = fma(x[i], col[i], acc)
    return acc


def incidence_over_costs(k, edges, costs):
    d = np.zeros((k, len(edges)))
    for e, (a, b) in enumerate(edges):
        d[a, e], d[b, e] = 1.0, -1.0
    return d / np.asarray(costs)


def main(samples=300):
    rng = np.random.default_rng(0)
    graphs = [(2, [(0, 1)]), (3, [(0, 1), (1, 2)]), (3, [(0, 1), (1, 2), (0, 2)]),
              (4, [(0, 1), (1, 2), (2, 3), (0, 3), (0, 2)]),
              (6, [(i, j) for i in range(6) for j in range(i + 1, 6)])]
    bad_total = 0
    for k, edges in graphs:
        ell = len(edges)
        coef = incidence_over_costs(k, edges, rng.uniform(0.5, 2.0, ell))
        for rows in (1000, 2_000_000):
            x = rng.random((rows, k))
            y = rng.random((rows, ell))
            gx = x @ coef
            dy = y @ (-coef.T)
            g_order = list(range(k))[::-1] if ell == 1 else list(range(k))
            bad_g = bad_d = 0
            for r in rng.integers(0, rows, samples):
                bad_g += sum(chain(x[r], coef[:, e], g_order) != gx[r, e] for e in range(ell))
                bad_d += sum(chain(y[r], -coef[c], range(ell)) != dy[r, c] for c in range(k))
            print(f"k={k} ell={ell} rows={rows}: grad mismatches {bad_g}, div mismatches {bad_d}")
            bad_total += bad_g + bad_d
    print("model holds" if bad_total == 0 else f"MODEL BROKEN: {bad_total} mismatches")
    return bad_total


if __name__ == "__main__":
    sys.exit(1 if main() else 0)

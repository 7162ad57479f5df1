"""Which summation order does NumPy's einsum use for the reference's block
norms (S/shrink.py:88-104: np.einsum over the contiguous payload axes)?

Model (payload.cuh np_sumsq): two lanes, multiply then add (no FMA); blocks
of 8 elements accumulate x[6+l]^2, x[4+l]^2, x[2+l]^2, x[l]^2 into lane l,
the rest two at a time, result lane0 + lane1.

    python tools/einsum_order.py     # 0 mismatches = the model holds
"""
import sys

import numpy as np


def np_sumsq(x):
    acc = [0.0, 0.0]
    i, n = 0, len(x)
    while n - i >= 8:
        for lane in (0, 1):
            t = acc[lane]
            for q in (3, 2, 1, 0):
                v = x[i + 2 * q + lane]
                t = v * v + t
            acc[lane] = t
        i += 8
    while i < n:
        for lane in (0, 1):
            if i + lane < n:
                v = x[i + lane]
                acc[lane] = v * v + acc[lane]
        i += 2
    return acc[0] + acc[1]


def main(cells=400):
    rng = np.random.default_rng(0)
    bad_total = 0
    for tail in [(2,), (3,), (5,), (6,), (2, 2), (2, 3), (2, 4), (2, 6), (2, 8), (15,), (21,),
                 (2, 3, 3), (2, 4, 4)]:
        x = rng.normal(size=(cells,) + tail)
        sub = "zabcd"[: 1 + len(tail)]
        ref = np.einsum(f"{sub},{sub}->z", x, x)
        flat = x.reshape(cells, -1)
        bad = sum(np_sumsq(list(flat[c])) != ref[c] for c in range(cells))
        print(f"payload {tail}: {bad} mismatches")
        bad_total += bad
    print("model holds" if bad_total == 0 else f"MODEL BROKEN: {bad_total}")
    return bad_total


if __name__ == "__main__":
    sys.exit(1 if main() else 0)

"""Loading the golden fixtures (tests/golden, written by tools/make_golden.py
from the reference) and replaying them through the oracle."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def index():
    return json.loads((GOLDEN / "index.json").read_text())


# generators of the BASELINE-size fixtures whose marginals are not stored
# (tools/make_golden.py marginals=False): the package's restated generators,
# checked against the sha256 of the reference's bytes on every load
_MARGINALS = {
    "B_vec256": lambda s: s.rgb_disk_pair(256),
    "B_vec256_a03": lambda s: s.rgb_disk_pair(256),
    "B_matr256": lambda s: s.matrix_blob_fixtures(256)[:2],
    "B_matc128": lambda s: s.blob_pair_k2(128),
}


def _sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    meta = index()[name]
    with np.load(GOLDEN / f"{name}.npz") as z:
        arrs = {k: z[k] for k in z.files}
    if "l0" not in arrs and name in _MARGINALS:
        from paper_1712_10279_b200 import synthetic

        l0, l1 = _MARGINALS[name](synthetic)
        assert _sha(l0) == meta["sha256"]["l0"] and _sha(l1) == meta["sha256"]["l1"], name
        arrs["l0"], arrs["l1"] = l0, l1
    return meta, arrs


def full_cases():
    return sorted(k for k, v in index().items() if v["full"])


def summary_cases():
    return sorted(k for k, v in index().items() if not v["full"])


def matrix_path(l0, l1, mats, norm_u, norm_w):
    """Real/complex path rule of S/solver.py:412-426."""
    diff = l0 - l1
    use_real = ("l1nuc" not in (norm_u, norm_w) and not np.any(diff.imag)
                and not np.any(np.asarray(mats).imag))
    if use_real:
        return np.ascontiguousarray(diff.real), np.ascontiguousarray(np.real(mats)), np.float64
    return diff, np.asarray(mats, dtype=np.complex128), np.complex128


def oracle_engine(meta, arrs, l0=None, l1=None):
    from oracle.pdhg import (OracleEngine, comm_lambda_max, graph_coef,
                             graph_lambda_max)

    cfg = meta["cfg"]
    l0 = arrs["l0"] if l0 is None else l0
    l1 = arrs["l1"] if l1 is None else l1
    n = l0.shape[0]
    kind = meta["kind"]
    tau = cfg.get("tau")
    if tau is None:
        tau = 1.0 if n <= 64 else 3.0
    common = dict(norm_u=cfg.get("norm_u", "l2"), norm_w=cfg.get("norm_w", "l1"),
                  alpha=cfg.get("alpha", 1.0), eps=cfg.get("eps_reg", 0.0))
    if kind == "scalar":
        return OracleEngine("scalar", l0 - l1, n, tau, **common)
    if kind == "vector":
        g = meta["graph"]
        coef = graph_coef(g["k"], g["edges"], g["costs"], g["orientations"])
        lam = graph_lambda_max(g["k"], g["edges"], g["costs"], g["orientations"])
        return OracleEngine("vector", l0 - l1, n, tau, chan=coef, lam_chan=lam, **common)
    mats = arrs["lindblad"]
    diff, m, dt = matrix_path(l0, l1, mats, common["norm_u"], common["norm_w"])
    lam = comm_lambda_max(mats)
    return OracleEngine("matrix", diff, n, tau, chan=m, lam_chan=lam, dtype=dt, **common)


def run_cfg(meta):
    cfg = meta["cfg"]
    return dict(tol_gap=cfg.get("tol_gap", 1e-3), tol_feas=cfg.get("tol_feas", 1e-5),
                max_iters=cfg.get("max_iters", 200_000), check_every=cfg.get("check_every", 100))

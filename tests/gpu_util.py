"""Helpers for the GPU parity tests: run a golden / oracle case through the
package's public API (the CUDA path)."""

from __future__ import annotations

import json
import os

import numpy as np

import paper_1712_10279_b200 as pk


def cfg_of(meta, **over):
    c = dict(meta["cfg"])
    c.update(over)
    return pk.SolverConfig(**c)


def lindblad_from(mats):
    return pk.LindbladSet(np.asarray(mats))


def graph_from(g):
    return pk.TransportGraph(g["k"], [tuple(e) for e in g["edges"]], g["costs"],
                             orientations=g["orientations"])


def solve_case(meta, l0, l1, lindblad=None, precision="f64", **over):
    cfg = cfg_of(meta, **over)
    kind = meta["kind"]
    if kind == "scalar":
        return pk.solve_scalar(pk.ScalarDensity(l0), pk.ScalarDensity(l1), cfg=cfg,
                               precision=precision)
    if kind == "vector":
        return pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), graph_from(meta["graph"]),
                               cfg=cfg, precision=precision)
    return pk.solve_matrix(pk.MatrixDensity(l0), pk.MatrixDensity(l1), lindblad_from(lindblad),
                           cfg=cfg, precision=precision)


def _log_err(err):
    """With OTFX_PARITY_LOG=<file>, record the worst relative error each test
    measured (the parity table in profiles/ is built from this log)."""
    path = os.environ.get("OTFX_PARITY_LOG")
    if path:
        test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
        with open(path, "a") as f:
            f.write(json.dumps({"test": test, "rel_err": err}) + "\n")


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    scale = float(np.max(np.abs(b))) if b.size else 0.0
    if scale == 0.0:
        err = float(np.max(np.abs(a))) if a.size else 0.0
    else:
        err = float(np.max(np.abs(a - b))) / scale
    _log_err(err)
    return err


def hist_array(report):
    return np.array([[h.iteration, h.primal, h.dual, h.gap_ratio, h.feas_residual, h.residual]
                     for h in report.history])


def hist_close(h, ref, rtol):
    """Compare history rows column by column relative to each column's scale."""
    assert h.shape == ref.shape, (h.shape, ref.shape)
    assert np.array_equal(h[:, 0], ref[:, 0])
    worst = 0.0
    for c in range(1, 6):
        fin = np.isfinite(ref[:, c])
        assert np.array_equal(np.isfinite(h[:, c]), fin)
        if fin.any():
            worst = max(worst, rel_err(h[fin, c], ref[fin, c]))
    assert worst <= rtol, worst
    return worst

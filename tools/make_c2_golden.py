"""BASELINE configs[1] ("vector-OMT 3-channel 256x256 to convergence") golden.

Runs the REFERENCE solver (S/solver.py:372-393, the `_run` loop of
S/solver.py:294-337) to convergence on ``rgb_disk_pair(GridSpec(256))`` with the
triangle graph, l12/l1, alpha = 1, the default tolerances (gap 1e-3, feas 1e-5)
and a pinned dual step tau.  The CLI bench value tau = 6 (S/cli.py:251-256)
does not converge within the default 200 000 iterations, so the
case is pinned at tau = default_tau(256) = 3 (S/solver.py:66-68).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tools/make_c2_golden.py 3.0

Writes tests/golden/C2_vec256_tau<tau>.npz (history, meta, final u/w/phi) and
an entry in tests/golden/c2_index.json (iterations, V, wall seconds, norms).
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

import otflux as of

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main(tau: float, max_iters: int = 400_000) -> None:
    l0, l1 = of.rgb_disk_pair(of.GridSpec(256))
    cfg = of.SolverConfig(tau=tau, norm_u="l12", norm_w="l1", alpha=1.0,
                          max_iters=max_iters, check_every=100)
    t0 = time.perf_counter()
    rep, st = of.solve_vector(l0, l1, of.triangle_graph(), cfg=cfg)
    dt = time.perf_counter() - t0
    hist = np.array([[h.iteration, h.primal, h.dual, h.gap_ratio, h.feas_residual, h.residual]
                     for h in rep.history], dtype=np.float64)
    tag = f"{tau:g}".replace(".", "p")
    name = f"C2_vec256_tau{tag}"
    np.savez_compressed(OUT / f"{name}.npz", history=hist,
                        meta=np.array([rep.iterations, int(rep.converged), rep.transport_value]),
                        ux=st.u.ux, uy=st.u.uy, w=st.w.values, phi=st.phi)
    idx_path = OUT / "c2_index.json"
    index = json.loads(idx_path.read_text()) if idx_path.exists() else {}
    index[name] = dict(
        tau=tau, norm_u="l12", norm_w="l1", alpha=1.0, tol_gap=cfg.tol_gap,
        tol_feas=cfg.tol_feas, max_iters=max_iters, check_every=100,
        iterations=rep.iterations, converged=bool(rep.converged),
        transport_value=rep.transport_value, reference_seconds=round(dt, 1),
        reference_s_per_iter=dt / max(rep.iterations, 1),
        norms=dict(ux=float(np.linalg.norm(st.u.ux)), uy=float(np.linalg.norm(st.u.uy)),
                   w=float(np.linalg.norm(st.w.values)), phi=float(np.linalg.norm(st.phi))),
        sha256={k: hashlib.sha256(np.ascontiguousarray(v.values).tobytes()).hexdigest()
                for k, v in (("l0", l0), ("l1", l1))})
    idx_path.write_text(json.dumps(index, indent=1, sort_keys=True) + "\n")
    print(name, rep.iterations, rep.converged, rep.transport_value, f"{dt:.1f}s")


if __name__ == "__main__":
    main(float(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 400_000)

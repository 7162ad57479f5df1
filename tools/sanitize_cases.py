"""Small solves through every execution path, for compute-sanitizer
(racecheck / synccheck / memcheck / initcheck):

  cluster   the on-chip cluster solve (st.async into peer DSMEM + mbarriers)
  register  the register-streamed sweep (one __syncthreads per row)
  tma       the TMA-streamed sweep (producer warp, full/empty mbarrier ring),
            fused check + speculative dual sweep and the flip-back
  heavy     the 6-consumer-warp 2-stage ring of the 3x3 complex payload
  slabs     a local 3-slab group on the overlapped schedule (edge stream +
            halo pack / transport / unpack + interior bands)
  matrix    2x2 complex l1nuc through the TMA ring

Each case checks its result against the oracle, so a run that the sanitizer
perturbs into a wrong answer also fails here.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1712_10279_b200 as pk  # noqa: E402
from oracle import pdhg  # noqa: E402
from paper_1712_10279_b200 import synthetic  # noqa: E402
from paper_1712_10279_b200.solver import build_engine, run_local  # noqa: E402


def _env(**kv):
    for k in ("OTFX_CLUSTER", "OTFX_TMA", "OTFX_OVERLAP"):
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in kv.items()})


def _vector(n, iters, ce):
    l0, l1 = synthetic.rgb_disk_pair(n)
    g = pk.triangle_graph((1.0, 1.3, 0.8))
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.05, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=iters, check_every=ce)
    rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), g, cfg=cfg)
    eng = pdhg.OracleEngine("vector", l0 - l1, n, 6.0, norm_u="l12", norm_w="l1", alpha=0.05,
                            chan=g.coefficients(), lam_chan=pk.lambda_max_graph(g))
    pdhg.oracle_run(eng, 1e-300, 1e-300, iters, ce)
    assert np.array_equal(st.phi, eng.phi), "phi differs from the oracle"
    return rep


def _matrix(n, k, norm, iters, ce):
    rng = np.random.default_rng(k)
    a = rng.normal(size=(2, n, n, k, k)) + 1j * rng.normal(size=(2, n, n, k, k))
    p = a @ np.conj(np.swapaxes(a, -1, -2))
    p /= np.sum(np.real(np.trace(p, axis1=-2, axis2=-1)), axis=(1, 2))[:, None, None, None, None]
    m = rng.normal(size=(2, k, k)) + 1j * rng.normal(size=(2, k, k))
    lind = pk.LindbladSet(0.5 * (m + np.conj(np.swapaxes(m, -1, -2))))
    cfg = pk.SolverConfig(tau=10.0, norm_u=norm, norm_w=norm, alpha=0.3, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=iters, check_every=ce)
    rep, st = pk.solve_matrix(pk.MatrixDensity(p[0]), pk.MatrixDensity(p[1]), lind, cfg=cfg)
    eng = pdhg.OracleEngine("matrix", p[0] - p[1], n, 10.0, norm_u=norm, norm_w=norm, alpha=0.3,
                            chan=lind.matrices, lam_chan=pk.lambda_max_L(lind),
                            dtype=np.complex128)
    pdhg.oracle_run(eng, 1e-300, 1e-300, iters, ce)
    err = float(np.max(np.abs(st.phi - eng.phi)) / np.max(np.abs(eng.phi)))
    assert err <= 1e-10, err
    return rep


def case_cluster():
    _env()
    _vector(48, 60, 20)


def case_register():
    _env(OTFX_CLUSTER=0, OTFX_TMA=0)
    _vector(96, 30, 10)


def case_tma():
    _env(OTFX_TMA=1)
    _vector(160, 30, 10)


def case_heavy():
    _env(OTFX_TMA=1)
    _matrix(64, 3, "l1nuc", 12, 5)


def case_matrix():
    _env(OTFX_TMA=1)
    _matrix(64, 2, "l1nuc", 12, 5)


def case_slabs():
    _env(OTFX_TMA=1, OTFX_OVERLAP=1)
    n, P = 192, 3
    l0, l1 = synthetic.rgb_disk_pair(n)
    g = pk.triangle_graph()
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.05, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=24, check_every=10)
    whole = build_engine("vector", n, cfg, graph=g)
    whole.set_marginals(l0, l1)
    whole.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
    ref = whole.get_state()
    whole.close()
    bounds = np.linspace(0, n, P + 1).astype(int)
    slabs, stream = [], None
    for r in range(P):
        e = build_engine("vector", n, cfg, graph=g, rows=(bounds[r], bounds[r + 1]), stream=stream)
        stream = e.stream
        e.set_marginals(l0[bounds[r]:bounds[r + 1]], l1[bounds[r]:bounds[r + 1]])
        slabs.append(e)
    run_local(slabs, cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
    got = [e.get_state() for e in slabs]
    for q, want in enumerate(ref):
        assert np.array_equal(np.concatenate([s[q] for s in got], axis=0), want), q
    for e in reversed(slabs):
        e.close()


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        CASES[name]()
        print(f"sanitize case {name}: ok", flush=True)

"""Full-iterate parity at the BASELINE sizes the bench quotes (configs[4] and
the north-star's 4096^2): the CUDA path through ``solve_vector`` against the
NumPy oracle (pinned bit-exactly to the reference, tests/test_oracle_golden.py)
run on the GPU box's host for a few iterations.

The vector path is bit-identical to the reference's operation order
(DESIGN.md §4), so u, w and phi must be EQUAL; the history rows differ only by
the summation order of the whole-grid reductions and are held to the
north-star's 1e-10 relative bound (BASELINE.json).  The oracle needs about
6.5 s per iteration at 4096^2 and 29 s at 8192^2 (22 GB RSS), so the
iteration counts stay small; the BASELINE C2/C3/C4 grids get full goldens
written by the reference itself (B_* fixtures, tests/test_gpu_parity.py).
"""

import numpy as np
import pytest

import gpu_util as g
import paper_1712_10279_b200 as pk
from oracle import pdhg
from paper_1712_10279_b200 import synthetic
from paper_1712_10279_b200.solver import build_engine

pytestmark = pytest.mark.gpu


def _run_both(n, iters, check_every, alpha, precision="f64"):
    l0, l1 = synthetic.rgb_disk_pair(n)
    graph = pk.triangle_graph()
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=alpha, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=iters, check_every=check_every)
    rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), graph, cfg=cfg,
                              precision=precision)
    eng = pdhg.OracleEngine("vector", l0 - l1, n, 6.0, norm_u="l12", norm_w="l1", alpha=alpha,
                            chan=graph.coefficients(), lam_chan=pk.lambda_max_graph(graph))
    del l0, l1
    _, it, hist = pdhg.oracle_run(eng, 1e-300, 1e-300, iters, check_every)
    assert rep.iterations == it == iters
    return rep, st, eng, np.array(hist)


@pytest.mark.parametrize("n,iters,check_every", [(4096, 4, 2), (8192, 2, 2)])
def test_baseline_size_iterates_equal_oracle(n, iters, check_every):
    """The bench workload through the public API from the zero state."""
    rep, st, eng, hist = _run_both(n, iters, check_every, alpha=1.0)
    g.hist_close(g.hist_array(rep), hist, 1e-10)
    assert np.array_equal(st.u.ux, eng.u[:, :, 0])
    assert np.array_equal(st.u.uy, eng.u[:, :, 1])
    assert np.array_equal(st.phi, eng.phi)
    assert np.array_equal(st.w.values, eng.w)
    # ghost entries (S/spatial.py:80-86)
    assert not np.any(st.u.ux[-1]) and not np.any(st.u.uy[:, -1])


@pytest.mark.parametrize("n,plain", [(4096, 3), (8192, 1)])
def test_baseline_size_random_state_equal_oracle(n, plain):
    """From the zero state at normalised mass the first iterations leave the
    channel flux at 0 (|grad_G phi| << alpha), so a random state of the
    magnitudes where both shrinks are partly active (|u| ~ mu-scaled, channel
    differences of phi ~ alpha) is loaded through the state API
    (S/solver.py:477-482) and stepped: `plain` iterations and one check
    iteration (R^k + evaluate), against the oracle from the same state."""
    rng = np.random.default_rng(n)
    l0, l1 = synthetic.rgb_disk_pair(n)
    graph = pk.triangle_graph((1.0, 1.3, 0.8))
    alpha = 0.3
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=alpha)
    eng = build_engine("vector", n, cfg, graph=graph)
    try:
        eng.set_marginals(l0, l1)
        mu, nu = eng.mu, eng.nu
        phi = rng.random((n, n, 3))
        u = rng.normal(scale=mu * n, size=(n, n, 2, 3))
        u[-1, :, 0] = 0.0
        u[:, -1, 1] = 0.0
        w = rng.normal(scale=nu, size=(n, n, 3))
        eng.set_state(u[:, :, 0], u[:, :, 1], w, phi)
        eng.step(plain)
        out = eng.step_check()
        ux, uy, w1, phi1 = eng.get_state()
    finally:
        eng.close()
    ora = pdhg.OracleEngine("vector", l0 - l1, n, 6.0, norm_u="l12", norm_w="l1", alpha=alpha,
                            chan=graph.coefficients(), lam_chan=pk.lambda_max_graph(graph))
    del l0, l1
    ora.u, ora.w, ora.phi = u, w, phi
    for _ in range(plain):
        ora.step()
    u0, w0, p0 = ora.u.copy(), ora.w.copy(), ora.phi.copy()
    ora.step()
    rk = ora.residual_from(u0, w0, p0)
    del u0, w0, p0
    want = ora.evaluate() + (rk,)
    assert np.array_equal(ux, ora.u[:, :, 0])
    assert np.array_equal(uy, ora.u[:, :, 1])
    assert np.array_equal(phi1, ora.phi)
    assert np.array_equal(w1, ora.w)
    act_w = np.count_nonzero(ora.w) / ora.w.size
    assert 0.05 < act_w < 0.95, act_w  # the w soft threshold cuts some entries, not all
    np.testing.assert_allclose(np.array(out), np.array(want), rtol=1e-10, atol=0)

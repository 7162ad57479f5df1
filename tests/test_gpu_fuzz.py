"""Seeded random parity sweep over the whole configuration space the engine
accepts: payload kind (scalar, k-channel vector, real-symmetric and complex
Hermitian matrix), every valid norm pairing, eps_reg, alpha, tau, grid sizes
down to 2x2, odd check cadences -- CUDA path (whichever execution path the
engine picks, plus the forced alternatives) against the NumPy oracle, which is
itself pinned bit-exact to the reference (tests/test_oracle_golden.py)."""

import numpy as np
import pytest

import gpu_util as g
import paper_1712_10279_b200 as pk
from oracle import pdhg

pytestmark = pytest.mark.gpu

VEC_NORMS = ["l2", "l12", "l1"]
MAT_NORMS = ["l2", "l12", "l1", "l1nuc"]


def _norm(rng, shape):
    v = rng.random(shape) + 0.05
    return v / v.sum()


def _psd(rng, n, k, complex_):
    a = rng.normal(size=(n, n, k, k))
    if complex_:
        a = a + 1j * rng.normal(size=(n, n, k, k))
    p = a @ np.conj(np.swapaxes(a, -1, -2))
    tr = np.sum(np.real(np.trace(p, axis1=2, axis2=3)))
    return (p / tr).astype(np.complex128)


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = ["scalar", "vector", "vector", "matrix_real", "matrix_complex"][seed % 5]
    n = int(rng.integers(2, 37))
    tau = float(rng.choice([0.7, 2.0, 6.0, 15.0]))
    alpha = float(rng.choice([0.05, 0.3, 1.0]))
    iters = int(rng.integers(25, 61))
    ce = int(rng.choice([7, 10, 25]))
    if kind in ("scalar", "vector"):
        nu, nw = str(rng.choice(VEC_NORMS)), str(rng.choice(["l2", "l1"]))
    elif kind == "matrix_real":  # l12 groups spatial fluxes only (S/shrink.py:70-76)
        nu, nw = str(rng.choice(MAT_NORMS[:3])), str(rng.choice(["l2", "l1"]))
    else:
        nu, nw = str(rng.choice(MAT_NORMS)), str(rng.choice(["l2", "l1", "l1nuc"]))
    nuclear = "l1nuc" in (nu, nw)
    eps = 0.0 if nuclear or rng.random() < 0.6 else float(rng.choice([1e-3, 0.02]))
    return rng, kind, n, tau, alpha, iters, ce, nu, nw, eps


def _run_case(seed):
    rng, kind, n, tau, alpha, iters, ce, nu, nw, eps = _case(seed)
    cfg = pk.SolverConfig(tau=tau, norm_u=nu, norm_w=nw, alpha=alpha, eps_reg=eps,
                          tol_gap=1e-300, tol_feas=1e-300, max_iters=iters, check_every=ce)
    if kind == "scalar":
        l0, l1 = _norm(rng, (n, n)), _norm(rng, (n, n))
        rep, st = pk.solve_scalar(pk.ScalarDensity(l0), pk.ScalarDensity(l1), cfg=cfg)
        eng = pdhg.OracleEngine("scalar", l0 - l1, n, tau, norm_u=nu, norm_w=nw, alpha=alpha,
                                eps=eps)
        tol = 1e-10
    elif kind == "vector":
        k = int(rng.integers(2, 5))
        edges = [(a, b) for a in range(k) for b in range(a + 1, k)]
        costs = [float(c) for c in rng.uniform(0.5, 2.0, len(edges))]
        graph = pk.TransportGraph(k, edges, costs)
        l0, l1 = _norm(rng, (n, n, k)), _norm(rng, (n, n, k))
        rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), graph, cfg=cfg)
        eng = pdhg.OracleEngine("vector", l0 - l1, n, tau, norm_u=nu, norm_w=nw, alpha=alpha,
                                eps=eps, chan=graph.coefficients(),
                                lam_chan=pk.lambda_max_graph(graph))
        tol = 1e-10
    else:
        cplx = kind == "matrix_complex"
        k = int(rng.integers(2, 4))
        l0, l1 = _psd(rng, n, k, cplx), _psd(rng, n, k, cplx)
        mats = rng.normal(size=(2, k, k))
        if cplx:
            mats = mats + 1j * rng.normal(size=(2, k, k))
        lind = pk.LindbladSet(0.5 * (mats + np.conj(np.swapaxes(mats, -1, -2))))
        rep, st = pk.solve_matrix(pk.MatrixDensity(l0), pk.MatrixDensity(l1), lind, cfg=cfg)
        real_path = st.phi.dtype == np.float64
        assert real_path == (not cplx and not ("l1nuc" in (nu, nw)))
        dt = np.float64 if real_path else np.complex128
        diff = (l0 - l1).real if real_path else (l0 - l1)
        chan = lind.matrices.real if real_path else lind.matrices
        eng = pdhg.OracleEngine("matrix", diff.astype(dt), n, tau, norm_u=nu, norm_w=nw,
                                alpha=alpha, eps=eps, chan=chan, lam_chan=pk.lambda_max_L(lind),
                                dtype=dt)
        tol = 1e-10
    _, _, hist = pdhg.oracle_run(eng, 1e-300, 1e-300, iters, ce)
    assert rep.iterations == iters
    g.hist_close(g.hist_array(rep), np.array(hist), tol)
    assert g.rel_err(st.phi, eng.phi) <= tol
    assert g.rel_err(st.u.ux, eng.u[:, :, 0]) <= tol
    if st.w is not None:
        assert g.rel_err(st.w.values, eng.w) <= tol
    if kind in ("scalar", "vector"):
        # same rounding sequence as the reference: equal bits
        assert np.array_equal(st.phi, eng.phi)
        assert np.array_equal(st.u.ux, eng.u[:, :, 0]) and np.array_equal(st.u.uy, eng.u[:, :, 1])
        if st.w is not None:
            assert np.array_equal(st.w.values, eng.w)


@pytest.mark.parametrize("path", ["default", "register", "tma"])
@pytest.mark.parametrize("seed", range(30))
def test_random_configuration_vs_oracle(monkeypatch, seed, path):
    if path == "register":
        monkeypatch.setenv("OTFX_CLUSTER", "0")
        monkeypatch.setenv("OTFX_TMA", "0")
    elif path == "tma":
        monkeypatch.setenv("OTFX_TMA", "1")
    _run_case(seed)

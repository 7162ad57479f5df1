"""Channel and Lindblad counts beyond the common cases: the reference's
TransportGraph (S/graph.py:23-70) takes any connected graph on k nodes and its
LindbladSet (S/lindblad.py:47-66) any ell Hermitian k x k matrices with a
nondegenerate gradient.  The engine instantiates vector payloads for
k = 2..8 (compiled, state in registers) and runs k = 9..32 (up to 128 edges)
on the runtime-size payload (csrc/dyn.cuh); matrix payloads are compiled for
k = 2..4 with ell <= 4, and k = 2, 3 with ell <= 8 (the eight Gell-Mann
matrices of su(3)), and run on the runtime-size matrix payload beyond that
(k <= 8, ell * block reals <= 256: su(4)'s 15 generators at k = 4).  Each is checked here against the oracle through every
execution path, and what lies outside is rejected with UnsupportedNormError
before any device work."""

import numpy as np
import pytest

import gpu_util as g
import paper_1712_10279_b200 as pk
from oracle import pdhg

pytestmark = pytest.mark.gpu

PATHS = {"default": {}, "register": {"OTFX_CLUSTER": "0", "OTFX_TMA": "0"},
         "tma": {"OTFX_TMA": "1"}}


def _norm(rng, shape):
    v = rng.random(shape) + 0.05
    return v / v.sum()


def gell_mann():
    """The eight Gell-Mann matrices (a basis of su(3))."""
    m = np.zeros((8, 3, 3), dtype=np.complex128)
    pairs = [(0, 1), (0, 2), (1, 2)]
    s = 0
    for a, b in pairs:
        m[s, a, b] = m[s, b, a] = 1.0
        s += 1
        m[s, a, b], m[s, b, a] = -1j, 1j
        s += 1
    m[6] = np.diag([1.0, -1.0, 0.0])
    m[7] = np.diag([1.0, 1.0, -2.0]) / np.sqrt(3.0)
    return m


def _psd(rng, n, k, complex_):
    a = rng.normal(size=(n, n, k, k))
    if complex_:
        a = a + 1j * rng.normal(size=(n, n, k, k))
    p = a @ np.conj(np.swapaxes(a, -1, -2))
    return (p / np.sum(np.real(np.trace(p, axis1=2, axis2=3)))).astype(np.complex128)


def _check(rep, st, eng, iters, ce, bit_exact):
    _, _, hist = pdhg.oracle_run(eng, 1e-300, 1e-300, iters, ce)
    assert rep.iterations == iters
    g.hist_close(g.hist_array(rep), np.array(hist), 1e-10)
    assert g.rel_err(st.phi, eng.phi) <= 1e-10
    assert g.rel_err(st.u.ux, eng.u[:, :, 0]) <= 1e-10
    assert g.rel_err(st.u.uy, eng.u[:, :, 1]) <= 1e-10
    assert g.rel_err(st.w.values, eng.w) <= 1e-10
    if bit_exact:
        assert np.array_equal(st.phi, eng.phi) and np.array_equal(st.w.values, eng.w)


@pytest.mark.parametrize("path", sorted(PATHS))
@pytest.mark.parametrize("k,graph_kind", [(7, "chain"), (7, "complete"), (8, "star"), (5, "chain")])
def test_vector_channel_counts(monkeypatch, path, k, graph_kind):
    for key, val in PATHS[path].items():
        monkeypatch.setenv(key, val)
    rng = np.random.default_rng(k * 10 + len(graph_kind))
    if graph_kind == "chain":
        edges = [(c, c + 1) for c in range(k - 1)]
    elif graph_kind == "star":
        edges = [(0, c) for c in range(1, k)]
    else:
        edges = [(a, b) for a in range(k) for b in range(a + 1, k)]
    graph = pk.TransportGraph(k, edges, rng.uniform(0.5, 2.0, len(edges)))
    n, iters, ce, tau, alpha = 40, 60, 20, 3.0, 0.05
    l0, l1 = _norm(rng, (n, n, k)), _norm(rng, (n, n, k))
    cfg = pk.SolverConfig(tau=tau, norm_u="l12", norm_w="l1", alpha=alpha, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=iters, check_every=ce)
    rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), graph, cfg=cfg)
    eng = pdhg.OracleEngine("vector", l0 - l1, n, tau, norm_u="l12", norm_w="l1", alpha=alpha,
                            chan=graph.coefficients(), lam_chan=pk.lambda_max_graph(graph))
    _check(rep, st, eng, iters, ce, bit_exact=False)
    if graph_kind != "star":
        assert np.count_nonzero(st.w.values) > 0  # the channel flux is active


@pytest.mark.parametrize("path", sorted(PATHS))
@pytest.mark.parametrize("case", ["gellmann_l2l1", "gellmann_nuc", "k2_ell6_real", "k3_ell5_real"])
def test_matrix_lindblad_counts(monkeypatch, path, case):
    for key, val in PATHS[path].items():
        monkeypatch.setenv(key, val)
    rng = np.random.default_rng(len(case))
    n, iters, ce, tau, alpha = 24, 40, 20, 10.0, 0.3
    if case.startswith("gellmann"):
        k, mats, cplx = 3, gell_mann(), True
        nu, nw = ("l1nuc", "l1nuc") if case.endswith("nuc") else ("l2", "l1")
    else:
        k = 2 if case.startswith("k2") else 3
        ell = 6 if k == 2 else 5
        a = rng.normal(size=(ell, k, k))
        mats, cplx = 0.5 * (a + np.swapaxes(a, -1, -2)), False
        nu, nw = "l2", "l1"
    lind = pk.LindbladSet(mats)
    assert lind.ell > 4
    l0, l1 = _psd(rng, n, k, cplx), _psd(rng, n, k, cplx)
    cfg = pk.SolverConfig(tau=tau, norm_u=nu, norm_w=nw, alpha=alpha, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=iters, check_every=ce)
    rep, st = pk.solve_matrix(pk.MatrixDensity(l0), pk.MatrixDensity(l1), lind, cfg=cfg)
    real_path = st.phi.dtype == np.float64
    assert real_path == (not cplx)
    dt = np.float64 if real_path else np.complex128
    diff = (l0 - l1).real if real_path else (l0 - l1)
    chan = lind.matrices.real if real_path else lind.matrices
    eng = pdhg.OracleEngine("matrix", diff.astype(dt), n, tau, norm_u=nu, norm_w=nw, alpha=alpha,
                            chan=chan, lam_chan=pk.lambda_max_L(lind), dtype=dt)
    assert st.w.values.dtype == dt  # real path: float64 w, as the reference
    _check(rep, st, eng, iters, ce, bit_exact=False)


@pytest.mark.parametrize("path", ["default", "tma"])
@pytest.mark.parametrize("k,graph_kind,norms,eps", [
    (9, "chain", ("l12", "l1"), 0.0), (12, "complete", ("l2", "l2"), 0.0),
    (16, "complete", ("l12", "l1"), 0.0), (10, "star", ("l1", "l1"), 0.01),
    (24, "chain", ("l2", "l1"), 0.0),
])
def test_vector_runtime_width(monkeypatch, path, k, graph_kind, norms, eps):
    """Graphs wider than the compiled policies (k > 8) run on the runtime-size
    payload (csrc/dyn.cuh): same operation order as the compiled vector path,
    so the iterates EQUAL the oracle's (which is pinned to the reference)."""
    for key, val in PATHS[path].items():
        monkeypatch.setenv(key, val)
    rng = np.random.default_rng(k * 7 + len(graph_kind))
    if graph_kind == "chain":
        edges = [(c, c + 1) for c in range(k - 1)]
    elif graph_kind == "star":
        edges = [(0, c) for c in range(1, k)]
    else:
        edges = [(a, b) for a in range(k) for b in range(a + 1, k)]
    graph = pk.TransportGraph(k, edges, rng.uniform(0.5, 2.0, len(edges)))
    n, iters, ce, tau, alpha = 36, 50, 25, 3.0, 0.05
    l0, l1 = _norm(rng, (n, n, k)), _norm(rng, (n, n, k))
    cfg = pk.SolverConfig(tau=tau, norm_u=norms[0], norm_w=norms[1], alpha=alpha, eps_reg=eps,
                          tol_gap=1e-300, tol_feas=1e-300, max_iters=iters, check_every=ce)
    rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), graph, cfg=cfg)
    eng = pdhg.OracleEngine("vector", l0 - l1, n, tau, norm_u=norms[0], norm_w=norms[1],
                            alpha=alpha, eps=eps, chan=graph.coefficients(),
                            lam_chan=pk.lambda_max_graph(graph))
    _check(rep, st, eng, iters, ce, bit_exact=True)
    if k == 9:
        assert np.count_nonzero(st.w.values) > 0  # the channel flux is active


@pytest.mark.parametrize("path", ["default", "tma"])
@pytest.mark.parametrize("k,ell,cplx,norms", [
    (4, 6, True, ("l1nuc", "l1nuc")), (4, 15, True, ("l2", "l1")), (5, 3, False, ("l2", "l1")),
    (5, 2, True, ("l1nuc", "l1nuc")), (6, 3, True, ("l1", "l2")), (2, 10, False, ("l12", "l1")),
])
def test_matrix_runtime_size(monkeypatch, path, k, ell, cplx, norms):
    """Matrix payloads beyond the compiled (k, ell) instantiations run on the
    runtime-size payload (csrc/dyn.cuh DynMat): packed layouts, commutators
    and the Jacobi eigen-shrink of the compiled policies with runtime k;
    held to the north star's 1e-10 against the oracle (which runs LAPACK)."""
    for key, val in PATHS[path].items():
        monkeypatch.setenv(key, val)
    rng = np.random.default_rng(k * 100 + ell)
    n, iters, ce, tau, alpha = 16, 30, 15, 10.0, 0.3
    a = rng.normal(size=(ell, k, k))
    if cplx:
        a = a + 1j * rng.normal(size=(ell, k, k))
        mats = 0.5 * (a + np.conj(np.swapaxes(a, -1, -2)))
    else:
        mats = 0.5 * (a + np.swapaxes(a, -1, -2))
    lind = pk.LindbladSet(mats.astype(np.complex128))
    l0, l1 = _psd(rng, n, k, cplx), _psd(rng, n, k, cplx)
    cfg = pk.SolverConfig(tau=tau, norm_u=norms[0], norm_w=norms[1], alpha=alpha,
                          tol_gap=1e-300, tol_feas=1e-300, max_iters=iters, check_every=ce)
    rep, st = pk.solve_matrix(pk.MatrixDensity(l0), pk.MatrixDensity(l1), lind, cfg=cfg)
    real_path = st.phi.dtype == np.float64
    assert real_path == (not cplx)
    dt = np.float64 if real_path else np.complex128
    diff = (l0 - l1).real if real_path else (l0 - l1)
    chan = lind.matrices.real if real_path else lind.matrices
    eng = pdhg.OracleEngine("matrix", diff.astype(dt), n, tau, norm_u=norms[0], norm_w=norms[1],
                            alpha=alpha, chan=chan, lam_chan=pk.lambda_max_L(lind), dtype=dt)
    _check(rep, st, eng, iters, ce, bit_exact=False)
    assert np.count_nonzero(st.w.values) > 0


@pytest.mark.parametrize("kind", ["vector", "matrix"])
def test_runtime_size_fp32(kind):
    """The fp32 build of the runtime-size payloads: objective within 1e-4 of
    the fp64 oracle at every check (the north star's fp32 bound)."""
    rng = np.random.default_rng(11)
    n, iters, ce = 24, 60, 20
    if kind == "vector":
        k = 12
        graph = pk.TransportGraph(k, [(c, c + 1) for c in range(k - 1)], rng.uniform(0.5, 2.0, k - 1))
        l0, l1 = _norm(rng, (n, n, k)), _norm(rng, (n, n, k))
        cfg = pk.SolverConfig(tau=3.0, norm_u="l12", norm_w="l1", alpha=0.05, tol_gap=1e-300,
                              tol_feas=1e-300, max_iters=iters, check_every=ce)
        rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), graph, cfg=cfg,
                                  precision="f32")
        eng = pdhg.OracleEngine("vector", l0 - l1, n, 3.0, norm_u="l12", norm_w="l1", alpha=0.05,
                                chan=graph.coefficients(), lam_chan=pk.lambda_max_graph(graph))
    else:
        k, ell = 5, 3
        a = rng.normal(size=(ell, k, k)) + 1j * rng.normal(size=(ell, k, k))
        lind = pk.LindbladSet(0.5 * (a + np.conj(np.swapaxes(a, -1, -2))))
        l0, l1 = _psd(rng, n, k, True), _psd(rng, n, k, True)
        cfg = pk.SolverConfig(tau=10.0, norm_u="l1nuc", norm_w="l1nuc", alpha=0.3,
                              tol_gap=1e-300, tol_feas=1e-300, max_iters=iters, check_every=ce)
        rep, st = pk.solve_matrix(pk.MatrixDensity(l0), pk.MatrixDensity(l1), lind, cfg=cfg,
                                  precision="f32")
        eng = pdhg.OracleEngine("matrix", l0 - l1, n, 10.0, norm_u="l1nuc", norm_w="l1nuc",
                                alpha=0.3, chan=lind.matrices, lam_chan=pk.lambda_max_L(lind),
                                dtype=np.complex128)
    _, _, hist = pdhg.oracle_run(eng, 1e-300, 1e-300, iters, ce)
    assert rep.iterations == iters
    assert g.rel_err(g.hist_array(rep)[:, 1], np.array(hist)[:, 1]) <= 1e-4


def test_runtime_width_slabs_match_one_engine():
    """The runtime-size payload under the multi-slab run loop (overlapped
    halo exchange, NCCL loopback transport): the slabs' state equals one
    engine's."""
    from paper_1712_10279_b200 import distributed as D
    from paper_1712_10279_b200.solver import build_engine, run_local

    rng = np.random.default_rng(5)
    k, n = 11, 96
    graph = pk.TransportGraph(k, [(c, c + 1) for c in range(k - 1)] + [(0, k - 1)],
                              rng.uniform(0.5, 2.0, k))
    l0, l1 = _norm(rng, (n, n, k)), _norm(rng, (n, n, k))
    cfg = pk.SolverConfig(tau=3.0, norm_u="l12", norm_w="l1", alpha=0.05, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=60, check_every=20)
    whole = build_engine("vector", n, cfg, graph=graph)
    whole.set_marginals(l0, l1)
    hist1, it1, _, _ = whole.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
    ref = whole.get_state()
    whole.close()
    loop = D.SlabCommunicator(pk.solver.nccl_unique_id(), 1, 0, 0)
    bounds, slabs, stream = [0, 40, n], [], None
    for r in range(2):
        e = build_engine("vector", n, cfg, graph=graph, rows=(bounds[r], bounds[r + 1]),
                         stream=stream)
        stream = e.stream
        e.set_marginals(l0[bounds[r]:bounds[r + 1]], l1[bounds[r]:bounds[r + 1]])
        slabs.append(e)
    hist2, it2, _ = run_local(slabs, cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every,
                              loopback=loop)
    assert it1 == it2
    g.hist_close(g.hist_array(pk.SolveReport(False, it1, 0.0, hist1)),
                 g.hist_array(pk.SolveReport(False, it2, 0.0, hist2)), 1e-12)
    got = [e.get_state() for e in slabs]
    for q, want in enumerate(ref):
        assert np.array_equal(np.concatenate([s[q] for s in got], axis=0), want), q
    for e in reversed(slabs):
        e.close()
    loop.close()


def test_outside_the_instantiations_is_rejected():
    rng = np.random.default_rng(0)
    # a 9x9 matrix payload is beyond the runtime-size matrix capacity (8)
    k9 = 9
    lind = pk.LindbladSet(np.stack([np.diag(np.arange(k9, dtype=float)),
                                    np.eye(k9, k=1) + np.eye(k9, k=-1)]).astype(np.complex128))
    m0, m1 = _psd(rng, 6, k9, False), _psd(rng, 6, k9, False)
    with pytest.raises(pk.UnsupportedNormError):
        pk.solve_matrix(pk.MatrixDensity(m0), pk.MatrixDensity(m1), lind,
                        cfg=pk.SolverConfig(max_iters=10))
    n = 8
    k = 33  # beyond the runtime-size payload's 32 channels
    graph = pk.TransportGraph(k, [(c, c + 1) for c in range(k - 1)], np.ones(k - 1))
    l0, l1 = _norm(rng, (n, n, k)), _norm(rng, (n, n, k))
    with pytest.raises(pk.UnsupportedNormError):
        pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), graph,
                        cfg=pk.SolverConfig(max_iters=10))

"""GPU behaviour tests mirroring the reference suite (T/test_solver.py) plus
oracle parity on seeded random inputs, determinism, slab decomposition and the
standalone metric helpers."""

import numpy as np
import pytest

import gpu_util as g
import paper_1712_10279_b200 as pk
from oracle import pdhg
from paper_1712_10279_b200 import synthetic
from paper_1712_10279_b200.solver import CudaEngine, build_engine, exchange_local

pytestmark = pytest.mark.gpu


def _norm_rand(rng, shape):
    v = rng.random(shape)
    return v / v.sum()


def _rand_herm_psd(rng, n, k):
    a = rng.normal(size=(n, n, k, k)) + 1j * rng.normal(size=(n, n, k, k))
    p = a @ np.conj(np.swapaxes(a, -1, -2))
    tr = np.sum(np.real(np.trace(p, axis1=2, axis2=3)))
    return pk.MatrixDensity(p / tr)


def _oracle_vector(l0, l1, graph, cfg, iters, check_every):
    n = l0.shape[0]
    tau = cfg.tau if cfg.tau is not None else pk.default_tau(n)
    eng = pdhg.OracleEngine("vector", l0 - l1, n, tau, norm_u=cfg.norm_u.value,
                            norm_w=cfg.norm_w.value, alpha=cfg.alpha, eps=cfg.eps_reg,
                            chan=graph.coefficients(), lam_chan=pk.lambda_max_graph(graph))
    conv, it, hist = pdhg.oracle_run(eng, 1e-300, 1e-300, iters, check_every)
    return eng, np.array(hist)


# ---------------------------------------------------------------------------
# oracle parity on random inputs, every vector norm pairing, odd sizes
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,k,norm_u,norm_w,alpha,eps", [
    (33, 3, "l12", "l1", 0.02, 0.0),
    (47, 3, "l2", "l2", 0.02, 0.0),
    (65, 3, "l1", "l1", 0.02, 0.0),
    (129, 3, "l12", "l1", 0.02, 0.01),
    (40, 4, "l2", "l1", 0.02, 0.0),
    (37, 2, "l1", "l2", 0.05, 0.0),
    (300, 3, "l12", "l1", 0.002, 0.0),
])
def test_vector_random_vs_oracle(rng, n, k, norm_u, norm_w, alpha, eps):
    l0 = _norm_rand(rng, (n, n, k))
    l1 = _norm_rand(rng, (n, n, k))
    if k == 3:
        graph = pk.triangle_graph((1.0, 1.3, 0.8))
    else:
        edges = [(i, i + 1) for i in range(k - 1)] + ([(0, k - 1)] if k > 2 else [])
        graph = pk.TransportGraph(k, edges, np.linspace(0.7, 1.4, len(edges)))
    cfg = pk.SolverConfig(tau=2.0, norm_u=norm_u, norm_w=norm_w, alpha=alpha, eps_reg=eps,
                          tol_gap=1e-300, tol_feas=1e-300, max_iters=150, check_every=50)
    rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), graph, cfg=cfg)
    eng, hist = _oracle_vector(l0, l1, graph, cfg, 150, 50)
    g.hist_close(g.hist_array(rep), hist, 1e-10)
    assert g.rel_err(st.u.ux, eng.u[:, :, 0]) <= 1e-10
    assert g.rel_err(st.u.uy, eng.u[:, :, 1]) <= 1e-10
    assert g.rel_err(st.phi, eng.phi) <= 1e-10
    assert g.rel_err(st.w.values, eng.w) <= 1e-10
    assert np.linalg.norm(eng.w) > 0


def test_large_grid_few_iterations_vs_oracle():
    """A 2048^2 rgb instance (the BASELINE C5 family) for 3 iterations."""
    l0, l1 = synthetic.rgb_disk_pair(2048)
    graph = pk.triangle_graph()
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.3, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=3, check_every=3)
    rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), graph, cfg=cfg)
    eng, hist = _oracle_vector(l0, l1, graph, cfg, 3, 3)
    g.hist_close(g.hist_array(rep), hist, 1e-10)
    assert g.rel_err(st.phi, eng.phi) <= 1e-10
    assert g.rel_err(st.u.ux, eng.u[:, :, 0]) <= 1e-10


@pytest.mark.parametrize("k,norm_u,norm_w", [(2, "l1nuc", "l1"), (3, "l1nuc", "l1nuc"),
                                             (3, "l2", "l1"), (2, "l12", "l2"), (4, "l1nuc", "l1nuc"),
                                             (4, "l2", "l1")])
def test_matrix_complex_random_vs_oracle(rng, k, norm_u, norm_w):
    n = 12
    a = _rand_herm_psd(rng, n, k)
    b = _rand_herm_psd(rng, n, k)
    mats = rng.normal(size=(2, k, k)) + 1j * rng.normal(size=(2, k, k))
    lind = pk.LindbladSet(0.5 * (mats + np.conj(np.swapaxes(mats, -1, -2))))
    cfg = pk.SolverConfig(tau=5.0, norm_u=norm_u, norm_w=norm_w, alpha=0.4, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=120, check_every=40)
    rep, st = pk.solve_matrix(a, b, lind, cfg=cfg)
    eng = pdhg.OracleEngine("matrix", a.values - b.values, n, 5.0, norm_u=norm_u, norm_w=norm_w,
                            alpha=0.4, chan=lind.matrices, lam_chan=pk.lambda_max_L(lind),
                            dtype=np.complex128)
    _, _, hist = pdhg.oracle_run(eng, 1e-300, 1e-300, 120, 40)
    g.hist_close(g.hist_array(rep), np.array(hist), 1e-10)
    assert g.rel_err(st.phi, eng.phi) <= 1e-10
    assert g.rel_err(st.w.values, eng.w) <= 1e-10
    assert np.linalg.norm(eng.w) > 0


# ---------------------------------------------------------------------------
# reference behaviour (T/test_solver.py)
# ---------------------------------------------------------------------------
def test_identical_marginals_immediate(rng):
    d = pk.normalize(pk.ScalarDensity(rng.random((8, 8))))
    rep, _ = pk.solve_scalar(d, d)
    assert rep.converged and rep.iterations == 0
    assert rep.transport_value == pytest.approx(0.0, abs=1e-12)
    v = pk.normalize(pk.VectorDensity(rng.random((6, 6, 3))))
    rep, _ = pk.solve_vector(v, v, pk.triangle_graph())
    assert rep.converged and rep.iterations == 0
    m0, _, _ = synthetic.matrix_blob_fixtures(5)
    rep, _ = pk.solve_matrix(pk.MatrixDensity(m0), pk.MatrixDensity(m0), pk.default_lindblad3())
    assert rep.converged and rep.transport_value == pytest.approx(0.0, abs=1e-12)


def test_mass_mismatch_rejected(rng):
    a = pk.normalize(pk.ScalarDensity(rng.random((6, 6))))
    b = pk.ScalarDensity(a.values * 1.5)
    with pytest.raises(pk.ValidationError):
        pk.solve_scalar(a, b)


def test_ghost_stays_zero(rng):
    a = pk.normalize(pk.ScalarDensity(rng.random((7, 7))))
    b = pk.normalize(pk.ScalarDensity(rng.random((7, 7))))
    _, st = pk.solve_scalar(a, b, cfg=pk.SolverConfig(max_iters=500))
    assert np.all(st.u.ux[-1, :] == 0) and np.all(st.u.uy[:, -1] == 0)
    l0, l1 = synthetic.rgb_disk_pair(130)
    _, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), pk.triangle_graph(),
                            cfg=pk.SolverConfig(max_iters=300, alpha=0.3))
    assert np.all(st.u.ux[-1] == 0) and np.all(st.u.uy[:, -1] == 0)


def test_deterministic_bitwise(rng):
    a = pk.normalize(pk.VectorDensity(rng.random((70, 70, 3))))
    b = pk.normalize(pk.VectorDensity(rng.random((70, 70, 3))))
    cfg = pk.SolverConfig(tau=3.0, max_iters=400, alpha=0.3)
    r1, s1 = pk.solve_vector(a, b, pk.triangle_graph(), cfg=cfg)
    r2, s2 = pk.solve_vector(a, b, pk.triangle_graph(), cfg=cfg)
    assert r1.transport_value == r2.transport_value and r1.iterations == r2.iterations
    assert np.array_equal(s1.phi, s2.phi) and np.array_equal(s1.u.ux, s2.u.ux)
    assert np.array_equal(s1.w.values, s2.w.values)


def test_nonconvergence_reported(rng):
    a = pk.normalize(pk.ScalarDensity(rng.random((8, 8))))
    b = pk.normalize(pk.ScalarDensity(rng.random((8, 8))))
    rep, _ = pk.solve_scalar(a, b, cfg=pk.SolverConfig(max_iters=5))
    assert not rep.converged and rep.iterations == 5


def test_matrix_structure_exact():
    m0, m1, _ = synthetic.matrix_blob_fixtures(8)
    cfg = pk.SolverConfig(tau=10.0, norm_u="l2", norm_w="l1")
    rep, st = pk.solve_matrix(pk.MatrixDensity(m0), pk.MatrixDensity(m1), pk.default_lindblad3(),
                              cfg=cfg)
    assert rep.converged
    phi = st.phi
    assert np.array_equal(phi, np.conj(np.swapaxes(phi, -1, -2)))
    wv = st.w.values
    assert np.array_equal(wv, -np.conj(np.swapaxes(wv, -1, -2)))
    ux = st.u.ux
    assert np.array_equal(ux, np.conj(np.swapaxes(ux, -1, -2)))
    res = [h.residual for h in rep.history if np.isfinite(h.residual)]
    assert all(r >= -1e-9 * max(res[0], 1.0) for r in res)
    for x, y in zip(res, res[1:]):
        assert y <= x * (1 + 1e-9) + 1e-15


def test_channel_swap_costs_alpha():
    v0 = np.zeros((4, 4, 3))
    v0[1, 1, 0] = 1.0
    v1 = np.zeros((4, 4, 3))
    v1[1, 1, 1] = 1.0
    cfg = pk.SolverConfig(norm_u="l1", norm_w="l1")
    rep, _ = pk.solve_vector(pk.VectorDensity(v0), pk.VectorDensity(v1), pk.triangle_graph(), cfg=cfg)
    assert rep.converged and rep.transport_value == pytest.approx(1.0, rel=0.02)


def test_regularized_nuclear_rejected():
    m0, m1, _ = synthetic.matrix_blob_fixtures(5)
    cfg = pk.SolverConfig(eps_reg=0.1, norm_u="l1nuc", norm_w="l1")
    with pytest.raises(pk.UnsupportedNormError):
        pk.solve_matrix(pk.MatrixDensity(m0), pk.MatrixDensity(m1), pk.default_lindblad3(), cfg=cfg)


# ---------------------------------------------------------------------------
# metric helpers on the device vs the oracle
# ---------------------------------------------------------------------------
def test_duality_gap_and_residual_vs_oracle(rng):
    n = 20
    a = pk.normalize(pk.VectorDensity(rng.random((n, n, 3))))
    b = pk.normalize(pk.VectorDensity(rng.random((n, n, 3))))
    gph = pk.triangle_graph()
    states = []
    for iters in (40, 41):
        _, st = pk.solve_vector(a, b, gph, cfg=pk.SolverConfig(max_iters=iters, check_every=1000,
                                                                alpha=0.3))
        states.append(st)
    mu, nu, tau = pk.step_sizes_vector(pk.GridSpec(n), gph, 1.0)
    r = pk.residual_Rk(states[0], states[1], mu, nu, tau, graph=gph)
    eng = pdhg.OracleEngine("vector", a.values - b.values, n, 1.0, norm_w="l1", alpha=0.3,
                            chan=gph.coefficients(), lam_chan=pk.lambda_max_graph(gph))
    eng.u = np.stack([states[1].u.ux, states[1].u.uy], axis=2)
    eng.w = states[1].w.values
    eng.phi = states[1].phi
    ref = eng.residual_from(np.stack([states[0].u.ux, states[0].u.uy], axis=2),
                            states[0].w.values, states[0].phi)
    assert r == pytest.approx(ref, rel=1e-10, abs=1e-18)
    assert r >= 0
    cfg = pk.SolverConfig(alpha=0.3)
    got = pk.duality_gap(states[1], a, b, cfg, graph=gph)
    want = eng.evaluate()
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-15)
    zero = pk.SolverState(u=states[1].u, w=states[1].w, phi=np.zeros_like(states[1].phi),
                          iteration=0, residual=0.0, primal_value=0.0, dual_value=0.0,
                          gap_ratio=0.0, feas_residual=0.0)
    p, d, gap, f = pk.duality_gap(zero, a, b, cfg, graph=gph)
    assert d == 0.0 and gap == pytest.approx(1.0)


# ---------------------------------------------------------------------------
# row-slab decomposition on one GPU: P engines stepped in lockstep with halo
# copies must reproduce the single-slab iterates bit for bit
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("P,n", [(2, 64), (3, 101), (4, 256)])
def test_local_slabs_bit_identical(P, n):
    l0, l1 = synthetic.rgb_disk_pair(n)
    gph = pk.triangle_graph()
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.3)
    whole = build_engine("vector", n, cfg, graph=gph)
    whole.set_marginals(l0, l1)
    whole.step(57)
    ref = whole.step_check()
    ux, uy, w, phi = whole.get_state()
    whole.close()
    bounds = np.linspace(0, n, P + 1).astype(int)
    slabs = []
    stream = None
    for r in range(P):
        e = build_engine("vector", n, cfg, graph=gph, rows=(bounds[r], bounds[r + 1]), stream=stream)
        stream = e.stream
        e.set_marginals(l0[bounds[r]:bounds[r + 1]], l1[bounds[r]:bounds[r + 1]])
        slabs.append(e)
    dn = float(np.sqrt(sum(e.diff_norm ** 2 for e in slabs)))
    for e in slabs:
        e.diff_norm = dn
    for it in range(58):
        for e in slabs:
            e.sweep(check=(it == 57))
        exchange_local(slabs)
    raws = [e.raw(with_residual=True) for e in slabs]
    tot = np.sum([r[:12] for r in raws], axis=0)
    mx = np.max([r[12:] for r in raws], axis=0)
    out = slabs[0].finalize(np.concatenate([tot, mx]))
    got = [e.get_state() for e in slabs]
    for q, ref_arr in enumerate((ux, uy, w, phi)):
        cat = np.concatenate([s[q] for s in got], axis=0)
        assert np.array_equal(cat, ref_arr), q
    np.testing.assert_allclose(out, ref, rtol=1e-12)
    for e in reversed(slabs):  # slab 0 owns the shared stream
        e.close()


# ---------------------------------------------------------------------------
# both sweep implementations (TMA-streamed default, register-streamed
# fallback) produce the same bits
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_tma_and_register_sweeps_identical(monkeypatch, precision):
    l0, l1 = synthetic.rgb_disk_pair(300)
    gph = pk.triangle_graph((1.0, 1.2, 0.9))
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.05, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=120, check_every=40)
    outs = []
    for tma in ("1", "0"):
        monkeypatch.setenv("OTFX_TMA", tma)
        eng = build_engine("vector", 300, cfg, graph=gph, precision=precision)
        assert (eng.info()["tma_stages"] > 0) == (tma == "1")
        eng.set_marginals(l0, l1)
        hist, it, conv, wall = eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
        outs.append((g.hist_array(pk.SolveReport(conv, it, 0.0, hist)), eng.get_state()))
        eng.close()
    (h1, s1), (h2, s2) = outs
    # iterates are bit-identical; the check scalars of the fused TMA check are
    # summed in a different order than the evaluate kernel's
    g.hist_close(h1, h2, 1e-12)
    for a, b in zip(s1, s2):
        np.testing.assert_array_equal(a, b)


def test_default_path_is_tma_streamed():
    cfg = pk.SolverConfig()
    eng = build_engine("vector", 1024, cfg, graph=pk.triangle_graph())
    inf = eng.info()
    eng.close()
    assert inf["tma_stages"] >= 3 and inf["tile_cols"] in (124, 248)


@pytest.mark.parametrize("kind", ["vector", "matrix"])
def test_fused_check_matches_evaluate_kernel(monkeypatch, kind):
    """The fused check (primal/feasibility in the check sweep, dual norms in
    the speculative next sweep) reports the same history as the separate
    evaluate kernel and stops on the same iterate."""
    if kind == "vector":
        l0, l1 = synthetic.rgb_disk_pair(40)
        args = dict(graph=pk.triangle_graph())
        cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.3, max_iters=20000)
        n, path = 40, None
    else:
        l0, l1 = synthetic.blob_pair_k2(24)
        args = dict(lindblad=pk.lindblad_pair_k2(), complex_path=True)
        cfg = pk.SolverConfig(tau=30.0, norm_u="l1nuc", norm_w="l1nuc", max_iters=3000)
        n, path = 24, None
    outs = []
    monkeypatch.setenv("OTFX_TMA", "1")  # the fused check runs on the TMA sweep
    for fused in ("1", "0"):
        monkeypatch.setenv("OTFX_FUSED_CHECK", fused)
        eng = build_engine(kind, n, cfg, **args)
        eng.set_marginals(l0, l1)
        hist, it, conv, _ = eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
        outs.append((g.hist_array(pk.SolveReport(conv, it, 0.0, hist)), it, conv, eng.get_state()))
        eng.close()
    (h1, it1, c1, s1), (h2, it2, c2, s2) = outs
    assert it1 == it2 and c1 == c2
    g.hist_close(h1, h2, 1e-12)
    for a, b in zip(s1, s2):
        np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------------------
# edge cases: minimum grids, wider channel graphs, more Lindblad matrices
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [2, 3, 5])
def test_tiny_grids_vs_oracle(rng, n):
    l0 = _norm_rand(rng, (n, n, 3))
    l1 = _norm_rand(rng, (n, n, 3))
    gph = pk.triangle_graph()
    cfg = pk.SolverConfig(tau=1.0, norm_u="l12", norm_w="l1", alpha=0.05, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=60, check_every=20)
    rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), gph, cfg=cfg)
    eng, hist = _oracle_vector(l0, l1, gph, cfg, 60, 20)
    g.hist_close(g.hist_array(rep), hist, 1e-10)
    assert g.rel_err(st.phi, eng.phi) <= 1e-10
    assert g.rel_err(st.u.uy, eng.u[:, :, 1]) <= 1e-10


@pytest.mark.parametrize("k", [5, 6, 8])
def test_wide_channel_graphs_vs_oracle(rng, k):
    n = 24
    l0 = _norm_rand(rng, (n, n, k))
    l1 = _norm_rand(rng, (n, n, k))
    edges = [(i, i + 1) for i in range(k - 1)] + [(0, k - 1), (0, k // 2)]
    gph = pk.TransportGraph(k, edges, np.linspace(0.6, 1.5, len(edges)))
    cfg = pk.SolverConfig(tau=2.0, norm_u="l2", norm_w="l1", alpha=0.02, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=80, check_every=40)
    rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), gph, cfg=cfg)
    eng, hist = _oracle_vector(l0, l1, gph, cfg, 80, 40)
    g.hist_close(g.hist_array(rep), hist, 1e-10)
    assert g.rel_err(st.phi, eng.phi) <= 1e-10
    assert g.rel_err(st.w.values, eng.w) <= 1e-10


@pytest.mark.parametrize("k,ell,norms,path", [
    (4, 2, ("l2", "l1"), "real"), (3, 3, ("l12", "l2"), "real"), (2, 4, ("l1", "l1"), "real"),
    (3, 3, ("l1nuc", "l1"), "complex"), (2, 3, ("l2", "l1nuc"), "complex"),
])
def test_matrix_more_lindblad_vs_oracle(rng, k, ell, norms, path):
    n = 10
    a = _rand_herm_psd(rng, n, k)
    b = _rand_herm_psd(rng, n, k)
    if path == "real":
        a = pk.MatrixDensity(np.real(a.values) + 0j)
        b = pk.MatrixDensity(np.real(b.values) + 0j)
        m = rng.normal(size=(ell, k, k))
        mats = 0.5 * (m + np.swapaxes(m, -1, -2)) + 0j
    else:
        m = rng.normal(size=(ell, k, k)) + 1j * rng.normal(size=(ell, k, k))
        mats = 0.5 * (m + np.conj(np.swapaxes(m, -1, -2)))
    lind = pk.LindbladSet(mats)
    cfg = pk.SolverConfig(tau=4.0, norm_u=norms[0], norm_w=norms[1], alpha=0.5, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=90, check_every=30)
    rep, st = pk.solve_matrix(a, b, lind, cfg=cfg)
    use_real = path == "real"
    diff = a.values - b.values
    eng = pdhg.OracleEngine("matrix", np.ascontiguousarray(diff.real) if use_real else diff, n, 4.0,
                            norm_u=norms[0], norm_w=norms[1], alpha=0.5,
                            chan=np.ascontiguousarray(np.real(lind.matrices)) if use_real else lind.matrices,
                            lam_chan=pk.lambda_max_L(lind),
                            dtype=np.float64 if use_real else np.complex128)
    _, _, hist = pdhg.oracle_run(eng, 1e-300, 1e-300, 90, 30)
    assert st.phi.dtype == (np.float64 if use_real else np.complex128)
    g.hist_close(g.hist_array(rep), np.array(hist), 1e-10)
    assert g.rel_err(st.phi, eng.phi) <= 1e-10
    assert g.rel_err(st.w.values, eng.w) <= 1e-10


@pytest.mark.parametrize("kind", ["matrix_real", "matrix_complex", "scalar"])
def test_local_slabs_other_payloads(kind):
    """Row-slab halo exchange for the matrix payloads (K^2 / K(K+1)/2 planes)
    and the scalar payload: bit-identical to one slab."""
    n, P = 30, 3
    if kind == "scalar":
        rng = np.random.default_rng(3)
        l0 = rng.random((n, n)); l0 /= l0.sum()
        l1 = rng.random((n, n)); l1 /= l1.sum()
        cfg = pk.SolverConfig(tau=2.0, norm_u="l2")
        args = {}
        bkind = "scalar"
    else:
        if kind == "matrix_real":
            l0, l1 = synthetic.matrix_blob_fixtures(n)[:2]
            cfg = pk.SolverConfig(tau=10.0, norm_u="l2", norm_w="l1")
            args = dict(lindblad=pk.default_lindblad3(), complex_path=False)
        else:
            l0, l1 = synthetic.blob_pair_k2(n)
            cfg = pk.SolverConfig(tau=10.0, norm_u="l1nuc", norm_w="l1nuc")
            args = dict(lindblad=pk.lindblad_pair_k2(), complex_path=True)
        bkind = "matrix"
    whole = build_engine(bkind, n, cfg, **args)
    whole.set_marginals(l0, l1)
    whole.step(23)
    ref = whole.get_state()
    whole.close()
    bounds = np.linspace(0, n, P + 1).astype(int)
    slabs, stream = [], None
    for r in range(P):
        e = build_engine(bkind, n, cfg, rows=(bounds[r], bounds[r + 1]), stream=stream, **args)
        stream = e.stream
        e.set_marginals(l0[bounds[r]:bounds[r + 1]], l1[bounds[r]:bounds[r + 1]])
        slabs.append(e)
    for _ in range(23):
        for e in slabs:
            e.sweep()
        exchange_local(slabs)
    got = [e.get_state() for e in slabs]
    for q, ref_arr in enumerate(ref):
        if ref_arr is None:
            continue
        cat = np.concatenate([s[q] for s in got], axis=0)
        assert np.array_equal(cat, ref_arr), q
    for e in reversed(slabs):
        e.close()


# ---------------------------------------------------------------------------
# the NCCL code path with a single rank (the pool has one GPU): dlopen, comm
# init, allreduce of the check scalars and masses, comm teardown; results must
# equal the engine without a communicator
# ---------------------------------------------------------------------------
def test_nccl_single_rank_path():
    from paper_1712_10279_b200 import distributed as D

    n = 300
    l0, l1 = synthetic.rgb_disk_pair(n)
    gph = pk.triangle_graph()
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.05, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=250, check_every=100)
    uid = pk.solver.nccl_unique_id()
    assert len(uid) == 128
    rep1, st1 = D.solve_vector_rows(l0, l1, gph, n, cfg, nranks=1, rank=0, unique_id=uid)
    rep2, st2 = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), gph, cfg=cfg)
    np.testing.assert_array_equal(g.hist_array(rep1), g.hist_array(rep2))
    np.testing.assert_array_equal(st1.phi, st2.phi)
    np.testing.assert_array_equal(st1.w.values, st2.w.values)
    # a communicator that outlives the engines of several solves
    comm = D.SlabCommunicator(pk.solver.nccl_unique_id(), 1, 0, 0)
    for _ in range(2):
        rep3, st3 = D.solve_vector_rows(l0, l1, gph, n, cfg, nranks=1, rank=0, comm=comm)
        np.testing.assert_array_equal(g.hist_array(rep3), g.hist_array(rep2))
        np.testing.assert_array_equal(st3.phi, st2.phi)
    comm.close()


@pytest.mark.parametrize("warps", ["4", "8"])
def test_tma_cta_widths_identical(monkeypatch, warps):
    """4- and 8-warp TMA sweeps (124 / 248 columns per CTA) give the same bits
    as the register sweep."""
    n = 700
    l0, l1 = synthetic.rgb_disk_pair(n)
    gph = pk.triangle_graph((1.0, 1.1, 0.9))
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.05, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=40, check_every=20)
    outs = []
    for tma in ("1", "0"):
        monkeypatch.setenv("OTFX_TMA", tma)
        monkeypatch.setenv("OTFX_TMA_WARPS", warps)
        eng = build_engine("vector", n, cfg, graph=gph)
        if tma == "1":
            assert eng.info()["tile_cols"] == 31 * int(warps)
        eng.set_marginals(l0, l1)
        eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
        outs.append(eng.get_state())
        eng.close()
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)




@pytest.mark.parametrize("warps", ["4", "8"])
def test_tma_heavy_complex_widths_identical(monkeypatch, warps):
    """3x3 complex-Hermitian l1nuc (226-255-register payload): the 8-warp
    self-producing / 2-stage TMA sweep and the 4-warp one with a producer warp
    give the same bits as the register sweep."""
    n = 600
    l0, l1 = synthetic.matrix_blob_fixtures(n)[:2]
    cfg = pk.SolverConfig(tau=30.0, norm_u="l1nuc", norm_w="l1nuc", tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=24, check_every=12)
    outs = []
    for tma in ("1", "0"):
        monkeypatch.setenv("OTFX_TMA", tma)
        monkeypatch.setenv("OTFX_TMA_WARPS", warps)
        eng = build_engine("matrix", n, cfg, lindblad=pk.default_lindblad3(), complex_path=True)
        if tma == "1":
            inf = eng.info()
            assert inf["tile_cols"] == 31 * int(warps)
            assert inf["tma_stages"] == (2 if warps == "8" else 4)
        eng.set_marginals(l0, l1)
        eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
        outs.append(eng.get_state())
        eng.close()
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n,rows", [(40, 1), (40, 3), (257, 1), (257, 5)])
def test_tma_heavy_self_produce_ragged(monkeypatch, n, rows):
    """8-warp self-producing ring (no producer warp: the last warp out of a
    slot issues its next stage) on ragged shapes -- one-row CTAs whose ring
    holds the whole band, a partial last CTA column, rows not dividing n --
    bit-identical to the register sweep, with checks (fused check and dual
    sweeps) on the way."""
    l0, l1 = synthetic.matrix_blob_fixtures(n)[:2]
    cfg = pk.SolverConfig(tau=30.0, norm_u="l1nuc", norm_w="l2", tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=14, check_every=5)
    outs = []
    for tma in ("1", "0"):
        monkeypatch.setenv("OTFX_TMA", tma)
        if tma == "1":
            monkeypatch.setenv("OTFX_TILE_ROWS", str(rows))
        else:
            monkeypatch.delenv("OTFX_TILE_ROWS", raising=False)
        eng = build_engine("matrix", n, cfg, lindblad=pk.default_lindblad3(), complex_path=True)
        if tma == "1":
            inf = eng.info()
            assert inf["tile_cols"] == 248 and inf["tile_rows"] == rows
        eng.set_marginals(l0, l1)
        h, it, conv, _ = eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
        outs.append((eng.get_state(), [(r.iteration, r.primal, r.dual, r.gap_ratio,
                                         r.feas_residual, r.residual) for r in h]))
        eng.close()
    for a, b in zip(outs[0][0], outs[1][0]):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_allclose(np.array(outs[0][1], dtype=float), np.array(outs[1][1], dtype=float),
                               rtol=1e-12, atol=0)


# ---------------------------------------------------------------------------
# on-chip cluster solve (small grids: whole run loop in one cluster launch)
# against the streamed per-iteration path: same iterates bit for bit, same
# history up to the reduction order of the check scalars, same stopping point
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,k,norm_u,norm_w,alpha,eps,precision,tol,iters", [
    (64, 3, "l12", "l1", 0.3, 0.0, "f64", 1e-300, 2000),   # BASELINE C1 shape, w active
    (37, 3, "l2", "l2", 0.05, 0.01, "f64", 1e-300, 333),
    (60, 3, "l1", "l1", 0.05, 0.0, "f64", 1e-300, 250),
    (32, 3, "l12", "l1", 1.0, 0.0, "f64", None, 200000),   # converges: early stop on device
    (50, 4, "l12", "l2", 0.05, 0.0, "f32", 1e-300, 300),
    (5, 2, "l12", "l1", 0.05, 0.0, "f64", 1e-300, 120),
    (1, 1, "l2", "l1", 1.0, 0.0, "f64", 1e-300, 150),      # scalar (n=33)
])
def test_cluster_solve_matches_streamed_path(monkeypatch, n, k, norm_u, norm_w, alpha, eps,
                                             precision, tol, iters):
    rng = np.random.default_rng(11)
    if k == 1:
        n = 33
        l0 = _norm_rand(rng, (n, n)); l1 = _norm_rand(rng, (n, n))
        kind, args = "scalar", {}
    elif k == 3 and n in (64, 32, 60):
        l0, l1 = synthetic.rgb_disk_pair(n)
        kind, args = "vector", dict(graph=pk.triangle_graph((1.0, 1.3, 0.8)))
    else:
        l0 = _norm_rand(rng, (n, n, k)); l1 = _norm_rand(rng, (n, n, k))
        edges = [(a, b) for a in range(k) for b in range(a + 1, k)]
        kind, args = "vector", dict(graph=pk.TransportGraph(k, edges, [1.0 + 0.1 * q for q in range(len(edges))]))
    kw = dict(tau=6.0, norm_u=norm_u, norm_w=norm_w, alpha=alpha, eps_reg=eps, max_iters=iters,
              check_every=100)
    if tol is not None:
        kw.update(tol_gap=tol, tol_feas=tol)
    cfg = pk.SolverConfig(**kw)
    outs = []
    for cl in ("1", "0"):
        monkeypatch.setenv("OTFX_CLUSTER", cl)
        eng = build_engine(kind, n, cfg, precision=precision, **args)
        assert (eng.info()["cluster_ctas"] > 0) == (cl == "1")
        eng.set_marginals(l0, l1)
        hist, it, conv, _ = eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
        st = eng.get_state()
        eng.step(7)  # plain iterations after the run, through the same path
        outs.append((g.hist_array(pk.SolveReport(conv, it, 0.0, hist)), it, conv, st,
                     eng.get_state()))
        eng.close()
    (h1, it1, c1, s1, t1), (h2, it2, c2, s2, t2) = outs
    assert it1 == it2 and c1 == c2
    if tol is None:
        assert c1 and it1 < iters
    g.hist_close(h1, h2, 1e-12)
    for a, b in zip(s1 + t1, s2 + t2):
        if a is not None:
            np.testing.assert_array_equal(a, b)


def test_cluster_solve_is_default_for_small_grids():
    for n, want in ((48, True), (64, True), (128, False), (1024, False)):
        eng = build_engine("vector", n, pk.SolverConfig(), graph=pk.triangle_graph())
        assert (eng.info()["cluster_ctas"] > 0) == want, n
        eng.close()


def test_pooled_engines_reuse_memory_and_release():
    """Engine memory comes from the library's stream-ordered pool: a second
    engine of the same size reuses the cached block (no stale state: the
    iterate starts from zero), and the cache can be trimmed."""
    l0, l1 = synthetic.rgb_disk_pair(300)
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", tol_gap=1e-300, tol_feas=1e-300,
                          max_iters=50, check_every=25)
    states = []
    for _ in range(2):
        rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), pk.triangle_graph(),
                                  cfg=cfg)
        states.append((rep.transport_value, st.phi))
    assert states[0][0] == states[1][0]
    np.testing.assert_array_equal(states[0][1], states[1][1])
    pk.release_cached_memory()


# ---------------------------------------------------------------------------
# the distributed run loop (fused checks, speculative dual sweep, stopping
# rule) over P row slabs of one grid on one GPU, with the TMA-streamed slab
# sweeps the multi-GPU bench runs: same iterates and history as one engine
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("transport", ["copy", "nccl"])
@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("P,n,force_tma,conv", [
    (2, 300, True, False), (3, 301, True, False), (2, 1100, False, False), (2, 32, True, True),
    (4, 900, True, False),
])
def test_local_slab_run_loop_matches_single_engine(monkeypatch, P, n, force_tma, conv, overlap,
                                                   transport):
    """overlap=1: edge bands + halo exchange on the high-priority stream,
    interior bands concurrently on the engine stream (the multi-GPU schedule).
    transport=nccl: the halo rows and the check scalars go through the
    ncclSend / ncclRecv / ncclAllReduce calls of the multi-GPU ranks, posted
    to a one-rank communicator (NCCL loopback on one GPU)."""
    from paper_1712_10279_b200 import distributed as D
    from paper_1712_10279_b200.solver import run_local
    loop = D.SlabCommunicator(pk.solver.nccl_unique_id(), 1, 0, 0) if transport == "nccl" else None
    monkeypatch.setenv("OTFX_OVERLAP", overlap)
    if force_tma:
        monkeypatch.setenv("OTFX_TMA", "1")
    l0, l1 = synthetic.rgb_disk_pair(n)
    gph = pk.triangle_graph((1.0, 1.2, 0.9))
    if conv:
        cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=1.0, max_iters=200000)
    else:
        cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.05, tol_gap=1e-300,
                              tol_feas=1e-300, max_iters=230, check_every=50)
    whole = build_engine("vector", n, cfg, graph=gph)
    assert whole.info()["tma_stages"] > 0
    whole.set_marginals(l0, l1)
    hist1, it1, c1, _ = whole.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
    ref = whole.get_state()
    whole.close()
    bounds = np.linspace(0, n, P + 1).astype(int)
    slabs, stream = [], None
    for r in range(P):
        e = build_engine("vector", n, cfg, graph=gph, rows=(bounds[r], bounds[r + 1]), stream=stream)
        assert e.info()["tma_stages"] > 0
        assert e.info()["halo_overlap"] == (1 if overlap == "1" and e.info()["grid_y"] >= 3 else 0)
        stream = e.stream
        e.set_marginals(l0[bounds[r]:bounds[r + 1]], l1[bounds[r]:bounds[r + 1]])
        slabs.append(e)
    # run_local combines the slabs' own-row ||diff|| itself (no override)
    hist2, it2, c2 = run_local(slabs, cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every,
                               loopback=loop)
    assert it1 == it2 and c1 == c2 == conv
    g.hist_close(g.hist_array(pk.SolveReport(c1, it1, 0.0, hist1)),
                 g.hist_array(pk.SolveReport(c2, it2, 0.0, hist2)), 1e-12)
    got = [e.get_state() for e in slabs]
    for q, ref_arr in enumerate(ref):
        cat = np.concatenate([s[q] for s in got], axis=0)
        assert np.array_equal(cat, ref_arr), q
    for e in reversed(slabs):
        e.close()
    if loop is not None:
        loop.close()


# ---------------------------------------------------------------------------
# the bench workload itself (BASELINE configs[4], vector 3-channel 8192^2):
# the TMA-streamed headline kernel (fused check + speculative dual sweep) and
# the register-streamed sweep (pinned bit-exact to the reference goldens at
# small sizes) give the same bits at full size; ghost entries stay zero
# ---------------------------------------------------------------------------
def test_bench_size_tma_matches_register_sweep(monkeypatch):
    n = 8192
    l0, l1 = synthetic.rgb_disk_pair(n)
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.3, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=5, check_every=2)
    outs = []
    for tma in ("1", "0"):
        monkeypatch.setenv("OTFX_TMA", tma)
        eng = build_engine("vector", n, cfg, graph=pk.triangle_graph())
        assert (eng.info()["tma_stages"] > 0) == (tma == "1")
        eng.set_marginals(l0, l1)
        hist, it, conv, _ = eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
        ux, uy, w, phi = eng.get_state()
        eng.close()
        assert it == 5 and not conv
        assert not ux[n - 1].any() and not uy[:, n - 1].any()  # ghost entries (S/spatial.py:80-86)
        outs.append((g.hist_array(pk.SolveReport(conv, it, 0.0, hist)), phi, w, ux))
        del uy
    (h1, p1, w1, x1), (h2, p2, w2, x2) = outs
    g.hist_close(h1, h2, 1e-12)
    assert np.array_equal(p1, p2) and np.array_equal(w1, w2) and np.array_equal(x1, x2)


def test_engine_timing_covers_ungraphed_runs(monkeypatch):
    """The bench's sweep timing also brackets plain iterations launched
    without a CUDA graph (the path a decomposed slab takes)."""
    monkeypatch.setenv("OTFX_GRAPHS", "0")
    l0, l1 = synthetic.rgb_disk_pair(600)
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", tol_gap=1e-300, tol_feas=1e-300,
                          max_iters=200, check_every=100)
    eng = build_engine("vector", 600, cfg, graph=pk.triangle_graph())
    eng.set_marginals(l0, l1)
    eng.timing(1)
    eng.run(1e-300, 1e-300, 200, 100)
    ms, iters = eng.timing(0)
    eng.close()
    assert iters >= 190 and ms > 0

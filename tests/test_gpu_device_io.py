"""Device-pointer hand-off (include/otfx.h *_device entry points): torch owns
the marginals and the returned state, the engine reads / writes them in place
(SURVEY §8(b) ownership row).  Results must be bit-identical to the host-array
path, which the parity tests pin to the reference."""

import numpy as np
import pytest
import torch

import gpu_util as g
import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import synthetic
from paper_1712_10279_b200.solver import build_engine

pytestmark = pytest.mark.gpu


def _same(rep_a, st_a, rep_b, st_b):
    assert rep_a.iterations == rep_b.iterations and rep_a.converged == rep_b.converged
    assert np.array_equal(g.hist_array(rep_a), g.hist_array(rep_b), equal_nan=True)
    assert np.array_equal(st_a.u.ux.cpu().numpy(), st_b.u.ux)
    assert np.array_equal(st_a.u.uy.cpu().numpy(), st_b.u.uy)
    assert np.array_equal(st_a.phi.cpu().numpy(), st_b.phi)
    if st_b.w is not None:
        assert st_a.w.values.dtype == {np.dtype(np.float64): torch.float64,
                                       np.dtype(np.complex128): torch.complex128}[st_b.w.values.dtype]
        assert np.array_equal(st_a.w.values.cpu().numpy(), st_b.w.values)


@pytest.mark.parametrize("n", [48, 300, 1024])
def test_vector_tensors_match_host_path(n):
    l0, l1 = synthetic.rgb_disk_pair(n)
    graph = pk.triangle_graph()
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.3, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=250, check_every=100)
    rep_h, st_h = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), graph, cfg=cfg)
    t0 = torch.from_numpy(l0).cuda()
    t1 = torch.from_numpy(l1).cuda()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):  # a non-default caller stream
        rep_d, st_d = pk.solve_tensors(t0, t1, graph, cfg=cfg)
    assert st_d.phi.is_cuda and st_d.phi.shape == (n, n, 3)
    _same(rep_d, st_d, rep_h, st_h)


@pytest.mark.parametrize("case", ["real3", "complex2"])
def test_matrix_tensors_match_host_path(case):
    if case == "real3":
        a, b = synthetic.matrix_blob_fixtures(40)[:2]
        lind = pk.default_lindblad3()
        cfg = pk.SolverConfig(tau=30.0, norm_u="l2", norm_w="l1", tol_gap=1e-300,
                              tol_feas=1e-300, max_iters=200, check_every=100)
    else:
        a, b = synthetic.blob_pair_k2(40)
        lind = pk.lindblad_pair_k2()
        cfg = pk.SolverConfig(tau=30.0, norm_u="l1nuc", norm_w="l1nuc", tol_gap=1e-300,
                              tol_feas=1e-300, max_iters=200, check_every=100)
    rep_h, st_h = pk.solve_matrix(pk.MatrixDensity(a), pk.MatrixDensity(b), lind, cfg=cfg)
    rep_d, st_d = pk.solve_tensors(torch.from_numpy(np.asarray(a, np.complex128)).cuda(),
                                   torch.from_numpy(np.asarray(b, np.complex128)).cuda(), lind,
                                   cfg=cfg)
    assert (st_d.phi.dtype == torch.float64) == (case == "real3")
    _same(rep_d, st_d, rep_h, st_h)


def test_scalar_tensors_match_host_path():
    a, b = synthetic.dirac_pair(33, (8, 16), (24, 16))
    cfg = pk.SolverConfig(tau=3.0, max_iters=300, tol_gap=1e-300, tol_feas=1e-300)
    rep_h, st_h = pk.solve_scalar(pk.ScalarDensity(a), pk.ScalarDensity(b), cfg=cfg)
    rep_d, st_d = pk.solve_tensors(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), cfg=cfg)
    assert st_d.w is None
    _same(rep_d, st_d, rep_h, st_h)


def test_state_device_roundtrip_and_step_equals_host():
    n = 700
    rng = np.random.default_rng(3)
    l0, l1 = synthetic.rgb_disk_pair(n)
    graph = pk.triangle_graph()
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.3)
    state = [rng.normal(size=(n, n, 3)) * s for s in (1e-7, 1e-7, 1e-3, 1e-2)]
    state[0][-1] = 0.0
    state[1][:, -1] = 0.0
    outs = []
    for device_io in (False, True):
        eng = build_engine("vector", n, cfg, graph=graph)
        try:
            if device_io:
                eng.set_marginals_device(torch.from_numpy(l0).cuda(), torch.from_numpy(l1).cuda())
                eng.set_state_device(*[torch.from_numpy(x).cuda() for x in state])
                back = [t.cpu().numpy() for t in eng.get_state_device()]
                assert all(np.array_equal(x, y) for x, y in zip(back, state))
            else:
                eng.set_marginals(l0, l1)
                eng.set_state(*state)
            eng.step(5)
            chk = eng.step_check()
            st = ([t.cpu().numpy() for t in eng.get_state_device()] if device_io
                  else list(eng.get_state()))
        finally:
            eng.close()
        outs.append((chk, st))
    assert outs[0][0] == outs[1][0]
    assert all(np.array_equal(x, y) for x, y in zip(outs[0][1], outs[1][1]))


def test_device_io_rejects_wrong_tensors():
    n = 32
    l0, l1 = synthetic.rgb_disk_pair(n)
    with pytest.raises(pk.ValidationError):
        pk.solve_tensors(torch.from_numpy(l0), torch.from_numpy(l1), pk.triangle_graph())
    eng = build_engine("vector", n, pk.SolverConfig(tau=6.0), graph=pk.triangle_graph())
    try:
        with pytest.raises(pk.ValidationError):
            eng.set_marginals_device(torch.from_numpy(l0).cuda().float(),
                                     torch.from_numpy(l1).cuda().float())
        with pytest.raises(pk.ValidationError):  # non-contiguous
            t = torch.from_numpy(l0).cuda().transpose(0, 1)
            eng.set_marginals_device(t, t)
    finally:
        eng.close()
    with pytest.raises(pk.ValidationError):  # mass mismatch, detected on the device sums
        pk.solve_tensors(torch.from_numpy(l0).cuda(), 2 * torch.from_numpy(l1).cuda(),
                         pk.triangle_graph())

"""The reference's acceptance criteria that exercise the solver path
(T/test_acceptance.py C04-C10), run on the B200 engine, against the values the
reference itself printed when run in the build container:

    C04 S = 0.50006 after 39,300 iterations       C05 V = 0.46124/0.46076/0.46129
    C06 V_l1 = 0.56470                            C09 matrix n=128: 3,200 iterations
    C07 M01 = 2.5 alpha, M02 = 0.3625 (alpha=0.1), 0.4034-0.4042 (alpha>=0.3)
"""

import numpy as np
import pytest

import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import synthetic

pytestmark = pytest.mark.gpu
GAP_TOL, FEAS_TOL = 1e-3, 1e-5


def check_health(report, label=""):
    """Criterion 9 screen (T/test_acceptance.py:23-34)."""
    res = [h.residual for h in report.history if np.isfinite(h.residual)]
    assert res, label
    scale = max(res[0], 1e-30)
    for a, b in zip(res, res[1:]):
        assert b <= a * (1 + 1e-9) + 1e-15 * scale, f"{label}: residual increased"
    assert min(res) >= -1e-9 * scale, f"{label}: negative residual"
    assert report.converged, f"{label}: did not converge"
    assert report.history[-1].gap_ratio <= GAP_TOL
    assert report.history[-1].feas_residual <= FEAS_TOL


def rgb(n, norm_u="l12", precision="f64"):
    l0, l1 = synthetic.rgb_disk_pair(n)
    cfg = pk.SolverConfig(tau=6.0, norm_u=norm_u, norm_w="l1", alpha=1.0)
    return pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), pk.triangle_graph(),
                           cfg=cfg, precision=precision)


def test_c04_dirac_distance():
    a, b = synthetic.dirac_pair(33, (8, 16), (24, 16))
    rep, _ = pk.solve_scalar(pk.ScalarDensity(a), pk.ScalarDensity(b),
                             cfg=pk.SolverConfig(norm_u="l2"))
    check_health(rep, "dirac")
    assert rep.transport_value == pytest.approx(0.50006, abs=5e-6)
    assert rep.iterations == 39_300


@pytest.mark.parametrize("n,value", [(32, 0.46124), (64, 0.46076), (128, 0.46129)])
def test_c05_grid_consistency(n, value):
    rep, _ = rgb(n)
    check_health(rep, f"rgb n={n}")
    assert rep.transport_value == pytest.approx(value, abs=5e-6)
    if n == 128:
        assert rep.iterations == 86_400


def test_c05_fp32_build_converged_value():
    """north_star: the fp32 build's converged W1 distance agrees to 1e-4."""
    r64, _ = rgb(64)
    r32, _ = rgb(64, precision="f32")
    assert r32.converged
    assert r32.transport_value == pytest.approx(r64.transport_value, rel=1e-4)


def test_c06_norm_ordering():
    rep, _ = rgb(32, norm_u="l1")
    check_health(rep, "l1")
    assert rep.transport_value == pytest.approx(0.56470, abs=5e-6)
    assert rep.transport_value >= 0.46124 * 1.03


def test_c07_alpha_sweep_values():
    """Reference behaviour: M01/alpha = 2.5 exactly-ish, M02 not constant
    (the reference's own C07 assertion fails on it; we reproduce the values)."""
    m0, m1, m2 = (pk.MatrixDensity(m) for m in synthetic.matrix_blob_fixtures(32))
    lind = pk.default_lindblad3()
    m02_ref = {0.1: 0.3625, 0.3: 0.4034, 1.0: 0.4042}
    for alpha in (0.1, 0.3, 1.0):
        cfg = pk.SolverConfig(tau=3.0, norm_u="l2", norm_w="l1", alpha=alpha)
        rep01, _ = pk.solve_matrix(m0, m1, lind, cfg=cfg)
        rep02, _ = pk.solve_matrix(m0, m2, lind, cfg=cfg)
        check_health(rep01, f"M01 alpha={alpha}")
        check_health(rep02, f"M02 alpha={alpha}")
        assert rep01.transport_value / alpha == pytest.approx(2.5, rel=2e-3)
        assert rep02.transport_value == pytest.approx(m02_ref[alpha], abs=5e-4)


def test_c08_metric_axioms():
    rng = np.random.default_rng(55)
    cfg = pk.SolverConfig(tau=3.0, norm_u="l12", norm_w="l1")
    dens = [pk.normalize(pk.VectorDensity(rng.random((8, 8, 3)))) for _ in range(3)]
    v = {}
    for i in range(3):
        for j in range(3):
            if i != j:
                rep, _ = pk.solve_vector(dens[i], dens[j], pk.triangle_graph(), cfg=cfg)
                check_health(rep, f"V({i},{j})")
                v[i, j] = rep.transport_value
    for i, j in ((0, 1), (0, 2), (1, 2)):
        assert v[i, j] == pytest.approx(v[j, i], rel=0.02)
    assert v[0, 2] <= (v[0, 1] + v[1, 2]) * 1.02


def test_c09_matrix_128_iterations():
    m0, m1, _ = synthetic.matrix_blob_fixtures(128)
    cfg = pk.SolverConfig(tau=30.0, norm_u="l2", norm_w="l1", alpha=1.0)
    rep, _ = pk.solve_matrix(pk.MatrixDensity(m0), pk.MatrixDensity(m1), pk.default_lindblad3(),
                             cfg=cfg)
    check_health(rep, "matrix n=128")
    assert rep.iterations == 3_200


def test_c10_quadratic_regularization():
    rng = np.random.default_rng(77)
    a = pk.normalize(pk.ScalarDensity(rng.random((16, 16))))
    b = pk.normalize(pk.ScalarDensity(rng.random((16, 16))))
    base, _ = pk.solve_scalar(a, b, cfg=pk.SolverConfig(tau=3.0))
    check_health(base, "base")
    values = []
    for eps in (1e-1, 1e-2, 1e-3):
        rep, _ = pk.solve_scalar(a, b, cfg=pk.SolverConfig(tau=3.0, eps_reg=eps))
        assert rep.converged
        assert rep.transport_value >= base.transport_value - GAP_TOL
        values.append(rep.transport_value)
    assert values[0] >= values[1] - 1e-9 and values[1] >= values[2] - 1e-9
    assert values[2] == pytest.approx(base.transport_value, rel=0.02)

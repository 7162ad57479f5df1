"""GPU parity: the CUDA path (through the public solve_* API and the C ABI)
against the reference's golden fixtures and the oracle.

Tolerances (BASELINE.json north_star): fp64 build <= 1e-10 relative on the
iterates and on the objective/history after the fixed iteration count; fp32
build <= 1e-4 relative on the objective.
"""

import numpy as np
import pytest

import golden_util as gu
import gpu_util as g
import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import synthetic

pytestmark = pytest.mark.gpu

F64_RTOL = 1e-10


@pytest.mark.parametrize("sweep", ["tma", "register", "cluster"])
@pytest.mark.parametrize("name", gu.full_cases())
def test_golden_full_fp64(name, sweep, monkeypatch):
    """Every iteration path against the reference's own iterates: the on-chip
    cluster solve (default for the small vector / scalar fixtures), the
    register-streamed sweep, and the TMA-streamed sweep."""
    monkeypatch.setenv("OTFX_TMA", "1" if sweep == "tma" else "0")
    monkeypatch.setenv("OTFX_CLUSTER", "1" if sweep == "cluster" else "0")
    meta, arrs = gu.load(name)
    rep, st = g.solve_case(meta, arrs["l0"], arrs["l1"], arrs.get("lindblad"))
    assert rep.iterations == meta["iterations"]
    assert rep.converged == meta["converged"]
    g.hist_close(g.hist_array(rep), arrs["history"], F64_RTOL)
    assert st.phi.dtype == np.dtype(meta["phi_dtype"])
    assert g.rel_err(st.u.ux, arrs["ux"]) <= F64_RTOL
    assert g.rel_err(st.u.uy, arrs["uy"]) <= F64_RTOL
    assert g.rel_err(st.phi, arrs["phi"]) <= F64_RTOL
    if "w" in arrs:
        assert st.w.values.shape == arrs["w"].shape
        assert g.rel_err(st.w.values, arrs["w"]) <= F64_RTOL
    if meta["kind"] in ("scalar", "vector"):
        # these paths follow the reference's rounding sequence exactly
        # (IEEE div/sqrt, no contraction, the BLAS order of the graph
        # operators): the reference's own iterates, bit for bit
        assert np.array_equal(st.u.ux, arrs["ux"]) and np.array_equal(st.u.uy, arrs["uy"])
        assert np.array_equal(st.phi, arrs["phi"])
        if "w" in arrs:
            assert np.array_equal(st.w.values, arrs["w"])


@pytest.mark.parametrize("name", gu.full_cases())
def test_golden_full_fp32(name):
    meta, arrs = gu.load(name)
    rep, st = g.solve_case(meta, arrs["l0"], arrs["l1"], arrs.get("lindblad"), precision="f32")
    assert rep.iterations == meta["iterations"]
    ref = arrs["history"]
    # objective (primal) within 1e-4 relative at every check
    assert g.rel_err(g.hist_array(rep)[:, 1], ref[:, 1]) <= 1e-4


SUMMARY_INPUTS = {
    "S_vec256": lambda: synthetic.rgb_disk_pair(256),
    "S_matr256": lambda: synthetic.matrix_blob_fixtures(256)[:2],
    "S_matc128": lambda: synthetic.blob_pair_k2(128),
    "S_vec32_conv": lambda: synthetic.rgb_disk_pair(32),
    "S_sca33_dirac_conv": lambda: synthetic.dirac_pair(33, (8, 16), (24, 16)),
}


@pytest.mark.parametrize("name", sorted(SUMMARY_INPUTS))
def test_golden_summary_fp64(name):
    """BASELINE configs C2/C3/C4 and the converged reference values."""
    meta, arrs = gu.load(name)
    l0, l1 = SUMMARY_INPUTS[name]()
    mats = arrs.get("lindblad")
    rep, st = g.solve_case(meta, l0, l1, mats)
    assert rep.iterations == meta["iterations"]
    assert rep.converged == meta["converged"]
    g.hist_close(g.hist_array(rep), arrs["history"], 1e-10)
    norms = meta["norms"]
    np.testing.assert_allclose(np.linalg.norm(st.phi), norms["phi"], rtol=1e-10)
    np.testing.assert_allclose(np.linalg.norm(st.u.ux), norms["ux"], rtol=1e-10)
    if norms["w"] > 0:
        np.testing.assert_allclose(np.linalg.norm(st.w.values), norms["w"], rtol=1e-10)


def test_converged_values_match_reference_acceptance():
    """C05 at n=32 (V = 0.46124) and the Dirac distance 0.5 (T/test_solver.py:70-77)."""
    meta, _ = gu.load("S_vec32_conv")
    l0, l1 = synthetic.rgb_disk_pair(32)
    rep, _ = g.solve_case(meta, l0, l1)
    assert rep.converged
    assert rep.transport_value == pytest.approx(0.46124, rel=1e-4)
    a, b = synthetic.dirac_pair(33, (8, 16), (24, 16))
    rep, _ = pk.solve_scalar(pk.ScalarDensity(a), pk.ScalarDensity(b), cfg=pk.SolverConfig(tau=3.0))
    assert rep.converged and rep.transport_value == pytest.approx(0.5, rel=0.02)

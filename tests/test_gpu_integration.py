"""The reference-side binding of INTEGRATION.md, executed: the UNMODIFIED
reference package (installed into baseline/_ref) builds its own
``_Engine`` (S/solver.py:179-205) and the ctypes stub
``integration/otflux_otfx.py``, loaded as ``otflux._otfx``, runs it on the B200
engine in place of ``_run`` (S/solver.py:294-337).  The result must equal the
reference's own CPU ``solve_vector`` (S/solver.py:372-393)."""

import importlib.util
import os
import sys

import numpy as np
import pytest

import gpu_util as g

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def otflux_with_binding():
    if not os.path.isdir(os.path.join(REF, "otflux")):
        pytest.skip("reference not installed into baseline/_ref (see DESIGN.md §10)")
    sys.path.insert(0, REF)
    try:
        import otflux
        from otflux import solver as ref_solver
    finally:
        sys.path.remove(REF)
    assert os.path.realpath(otflux.__file__).startswith(os.path.realpath(REF))
    spec = importlib.util.spec_from_file_location(
        "otflux._otfx", os.path.join(ROOT, "integration", "otflux_otfx.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["otflux._otfx"] = mod
    spec.loader.exec_module(mod)
    os.environ["OTFX_LIB"] = os.path.join(ROOT, "paper_1712_10279_b200", "libotfx.so")
    return otflux, ref_solver, mod


@pytest.mark.parametrize("n,alpha,iters", [(64, 0.3, 2000), (48, 1.0, 700)])
def test_reference_solve_vector_with_gpu_run(otflux_with_binding, n, alpha, iters):
    otflux, ref_solver, binding = otflux_with_binding
    l0, l1 = otflux.rgb_disk_pair(otflux.GridSpec(n))
    graph = otflux.triangle_graph()
    cfg = otflux.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=alpha,
                              tol_gap=1e-300, tol_feas=1e-300, max_iters=iters, check_every=100)
    # the reference, unchanged, on the CPU
    rep_ref, st_ref = otflux.solve_vector(l0, l1, graph, cfg=cfg)
    # the maintainer's change: the same engine, _run replaced by the binding
    engine = ref_solver._engine_for("vector", l0, l1, cfg, graph=graph)
    rep, st = binding.run_vector_on_gpu(engine, graph, l0, l1)
    assert type(rep) is type(rep_ref) and type(st) is type(st_ref)
    assert rep.iterations == rep_ref.iterations == iters
    assert rep.converged == rep_ref.converged
    h = np.array([[p.iteration, p.primal, p.dual, p.gap_ratio, p.feas_residual, p.residual]
                  for p in rep.history])
    href = np.array([[p.iteration, p.primal, p.dual, p.gap_ratio, p.feas_residual, p.residual]
                     for p in rep_ref.history])
    g.hist_close(h, href, 1e-10)
    # the vector path follows the reference's operation order: equal iterates
    assert np.array_equal(st.u.ux, st_ref.u.ux)
    assert np.array_equal(st.u.uy, st_ref.u.uy)
    assert np.array_equal(st.phi, st_ref.phi)
    assert np.array_equal(st.w.values, st_ref.w.values)
    if alpha < 1:
        assert np.linalg.norm(st_ref.w.values) > 0
    assert rep.transport_value == pytest.approx(rep_ref.transport_value, rel=1e-10)


def test_reference_converged_solve_with_gpu_run(otflux_with_binding):
    """C05 at n = 32 to convergence (T/test_acceptance.py C05): identical
    iteration count and value."""
    otflux, ref_solver, binding = otflux_with_binding
    l0, l1 = otflux.rgb_disk_pair(otflux.GridSpec(32))
    graph = otflux.triangle_graph()
    cfg = otflux.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1")
    rep_ref, _ = otflux.solve_vector(l0, l1, graph, cfg=cfg)
    engine = ref_solver._engine_for("vector", l0, l1, cfg, graph=graph)
    rep, _ = binding.run_vector_on_gpu(engine, graph, l0, l1)
    assert rep.converged and rep_ref.converged
    assert rep.iterations == rep_ref.iterations
    assert rep.transport_value == pytest.approx(rep_ref.transport_value, rel=1e-10)


def test_c_only_caller_matches_python_path(tmp_path):
    """integration/otfx_scalar_example.c drives the engine through the C ABI
    alone (create, set_marginals, run, history, destroy) on the reference's
    Dirac-pair fixture (T/test_solver.py:70-77): same iteration count and the
    same W1 bits as solve_scalar, and W1 = 0.5 within the reference's 2 %."""
    import shutil
    import subprocess
    from pathlib import Path

    import paper_1712_10279_b200 as pk

    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    root = Path(__file__).resolve().parent.parent
    lib_dir = str(root / "paper_1712_10279_b200")
    exe = tmp_path / "ex"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", f"-I{root / 'include'}",
                    str(root / "integration" / "otfx_scalar_example.c"), f"-L{lib_dir}",
                    "-l:libotfx.so", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    iters, conv, w1 = int(out[0]), int(out[1]), float(out[2])
    a, b = pk.dirac_pair(pk.GridSpec(33), (8, 16), (24, 16))
    rep, _ = pk.solve_scalar(a, b, cfg=pk.SolverConfig(tau=3.0))
    assert conv == 1 and rep.converged
    assert iters == rep.iterations
    assert w1 == rep.transport_value
    assert abs(w1 - 0.5) <= 0.02 * 0.5

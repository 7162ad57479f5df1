"""CPU tests of the host layer: the C ABI library loads and exports every
symbol include/otfx.h declares (no compute calls), configuration and input
validation mirror the reference (T/test_solver.py:23-59, T/test_graph.py,
T/test_lindblad.py), and the product path fails loudly without a GPU."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import _lib
from paper_1712_10279_b200.distributed import halo_plan, slab_bounds

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "otfx.h").read_text()
    names = sorted(set(re.findall(r"^\s*(?:int|const char\*|void\*)\s+(otfx_\w+)\(", header, re.M)))
    assert len(names) >= 20
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)
    assert _lib.load().otfx_abi_version() == 2


def test_error_codes_map_to_reference_exceptions():
    with pytest.raises(pk.ValidationError):
        _lib.check(_lib.EINVAL)
    with pytest.raises(pk.UnsupportedNormError):
        _lib.check(_lib.EUNSUPPORTED)
    with pytest.raises(pk.NumericalError):
        _lib.check(_lib.ECUDA)


def test_no_gpu_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    a = pk.normalize(pk.ScalarDensity(np.random.default_rng(0).random((6, 6))))
    with pytest.raises(pk.NumericalError):
        pk.solve_scalar(a, a)


class TestStepSizes:
    def test_scalar_values(self):
        mu, tau = pk.step_sizes_scalar(pk.GridSpec(33), 1.0)
        assert mu == pytest.approx(1 / 16384)
        mu, _ = pk.step_sizes_scalar(pk.GridSpec(2), 2.0)
        assert mu == pytest.approx(1 / 32)

    def test_vector_values(self):
        g = pk.TransportGraph(2, [(0, 1)], [1.0])
        mu, nu, tau = pk.step_sizes_vector(pk.GridSpec(33), g, 1.0)
        assert mu == pytest.approx(1 / 32768) and nu == pytest.approx(1 / 8)

    def test_vector_combined_bound_half(self):
        g = pk.triangle_graph((1.0, 2.0, 0.7))
        grid = pk.GridSpec(9)
        for tau in (0.5, 1.0, 4.0):
            mu, nu, _ = pk.step_sizes_vector(grid, g, tau)
            total = tau * mu * 8.0 * (grid.n - 1) ** 2 + tau * nu * pk.lambda_max_graph(g)
            assert total == pytest.approx(0.5)

    def test_matrix_uses_operator_bound(self):
        L = pk.default_lindblad3()
        mu, nu, tau = pk.step_sizes_matrix(pk.GridSpec(9), L, 2.0)
        assert nu == pytest.approx(1 / (4 * 2.0 * pk.lambda_max_L(L)))

    def test_rejects_bad_tau(self):
        with pytest.raises(pk.ValidationError):
            pk.step_sizes_scalar(pk.GridSpec(4), 0.0)


def test_config_validation():
    for bad in (dict(tau=0.0), dict(tol_gap=0), dict(max_iters=0), dict(alpha=-1),
                dict(eps_reg=-0.1), dict(check_every=0)):
        with pytest.raises(pk.ValidationError):
            pk.SolverConfig(**bad)
    with pytest.raises(ValueError):
        pk.SolverConfig(norm_u="l3")
    assert pk.SolverConfig().norm_w == pk.NormFamily.L1
    assert pk.default_tau(64) == 1.0 and pk.default_tau(65) == 3.0


def test_input_validation_before_device(rng):
    d = pk.normalize(pk.VectorDensity(rng.random((5, 5, 2))))
    with pytest.raises(pk.ValidationError):
        pk.solve_vector(d, d, pk.triangle_graph())
    s = pk.normalize(pk.ScalarDensity(rng.random((5, 5))))
    with pytest.raises(pk.ValidationError):
        pk.solve_scalar(s, pk.normalize(pk.ScalarDensity(rng.random((6, 6)))))
    with pytest.raises(pk.UnsupportedNormError):
        pk.solve_scalar(s, s, cfg=pk.SolverConfig(norm_u="l1nuc"))
    v = pk.normalize(pk.VectorDensity(rng.random((5, 5, 3))))
    with pytest.raises(pk.UnsupportedNormError):
        pk.solve_vector(v, v, pk.triangle_graph(), cfg=pk.SolverConfig(norm_w="l12"))
    vals = np.zeros((4, 4, 2, 2), dtype=complex)
    vals[0, 0] = np.eye(2)
    m = pk.normalize(pk.MatrixDensity(vals))
    with pytest.raises(pk.ValidationError):
        pk.solve_matrix(m, m, pk.default_lindblad3())
    m3 = pk.MatrixDensity(np.tile(np.eye(3, dtype=complex) / 75.0, (5, 5, 1, 1)))
    with pytest.raises(pk.UnsupportedNormError):
        pk.solve_matrix(m3, m3, pk.default_lindblad3(),
                        cfg=pk.SolverConfig(eps_reg=0.1, norm_u="l1nuc"))
    with pytest.raises(pk.ValidationError):
        pk.solve_scalar(s, pk.ScalarDensity(s.values), grid=pk.GridSpec(7))


def test_value_type_validation():
    with pytest.raises(pk.ValidationError):
        pk.GridSpec(1)
    with pytest.raises(pk.ValidationError):
        pk.ScalarDensity(-np.ones((3, 3)))
    with pytest.raises(pk.ValidationError):
        pk.MatrixDensity(np.tile(np.array([[1, 1j], [0, 1]]), (3, 3, 1, 1)))
    with pytest.raises(pk.ValidationError):
        pk.FluxField(np.ones((3, 3)), np.zeros((3, 3)))
    with pytest.raises(pk.ValidationError):
        pk.LindbladSet(np.diag([1.0, 2.0, 0.0]).astype(complex)[None])
    with pytest.raises(pk.ValidationError):
        pk.TransportGraph(3, [(0, 1)], [1.0])  # disconnected
    with pytest.raises(pk.ValidationError):
        pk.TransportGraph(2, [(0, 1)], [0.0])


def test_graph_and_lindblad_setup_match_reference_numbers():
    g = pk.triangle_graph()
    assert pk.lambda_max_graph(g) == pytest.approx(3.0)
    D = g.incidence
    assert np.array_equal(D.sum(axis=0), np.zeros(3))
    flipped = pk.TransportGraph(3, g.edges, g.costs, orientations=[-1, -1, -1])
    assert np.array_equal(flipped.coefficients(), -g.coefficients())
    L = pk.default_lindblad3()
    assert L.k == 3 and L.ell == 2
    assert pk.lambda_max_L(L) > 0


@pytest.mark.parametrize("n,P", [(10, 1), (10, 3), (8192, 8), (11586, 2), (23168, 8), (7, 7)])
def test_slab_bounds_cover_grid(n, P):
    b = slab_bounds(n, P)
    assert b[0] == 0 and b[-1] == n and len(b) == P + 1
    sizes = np.diff(b)
    assert sizes.min() >= 1 and sizes.max() - sizes.min() <= 1
    plan = halo_plan(n, P)
    for r, p in enumerate(plan):
        assert p["rows"] == (b[r], b[r + 1])
        if r > 0:
            assert p["top"]["row"] == b[r] - 1 and p["top"]["src"] == r - 1
            assert plan[r - 1]["rows"][1] - 1 == p["top"]["row"]
        if r < P - 1:
            assert p["bottom"]["row"] == b[r + 1] == plan[r + 1]["rows"][0]
    with pytest.raises(ValueError):
        slab_bounds(3, 4)


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the CPU reference arm the driver runs): one
    JSON line with the contract keys on rank 0; other ranks exit 0 silently."""
    import json
    import os
    import subprocess
    import sys

    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
           "--warmup", "1", "--ref-n", "48", "--n", "48"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, check=True)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    # the unmodified reference from baseline/_ref when installed,
    # else the NumPy port
    installed = (ROOT / "baseline" / "_ref" / "otflux").is_dir()
    assert line["cpu_baseline"]["kind"] == ("reference" if installed else "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["config"]["sample_n"] == 48
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env,
                         check=True)
    assert out.stdout.strip() == ""


def test_host_prefault_touches_buffer_without_gpu():
    """otfx_host_prefault is host-only (no device call): it writes one zero
    per 4 KiB page of the buffer and leaves a null/empty request alone."""
    lib = _lib.load()
    a = np.full(3 * 4096 // 8 + 5, 7.0)
    _lib.check(lib.otfx_host_prefault(a.ctypes.data, a.nbytes))
    b = a.view(np.uint8)
    assert b[0] == 0 and b[4096] == 0 and b[8192] == 0
    assert b[1] == np.float64(7.0).tobytes()[1]
    _lib.check(lib.otfx_host_prefault(None, 0))
    with pytest.raises(pk.ValidationError):
        _lib.check(lib.otfx_host_prefault(None, 8))


def test_c_abi_header_compiles_and_links_from_c(tmp_path):
    """include/otfx.h is plain C (C99, -Wall -Werror) and C++, and a C program
    links against libotfx.so and calls into it -- the boundary a cgo / JNI /
    ctypes binding of the reference would use (no device work: the ABI version
    and the last-error string)."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    src = tmp_path / "abi.c"
    src.write_text(
        '#include <stdio.h>\n#include "otfx.h"\n'
        "int main(void) {\n"
        "  otfx_engine_desc d;\n"
        "  (void)d;\n"
        '  printf("%d %s\\n", otfx_abi_version(), otfx_last_error());\n'
        "  return 0;\n}\n")
    lib_dir = str(ROOT / "paper_1712_10279_b200")
    inc = str(ROOT / "include")
    exe = tmp_path / "abi"
    for comp, std in (("gcc", "-std=c99"), ("g++", "-std=c++17")):
        if shutil.which(comp) is None:
            continue
        subprocess.run([comp, std, "-Wall", "-Werror", "-x", "c" if comp == "gcc" else "c++",
                        str(src), f"-I{inc}", f"-L{lib_dir}", "-l:libotfx.so",
                        f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True, capture_output=True,
                       text=True)
        out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
        assert out.split()[0] == str(_lib.load().otfx_abi_version())


def test_c_example_builds(tmp_path):
    """integration/otfx_scalar_example.c (a C-only caller of the engine) builds
    against include/otfx.h and libotfx.so; tests/test_gpu_integration.py runs it."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    lib_dir = str(ROOT / "paper_1712_10279_b200")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", f"-I{ROOT / 'include'}",
                    str(ROOT / "integration" / "otfx_scalar_example.c"), f"-L{lib_dir}",
                    "-l:libotfx.so", f"-Wl,-rpath,{lib_dir}", "-o", str(tmp_path / "ex")],
                   check=True, capture_output=True, text=True)

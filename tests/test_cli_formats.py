"""CPU tests of the CLI front end and its file formats:
OMTF / graph / Lindblad files written by the reference are read identically
and re-written byte for byte; argument and input errors map to the
reference's exit codes without touching a GPU."""

import contextlib
import io
import json
from pathlib import Path

import numpy as np

import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import omtf
from paper_1712_10279_b200.cli import main


def _cli(args):
    """Run the CLI in-process: (exit code, stdout + stderr)."""
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(buf):
        code = main([str(a) for a in args])
    return code, buf.getvalue()

G = Path(__file__).resolve().parent / "golden" / "omtf"


def test_omtf_round_trip_byte_identical(tmp_path):
    for name in ("scalar5", "vector4", "matrix_real6", "matrix_cplx3"):
        d = omtf.read_omtf(G / f"{name}.omtf")
        out = tmp_path / f"{name}.omtf"
        omtf.write_omtf(out, d)
        assert out.read_bytes() == (G / f"{name}.omtf").read_bytes(), name
    assert isinstance(omtf.read_omtf(G / "vector4.omtf"), pk.VectorDensity)
    m = omtf.read_omtf(G / "matrix_cplx3.omtf")
    assert m.values.shape == (3, 3, 2, 2) and np.any(m.values.imag)


def test_graph_and_lindblad_files(tmp_path):
    g = omtf.load_graph(G / "triangle.json")
    assert g.k == 3 and list(g.costs) == [1.0, 2.0, 0.5]
    omtf.save_graph(tmp_path / "g.json", g)
    assert json.loads((tmp_path / "g.json").read_text()) == json.loads((G / "triangle.json").read_text())
    L = omtf.load_lindblad(G / "lindblad3.json")
    assert np.array_equal(L.matrices, pk.default_lindblad3().matrices)
    omtf.save_lindblad(tmp_path / "l.json", L)
    assert json.loads((tmp_path / "l.json").read_text()) == json.loads((G / "lindblad3.json").read_text())


def test_cli_input_errors_exit_2(tmp_path):
    code, output = _cli(["solve", "vector", "--lambda0", str(tmp_path / "missing.omtf"),
                                  "--lambda1", str(G / "vector4.omtf"), "--graph",
                                  str(G / "triangle.json")])
    assert code == 2 and "not found" in output
    code, output = _cli(["solve", "vector", "--lambda0", str(G / "vector4.omtf"),
                                  "--lambda1", str(G / "vector4.omtf")])
    assert code == 2 and "--graph" in output
    code, output = _cli(["solve", "matrix", "--lambda0", str(G / "vector4.omtf"),
                                  "--lambda1", str(G / "vector4.omtf"), "--lindblad",
                                  str(G / "lindblad3.json")])
    assert code == 2
    code, output = _cli(["bench", "--suite", "vector", "--sizes", ",",
                                  "--out", str(tmp_path / "t.csv")])
    assert code == 2


def test_graph_info():
    code, output = _cli(["graph-info", "--graph", str(G / "triangle.json")])
    assert code == 0
    assert "nodes: 3, edges: 3" in output and "lambda_max" in output

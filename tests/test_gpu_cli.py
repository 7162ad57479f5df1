"""GPU tests of the CLI front end: the reference's bench / solve / table2
outputs (S/cli.py:160-357) produced by the B200 engine."""

import csv
import contextlib
import io
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import omtf, synthetic
from paper_1712_10279_b200.cli import main


def _cli(args):
    """Run the CLI in-process: (exit code, stdout + stderr)."""
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(buf):
        code = main([str(a) for a in args])
    return code, buf.getvalue()

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden" / "omtf"


def test_cli_bench_vector_matches_api(tmp_path):
    out = tmp_path / "t.csv"
    code, output = _cli(["bench", "--suite", "vector", "--sizes", "16,24",
                                  "--max-iters", "700", "--out", str(out)])
    assert code == 0, output
    rows = list(csv.DictReader(open(out)))
    assert list(rows[0].keys()) == ["n", "iterations", "time_per_iter_s", "total_time_s", "tau",
                                    "transport_value"]
    l0, l1 = synthetic.rgb_disk_pair(16)
    rep, _ = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), pk.triangle_graph(),
                             cfg=pk.SolverConfig(tau=6.0, max_iters=700, norm_u="l12",
                                                 norm_w="l1"))
    assert int(rows[0]["iterations"]) == rep.iterations
    assert float(rows[0]["transport_value"]) == pytest.approx(rep.transport_value, rel=1e-12)


def test_cli_bench_matrix(tmp_path):
    out = tmp_path / "m.csv"
    code, output = _cli(["bench", "--suite", "matrix", "--sizes", "8",
                                  "--out", str(out)])
    assert code == 0, output
    rows = list(csv.DictReader(open(out)))
    assert float(rows[0]["tau"]) == 10.0 and int(rows[0]["iterations"]) > 0


def test_cli_solve_artifacts(tmp_path):
    l0, l1 = synthetic.rgb_disk_pair(12)
    omtf.write_omtf(tmp_path / "a.omtf", pk.VectorDensity(l0))
    omtf.write_omtf(tmp_path / "b.omtf", pk.VectorDensity(l1))
    args = ["solve", "vector", "--lambda0", str(tmp_path / "a.omtf"), "--lambda1",
            str(tmp_path / "b.omtf"), "--graph", str(G / "triangle.json"), "--tau", "3",
            "--out-metrics", str(tmp_path / "m.json"), "--out-flux", str(tmp_path / "flux"),
            "--out-quiver", str(tmp_path / "q.csv")]
    code, output = _cli(args)
    assert code == 0, output
    m = json.loads((tmp_path / "m.json").read_text())
    assert m["converged"] and m["config"]["tau"] == 3.0 and m["kind"] == "vector"
    assert (tmp_path / "flux.ux.omtf").read_bytes()[:5] == b"OMTF1"
    assert sum(1 for _ in open(tmp_path / "q.csv")) == 1 + 3 * 12 * 12
    # non-convergence -> exit 1
    code, output = _cli(args[:-6] + ["--max-iters", "3"])
    assert code == 1


def test_cli_solve_matrix_from_reference_files(tmp_path):
    m = omtf.read_omtf(G / "matrix_real6.omtf")
    omtf.write_omtf(tmp_path / "b.omtf", pk.MatrixDensity(m.values[:, ::-1].copy()))
    code, output = _cli(["solve", "matrix", "--lambda0", str(G / "matrix_real6.omtf"),
                                  "--lambda1", str(tmp_path / "b.omtf"), "--lindblad",
                                  str(G / "lindblad3.json"), "--tau", "10", "--max-iters", "500"])
    assert code in (0, 1), output
    assert "matrix: value=" in output

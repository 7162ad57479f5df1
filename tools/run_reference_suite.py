"""Run the reference's own test modules against the drop-in on a GPU box:
``otflux`` (and ``otflux.errors``) are aliased to this package before pytest
collects, so every ``of.solve_*`` in those tests runs the CUDA engine.  The
modules come from baseline/_ref/tests_ref (tools/stage_reference_tests.sh; not
committed).  Writes a per-test outcome summary to gpurun_out/ref_suite.json.

    python tools/run_reference_suite.py [test_solver.py test_acceptance.py ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pytest  # noqa: E402

import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200 import errors  # noqa: E402

# The reference's exact LP oracle (S/lp.py, SciPy HiGHS) is a checker the
# tests compare the solver against, not part of the solver: borrow the real
# one from baseline/_ref (converting the value objects it type-checks), then
# alias the name ``otflux`` to the drop-in.
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, REF)
import otflux as _ref  # noqa: E402

for _name in [m for m in sys.modules if m == "otflux" or m.startswith("otflux.")]:
    sys.modules["_reference_" + _name] = sys.modules.pop(_name)
sys.path.remove(REF)


def lp_oracle(lambda0, lambda1, grid=None, graph=None, **kw):
    conv = {pk.ScalarDensity: _ref.ScalarDensity, pk.VectorDensity: _ref.VectorDensity}
    a, b = conv[type(lambda0)](lambda0.values), conv[type(lambda1)](lambda1.values)
    g = None if graph is None else _ref.TransportGraph(graph.k, graph.edges, graph.costs,
                                                         graph.orientations)
    rg = None if grid is None else _ref.GridSpec(grid.n)
    return _ref.lp_oracle(a, b, grid=rg, graph=g, **kw)


pk.lp_oracle = lp_oracle
sys.modules["otflux"] = pk
sys.modules["otflux.errors"] = errors
# the reference's LP / prox oracles import cvxpy, absent here: a stub lets the
# modules import (SURVEY §8(c) ran them the same way); tests that call cvxpy
# fail and are reported as such
if "cvxpy" not in sys.modules:
    import types

    class _Absent(types.ModuleType):
        def __getattr__(self, name):
            if name.startswith("__"):
                raise AttributeError(name)
            return _Absent(f"{self.__name__}.{name}")

        def __call__(self, *a, **k):
            raise ImportError("cvxpy is not installed (reference LP / prox oracle)")

    sys.modules["cvxpy"] = _Absent("cvxpy")

TESTS = os.path.join(ROOT, "baseline", "_ref", "tests_ref")


class Collect:
    def __init__(self):
        self.rows = []

    def pytest_runtest_logreport(self, report):
        if report.when == "call" or report.outcome != "passed":
            msg = ""
            if report.outcome != "passed" and report.longrepr is not None:
                text = str(report.longrepr).strip().splitlines()
                msg = next((ln for ln in reversed(text) if ln.startswith("E ")), text[-1] if text else "")
            self.rows.append({"test": report.nodeid, "when": report.when,
                              "outcome": report.outcome, "reason": msg[:300]})


def main():
    mods = sys.argv[1:] or ["test_solver.py", "test_acceptance.py"]
    c = Collect()
    rc = pytest.main([os.path.join(TESTS, m) for m in mods] +
                     ["-q", "-p", "no:cacheprovider", "--rootdir", TESTS], plugins=[c])
    calls = [r for r in c.rows if r["when"] == "call"]
    summary = {"modules": mods, "rc": int(rc),
               "passed": sum(r["outcome"] == "passed" for r in calls),
               "failed": sum(r["outcome"] == "failed" for r in c.rows),
               "skipped": sum(r["outcome"] == "skipped" for r in c.rows),
               "rows": c.rows}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "ref_suite.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "rows"}))


if __name__ == "__main__":
    main()

"""BASELINE configs[1] ("vector-OMT 3-channel 256x256 to convergence") at the
reference's own termination rule (S/solver.py:294-337).

The reference, run in the build container by tools/make_c2_golden.py on
rgb_disk_pair(256) with the triangle graph, l12/l1, alpha = 1 and the default
tolerances, does NOT meet the gap/feasibility test within 400 000 iterations at
tau = 3 (default_tau(256)) or tau = 1.5 (tests/golden/c2_index.json: 6 175 s
and 6 189 s of CPU).  The CUDA path must reproduce that outcome exactly: the same
400 000 iterations, converged = False, all 4 001 history rows and the final
u, w, phi within the north star's 1e-10 relative bound (in practice the vector
path is bit-identical, so the state is also checked for equality where it is).
"""

import json

import numpy as np
import pytest

import gpu_util as g
import paper_1712_10279_b200 as pk
from golden_util import GOLDEN
from paper_1712_10279_b200 import synthetic

pytestmark = pytest.mark.gpu

_INDEX = json.loads((GOLDEN / "c2_index.json").read_text())


@pytest.mark.parametrize("name", sorted(_INDEX))
def test_c2_run_matches_reference(name):
    meta = _INDEX[name]
    l0, l1 = synthetic.rgb_disk_pair(256)
    import hashlib

    for key, arr in (("l0", l0), ("l1", l1)):
        assert hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest() == meta["sha256"][key]
    with np.load(GOLDEN / f"{name}.npz") as z:
        ref = {k: z[k] for k in z.files}
    cfg = pk.SolverConfig(tau=meta["tau"], norm_u=meta["norm_u"], norm_w=meta["norm_w"],
                          alpha=meta["alpha"], tol_gap=meta["tol_gap"], tol_feas=meta["tol_feas"],
                          max_iters=meta["max_iters"], check_every=meta["check_every"])
    rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), pk.triangle_graph(),
                              cfg=cfg)
    assert rep.iterations == meta["iterations"] == int(ref["meta"][0])
    assert rep.converged == meta["converged"] == bool(ref["meta"][1])
    assert abs(rep.transport_value - meta["transport_value"]) <= 1e-10 * abs(meta["transport_value"])
    g.hist_close(g.hist_array(rep), ref["history"], 1e-10)
    for got, want in ((st.u.ux, ref["ux"]), (st.u.uy, ref["uy"]), (st.phi, ref["phi"]),
                      (st.w.values, ref["w"])):
        assert got.shape == want.shape
        assert g.rel_err(got, want) <= 1e-10

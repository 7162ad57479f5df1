"""Pin the CPU oracle to the reference: replay every golden fixture through
oracle.pdhg and compare with what the reference produced (tools/make_golden.py).

The oracle mirrors the reference's NumPy operation order, so iterates and
history must agree to the last few ulps (we allow 1e-12 relative to absorb
BLAS summation-order differences between machines)."""

import hashlib

import numpy as np
import pytest

import golden_util as gu
from oracle.pdhg import oracle_run

FAST_SUMMARY = ["S_vec32_conv"]


def _rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) / den if a.size else 0.0


# the BASELINE-size matrix fixtures take minutes through the NumPy oracle; the
# GPU tests compare the CUDA path with them directly
SLOW_FULL = {"B_matr256", "B_matc128"}


@pytest.mark.parametrize("name", [c for c in gu.full_cases() if c not in SLOW_FULL])
def test_oracle_matches_reference(name):
    meta, arrs = gu.load(name)
    eng = gu.oracle_engine(meta, arrs)
    conv, it, hist = oracle_run(eng, **gu.run_cfg(meta))
    assert it == meta["iterations"]
    hist = np.array(hist)
    ref = arrs["history"]
    assert hist.shape == ref.shape
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(hist), fin)
    assert _rel(hist[fin], ref[fin]) < 1e-12
    assert _rel(eng.u[:, :, 0], arrs["ux"]) < 1e-12
    assert _rel(eng.u[:, :, 1], arrs["uy"]) < 1e-12
    assert _rel(eng.phi, arrs["phi"]) < 1e-12
    if "w" in arrs:
        assert _rel(eng.w, arrs["w"]) < 1e-12


@pytest.mark.parametrize("name", FAST_SUMMARY)
def test_oracle_summary(name):
    from paper_1712_10279_b200 import synthetic

    meta, arrs = gu.load(name)
    l0, l1 = synthetic.rgb_disk_pair(32)
    eng = gu.oracle_engine(meta, arrs, l0=l0, l1=l1)
    conv, it, hist = oracle_run(eng, **gu.run_cfg(meta))
    assert it == meta["iterations"]
    assert conv == meta["converged"]
    np.testing.assert_allclose(hist[-1][1], meta["transport_value"], rtol=1e-12)


def test_generators_match_reference_bytes():
    """The package's synthetic generators reproduce the reference generators
    bit-for-bit (sha256 of the marginals recorded by tools/make_golden.py)."""
    from paper_1712_10279_b200 import synthetic

    idx = gu.index()
    made = {
        "S_vec256": synthetic.rgb_disk_pair(256),
        "S_vec32_conv": synthetic.rgb_disk_pair(32),
        "S_matr256": synthetic.matrix_blob_fixtures(256)[:2],
        "S_matc128": synthetic.blob_pair_k2(128),
        "S_sca33_dirac_conv": synthetic.dirac_pair(33, (8, 16), (24, 16)),
    }
    for name, (a, b) in made.items():
        for arr, key in ((a, "l0"), (b, "l1")):
            h = hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()
            assert h == idx[name]["sha256"][key], (name, key)


def test_blas_rounding_model_of_graph_operators():
    """The CUDA graph operators reproduce NumPy/OpenBLAS's fused multiply-add
    order for S/graph.py:105-123 (tools/blas_order.py); pin the model on this
    host's BLAS."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    import blas_order

    assert blas_order.main(samples=40) == 0


def test_einsum_summation_model_of_block_norms():
    """The CUDA block norms reproduce np.einsum's summation order for
    S/shrink.py:88-104 (tools/einsum_order.py); pin the model here."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    import einsum_order

    assert einsum_order.main(cells=100) == 0

"""Sweep time of the TMA kernel for several payloads / sizes (engine events),
used to pick the CTA row split (OTFX_MIN_WAVES)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200 import synthetic  # noqa: E402
from paper_1712_10279_b200.solver import build_engine  # noqa: E402

PEAK = 6541.5e9
cases = [("vec f64 8192", "vector", 8192, "f64", 216), ("vec f64 4096", "vector", 4096, "f64", 216),
         ("vec f32 4096", "vector", 4096, "f32", 108), ("vec f32 8192", "vector", 8192, "f32", 108),
         ("vec f64 2048", "vector", 2048, "f64", 216),
         ("C4 2048", "matrix_real", 2048, "f64", 432), ("C3 2048", "matrix_cplx", 2048, "f64", 352),
         ("C4 4096", "matrix_real", 4096, "f64", 432)]
out = {}
for name, kind, n, prec, bpc in cases:
    if kind == "vector":
        l0, l1 = synthetic.rgb_disk_pair(n)
        cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1")
        eng = build_engine("vector", n, cfg, graph=pk.triangle_graph(), precision=prec)
    elif kind == "matrix_real":
        l0, l1 = synthetic.matrix_blob_fixtures(n)[:2]
        cfg = pk.SolverConfig(tau=30.0, norm_u="l2", norm_w="l1")
        eng = build_engine("matrix", n, cfg, lindblad=pk.default_lindblad3(), complex_path=False)
    else:
        l0, l1 = synthetic.blob_pair_k2(n)
        cfg = pk.SolverConfig(tau=30.0, norm_u="l1nuc", norm_w="l1nuc")
        eng = build_engine("matrix", n, cfg, lindblad=pk.lindblad_pair_k2(), complex_path=True)
    eng.set_marginals(l0, l1)
    eng.run(1e-300, 1e-300, 200, 100)
    eng.timing(1)
    eng.run(1e-300, 1e-300, 300, 100)
    ms, it = eng.timing(0)
    inf = eng.info()
    eng.close()
    per = ms / it * 1e-3
    out[name] = dict(frac=round(bpc * n * n / per / PEAK, 4), R=inf["tile_rows"], gy=inf["grid_y"],
                     gx=inf["grid_x"])
print(json.dumps(out))

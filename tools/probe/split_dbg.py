"""Probe: run the U/W-split sweep variants one at a time (plain, check,
dual via run) and report which one fails."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import synthetic
from paper_1712_10279_b200.solver import build_engine
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
what = sys.argv[2] if len(sys.argv) > 2 else "plain"
l0, l1 = synthetic.matrix_blob_fixtures(n)[:2]
cfg = pk.SolverConfig(tau=30.0, norm_u="l2", norm_w="l1")
eng = build_engine("matrix", n, cfg, lindblad=pk.default_lindblad3(), complex_path=True)
inf = eng.info()
print({k: inf[k] for k in ("tile_cols", "tile_rows", "grid_x", "grid_y", "tma_stages", "smem_bytes", "regs_plain")}, flush=True)
eng.set_marginals(l0, l1)
if what == "plain":
    eng.sweep(check=False); eng.sync(); print("plain sweep ok", flush=True)
elif what == "check":
    eng.sweep(check=True); eng.sync(); print("check sweep ok", flush=True)
else:
    print(eng.run(1e-300, 1e-300, 250, 100)[1], flush=True)
eng.close()

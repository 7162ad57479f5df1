"""One on-chip cluster solve (vector 3-channel, BASELINE C1 shape) for ncu."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200 import synthetic  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
l0, l1 = synthetic.rgb_disk_pair(n)
cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=1.0, tol_gap=1e-300,
                      tol_feas=1e-300, max_iters=iters, check_every=100)
rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), pk.triangle_graph(), cfg=cfg)
print(n, iters, rep.iterations, rep.transport_value, np.linalg.norm(st.phi))

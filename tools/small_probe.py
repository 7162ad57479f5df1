"""One BASELINE C2-sized solve (vector 3-channel 256^2, 400 iterations) for an ncu launch list of the small-grid register sweep."""
import sys
sys.path.insert(0, ".")
import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import synthetic
from paper_1712_10279_b200.solver import build_engine
n = 256
l0, l1 = synthetic.rgb_disk_pair(n)
cfg = pk.SolverConfig(tau=3.0, norm_u="l12", norm_w="l1", tol_gap=1e-300, tol_feas=1e-300,
                      max_iters=400, check_every=100)
eng = build_engine("vector", n, cfg, graph=pk.triangle_graph())
eng.set_marginals(l0, l1)
eng.run(1e-300, 1e-300, 400, 100)
print(eng.info())
eng.close()

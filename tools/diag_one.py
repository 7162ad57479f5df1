import sys
sys.path.insert(0, ".")
import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import synthetic
n = int(sys.argv[1]); prec = sys.argv[2]
l0, l1 = synthetic.rgb_disk_pair(n)
cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.3, tol_gap=1e-300,
                      tol_feas=1e-300, max_iters=4, check_every=2)
rep, st = pk.solve_vector(pk.VectorDensity(l0), pk.VectorDensity(l1), pk.triangle_graph(),
                          cfg=cfg, precision=prec)
print("OK", rep.transport_value)

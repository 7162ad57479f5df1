"""One matrix-payload run for ncu: C3 family (2x2 complex, l1nuc/l1nuc) or C4
family (3x3 real symmetric, l2/l1) at n x n, fp64."""
import sys

sys.path.insert(0, ".")
import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200 import synthetic  # noqa: E402
from paper_1712_10279_b200.solver import build_engine  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
if fam == "c3":
    l0, l1 = synthetic.blob_pair_k2(n)
    lind, norms, cplx = pk.lindblad_pair_k2(), ("l1nuc", "l1nuc"), True
elif fam == "c3k3":
    l0, l1 = synthetic.matrix_blob_fixtures(n)[:2]
    lind, norms, cplx = pk.default_lindblad3(), ("l1nuc", "l1nuc"), True
else:
    l0, l1 = synthetic.matrix_blob_fixtures(n)[:2]
    lind, norms, cplx = pk.default_lindblad3(), ("l2", "l1"), False
cfg = pk.SolverConfig(tau=30.0, norm_u=norms[0], norm_w=norms[1])
eng = build_engine("matrix", n, cfg, lindblad=lind, complex_path=cplx)
eng.set_marginals(l0, l1)
eng.step(iters)
print(fam, n, iters, eng.evaluate(), eng.info())
eng.close()

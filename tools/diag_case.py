import sys, os, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1712_10279_b200 as pk
from oracle import pdhg
rng = np.random.default_rng(12345)
def rpsd(n,k):
    a = rng.normal(size=(n, n, k, k)) + 1j * rng.normal(size=(n, n, k, k))
    p = a @ np.conj(np.swapaxes(a, -1, -2)); return pk.MatrixDensity(p / np.sum(np.real(np.trace(p, axis1=2, axis2=3))))
k, ell, n = int(sys.argv[1]), int(sys.argv[2]), 10
a = rpsd(n,k); b = rpsd(n,k)
a = pk.MatrixDensity(np.real(a.values)+0j); b = pk.MatrixDensity(np.real(b.values)+0j)
m = rng.normal(size=(ell, k, k)); mats = 0.5*(m+np.swapaxes(m,-1,-2))+0j
lind = pk.LindbladSet(mats)
nu, nw = sys.argv[3], sys.argv[4]
cfg = pk.SolverConfig(tau=4.0, norm_u=nu, norm_w=nw, alpha=0.5, tol_gap=1e-300, tol_feas=1e-300, max_iters=90, check_every=30)
rep, st = pk.solve_matrix(a, b, lind, cfg=cfg)
diff = a.values - b.values
eng = pdhg.OracleEngine("matrix", np.ascontiguousarray(diff.real), n, 4.0, norm_u=nu, norm_w=nw, alpha=0.5, chan=np.ascontiguousarray(np.real(lind.matrices)), lam_chan=pk.lambda_max_L(lind), dtype=np.float64)
_, _, hist = pdhg.oracle_run(eng, 1e-300, 1e-300, 90, 30)
print("gpu", [(h.iteration, h.primal, h.dual, h.feas_residual, h.residual) for h in rep.history])
print("cpu", [h[:3]+h[4:] for h in hist])
print("phi err", np.max(np.abs(st.phi-eng.phi)), np.max(np.abs(eng.phi)), "w err", np.max(np.abs(st.w.values.real - eng.w)), "u err", np.max(np.abs(st.u.ux-eng.u[:,:,0])))

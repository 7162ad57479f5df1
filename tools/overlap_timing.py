"""Cost of the overlapped halo schedule on one GPU: P row slabs of an n x n
vector grid run by the local group loop (edge bands + exchange on the
high-priority stream, interior concurrently) vs the serial schedule vs one
engine.  Device time per iteration from CUDA events."""
import json
import os
import subprocess
import sys

SNIP = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import synthetic
from paper_1712_10279_b200.solver import build_engine, run_local
n, P, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
l0, l1 = synthetic.rgb_disk_pair(n)
cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", tol_gap=1e-300, tol_feas=1e-300,
                      max_iters=iters, check_every=100)
s = torch.cuda.Stream()
bounds = np.linspace(0, n, P + 1).astype(int)
engs = [build_engine("vector", n, cfg, graph=pk.triangle_graph(), rows=(bounds[r], bounds[r + 1]),
                     stream=s.cuda_stream) for r in range(P)]
for r, e in enumerate(engs):
    e.set_marginals(l0[bounds[r]:bounds[r + 1]], l1[bounds[r]:bounds[r + 1]])
run_local(engs, 1e-300, 1e-300, 100, 100)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
if P == 1:
    engs[0].run(1e-300, 1e-300, iters, 100)
else:
    run_local(engs, 1e-300, 1e-300, iters, 100)
b.record(s)
torch.cuda.synchronize()
print(json.dumps(dict(n=n, P=P, ms_per_iter=a.elapsed_time(b) / iters,
                      overlap=engs[0].info()["halo_overlap"])))
'''
for P, env in [(1, {}), (2, {"OTFX_OVERLAP": "0"}), (2, {"OTFX_OVERLAP": "1"}),
               (4, {"OTFX_OVERLAP": "0"}), (4, {"OTFX_OVERLAP": "1"})]:
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SNIP, "8192", str(P), "300"], env=e,
                       capture_output=True, text=True, timeout=600)
    print(json.dumps(env), (r.stdout.strip().splitlines() or [r.stderr[-400:]])[-1], flush=True)

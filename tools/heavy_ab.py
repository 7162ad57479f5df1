"""Timing of the heavy complex-Hermitian sweep: 3x3 complex payloads (default
Lindblad pair), l1nuc/l1nuc and l2/l1, fp64, at 1024^2 and 2048^2.  Prints
ms/iteration from the engine's CUDA events, the HBM roofline fraction
(compulsory bytes (7 + 2 ell) K^2 * 8 per cell) and a digest of the iterate
after 250 iterations (for A/B runs of kernel variants: equal digests = equal
iterates).  Round-2 A/B of a U/W warp-split variant:
profiles/r02_heavy_split_ab.md."""
import json
import os
import subprocess
import sys

SNIP = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import synthetic
from paper_1712_10279_b200.solver import build_engine
n, nu, nw, iters = int(sys.argv[1]), sys.argv[2], sys.argv[3], int(sys.argv[4])
l0, l1 = synthetic.matrix_blob_fixtures(n)[:2]
lind = pk.default_lindblad3()
cfg = pk.SolverConfig(tau=30.0, norm_u=nu, norm_w=nw)
s = torch.cuda.Stream()
eng = build_engine("matrix", n, cfg, lindblad=lind, complex_path=True, stream=s.cuda_stream)
eng.set_marginals(l0, l1)
h, it, conv, wall = eng.run(1e-300, 1e-300, 250, 100)
st = eng.get_state()
import hashlib
dig = hashlib.sha256(b"".join(np.ascontiguousarray(a).tobytes() for a in st)).hexdigest()[:16]
eng.timing(1)
eng.run(1e-300, 1e-300, iters, 100)
ms, sw = eng.timing(0)
info = eng.info()
eng.close()
per = ms / sw
words = (7 + 2 * 2) * 9
print(json.dumps(dict(n=n, norms=f"{nu}/{nw}", ms_per_iter=per, frac=words * 8 * n * n / (per * 1e-3) / 6538.6e9,
                      regs=[info["regs_plain"], info["regs_check"]], tile=info["tile_cols"],
                      grid=[info["grid_x"], info["grid_y"]], stages=info["tma_stages"],
                      smem=info["smem_bytes"], digest=dig, primal=h[-1].primal)))
'''
for n in (1024, 2048):
    for norms in (("l1nuc", "l1nuc"), ("l2", "l1")):
        r = subprocess.run([sys.executable, "-c", SNIP, str(n), *norms, "400"],
                           env=dict(os.environ), capture_output=True, text=True, timeout=900)
        print((r.stdout.strip().splitlines() or [r.stderr[-600:]])[-1], flush=True)

"""Device time per iteration and achieved algorithmic bandwidth of the matrix
payloads at grid sizes where HBM (not launch latency) should bound them."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200 import synthetic  # noqa: E402
from paper_1712_10279_b200.solver import build_engine  # noqa: E402

PEAK = 6541.5e9
cases = [
    ("C4 3x3 real l2/l1", 2048, lambda n: synthetic.matrix_blob_fixtures(n)[:2], pk.default_lindblad3(),
     ("l2", "l1"), False, lambda: (7 * 6 + 2 * 2 * 3)),
    ("C3 2x2 cplx l1nuc", 2048, synthetic.blob_pair_k2, pk.lindblad_pair_k2(), ("l1nuc", "l1nuc"),
     True, lambda: (7 + 2 * 2) * 4),
    ("3x3 cplx l1nuc", 1024, lambda n: synthetic.matrix_blob_fixtures(n)[:2], pk.default_lindblad3(),
     ("l1nuc", "l1nuc"), True, lambda: (7 + 2 * 2) * 9),
    ("3x3 cplx l2/l1", 1024, lambda n: synthetic.matrix_blob_fixtures(n)[:2], pk.default_lindblad3(),
     ("l2", "l1"), True, lambda: (7 + 2 * 2) * 9),
]
for name, n, gen, lind, norms, cplx, words in cases:
    l0, l1 = gen(n)
    cfg = pk.SolverConfig(tau=30.0, norm_u=norms[0], norm_w=norms[1], tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=200, check_every=100)
    s = torch.cuda.Stream()
    eng = build_engine("matrix", n, cfg, lindblad=lind, complex_path=cplx, stream=s.cuda_stream)
    eng.set_marginals(l0, l1)
    eng.run(1e-300, 1e-300, 200, 100)
    eng.timing(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    eng.run(1e-300, 1e-300, 400, 100)
    b.record(s)
    torch.cuda.synchronize()
    pms, pit = eng.timing(0)
    inf = eng.info()
    eng.close()
    per = pms / pit * 1e-3
    balg = words() * 8 * n * n
    print(json.dumps(dict(case=name, n=n, ms_per_iter=per * 1e3, step_ms=a.elapsed_time(b) / 400,
                          gbs=balg / per / 1e9, frac=balg / per / PEAK, tma=inf["tma_stages"],
                          regs=[inf["regs_plain"], inf["regs_check"]], smem=inf["smem_bytes"])),
          flush=True)

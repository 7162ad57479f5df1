"""4x4 complex-Hermitian payload (two qubits), l2/l1 and l1nuc, ell = 2 and 4,
fp64: ms per iteration (engine CUDA events), roofline fraction, sweep path."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200.solver import build_engine  # noqa: E402

PEAK = 6538.6e9
rng = np.random.default_rng(0)
n, K = int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 4
m = rng.normal(size=(n, n, K, K)) + 1j * rng.normal(size=(n, n, K, K))
m = m @ np.conj(np.swapaxes(m, -1, -2))
m /= np.real(np.trace(m, axis1=2, axis2=3)).sum()
for ell in (2, 4):
    a = rng.normal(size=(ell, K, K)) + 1j * rng.normal(size=(ell, K, K))
    lind = pk.LindbladSet(0.5 * (a + np.conj(np.swapaxes(a, -1, -2))))
    for norms in (("l2", "l1"), ("l1nuc", "l1nuc")):
        cfg = pk.SolverConfig(tau=10.0, norm_u=norms[0], norm_w=norms[1])
        s = torch.cuda.Stream()
        eng = build_engine("matrix", n, cfg, lindblad=lind, complex_path=True, stream=s.cuda_stream)
        eng.set_marginals(m, m[::-1].copy())
        eng.run(1e-300, 1e-300, 60, 30)
        eng.timing(1)
        eng.run(1e-300, 1e-300, 120, 60)
        ms, sw = eng.timing(0)
        per = ms / sw
        inf = eng.info()
        eng.close()
        byt = (7 + 2 * ell) * K * K * 8
        print(json.dumps(dict(ell=ell, norms="/".join(norms), n=n, ms=round(per, 4),
                              frac=round(byt * n * n / (per * 1e-3) / PEAK, 3),
                              tma=inf["tma_stages"], tile=inf["tile_cols"])))

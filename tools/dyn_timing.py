"""Device time per iteration of the runtime-size payloads (csrc/dyn.cuh) next
to a compiled payload of similar width: vector k = 8 (compiled) vs k = 9, 12,
16 (runtime), matrix 4x4 complex l = 4 (compiled) vs l = 6 (runtime), fp64,
engine CUDA events over plain iterations; roofline vs compulsory bytes."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200.solver import build_engine  # noqa: E402

PEAK = 6538.6e9
out = []
rng = np.random.default_rng(0)
for k in (8, 9, 12, 16):
    n = 1024
    g = pk.TransportGraph(k, [(c, c + 1) for c in range(k - 1)], np.ones(k - 1))
    cfg = pk.SolverConfig(tau=3.0, norm_u="l12", norm_w="l1", alpha=0.1)
    s = torch.cuda.Stream()
    eng = build_engine("vector", n, cfg, graph=g, stream=s.cuda_stream)
    v = rng.random((n, n, k)) + 0.1
    v /= v.sum()
    w = rng.random((n, n, k)) + 0.1
    w /= w.sum()
    eng.set_marginals(v, w)
    eng.run(1e-300, 1e-300, 200, 100)
    eng.timing(1)
    eng.run(1e-300, 1e-300, 400, 100)
    ms, sw = eng.timing(0)
    per = ms / sw
    ell = k - 1
    byt = (7 * k + 2 * ell) * 8
    out.append(dict(payload=f"vector k={k} chain", n=n, ms_per_iter=round(per, 4),
                    frac=round(byt * n * n / (per * 1e-3) / PEAK, 3), runtime_size=k > 8))
    eng.close()
for ell in (4, 6):
    n, K = 512, 4
    a = rng.normal(size=(ell, K, K)) + 1j * rng.normal(size=(ell, K, K))
    lind = pk.LindbladSet(0.5 * (a + np.conj(np.swapaxes(a, -1, -2))))
    cfg = pk.SolverConfig(tau=10.0, norm_u="l2", norm_w="l1")
    s = torch.cuda.Stream()
    eng = build_engine("matrix", n, cfg, lindblad=lind, complex_path=True, stream=s.cuda_stream)
    m = rng.normal(size=(n, n, K, K)) + 1j * rng.normal(size=(n, n, K, K))
    m = m @ np.conj(np.swapaxes(m, -1, -2))
    m /= np.real(np.trace(m, axis1=2, axis2=3)).sum()
    eng.set_marginals(m, m[::-1].copy())
    eng.run(1e-300, 1e-300, 100, 50)
    eng.timing(1)
    eng.run(1e-300, 1e-300, 200, 100)
    ms, sw = eng.timing(0)
    per = ms / sw
    byt = (7 + 2 * ell) * K * K * 8
    out.append(dict(payload=f"matrix 4x4 complex l2/l1 ell={ell}", n=n, ms_per_iter=round(per, 4),
                    frac=round(byt * n * n / (per * 1e-3) / PEAK, 3), runtime_size=ell > 4))
    eng.close()
print(json.dumps(out, indent=1))

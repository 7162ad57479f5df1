"""Cost of the host round trip per check on small grids: the same number of
iterations of vector 3-channel 256^2 (BASELINE C2 grid) with check_every = 100
(the reference's cadence) vs one check at the end; CUDA events on the engine
stream around eng.run (the check syncs are inside)."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200 import synthetic  # noqa: E402
from paper_1712_10279_b200.solver import build_engine  # noqa: E402

out = {}
for n in (128, 256):
    l0, l1 = synthetic.rgb_disk_pair(n)
    cfg = pk.SolverConfig(tau=3.0, norm_u="l12", norm_w="l1")
    s = torch.cuda.Stream()
    eng = build_engine("vector", n, cfg, graph=pk.triangle_graph(), stream=s.cuda_stream)
    eng.set_marginals(l0, l1)
    iters = 20000
    for ce in (100, iters):
        eng.run(1e-300, 1e-300, 2 * ce if ce < iters else iters, ce)  # warm-up / graph capture
        eng.zero_state()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        eng.run(1e-300, 1e-300, iters, ce)
        b.record(s)
        torch.cuda.synchronize()
        out[f"{n}_ce{ce}"] = a.elapsed_time(b) * 1e3 / iters
    eng.close()
print(json.dumps({k: round(v, 3) for k, v in out.items()}))

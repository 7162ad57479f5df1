"""Per-iteration device time of the plain-iteration CUDA graphs vs the number
of sweeps captured per graph (eng.step(count) launches one graph of `count`
sweeps), small grids where launch overhead matters; vector 3-channel fp64."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200 import synthetic  # noqa: E402
from paper_1712_10279_b200.solver import build_engine  # noqa: E402

out = {}
for n in [int(a) for a in (sys.argv[1:] or ["128", "256"])]:
    l0, l1 = synthetic.rgb_disk_pair(n)
    cfg = pk.SolverConfig(tau=3.0, norm_u="l12", norm_w="l1")
    s = torch.cuda.Stream()
    eng = build_engine("vector", n, cfg, graph=pk.triangle_graph(), stream=s.cuda_stream)
    eng.set_marginals(l0, l1)
    total = 12000
    for count in (4, 8, 16, 32, 64, 100, 200, 500, 2000):
        reps = total // count
        eng.step(count)
        eng.step(count)  # both ping-pong parities captured
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            eng.step(count)
        b.record(s)
        torch.cuda.synchronize()
        out[f"{n}_{count}"] = round(a.elapsed_time(b) * 1e3 / (reps * count), 3)
    eng.close()
print(json.dumps(out))

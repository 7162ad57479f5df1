"""Host<->device state transfer timing of one 8192^2 vector engine (fp64):
set_marginals (H2D 3.2 GB) and get_state (D2H 6.4 GB), best of 3."""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1712_10279_b200 as pk  # noqa: E402
from paper_1712_10279_b200 import synthetic  # noqa: E402
from paper_1712_10279_b200.solver import build_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
l0, l1 = synthetic.rgb_disk_pair(n)
cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1")
eng = build_engine("vector", n, cfg, graph=pk.triangle_graph())
up, down, down_pre = [], [], []
for _ in range(3):
    t = time.perf_counter(); eng.set_marginals(l0, l1); eng.sync(); up.append(time.perf_counter() - t)
    t = time.perf_counter(); st = eng.get_state(); down.append(time.perf_counter() - t)
    del st
    out = eng.get_state()  # reuse already-faulted arrays
    t = time.perf_counter(); eng._lib.otfx_engine_get_state(eng._h, *[a.ctypes.data if a is not None else None for a in out]); down_pre.append(time.perf_counter() - t)
eng.close()
print(f"threads={os.environ.get('OMP_NUM_THREADS', 'default')} cpus={os.cpu_count()} "
      f"upload {min(up):.4f} s  download(fresh arrays) {min(down):.4f} s  "
      f"download(faulted arrays) {min(down_pre):.4f} s")

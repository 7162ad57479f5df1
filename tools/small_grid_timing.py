"""Device time per iteration of small-grid solves (BASELINE C1/C2 sizes) under
the engine's tuning knobs; used to pick the small-grid launch geometry."""
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
out = {}
import os
sizes = [int(x) for x in os.environ.get("SIZES", "48,64,80,128").split(",")]
for n, iters in ((m, 2000) for m in sizes):
    l0, l1 = synthetic.rgb_disk_pair(n)
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", tol_gap=1e-300, tol_feas=1e-300,
                          max_iters=iters, check_every=100)
    s = torch.cuda.Stream()
    eng = build_engine("vector", n, cfg, graph=pk.triangle_graph(), stream=s.cuda_stream)
    eng.set_marginals(l0, l1)
    eng.run(1e-300, 1e-300, 300, 100)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); eng.run(1e-300, 1e-300, iters, 100); b.record(s); torch.cuda.synchronize()
    inf = eng.info()
    out[n] = dict(us_per_iter=1e3 * a.elapsed_time(b) / iters, tile=[inf["tile_cols"], inf["tile_rows"]],
                  grid=[inf["grid_x"], inf["grid_y"]], cluster=inf["cluster_ctas"])
    eng.close()
print(json.dumps(out))
'''
variants = [json.loads(a) for a in sys.argv[1:]] or [{}, {"OTFX_CLUSTER_CTAS": "8"},
                                                      {"OTFX_CLUSTER": "0"}]
for env in variants:
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SNIP], env=e, capture_output=True, text=True,
                       timeout=300)
    print(json.dumps(env), (r.stdout.strip().splitlines() or [r.stderr[-300:]])[-1], flush=True)

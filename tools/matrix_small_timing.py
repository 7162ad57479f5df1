"""Device time per iteration of the BASELINE matrix configs at their own sizes
(C3: 2x2 complex l1nuc 128^2; C4: 3x3 real l2/l1 256^2) under the engine's
geometry knobs; used to pick the small-grid launch geometry."""
import json
import os
import subprocess
import sys

SNIP = r'''
import sys, json, torch
sys.path.insert(0, ".")
import paper_1712_10279_b200 as pk
from paper_1712_10279_b200 import synthetic
from paper_1712_10279_b200.solver import build_engine
out = {}
cases = {"C3": (128, synthetic.blob_pair_k2, pk.lindblad_pair_k2(), ("l1nuc", "l1nuc"), True, 300),
         "C4": (256, lambda n: synthetic.matrix_blob_fixtures(n)[:2], pk.default_lindblad3(),
                ("l2", "l1"), False, 500)}
for name, (n, gen, lind, norms, cplx, iters) in cases.items():
    l0, l1 = gen(n)
    cfg = pk.SolverConfig(tau=30.0, norm_u=norms[0], norm_w=norms[1], tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=iters, check_every=100)
    s = torch.cuda.Stream()
    eng = build_engine("matrix", n, cfg, lindblad=lind, complex_path=cplx, stream=s.cuda_stream)
    eng.set_marginals(l0, l1)
    eng.run(1e-300, 1e-300, 200, 100)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); eng.run(1e-300, 1e-300, iters, 100); b.record(s); torch.cuda.synchronize()
    inf = eng.info()
    out[name] = dict(us_per_iter=round(1e3 * a.elapsed_time(b) / iters, 2),
                     tile=[inf["tile_cols"], inf["tile_rows"]], grid=[inf["grid_x"], inf["grid_y"]],
                     tma=inf["tma_stages"], regs=[inf["regs_plain"], inf["regs_check"]])
    eng.close()
print(json.dumps(out))
'''
variants = [json.loads(a) for a in sys.argv[1:]] or [{}, {"OTFX_TILE_COLS": "64"}, {"OTFX_TILE_COLS": "32"}, {"OTFX_TILE_ROWS": "2"},
            {"OTFX_TMA": "1"}, {"OTFX_TMA": "1", "OTFX_TILE_ROWS": "2"},
            {"OTFX_TMA": "1", "OTFX_TILE_ROWS": "4"}, {"OTFX_GRAPHS": "0"}]
for env in variants:
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SNIP], env=e, capture_output=True, text=True,
                       timeout=300)
    print(json.dumps(env), (r.stdout.strip().splitlines() or [r.stderr[-300:]])[-1], flush=True)

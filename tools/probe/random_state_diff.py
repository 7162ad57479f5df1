"""Probe: where does a random-state step differ from the oracle? (diagnostic)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1712_10279_b200 as pk
from oracle import pdhg
from paper_1712_10279_b200 import synthetic
from paper_1712_10279_b200.solver import build_engine

for n in [int(a) for a in sys.argv[1:]] or [64, 300]:
    rng = np.random.default_rng(n)
    l0, l1 = synthetic.rgb_disk_pair(n)
    graph = pk.triangle_graph((1.0, 1.3, 0.8))
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.3)
    for env in ({}, {"OTFX_TMA": "0", "OTFX_CLUSTER": "0"}, {"OTFX_TMA": "1"}):
        import os
        os.environ.pop("OTFX_TMA", None); os.environ.pop("OTFX_CLUSTER", None)
        os.environ.update(env)
        eng = build_engine("vector", n, cfg, graph=graph)
        eng.set_marginals(l0, l1)
        phi = rng.random((n, n, 3)) if True else None
        rng = np.random.default_rng(n)
        phi = rng.random((n, n, 3))
        u = rng.normal(scale=eng.mu * n, size=(n, n, 2, 3))
        u[-1, :, 0] = 0.0
        u[:, -1, 1] = 0.0
        w = rng.normal(scale=eng.nu, size=(n, n, 3))
        eng.set_state(u[:, :, 0], u[:, :, 1], w, phi)
        ux0, uy0, w0, phi0 = eng.get_state()
        print(n, env, "roundtrip equal:", np.array_equal(ux0, u[:, :, 0]), np.array_equal(uy0, u[:, :, 1]),
              np.array_equal(w0, w), np.array_equal(phi0, phi))
        eng.step(1)
        ux, uy, w1, phi1 = eng.get_state()
        eng.close()
        ora = pdhg.OracleEngine("vector", l0 - l1, n, 6.0, norm_u="l12", norm_w="l1", alpha=0.3,
                                chan=graph.coefficients(), lam_chan=pk.lambda_max_graph(graph))
        ora.u, ora.w, ora.phi = u.copy(), w.copy(), phi.copy()
        ora.step()
        for name, a, b in (("ux", ux, ora.u[:, :, 0]), ("uy", uy, ora.u[:, :, 1]), ("w", w1, ora.w),
                           ("phi", phi1, ora.phi)):
            d = a != b
            idx = np.argwhere(d)
            rel = np.max(np.abs(a - b)) / np.max(np.abs(b))
            print(f"  {name}: {d.sum()} differ of {d.size}, max rel {rel:.3e}",
                  idx[:5].tolist() if len(idx) else "")
            if len(idx):
                i = tuple(idx[0])
                print("    got", repr(a[i]), "want", repr(b[i]))

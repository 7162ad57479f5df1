"""Generate the golden parity fixtures under tests/golden/ from the REFERENCE.

Run in the build container (the reference is importable there, not on the GPU
box):

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py

Every case drives the reference's public entry points (``solve_scalar``,
``solve_vector``, ``solve_matrix`` -- S/solver.py:359-435) for an exact
iteration count (tolerances 1e-300, ``max_iters`` = N, as SURVEY.md App. A
prescribes), and stores the marginals, the configuration, the final state
(u, w, phi) and the check history.  "summary" cases at the BASELINE sizes store
the history and state norms only, to keep the fixtures small.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

import otflux as of

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def lindblad_k2():
    return of.LindbladSet(np.stack([np.diag([1.0, -1.0]).astype(complex),
                                    np.array([[0, 1], [1, 0]], dtype=complex)]))


def blob2(n):
    grid = of.GridSpec(n)
    a = of.gen_matrix_blobs([of.BlobSpec((0.3, 0.5), 0.15, np.diag([1.0, 0.0]))], grid)
    b = of.gen_matrix_blobs([of.BlobSpec((0.3, 0.5), 0.15,
                                         np.array([[0.5, 0.5j], [-0.5j, 0.5]]))], grid)
    return a, b


def random_psd_field(rng, n, k):
    a = rng.normal(size=(n, n, k, k)) + 1j * rng.normal(size=(n, n, k, k))
    psd = a @ np.conj(np.swapaxes(a, -1, -2))
    return of.normalize(of.MatrixDensity(psd))


def k4_graph():
    return of.TransportGraph(4, [(0, 1), (1, 2), (2, 3), (0, 3), (0, 2)],
                             [1.0, 2.0, 0.5, 1.5, 0.7], orientations=[1, -1, 1, -1, 1])


def cases():
    rng = np.random.default_rng(12345)
    out = []

    def add(name, kind, l0, l1, chan, cfg, full=True, note="", marginals=True):
        out.append(dict(name=name, kind=kind, l0=l0, l1=l1, chan=chan, cfg=cfg,
                        full=full, note=note, marginals=marginals))

    tri = of.triangle_graph()
    l0, l1 = of.rgb_disk_pair(of.GridSpec(64))
    add("vec64_a1", "vector", l0, l1, tri,
        dict(tau=6.0, norm_u="l12", norm_w="l1", alpha=1.0, max_iters=2000, check_every=500),
        note="BASELINE C1: rgb_disk_pair 64^2, exactly 2000 iterations")
    add("vec64_a03", "vector", l0, l1, tri,
        dict(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.3, max_iters=2000, check_every=500),
        note="C1 with alpha=0.3 so that w != 0")
    a = of.normalize(of.VectorDensity(rng.random((12, 12, 4))))
    b = of.normalize(of.VectorDensity(rng.random((12, 12, 4))))
    add("vec12_k4_l2l2_eps", "vector", a, b, k4_graph(),
        dict(tau=2.0, norm_u="l2", norm_w="l2", alpha=0.5, eps_reg=0.01, max_iters=300,
             check_every=100), note="k=4 graph, costs != 1, flipped orientations, eps>0")
    s0, s1 = of.rgb_disk_pair(of.GridSpec(16))
    add("vec16_l1l1", "vector", s0, s1, tri,
        dict(tau=3.0, norm_u="l1", norm_w="l1", alpha=0.3, max_iters=400, check_every=100))
    a = of.normalize(of.VectorDensity(rng.random((9, 9, 2))))
    b = of.normalize(of.VectorDensity(rng.random((9, 9, 2))))
    add("vec9_k2_l2l1_eps", "vector", a, b, of.TransportGraph(2, [(0, 1)], [0.8]),
        dict(tau=1.0, norm_u="l2", norm_w="l1", alpha=2.0, eps_reg=0.05, max_iters=150,
             check_every=50))
    da, db = of.dirac_pair(of.GridSpec(17), (4, 8), (12, 8))
    add("sca17_dirac", "scalar", da, db, None,
        dict(tau=3.0, norm_u="l2", max_iters=500, check_every=100))
    a = of.normalize(of.ScalarDensity(rng.random((9, 9))))
    b = of.normalize(of.ScalarDensity(rng.random((9, 9))))
    add("sca9_l1_eps", "scalar", a, b, None,
        dict(tau=1.0, norm_u="l1", eps_reg=0.05, max_iters=300, check_every=100))
    add("sca9_l12", "scalar", a, b, None,
        dict(tau=2.0, norm_u="l12", max_iters=200, check_every=100))
    m0, m1, m2 = of.matrix_blob_fixtures(of.GridSpec(24))
    L3 = of.default_lindblad3()
    add("matr24_l2l1", "matrix", m0, m1, L3,
        dict(tau=30.0, norm_u="l2", norm_w="l1", alpha=1.0, max_iters=300, check_every=100),
        note="real-symmetric path, DTI fixtures (C4 shape)")
    add("matr24_l12l2_shift", "matrix", m0, m2, L3,
        dict(tau=10.0, norm_u="l12", norm_w="l2", alpha=0.5, max_iters=200, check_every=100))
    add("matr24_l1l1_eps", "matrix", m0, m1, L3,
        dict(tau=10.0, norm_u="l1", norm_w="l1", alpha=0.7, eps_reg=0.02, max_iters=200,
             check_every=100))
    c0, c1 = blob2(24)
    add("matc24_k2_nuc", "matrix", c0, c1, lindblad_k2(),
        dict(tau=30.0, norm_u="l1nuc", norm_w="l1nuc", alpha=1.0, max_iters=300, check_every=100),
        note="complex Hermitian 2x2, eig shrink (C3 shape)")
    add("matc24_k2_l2l1", "matrix", c0, c1, lindblad_k2(),
        dict(tau=30.0, norm_u="l2", norm_w="l1", alpha=1.0, max_iters=200, check_every=100),
        note="complex path without nuclear norms (diff has imaginary part)")
    p0 = random_psd_field(rng, 10, 3)
    p1 = random_psd_field(rng, 10, 3)
    add("matc10_k3_nuc", "matrix", p0, p1, L3,
        dict(tau=10.0, norm_u="l1nuc", norm_w="l1nuc", alpha=0.3, max_iters=200, check_every=100),
        note="complex Hermitian 3x3, eig shrink both fluxes")
    add("matc10_k3_nucl1", "matrix", p0, p1, L3,
        dict(tau=10.0, norm_u="l1nuc", norm_w="l1", alpha=1.0, max_iters=200, check_every=100))
    add("matc10_k3_l12l2_eps", "matrix", p0, p1, L3,
        dict(tau=5.0, norm_u="l12", norm_w="l2", alpha=1.0, eps_reg=0.01, max_iters=150,
             check_every=50))
    q0 = random_psd_field(rng, 8, 2)
    q1 = random_psd_field(rng, 8, 2)
    add("matc8_k2_nuc_rand", "matrix", q0, q1, lindblad_k2(),
        dict(tau=3.0, norm_u="l1nuc", norm_w="l1nuc", alpha=0.5, max_iters=200, check_every=100))
    # -- summary-only cases at the BASELINE sizes --------------------------
    g0, g1 = of.rgb_disk_pair(of.GridSpec(256))
    add("S_vec256", "vector", g0, g1, tri,
        dict(tau=6.0, norm_u="l12", norm_w="l1", alpha=1.0, max_iters=400, check_every=100),
        full=False, note="C2 grid, 400 iterations")
    M0, M1, _ = of.matrix_blob_fixtures(of.GridSpec(256))
    add("S_matr256", "matrix", M0, M1, L3,
        dict(tau=30.0, norm_u="l2", norm_w="l1", alpha=1.0, max_iters=500, check_every=100),
        full=False, note="C4: 3x3 DTI 256^2, 500 iterations")
    C0, C1 = blob2(128)
    add("S_matc128", "matrix", C0, C1, lindblad_k2(),
        dict(tau=30.0, norm_u="l1nuc", norm_w="l1nuc", alpha=1.0, max_iters=300, check_every=100),
        full=False, note="C3: 2x2 complex 128^2 l1nuc, 300 iterations")
    # -- full-state cases at the BASELINE sizes (the marginals are not stored:
    # the tests regenerate them with paper_1712_10279_b200.synthetic and check
    # the sha256 digests recorded here against the reference's bytes) -------
    add("B_vec256", "vector", g0, g1, tri,
        dict(tau=6.0, norm_u="l12", norm_w="l1", alpha=1.0, max_iters=400, check_every=100),
        marginals=False, note="BASELINE C2 grid: full state after 400 iterations")
    add("B_vec256_a03", "vector", g0, g1, tri,
        dict(tau=6.0, norm_u="l12", norm_w="l1", alpha=0.3, max_iters=400, check_every=100),
        marginals=False, note="BASELINE C2 grid at alpha=0.3 (w != 0), 400 iterations")
    add("B_matr256", "matrix", M0, M1, L3,
        dict(tau=30.0, norm_u="l2", norm_w="l1", alpha=1.0, max_iters=500, check_every=100),
        marginals=False, note="BASELINE C4: full state after 500 iterations")
    add("B_matc128", "matrix", C0, C1, lindblad_k2(),
        dict(tau=30.0, norm_u="l1nuc", norm_w="l1nuc", alpha=1.0, max_iters=300, check_every=100),
        marginals=False, note="BASELINE C3: full state after 300 iterations")
    r0, r1 = of.rgb_disk_pair(of.GridSpec(32))
    add("S_vec32_conv", "vector", r0, r1, tri,
        dict(tau=6.0, norm_u="l12", norm_w="l1", alpha=1.0), full=False,
        note="C05 at n=32 run to convergence with the default tolerances")
    add("S_sca33_dirac_conv", "scalar", *of.dirac_pair(of.GridSpec(33), (8, 16), (24, 16)), None,
        dict(tau=3.0), full=False, note="T/test_solver.py:70-77 Dirac pair to convergence")
    return out


def run_case(c):
    cfg = dict(c["cfg"])
    if "max_iters" in cfg and c["name"] not in ("S_vec32_conv",):
        cfg.setdefault("tol_gap", 1e-300)
        cfg.setdefault("tol_feas", 1e-300)
    scfg = of.SolverConfig(**cfg)
    t0 = time.perf_counter()
    if c["kind"] == "scalar":
        rep, st = of.solve_scalar(c["l0"], c["l1"], cfg=scfg)
    elif c["kind"] == "vector":
        rep, st = of.solve_vector(c["l0"], c["l1"], c["chan"], cfg=scfg)
    else:
        rep, st = of.solve_matrix(c["l0"], c["l1"], c["chan"], cfg=scfg)
    dt = time.perf_counter() - t0
    return cfg, rep, st, dt


def main(names=None):
    OUT.mkdir(parents=True, exist_ok=True)
    index = {}
    for c in cases():
        if names and c["name"] not in names:
            continue
        cfg, rep, st, dt = run_case(c)
        hist = np.array([[h.iteration, h.primal, h.dual, h.gap_ratio, h.feas_residual,
                          h.residual] for h in rep.history], dtype=np.float64)
        arrs = dict(history=hist,
                    meta=np.array([rep.iterations, int(rep.converged), rep.transport_value]))
        wv = None if st.w is None else st.w.values
        import hashlib
        digests = {nm: hashlib.sha256(np.ascontiguousarray(c[nm].values).tobytes()).hexdigest()
                   for nm in ("l0", "l1")}
        norms = dict(ux=float(np.linalg.norm(st.u.ux)), uy=float(np.linalg.norm(st.u.uy)),
                     phi=float(np.linalg.norm(st.phi)),
                     w=0.0 if wv is None else float(np.linalg.norm(wv)))
        if c["full"]:
            arrs.update(ux=st.u.ux, uy=st.u.uy, phi=st.phi)
            if c["marginals"]:
                arrs.update(l0=c["l0"].values, l1=c["l1"].values)
            if wv is not None:
                arrs["w"] = wv
        chan = None
        if c["kind"] == "vector":
            g = c["chan"]
            chan = dict(k=g.k, edges=[list(e) for e in g.edges], costs=list(map(float, g.costs)),
                        orientations=list(map(float, g.orientations)))
        elif c["kind"] == "matrix":
            m = c["chan"].matrices
            arrs["lindblad"] = m
        np.savez_compressed(OUT / f"{c['name']}.npz", **arrs)
        index[c["name"]] = dict(kind=c["kind"], cfg=cfg, graph=chan, full=c["full"],
                                note=c["note"], marginals=c["marginals"],
                                iterations=rep.iterations,
                                converged=bool(rep.converged),
                                transport_value=rep.transport_value, norms=norms,
                                phi_dtype=str(st.phi.dtype), seconds=round(dt, 2),
                                sha256=digests)
        print(f"{c['name']:24s} it={rep.iterations:6d} V={rep.transport_value:.12g} "
              f"|w|={norms['w']:.3g} {dt:.1f}s", flush=True)
    idx_path = OUT / "index.json"
    old = json.loads(idx_path.read_text()) if idx_path.exists() else {}
    old.update(index)
    idx_path.write_text(json.dumps(old, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:] or None)

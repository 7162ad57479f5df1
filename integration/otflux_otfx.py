"""ctypes binding of libotfx.so (include/otfx.h) as an otflux maintainer would
add it to the REFERENCE package: ``otflux/_otfx.py``.

``run_vector_on_gpu(engine, graph, lambda0, lambda1)`` replaces
``_run(engine)`` (S/solver.py:294-337) in ``solve_vector``
(S/solver.py:372-393): the reference builds its ``_Engine`` exactly as today
(step sizes mu, nu, tau, inv_dx; S/solver.py:179-205), and the B200 engine
runs the whole check-cadence loop and returns the reference's own
``SolveReport`` / ``SolverState``.  It uses nothing but ctypes and NumPy, so it
can live inside otflux unchanged; ``tests/test_gpu_integration.py`` loads it
into the unmodified reference (baseline/_ref) and checks the result against
the reference's own CPU ``solve_vector``.

The library is found through ``OTFX_LIB`` (a path) or the loader's search
path (``libotfx.so``).
"""

import ctypes as C
import os

import numpy as np


class _Desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dtype", C.c_int32), ("n", C.c_int32), ("k", C.c_int32),
                ("ell", C.c_int32), ("norm_u", C.c_int32), ("norm_w", C.c_int32),
                ("device", C.c_int32), ("row_begin", C.c_int32), ("row_end", C.c_int32),
                ("tau", C.c_double), ("mu", C.c_double), ("nu", C.c_double),
                ("alpha", C.c_double), ("eps_reg", C.c_double), ("inv_dx", C.c_double),
                ("chan", C.POINTER(C.c_double)), ("stream", C.c_void_p)]


class _Hist(C.Structure):
    _fields_ = [(f, C.c_double) for f in
                ("iteration", "primal", "dual", "gap_ratio", "feas_residual", "residual")]


class _Run(C.Structure):
    _fields_ = [("tol_gap", C.c_double), ("tol_feas", C.c_double),
                ("max_iters", C.c_int64), ("check_every", C.c_int64)]


_NORM = {"l2": 0, "l12": 1, "l1": 2, "l1nuc": 3}
_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = C.CDLL(os.environ.get("OTFX_LIB", "libotfx.so"))
        lib.otfx_last_error.restype = C.c_char_p
        _lib = lib
    return _lib


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"otfx error {rc}: {_load().otfx_last_error().decode()}")


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def run_vector_on_gpu(engine, graph, lambda0, lambda1, device=0):
    """Replacement for solver._run(engine) for the vector kind: same
    SolveReport / SolverState, computed by the B200 engine."""
    from .fields import FluxField, GraphFlux
    from .solver import HistoryPoint, SolveReport, SolverState

    lib = _load()
    cfg, n = engine.cfg, engine.grid.n
    coef = np.ascontiguousarray(graph._incidence_over_costs, dtype=np.float64)  # D/c, k x ell
    d = _Desc(1, 0, n, graph.k, graph.num_edges, _NORM[cfg.norm_u.value],
              _NORM[cfg.norm_w.value], device, 0, n, engine.tau, engine.mu, engine.nu,
              cfg.alpha, cfg.eps_reg, engine.inv_dx,
              coef.ctypes.data_as(C.POINTER(C.c_double)), None)
    h = C.c_void_p()
    _check(lib.otfx_engine_create(C.byref(d), C.byref(h)))
    try:
        m = (C.c_double * 2)()
        a = np.ascontiguousarray(lambda0.values, dtype=np.float64)
        b = np.ascontiguousarray(lambda1.values, dtype=np.float64)
        _check(lib.otfx_engine_set_marginals(h, _ptr(a), _ptr(b), m))
        cap = cfg.max_iters // cfg.check_every + 3
        hist = (_Hist * cap)()
        nh, it, conv, wall = C.c_int64(), C.c_int64(), C.c_int(), C.c_double()
        _check(lib.otfx_engine_run(h, C.byref(_Run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters,
                                                   cfg.check_every)), hist, C.c_int64(cap),
                                   C.byref(nh), C.byref(it), C.byref(conv), C.byref(wall)))
        ux = np.empty((n, n, graph.k))
        uy = np.empty_like(ux)
        phi = np.empty_like(ux)
        w = np.empty((n, n, graph.num_edges))
        _check(lib.otfx_engine_get_state(h, _ptr(ux), _ptr(uy), _ptr(w), _ptr(phi)))
    finally:
        lib.otfx_engine_destroy(h)
    history = [HistoryPoint(int(p.iteration), p.primal, p.dual, p.gap_ratio,
                            p.feas_residual, p.residual) for p in hist[: nh.value]]
    last = history[-1]
    report = SolveReport(bool(conv.value), it.value, last.primal, history, wall.value)
    state = SolverState(FluxField(ux, uy), GraphFlux(w), phi, it.value, last.residual,
                        last.primal, last.dual, last.gap_ratio, last.feas_residual)
    return report, state

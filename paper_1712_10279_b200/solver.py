"""Drop-in solver entry points running the PDHG iteration on a B200.

Public surface (same names, signatures, return types and errors as the
reference ``otflux.solver``, S/solver.py:66-526):

    solve_scalar, solve_vector, solve_matrix      -> (SolveReport, SolverState)
    SolverConfig, SolveReport, SolverState, HistoryPoint
    duality_gap, residual_Rk, step_sizes_*, default_tau

The reference runs its ``_Engine`` (S/solver.py:175-291) in NumPy; here the
engine is ``CudaEngine``, a thin wrapper over the C ABI of libotfx.so
(include/otfx.h) whose iteration, check reductions and run loop execute on the
device.  Optional keyword arguments outside the reference signature select the
precision ("f64" default, bit-faithful to the reference's rounding order; or
"f32") and the device; ``SolverConfig`` itself is unchanged so the config echo
stays identical.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .errors import UnsupportedNormError, ValidationError
from .fields import (FluxField, GraphFlux, GridSpec, QuantumFlux, _trusted)
from .graph import TransportGraph, lambda_max_graph
from .lindblad import LindbladSet, lambda_max_L

# returned states at least this large are allocated and pre-faulted on a host
# thread during the run (_solve)
_PREFAULT_BYTES = 256 << 20

MASS_MISMATCH_TOL = 1e-9
_TINY = np.finfo(np.float64).tiny


class NormFamily(str, Enum):
    L2 = "l2"
    L12 = "l12"
    L1 = "l1"
    L1NUC = "l1nuc"


def validate_norm(family, kind: str, role: str) -> None:
    """Family / payload pairing rules of S/shrink.py:70-76."""
    family = NormFamily(family)
    if family == NormFamily.L1NUC and kind != "matrix":
        raise UnsupportedNormError("nuclear norm requires a matrix payload")
    if family == NormFamily.L12 and role != "u":
        raise UnsupportedNormError("row-grouped norm applies only to spatial fluxes")


def default_tau(n: int) -> float:
    """1 up to n = 64, 3 from there on (S/solver.py:66-68)."""
    return 1.0 if n <= 64 else 3.0


def step_sizes_scalar(grid: GridSpec, tau: float):
    if tau <= 0:
        raise ValidationError("tau must be positive")
    return 1.0 / (16.0 * tau * (grid.n - 1) ** 2), tau


def step_sizes_vector(grid: GridSpec, graph: TransportGraph, tau: float):
    if tau <= 0:
        raise ValidationError("tau must be positive")
    return (1.0 / (32.0 * tau * (grid.n - 1) ** 2),
            1.0 / (4.0 * tau * lambda_max_graph(graph)), tau)


def step_sizes_matrix(grid: GridSpec, lindblad: LindbladSet, tau: float):
    if tau <= 0:
        raise ValidationError("tau must be positive")
    return (1.0 / (32.0 * tau * (grid.n - 1) ** 2),
            1.0 / (4.0 * tau * lambda_max_L(lindblad)), tau)


@dataclass
class SolverConfig:
    """Same fields, defaults and validation as S/solver.py:97-130."""

    tau: float | None = None
    tol_gap: float = 1e-3
    tol_feas: float = 1e-5
    max_iters: int = 200_000
    alpha: float = 1.0
    norm_u: NormFamily = NormFamily.L2
    norm_w: NormFamily = NormFamily.L1
    eps_reg: float = 0.0
    check_every: int = 100

    def __post_init__(self):
        self.norm_u = NormFamily(self.norm_u)
        self.norm_w = NormFamily(self.norm_w)
        if self.tau is not None and self.tau <= 0:
            raise ValidationError("tau must be positive")
        if self.tol_gap <= 0 or self.tol_feas <= 0:
            raise ValidationError("tolerances must be positive")
        if self.max_iters < 1 or self.check_every < 1:
            raise ValidationError("max_iters and check_every must be >= 1")
        if self.alpha <= 0:
            raise ValidationError("alpha must be positive")
        if self.eps_reg < 0:
            raise ValidationError("eps_reg must be nonnegative")


@dataclass
class HistoryPoint:
    iteration: int
    primal: float
    dual: float
    gap_ratio: float
    feas_residual: float
    residual: float


@dataclass
class SolveReport:
    converged: bool
    iterations: int
    transport_value: float
    history: list = field(default_factory=list)
    wall_time: float = 0.0


@dataclass
class SolverState:
    u: FluxField
    w: object
    phi: np.ndarray
    iteration: int
    residual: float
    primal_value: float
    dual_value: float
    gap_ratio: float
    feas_residual: float


# ---------------------------------------------------------------------------
# the device engine
# ---------------------------------------------------------------------------


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


class CudaEngine:
    """Device counterpart of the reference ``_Engine`` protocol
    (S/solver.py:175-291): ``set_marginals``/``set_diff`` (constructor data),
    ``step``, ``evaluate``, ``step_check`` (step + residual_from + evaluate),
    ``run`` (the whole ``_run`` loop), ``get_state``/``set_state``.

    kind: "scalar" | "vector" | "matrix_real" | "matrix_complex".  For a row
    slab pass ``rows=(row_begin, row_end)``; arrays then cover those rows only.
    """

    def __init__(self, kind, n, *, tau, mu, nu=None, k=1, ell=0, chan=None, norm_u="l2",
                 norm_w="l1", alpha=1.0, eps=0.0, precision="f64", device=0, rows=None,
                 stream=None):
        lib = _lib.load()
        self.kind = kind
        self.n = n
        self.k = k
        self.ell = ell
        self.rows = (0, n) if rows is None else tuple(rows)
        self.precision = precision
        self.tau, self.mu, self.nu = tau, mu, nu
        if kind == "vector":
            coef = np.ascontiguousarray(chan, dtype=np.float64)
        elif kind.startswith("matrix"):
            coef = np.ascontiguousarray(chan, dtype=np.complex128).view(np.float64)
        else:
            coef = None
        self._coef = coef
        d = _lib.EngineDesc()
        d.kind = _lib.KIND[kind]
        d.dtype = _lib.DTYPE[precision]
        d.n, d.k, d.ell = n, k, ell
        d.norm_u = _lib.NORM[NormFamily(norm_u).value]
        d.norm_w = _lib.NORM[NormFamily(norm_w).value]
        d.device = int(device)
        d.row_begin, d.row_end = self.rows
        d.tau, d.mu = float(tau), float(mu)
        d.nu = float(nu) if nu is not None else 0.0
        d.alpha, d.eps_reg = float(alpha), float(eps)
        d.inv_dx = 1.0 / GridSpec(n).dx  # S/solver.py:183
        d.chan = coef.ctypes.data_as(C.POINTER(C.c_double)) if coef is not None else None
        d.stream = stream
        self._desc = d
        h = C.c_void_p()
        _lib.check(lib.otfx_engine_create(C.byref(d), C.byref(h)))
        self._h = h
        self._lib = lib

    # -- lifecycle ----------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.otfx_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def info(self):
        inf = _lib.EngineInfo()
        _lib.check(self._lib.otfx_engine_get_info(self._h, C.byref(inf)))
        return {f: getattr(inf, f) for f, _ in inf._fields_}

    @property
    def stream(self):
        return self._lib.otfx_engine_stream(self._h)

    # -- payload shapes -------------------------------------------------------
    @property
    def nrows(self):
        return self.rows[1] - self.rows[0]

    def _pshape(self):
        if self.kind == "scalar":
            return ()
        if self.kind == "vector":
            return (self.k,)
        return (self.k, self.k)

    def _pdtype(self):
        return np.complex128 if self.kind == "matrix_complex" else np.float64

    def _wdtype(self):
        """w is real for the vector and real-symmetric matrix paths (the
        reference's real engine holds w as float64, S/solver.py:414-432)."""
        return np.complex128 if self.kind == "matrix_complex" else np.float64

    def _wshape(self):
        if self.kind == "vector":
            return (self.ell,)
        return (self.ell, self.k, self.k)

    # -- data ---------------------------------------------------------------
    def set_marginals(self, l0, l1):
        """Upload the marginals (rows of this slab) and form diff on the device;
        returns the total masses (S/solver.py:351-355)."""
        dt = np.complex128 if self.kind.startswith("matrix") else np.float64
        a = np.ascontiguousarray(l0, dtype=dt)
        b = np.ascontiguousarray(l1, dtype=dt)
        m = (C.c_double * 2)()
        _lib.check(self._lib.otfx_engine_set_marginals(self._h, _ptr(a), _ptr(b), m))
        return m[0], m[1]

    def set_diff(self, diff):
        a = np.ascontiguousarray(diff, dtype=self._pdtype())
        _lib.check(self._lib.otfx_engine_set_diff(self._h, _ptr(a)))

    @property
    def diff_norm(self):
        v = C.c_double()
        _lib.check(self._lib.otfx_engine_diff_norm(self._h, C.byref(v), None))
        return v.value

    @diff_norm.setter
    def diff_norm(self, value):
        v = C.c_double(float(value))
        _lib.check(self._lib.otfx_engine_diff_norm(self._h, None, C.byref(v)))

    def zero_state(self):
        _lib.check(self._lib.otfx_engine_zero_state(self._h))

    def set_state(self, ux, uy, w, phi):
        pdt = self._pdtype()
        ux = np.ascontiguousarray(ux, dtype=pdt)
        uy = np.ascontiguousarray(uy, dtype=pdt)
        phi = np.ascontiguousarray(phi, dtype=pdt)
        if w is not None:
            w = np.ascontiguousarray(w, dtype=self._wdtype())
        _lib.check(self._lib.otfx_engine_set_state(self._h, _ptr(ux), _ptr(uy), _ptr(w), _ptr(phi)))

    def alloc_state(self, prefault=False):
        """Host arrays for get_state (reference shapes and dtypes,
        S/fields.py:265-289).  prefault=True takes their page faults now
        (otfx_host_prefault), e.g. from a thread while run() is on the GPU."""
        shape = (self.nrows, self.n) + self._pshape()
        pdt = self._pdtype()
        ux = np.empty(shape, pdt)
        uy = np.empty(shape, pdt)
        phi = np.empty(shape, pdt)
        w = None
        if self.kind != "scalar":
            w = np.empty((self.nrows, self.n) + self._wshape(), self._wdtype())
        if prefault:
            for a in (ux, uy, w, phi):
                if a is not None:
                    _lib.check(self._lib.otfx_host_prefault(_ptr(a), a.nbytes))
        return ux, uy, w, phi

    def state_nbytes(self):
        cells = self.nrows * self.n
        per = int(np.prod(self._pshape(), dtype=np.int64)) * np.dtype(self._pdtype()).itemsize
        wb = 0
        if self.kind != "scalar":
            wb = int(np.prod(self._wshape(), dtype=np.int64)) * np.dtype(self._wdtype()).itemsize
        return cells * (3 * per + wb)

    def prefault_async(self):
        """Start allocating + pre-faulting the state arrays on a host thread
        (large states only).  Returns a callable that joins and yields the
        arrays for get_state(out=...), or None."""
        if self.state_nbytes() < _PREFAULT_BYTES:
            return lambda: None
        box = []
        th = threading.Thread(target=lambda: box.append(self.alloc_state(prefault=True)))
        th.start()

        def join():
            th.join()
            return box[0] if box else None
        return join

    def get_state(self, out=None):
        ux, uy, w, phi = out if out is not None else self.alloc_state()
        _lib.check(self._lib.otfx_engine_get_state(self._h, _ptr(ux), _ptr(uy), _ptr(w), _ptr(phi)))
        return ux, uy, w, phi

    # -- device-pointer hand-off (torch CUDA tensors) --------------------------
    def _torch_stream(self, stream):
        import torch

        if stream is None:
            stream = torch.cuda.current_stream(self._desc.device)
        return C.c_void_p(stream.cuda_stream)

    def _tensor_ptr(self, t, dtype):
        """data_ptr of a contiguous CUDA tensor of the engine's device in the
        reference layout (complex128 tensors are interleaved doubles)."""
        import torch

        if t is None:
            return None
        want = torch.complex128 if dtype == np.complex128 else torch.float64
        if not (t.is_cuda and t.dtype == want and t.is_contiguous()
                and t.device.index == self._desc.device):
            raise ValidationError(
                f"expected a contiguous {want} tensor on cuda:{self._desc.device}, got "
                f"{t.dtype} on {t.device} (contiguous={t.is_contiguous()})")
        return C.c_void_p(t.data_ptr())

    def set_marginals_device(self, l0, l1, stream=None):
        """set_marginals for torch CUDA tensors (read in place on the device)."""
        dt = np.complex128 if self.kind.startswith("matrix") else np.float64
        m = (C.c_double * 2)()
        _lib.check(self._lib.otfx_engine_set_marginals_device(
            self._h, self._tensor_ptr(l0, dt), self._tensor_ptr(l1, dt), m,
            self._torch_stream(stream)))
        return m[0], m[1]

    def set_state_device(self, ux, uy, w, phi, stream=None):
        pdt = self._pdtype()
        wdt = self._wdtype()
        _lib.check(self._lib.otfx_engine_set_state_device(
            self._h, self._tensor_ptr(ux, pdt), self._tensor_ptr(uy, pdt),
            self._tensor_ptr(w, wdt), self._tensor_ptr(phi, pdt), self._torch_stream(stream)))

    def alloc_state_device(self):
        """torch CUDA tensors for get_state_device (reference shapes / dtypes)."""
        import torch

        dev = torch.device("cuda", self._desc.device)
        shape = (self.nrows, self.n) + self._pshape()
        pdt = torch.complex128 if self._pdtype() == np.complex128 else torch.float64
        ux = torch.empty(shape, dtype=pdt, device=dev)
        uy = torch.empty_like(ux)
        phi = torch.empty_like(ux)
        w = None
        if self.kind != "scalar":
            wdt = torch.complex128 if self._wdtype() == np.complex128 else torch.float64
            w = torch.empty((self.nrows, self.n) + self._wshape(), dtype=wdt, device=dev)
        return ux, uy, w, phi

    def get_state_device(self, out=None, stream=None):
        """The current iterate written into torch CUDA tensors on the caller's
        stream order (no host round trip)."""
        ux, uy, w, phi = out if out is not None else self.alloc_state_device()
        pdt = self._pdtype()
        wdt = self._wdtype()
        _lib.check(self._lib.otfx_engine_get_state_device(
            self._h, self._tensor_ptr(ux, pdt), self._tensor_ptr(uy, pdt),
            self._tensor_ptr(w, wdt), self._tensor_ptr(phi, pdt), self._torch_stream(stream)))
        return ux, uy, w, phi

    # -- iteration ------------------------------------------------------------
    def step(self, iters=1):
        _lib.check(self._lib.otfx_engine_step(self._h, int(iters)))

    def sweep(self, check=False):
        _lib.check(self._lib.otfx_engine_sweep(self._h, 1 if check else 0))

    def evaluate(self):
        out = (C.c_double * 4)()
        _lib.check(self._lib.otfx_engine_evaluate(self._h, out))
        return tuple(out)

    def step_check(self):
        out = (C.c_double * 5)()
        _lib.check(self._lib.otfx_engine_step_check(self._h, out))
        return tuple(out)

    def raw(self, with_residual=False):
        out = (C.c_double * _lib.NRAW)()
        _lib.check(self._lib.otfx_engine_raw(self._h, 1 if with_residual else 0, out))
        return np.array(out)

    def finalize(self, raw):
        raw = np.ascontiguousarray(raw, dtype=np.float64)
        out = (C.c_double * 5)()
        _lib.check(self._lib.otfx_engine_finalize(
            self._h, raw.ctypes.data_as(C.POINTER(C.c_double)), out))
        return tuple(out)

    def timing(self, enable=-1):
        """Device time of the plain-iteration graphs since the last reset:
        enable=1 reset+start, 0 reset+stop, -1 read.  Returns (ms, sweeps)."""
        ms, cnt = C.c_double(), C.c_int64()
        _lib.check(self._lib.otfx_engine_timing(self._h, int(enable), C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def sync(self):
        _lib.check(self._lib.otfx_engine_sync(self._h))

    def run(self, tol_gap, tol_feas, max_iters, check_every):
        """The _run loop (S/solver.py:294-337) on the device."""
        cap = _history_cap(max_iters, check_every)
        hist = (_lib.HistoryPointC * cap)()
        cfg = _lib.RunConfig(tol_gap, tol_feas, int(max_iters), int(check_every))
        nh, it = C.c_int64(), C.c_int64()
        conv, wall = C.c_int(), C.c_double()
        _lib.check(self._lib.otfx_engine_run(self._h, C.byref(cfg), hist, cap, C.byref(nh),
                                             C.byref(it), C.byref(conv), C.byref(wall)))
        history = _history(self._lib, self._h, hist, cap, nh.value)
        return history, it.value, bool(conv.value), wall.value

    def attach_nccl(self, unique_id: bytes, nranks: int, rank: int):
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        _lib.check(self._lib.otfx_engine_attach_nccl(self._h, buf, nranks, rank))

    def attach_comm(self, comm):
        """Use a SlabCommunicator (distributed.py) that outlives this engine."""
        _lib.check(self._lib.otfx_engine_attach_comm(self._h, comm.handle))


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _lib.check(_lib.load().otfx_nccl_unique_id(buf))
    return bytes(buf)


def run_local(engines, tol_gap, tol_feas, max_iters, check_every, loopback=None):
    """The run loop over the row-slab engines of one grid on one device, in
    lockstep with local halo copies (the single-GPU stand-in for NCCL ranks).
    loopback: a one-rank SlabCommunicator; the halo transport and the check
    allreduces then go through NCCL send / recv / allreduce to that rank."""
    cap = _history_cap(max_iters, check_every)
    hist = (_lib.HistoryPointC * cap)()
    cfg = _lib.RunConfig(tol_gap, tol_feas, int(max_iters), int(check_every))
    nh, it, conv = C.c_int64(), C.c_int64(), C.c_int()
    arr = (C.c_void_p * len(engines))(*[e.handle for e in engines])
    lib = _lib.load()
    _lib.check(lib.otfx_engines_run_local_nccl(arr, len(engines),
                                               loopback.handle if loopback else None,
                                               C.byref(cfg), hist, cap, C.byref(nh),
                                               C.byref(it), C.byref(conv)))
    history = _history(lib, engines[0].handle, hist, cap, nh.value)
    return history, it.value, bool(conv.value)


def _history_cap(max_iters, check_every):
    """Initial history buffer: enough for every check of the run, but bounded
    (the engine keeps the whole history; a longer one is fetched after)."""
    return int(min(max_iters // check_every + 3, 1 << 16))


def _history(lib, handle, hist, cap, total):
    if total > cap:
        hist = (_lib.HistoryPointC * total)()
        got = C.c_int64()
        _lib.check(lib.otfx_engine_history(handle, hist, total, C.byref(got)))
    return [HistoryPoint(int(h.iteration), h.primal, h.dual, h.gap_ratio, h.feas_residual,
                         h.residual) for h in hist[:total]]


def exchange_local(engines):
    arr = (C.c_void_p * len(engines))(*[e.handle for e in engines])
    _lib.check(_lib.load().otfx_engine_exchange_local(arr, len(engines)))


# ---------------------------------------------------------------------------
# problem setup shared by the public entry points
# ---------------------------------------------------------------------------


def _values(d):
    return np.asarray(d.values)


def _check_pair(l0, l1, grid):
    """Type / shape / grid checks of S/solver.py:340-356 (the mass check runs
    on the device right after upload, see _finish_mass_check)."""
    if type(l0) is not type(l1):
        raise ValidationError(f"marginals must share a type, got {type(l0)}/{type(l1)}")
    v0, v1 = _values(l0), _values(l1)
    if v0.shape != v1.shape:
        raise ValidationError(f"marginal shapes differ: {v0.shape} vs {v1.shape}")
    n = v0.shape[0]
    if grid is None:
        grid = GridSpec(n)
    elif grid.n != n:
        raise ValidationError(f"grid n={grid.n} does not match fields with n={n}")
    return grid


def _mass_check(m0, m1):
    if abs(m0 - m1) > MASS_MISMATCH_TOL:
        raise ValidationError(
            f"mass mismatch |{m0:.12g} - {m1:.12g}| > {MASS_MISMATCH_TOL:g}: infeasible")


def _reject_regularized_nuclear(cfg):
    if cfg.eps_reg > 0 and NormFamily.L1NUC in (cfg.norm_u, cfg.norm_w):
        raise UnsupportedNormError("eps_reg > 0 has no closed-form prox for the nuclear family")


def _tau(cfg, n):
    return cfg.tau if cfg.tau is not None else default_tau(n)


def _matrix_use_real(l0v, l1v, mats, cfg):
    """Real/complex path rule of S/solver.py:412-419."""
    return (NormFamily.L1NUC not in (cfg.norm_u, cfg.norm_w)
            and not np.any(l0v.imag != l1v.imag)
            and not np.any(np.asarray(mats).imag))


def build_engine(kind, n, cfg, graph=None, lindblad=None, precision="f64", device=0, rows=None,
                 complex_path=None, stream=None):
    """Construct the CudaEngine for one solve (the reference's _Engine
    constructor + set_channel_bound, S/solver.py:179-205, 386-392, 427-434)."""
    tau = _tau(cfg, n)
    common = dict(tau=tau, norm_u=cfg.norm_u.value, norm_w=cfg.norm_w.value, alpha=cfg.alpha,
                  eps=cfg.eps_reg, precision=precision, device=device, rows=rows, stream=stream)
    if kind == "scalar":
        mu = 1.0 / (16.0 * tau * (n - 1) ** 2)
        return CudaEngine("scalar", n, mu=mu, **common)
    mu = 1.0 / (32.0 * tau * (n - 1) ** 2)
    if kind == "vector":
        nu = 1.0 / (4.0 * tau * lambda_max_graph(graph))
        return CudaEngine("vector", n, mu=mu, nu=nu, k=graph.k, ell=graph.num_edges,
                          chan=graph.coefficients(), **common)
    mats = lindblad.matrices
    nu = 1.0 / (4.0 * tau * lambda_max_L(lindblad))
    kname = "matrix_complex" if complex_path else "matrix_real"
    chan = np.asarray(mats, dtype=np.complex128)
    if not complex_path:
        chan = np.real(chan).astype(np.complex128)
    return CudaEngine(kname, n, mu=mu, nu=nu, k=lindblad.k, ell=lindblad.ell, chan=chan, **common)


def _pack_state(engine, it, rk, primal, dual, gap, feas, out=None):
    ux, uy, w, phi = engine.get_state(out)
    if engine.kind == "scalar":
        wobj = None
    elif engine.kind == "vector":
        wobj = _trusted(GraphFlux, values=w)
    else:
        wobj = _trusted(QuantumFlux, values=w)
    return SolverState(u=_trusted(FluxField, ux=ux, uy=uy), w=wobj, phi=phi, iteration=it,
                       residual=rk, primal_value=primal, dual_value=dual, gap_ratio=gap,
                       feas_residual=feas)


def _solve(engine, l0v, l1v, cfg):
    try:
        m0, m1 = engine.set_marginals(l0v, l1v)
        _mass_check(m0, m1)
        # large states: the returned arrays are allocated and their page faults
        # taken on a host thread while the run occupies the GPU (the ctypes call
        # releases the GIL), so the download is bound by the copies alone
        join = engine.prefault_async()
        try:
            history, it, conv, wall = engine.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters,
                                                 cfg.check_every)
        finally:
            out = join()
        last = history[-1]
        report = SolveReport(conv, it, last.primal, history, wall)
        state = _pack_state(engine, it, last.residual, last.primal, last.dual, last.gap_ratio,
                            last.feas_residual, out)
        return report, state
    finally:
        engine.close()


# ---------------------------------------------------------------------------
# public entry points (S/solver.py:359-435)
# ---------------------------------------------------------------------------


def solve_scalar(lambda0, lambda1, grid: GridSpec | None = None, cfg: SolverConfig | None = None,
                 *, precision="f64", device=0):
    """Transport distance between scalar densities; returns (report, state)."""
    cfg = cfg if cfg is not None else SolverConfig()
    grid = _check_pair(lambda0, lambda1, grid)
    validate_norm(cfg.norm_u, "scalar", "u")
    _reject_regularized_nuclear(cfg)
    eng = build_engine("scalar", grid.n, cfg, precision=precision, device=device)
    return _solve(eng, _values(lambda0), _values(lambda1), cfg)


def solve_vector(lambda0, lambda1, graph: TransportGraph, grid: GridSpec | None = None,
                 cfg: SolverConfig | None = None, *, precision="f64", device=0):
    """Transport distance between k-channel densities over a channel graph."""
    cfg = cfg if cfg is not None else SolverConfig()
    grid = _check_pair(lambda0, lambda1, grid)
    k = _values(lambda0).shape[2]
    if graph.k != k:
        raise ValidationError(f"graph has {graph.k} nodes but densities have k={k}")
    validate_norm(cfg.norm_u, "vector", "u")
    validate_norm(cfg.norm_w, "vector", "w")
    _reject_regularized_nuclear(cfg)
    eng = build_engine("vector", grid.n, cfg, graph=graph, precision=precision, device=device)
    return _solve(eng, _values(lambda0), _values(lambda1), cfg)


def solve_matrix(Lambda0, Lambda1, lindblad: LindbladSet, grid: GridSpec | None = None,
                 cfg: SolverConfig | None = None, *, precision="f64", device=0):
    """Transport distance between Hermitian-PSD matrix densities."""
    cfg = cfg if cfg is not None else SolverConfig()
    grid = _check_pair(Lambda0, Lambda1, grid)
    k = _values(Lambda0).shape[2]
    if lindblad.k != k:
        raise ValidationError(f"matrix set has dim {lindblad.k} but densities have k={k}")
    validate_norm(cfg.norm_u, "matrix", "u")
    validate_norm(cfg.norm_w, "matrix", "w")
    _reject_regularized_nuclear(cfg)
    l0v = _values(Lambda0).astype(np.complex128, copy=False)
    l1v = _values(Lambda1).astype(np.complex128, copy=False)
    use_real = _matrix_use_real(l0v, l1v, lindblad.matrices, cfg)
    eng = build_engine("matrix", grid.n, cfg, lindblad=lindblad, precision=precision,
                       device=device, complex_path=not use_real)
    return _solve(eng, l0v, l1v, cfg)


def solve_tensors(lambda0, lambda1, channels=None, cfg: SolverConfig | None = None, *,
                  precision="f64"):
    """``solve_scalar`` / ``solve_vector`` / ``solve_matrix`` for marginals
    already resident on a GPU as torch tensors (SURVEY §8(b) ownership row:
    torch owns the tensors, the engine reads them in place).

    The kind follows the tensor rank, as the reference's density types do
    (S/fields.py:183-229): (n, n) scalar, (n, n, k) vector with ``channels`` a
    TransportGraph, (n, n, k, k) matrix with ``channels`` a LindbladSet.
    Validation, step sizes, the real/complex matrix rule (S/solver.py:412-419)
    and the run loop are those of the host entry points; the returned
    SolverState holds torch tensors on the marginals' device (same shapes and
    dtypes as the NumPy arrays of the host path), written by the engine
    without a host round trip."""
    import torch

    cfg = cfg if cfg is not None else SolverConfig()
    for t in (lambda0, lambda1):
        if not (isinstance(t, torch.Tensor) and t.is_cuda):
            raise ValidationError("solve_tensors expects torch CUDA tensors")
    if lambda0.shape != lambda1.shape:
        raise ValidationError(f"marginal shapes differ: {tuple(lambda0.shape)} vs "
                              f"{tuple(lambda1.shape)}")
    if lambda0.device != lambda1.device:
        raise ValidationError("marginals on different devices")
    nd = lambda0.dim()
    if nd < 2 or lambda0.shape[0] != lambda0.shape[1]:
        raise ValidationError(f"expected a square grid, got shape {tuple(lambda0.shape)}")
    n = lambda0.shape[0]
    device = lambda0.device.index or 0
    _reject_regularized_nuclear(cfg)
    if nd == 2:
        validate_norm(cfg.norm_u, "scalar", "u")
        eng = build_engine("scalar", n, cfg, precision=precision, device=device)
        a, b = lambda0.to(torch.float64).contiguous(), lambda1.to(torch.float64).contiguous()
    elif nd == 3:
        if not isinstance(channels, TransportGraph) or channels.k != lambda0.shape[2]:
            raise ValidationError("vector marginals need a TransportGraph with k = shape[2]")
        validate_norm(cfg.norm_u, "vector", "u")
        validate_norm(cfg.norm_w, "vector", "w")
        eng = build_engine("vector", n, cfg, graph=channels, precision=precision, device=device)
        a, b = lambda0.to(torch.float64).contiguous(), lambda1.to(torch.float64).contiguous()
    elif nd == 4:
        if not isinstance(channels, LindbladSet) or channels.k != lambda0.shape[2]:
            raise ValidationError("matrix marginals need a LindbladSet with k = shape[2]")
        validate_norm(cfg.norm_u, "matrix", "u")
        validate_norm(cfg.norm_w, "matrix", "w")
        a = lambda0.to(torch.complex128).contiguous()
        b = lambda1.to(torch.complex128).contiguous()
        use_real = (NormFamily.L1NUC not in (cfg.norm_u, cfg.norm_w)
                    and not bool(torch.any(a.imag != b.imag))
                    and not np.any(np.asarray(channels.matrices).imag))
        eng = build_engine("matrix", n, cfg, lindblad=channels, precision=precision,
                           device=device, complex_path=not use_real)
    else:
        raise ValidationError(f"unsupported marginal rank {nd}")
    try:
        m0, m1 = eng.set_marginals_device(a, b)
        _mass_check(m0, m1)
        history, it, conv, wall = eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters,
                                          cfg.check_every)
        last = history[-1]
        report = SolveReport(conv, it, last.primal, history, wall)
        ux, uy, w, phi = eng.get_state_device()
        if eng.kind == "scalar":
            wobj = None
        elif eng.kind == "vector":
            wobj = _trusted(GraphFlux, values=w)
        else:
            wobj = _trusted(QuantumFlux, values=w)
        state = SolverState(u=_trusted(FluxField, ux=ux, uy=uy), w=wobj, phi=phi, iteration=it,
                            residual=last.residual, primal_value=last.primal,
                            dual_value=last.dual, gap_ratio=last.gap_ratio,
                            feas_residual=last.feas_residual)
        return report, state  # close() drains the engine stream before freeing
    finally:
        eng.close()


# ---------------------------------------------------------------------------
# standalone metric helpers (S/solver.py:450-526)
# ---------------------------------------------------------------------------


def _kind_of(d):
    v = _values(d)
    return {2: "scalar", 3: "vector", 4: "matrix"}[v.ndim]


def duality_gap(state: SolverState, lambda0, lambda1, cfg: SolverConfig,
                graph: TransportGraph | None = None, lindblad: LindbladSet | None = None,
                *, precision="f64", device=0):
    """(primal, dual, gap_ratio, feas_residual) of an arbitrary state, on the
    device.  Matrix states use the complex path, as _engine_for does
    (S/solver.py:465-474)."""
    grid = _check_pair(lambda0, lambda1, None)
    kind = _kind_of(lambda0)
    l0v, l1v = _values(lambda0), _values(lambda1)
    eng = build_engine(kind, grid.n, cfg, graph=graph, lindblad=lindblad, precision=precision,
                       device=device, complex_path=True)
    try:
        if kind == "matrix":
            l0v = l0v.astype(np.complex128, copy=False)
            l1v = l1v.astype(np.complex128, copy=False)
        m0, m1 = eng.set_marginals(l0v, l1v)
        _mass_check(m0, m1)
        w = None if state.w is None else np.asarray(state.w.values)
        eng.set_state(state.u.ux, state.u.uy, w, state.phi)
        return eng.evaluate()
    finally:
        eng.close()


def residual_Rk(state_prev: SolverState, state_next: SolverState, mu: float, nu: float | None,
                tau: float, grid: GridSpec | None = None, graph: TransportGraph | None = None,
                lindblad: LindbladSet | None = None, *, precision="f64", device=0):
    """Fixed-point residual between consecutive iterates (S/solver.py:501-526):
    ||du||^2/mu + ||dw||^2/nu + ||dphi||^2/tau - 2 <dphi, div_x du + div_c dw>,
    computed by the engine's residual kernel on the device."""
    n = state_next.u.n if grid is None else grid.n
    has_w = state_next.w is not None
    if has_w and nu is None:
        raise ValidationError("nu is required when a channel flux is present")
    wv = np.asarray(state_next.w.values) if has_w else None
    if not has_w:
        kind, extra = "scalar", {}
    elif wv.ndim == 3:
        if graph is None:
            raise ValidationError("graph is required for a graph flux")
        kind = "vector"
        extra = dict(k=graph.k, ell=graph.num_edges, chan=graph.coefficients())
    else:
        if lindblad is None:
            raise ValidationError("lindblad set is required for a quantum flux")
        kind = "matrix_complex"
        extra = dict(k=lindblad.k, ell=lindblad.ell,
                     chan=np.asarray(lindblad.matrices, dtype=np.complex128))
    if kind == "scalar" and np.asarray(state_next.phi).ndim == 3:
        raise ValidationError("vector states need a graph flux")
    eng = CudaEngine(kind, n, tau=tau, mu=mu, nu=nu if has_w else None, precision=precision,
                     device=device, **extra)
    try:
        pdt = eng._pdtype()
        wdt = eng._wdtype()
        arrs = []
        for st in (state_prev, state_next):
            w = None if st.w is None else np.ascontiguousarray(st.w.values, dtype=wdt)
            arrs += [np.ascontiguousarray(st.u.ux, dtype=pdt), np.ascontiguousarray(st.u.uy, dtype=pdt),
                     w, np.ascontiguousarray(st.phi, dtype=pdt)]
        out = C.c_double()
        _lib.check(eng._lib.otfx_engine_residual_between(eng.handle, *[_ptr(a) for a in arrs],
                                                          C.byref(out)))
        return out.value
    finally:
        eng.close()

"""ctypes binding of libotfx.so (include/otfx.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (make -C
paper_1712_10279_b200/csrc).  There is no fallback: if the library is missing
or no CUDA device is present, every entry point raises NumericalError.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import NumericalError, UnsupportedNormError, ValidationError

LIB_PATH = Path(__file__).resolve().parent / "libotfx.so"

OK, EINVAL, EUNSUPPORTED, ECUDA, ENCCL, ENOMEM = 0, -1, -2, -3, -4, -5
KIND = {"scalar": 0, "vector": 1, "matrix_real": 2, "matrix_complex": 3}
NORM = {"l2": 0, "l12": 1, "l1": 2, "l1nuc": 3}
DTYPE = {"f64": 0, "f32": 1}
NRAW = 14


class EngineDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("dtype", C.c_int32), ("n", C.c_int32), ("k", C.c_int32),
        ("ell", C.c_int32), ("norm_u", C.c_int32), ("norm_w", C.c_int32), ("device", C.c_int32),
        ("row_begin", C.c_int32), ("row_end", C.c_int32),
        ("tau", C.c_double), ("mu", C.c_double), ("nu", C.c_double), ("alpha", C.c_double),
        ("eps_reg", C.c_double), ("inv_dx", C.c_double),
        ("chan", C.POINTER(C.c_double)), ("stream", C.c_void_p),
    ]


class HistoryPointC(C.Structure):
    _fields_ = [(f, C.c_double) for f in
                ("iteration", "primal", "dual", "gap_ratio", "feas_residual", "residual")]


class RunConfig(C.Structure):
    _fields_ = [("tol_gap", C.c_double), ("tol_feas", C.c_double),
                ("max_iters", C.c_int64), ("check_every", C.c_int64)]


class EngineInfo(C.Structure):
    _fields_ = [("state_bytes", C.c_int64), ("total_bytes", C.c_int64),
                ("np", C.c_int32), ("nws", C.c_int32), ("lmax", C.c_int32), ("pitch", C.c_int32),
                ("tile_cols", C.c_int32), ("tile_rows", C.c_int32), ("grid_x", C.c_int32),
                ("grid_y", C.c_int32), ("regs_plain", C.c_int32), ("regs_check", C.c_int32),
                ("graphs", C.c_int32), ("tma_stages", C.c_int32), ("smem_bytes", C.c_int32),
                ("cluster_ctas", C.c_int32), ("halo_overlap", C.c_int32)]


_P = C.c_void_p
_DP = C.POINTER(C.c_double)
SIGNATURES = {
    "otfx_abi_version": (C.c_int, []),
    "otfx_last_error": (C.c_char_p, []),
    "otfx_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "otfx_release_cached_memory": (C.c_int, []),
    "otfx_host_prefault": (C.c_int, [_P, C.c_size_t]),
    "otfx_engine_create": (C.c_int, [C.POINTER(EngineDesc), C.POINTER(_P)]),
    "otfx_engine_destroy": (C.c_int, [_P]),
    "otfx_engine_get_info": (C.c_int, [_P, C.POINTER(EngineInfo)]),
    "otfx_engine_set_marginals": (C.c_int, [_P, _P, _P, _DP]),
    "otfx_engine_set_marginals_device": (C.c_int, [_P, _P, _P, _DP, _P]),
    "otfx_engine_set_state_device": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "otfx_engine_get_state_device": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "otfx_engine_set_diff": (C.c_int, [_P, _P]),
    "otfx_engine_diff_norm": (C.c_int, [_P, _DP, _DP]),
    "otfx_engine_zero_state": (C.c_int, [_P]),
    "otfx_engine_set_state": (C.c_int, [_P, _P, _P, _P, _P]),
    "otfx_engine_get_state": (C.c_int, [_P, _P, _P, _P, _P]),
    "otfx_engine_step": (C.c_int, [_P, C.c_int64]),
    "otfx_engine_evaluate": (C.c_int, [_P, _DP]),
    "otfx_engine_step_check": (C.c_int, [_P, _DP]),
    "otfx_engine_run": (C.c_int, [_P, C.POINTER(RunConfig), C.POINTER(HistoryPointC), C.c_int64,
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int), _DP]),
    "otfx_engines_run_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.POINTER(RunConfig),
                                         C.POINTER(HistoryPointC), C.c_int64,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int)]),
    "otfx_engines_run_local_nccl": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, _P,
                                              C.POINTER(RunConfig), C.POINTER(HistoryPointC),
                                              C.c_int64, C.POINTER(C.c_int64),
                                              C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "otfx_engine_history": (C.c_int, [_P, C.POINTER(HistoryPointC), C.c_int64,
                                      C.POINTER(C.c_int64)]),
    "otfx_engine_residual_between": (C.c_int, [_P] + [_P] * 8 + [_DP]),
    "otfx_engine_sweep": (C.c_int, [_P, C.c_int]),
    "otfx_engine_raw": (C.c_int, [_P, C.c_int, _DP]),
    "otfx_engine_finalize": (C.c_int, [_P, _DP, _DP]),
    "otfx_engine_exchange_local": (C.c_int, [C.POINTER(_P), C.c_int]),
    "otfx_nccl_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
    "otfx_engine_attach_nccl": (C.c_int, [_P, C.POINTER(C.c_ubyte), C.c_int, C.c_int]),
    "otfx_comm_create": (C.c_int, [C.POINTER(C.c_ubyte), C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_void_p)]),
    "otfx_comm_destroy": (C.c_int, [_P]),
    "otfx_engine_attach_comm": (C.c_int, [_P, _P]),
    "otfx_engine_timing": (C.c_int, [_P, C.c_int, _DP, C.POINTER(C.c_int64)]),
    "otfx_engine_sync": (C.c_int, [_P]),
    "otfx_engine_stream": (C.c_void_p, [_P]),
}

_lib = None


def load():
    """Load libotfx.so (once).  Raises NumericalError when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("OTFX_LIB", str(LIB_PATH))
    if not os.path.exists(path):
        raise NumericalError(
            f"libotfx.so not built ({path}); run __graft_entry__.build() -- there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int):
    if rc == OK:
        return
    msg = load().otfx_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise ValidationError(msg)
    if rc == EUNSUPPORTED:
        raise UnsupportedNormError(msg)
    raise NumericalError(f"otfx error {rc}: {msg}")


def release_cached_memory() -> None:
    """Give the engine memory pool's cached blocks back to the driver."""
    check(load().otfx_release_cached_memory())


def device_count() -> int:
    c = C.c_int(0)
    check(load().otfx_device_count(C.byref(c)))
    return c.value

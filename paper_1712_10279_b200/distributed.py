"""Row-slab domain decomposition over several GPUs (one process per GPU).

Rank r owns global rows [bounds[r], bounds[r+1]) of the n x n grid; columns
are never split (coalescing is preserved).  Every iteration the engine
exchanges one halo row each way over NCCL (send/recv on NVLink / NVSwitch):
the first owned phi row goes up, the last owned (phi, u) rows go down
(include/otfx.h, engine.cu exchange_nccl).  Check iterations allreduce the
14 raw scalars (SUM for the 12 sums, MAX for the two dual-norm maxima), so
every rank takes the same convergence decision.  Iterates are bit-identical
to the single-GPU run; only the scalar reductions change order.

The reference has no parallelism beyond BLAS threads; the
decomposition follows the paper's per-pixel split.
"""

from __future__ import annotations

import numpy as np

import ctypes as C

from . import _lib
from .solver import (SolverConfig, _mass_check, _pack_state, SolveReport, build_engine,
                     nccl_unique_id, validate_norm)


def slab_bounds(n: int, nranks: int) -> list[int]:
    """Balanced row split: the first n % nranks slabs get one extra row."""
    if nranks < 1 or nranks > n:
        raise ValueError(f"cannot split {n} rows over {nranks} ranks")
    base, extra = divmod(n, nranks)
    out = [0]
    for r in range(nranks):
        out.append(out[-1] + base + (1 if r < extra else 0))
    return out


def halo_plan(n: int, nranks: int):
    """Per rank: owned rows, the global row of each ghost and its source rank.
    top ghost  = row_begin-1 (phi and u), filled from rank-1's last row;
    bottom ghost = row_end (phi only), filled from rank+1's first row."""
    b = slab_bounds(n, nranks)
    plan = []
    for r in range(nranks):
        plan.append(dict(rank=r, rows=(b[r], b[r + 1]),
                         top=None if r == 0 else dict(row=b[r] - 1, src=r - 1, fields=("phi", "u")),
                         bottom=None if r == nranks - 1 else dict(row=b[r + 1], src=r + 1,
                                                                   fields=("phi",))))
    return plan


def share_unique_id(dist, rank):
    """Create the NCCL unique id on rank 0 and broadcast it with
    torch.distributed (any backend)."""
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


class SlabCommunicator:
    """An NCCL communicator for this rank's slab that outlives the engines of a
    series of solves (the NCCL setup is paid once, not per solve)."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int, device: int = 0):
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        _lib.check(_lib.load().otfx_comm_create(buf, nranks, rank, device, C.byref(h)))
        self.handle = h
        self.nranks, self.rank, self.device = nranks, rank, device

    def close(self):
        if self.handle:
            _lib.check(_lib.load().otfx_comm_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_vector_slab_engine(n, graph, cfg: SolverConfig, *, nranks, rank, unique_id=None,
                            precision="f64", device=0, stream=None, comm=None):
    validate_norm(cfg.norm_u, "vector", "u")
    validate_norm(cfg.norm_w, "vector", "w")
    b = slab_bounds(n, nranks)
    eng = build_engine("vector", n, cfg, graph=graph, precision=precision, device=device,
                       rows=(b[rank], b[rank + 1]), stream=stream)
    if comm is not None:
        if (comm.nranks, comm.rank) != (nranks, rank):
            eng.close()
            raise ValueError("communicator was created for another rank layout")
        eng.attach_comm(comm)
    elif nranks > 1:
        eng.attach_nccl(unique_id, nranks, rank)
    return eng


def solve_vector_rows(l0_rows, l1_rows, graph, n, cfg: SolverConfig | None = None, *, nranks,
                      rank, unique_id=None, precision="f64", device=0, comm=None):
    """Distributed solve_vector: this rank passes its rows of the marginals and
    gets (report, state-of-its-rows); the report is identical on all ranks.
    Either a fresh NCCL unique id (a communicator per call) or a
    SlabCommunicator reused across calls."""
    cfg = cfg if cfg is not None else SolverConfig()
    eng = make_vector_slab_engine(n, graph, cfg, nranks=nranks, rank=rank, unique_id=unique_id,
                                  precision=precision, device=device, comm=comm)
    try:
        m0, m1 = eng.set_marginals(np.asarray(l0_rows), np.asarray(l1_rows))
        _mass_check(m0, m1)
        join = eng.prefault_async()  # state arrays faulted in during the run
        try:
            history, it, conv, wall = eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters,
                                              cfg.check_every)
        finally:
            out = join()
        last = history[-1]
        rep = SolveReport(conv, it, last.primal, history, wall)
        st = _pack_state(eng, it, last.residual, last.primal, last.dual, last.gap_ratio,
                         last.feas_residual, out)
        return rep, st
    finally:
        eng.close()

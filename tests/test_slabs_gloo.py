"""World-size-2 (and 3) CPU test of the row-slab decomposition with the gloo
backend: each rank steps its slab (plus one ghost row each side) with the
oracle and exchanges halo rows exactly as distributed.halo_plan prescribes
(and as engine.cu exchange_nccl implements over NCCL).  The gathered iterates
must equal the single-process oracle run bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

N, ITERS = 23, 40


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    from oracle.pdhg import OracleEngine, graph_coef, graph_lambda_max
    from paper_1712_10279_b200 import synthetic

    l0, l1 = synthetic.rgb_disk_pair(N)
    edges, costs = [(0, 1), (0, 2), (1, 2)], [1.0, 1.0, 1.0]
    mk = lambda diff: OracleEngine("vector", diff, N, 6.0, norm_u="l12", norm_w="l1", alpha=0.3,
                                   chan=graph_coef(3, edges, costs),
                                   lam_chan=graph_lambda_max(3, edges, costs))
    return l0 - l1, mk


def _worker(rank, world, port, out):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1712_10279_b200.distributed import halo_plan

    diff, mk = _problem()
    plan = halo_plan(N, world)[rank]
    r0, r1 = plan["rows"]
    e0, e1 = max(r0 - 1, 0), min(r1 + 1, N)  # extended block with ghost rows
    eng = mk(diff[e0:e1])
    eng.u = np.zeros((e1 - e0, N, 2, 3))
    eng.w = np.zeros((e1 - e0, N, 3))
    eng.phi = np.zeros((e1 - e0, N, 3))
    own = slice(r0 - e0, r1 - e0)
    for _ in range(ITERS):
        eng.step()
        reqs, bufs = [], {}
        if plan["top"] is not None:  # send first phi row up; receive (phi, u) ghost
            reqs.append(dist.isend(torch.from_numpy(eng.phi[own][0].copy()), rank - 1))
            bufs["tp"] = torch.empty(N, 3, dtype=torch.float64)
            bufs["tu"] = torch.empty(N, 2, 3, dtype=torch.float64)
            reqs.append(dist.irecv(bufs["tp"], rank - 1))
            reqs.append(dist.irecv(bufs["tu"], rank - 1))
        if plan["bottom"] is not None:  # send last (phi, u) rows down; receive phi ghost
            reqs.append(dist.isend(torch.from_numpy(eng.phi[own][-1].copy()), rank + 1))
            reqs.append(dist.isend(torch.from_numpy(eng.u[own][-1].copy()), rank + 1))
            bufs["bp"] = torch.empty(N, 3, dtype=torch.float64)
            reqs.append(dist.irecv(bufs["bp"], rank + 1))
        for r in reqs:
            r.wait()
        if "tp" in bufs:
            eng.phi[0] = bufs["tp"].numpy()
            eng.u[0] = bufs["tu"].numpy()
        if "bp" in bufs:
            eng.phi[-1] = bufs["bp"].numpy()
    np.savez(out % rank, u=eng.u[own], w=eng.w[own], phi=eng.phi[own])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slabs_match_single_process(tmp_path, world):
    from oracle.pdhg import oracle_run  # noqa: F401

    out = str(tmp_path / "rank%d.npz")
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    diff, mk = _problem()
    ref = mk(diff)
    for _ in range(ITERS):
        ref.step()
    parts = [np.load(out % r) for r in range(world)]
    for key, arr in (("u", ref.u), ("w", ref.w), ("phi", ref.phi)):
        got = np.concatenate([p[key] for p in parts], axis=0)
        assert np.array_equal(got, arr), key
    assert np.linalg.norm(ref.w) > 0

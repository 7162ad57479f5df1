#!/usr/bin/env python
"""Benchmark of the PDHG hot path (BASELINE.json metric: "PDHG grid-cell
updates/sec and % HBM roofline at 1/2/4/8 B200 vs CPU ref").

Workload: BASELINE configs[4], vector-OMT 3-channel (RGB disks of the
reference's rgb_disk_pair generator, triangle graph, l12/l1, alpha=1, tau=6),
row-slab sharded; weak scaling keeps ~8192^2 cells per GPU (global n =
8192*sqrt(N), rounded to a multiple of N).  One bench "step" is one check
period of the reference run loop (S/solver.py:303-315): 99 plain iterations
plus one check iteration with R^k and the primal/dual/feasibility evaluation.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: launched by torchrun, one process per GPU, NCCL.  Timing: CUDA
events on the engine stream, barrier + synchronize around the timed region,
max over ranks.  The state (14.5 GB at 8192^2 fp64) is far larger than L2, so
no flush is needed between iterations.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "PDHG grid-cell updates/sec and % HBM roofline at 1/2/4/8 B200 vs CPU ref"
UNIT = "cell-updates/s"
K_CH, ELL = 3, 3


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--precision", choices=["f64", "f32"], default="f64")
    p.add_argument("--n", "--side", type=int, default=8192,
                   help="grid side per GPU (weak scaling)")
    p.add_argument("--iters-per-step", type=int, default=100)
    # one e2e call = a 2000-iteration solve, the fixed count of BASELINE configs[0]
    p.add_argument("--e2e-iters", type=int, default=2000)
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--ref-n", type=int, default=2048, help="CPU sample grid side")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--ref-seconds", type=float, default=75.0,
                   help="bound on the timed sample of the reference arm")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the BASELINE configs[0..3] side measurements")
    p.add_argument("--dist", action="store_true",
                   help="take the multi-rank code path (process group, NCCL id broadcast, "
                        "slab communicator, solve_vector_rows) even at world size 1, under "
                        "torchrun: the one-GPU check of what an N-GPU run executes")
    return p.parse_args()


def global_n(n1, world):
    n = int(round(n1 * math.sqrt(world)))
    return max(world, n - n % world)


def bytes_per_cell(precision):
    t = 8 if precision == "f64" else 4
    return (7 * K_CH + 2 * ELL) * t  # compulsory: read u,w,phi,diff; write u,w,phi


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Samples SM clocks and clock-event reasons with NVML while running."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, device):
        self.samples, self.reasons = [], set()
        self.stop_flag = False
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self.stop_flag:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = get_reasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_flag = True
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_baseline(ref_n, seconds, max_steps=None):
    """The oracle (NumPy port of the reference engine) on the host cores."""
    from threadpoolctl import threadpool_limits

    from oracle.pdhg import OracleEngine, graph_coef
    import paper_1712_10279_b200 as pk
    from paper_1712_10279_b200 import synthetic

    l0, l1 = synthetic.rgb_disk_pair(ref_n)
    g = pk.triangle_graph()
    cores = os.cpu_count() or 1
    with threadpool_limits(limits=cores):
        eng = OracleEngine("vector", l0 - l1, ref_n, 6.0, norm_u="l12", norm_w="l1", alpha=1.0,
                           chan=graph_coef(3, g.edges, g.costs), lam_chan=pk.lambda_max_graph(g))
        eng.step()
        t0 = time.perf_counter()
        steps = 0
        while True:
            eng.step()
            steps += 1
            el = time.perf_counter() - t0
            if el >= seconds or (max_steps and steps >= max_steps):
                break
    return dict(value=ref_n * ref_n * steps / el, unit=UNIT, cores=cores, kind="port",
                sample=f"{steps} PDHG iterations of oracle/pdhg.py (NumPy restatement of "
                       f"S/solver.py:220-240, fp64) on rgb_disk_pair({ref_n}) (1/{(8192 // ref_n) ** 2}"
                       f" of the 8192^2 cells), {el:.1f} s; NumPy elementwise is single-threaded, "
                       f"BLAS pool = {cores} threads")


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _import_reference():
    """The unmodified reference package (otflux) installed into baseline/_ref
    (DESIGN.md §10); None when it is absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "otflux")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import otflux  # noqa: F401
        from otflux import solver as ref_solver
    except Exception:
        return None
    return otflux, ref_solver


def run_reference(args):
    """The reference's own CPU engine on the bench workload: otflux's
    ``_engine_for("vector", ...)`` (S/solver.py:450-464) stepped with
    ``_Engine.step()`` (S/solver.py:220-240) at the grid our arm runs per GPU
    (8192^2 rgb_disk_pair from the reference's own generator,
    S/problems.py:175-185), BLAS pool = all host cores.  One reference step at
    8192^2 takes ~30 s, so the timed sample is bounded by --ref-seconds
    (at least 2 steps, at most --steps) after one warm-up step; the line says
    how many steps were timed.  Falls back to the NumPy port (oracle/) at
    --ref-n when baseline/_ref is missing."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits

    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    n = global_n(args.n, world)
    cores = os.cpu_count() or 1
    ref = _import_reference()
    if ref is not None:
        otflux, ref_solver = ref
        n_ref = args.n
        l0, l1 = otflux.rgb_disk_pair(otflux.GridSpec(n_ref))
        cfg = otflux.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=1.0,
                                  check_every=args.iters_per_step)
        kind = "reference"
        with threadpool_limits(limits=cores):
            eng = ref_solver._engine_for("vector", l0, l1, cfg, graph=otflux.triangle_graph())
            del l0, l1
            step = eng.step
            what = (f"otflux (baseline/_ref, unmodified) _Engine.step() at {n_ref}^2, "
                    f"{cores} BLAS threads")
            _time_reference(args, step, n_ref, n, world, cores, kind, what)
        return
    from oracle.pdhg import OracleEngine, graph_coef
    import paper_1712_10279_b200 as pk
    from paper_1712_10279_b200 import synthetic

    n_ref = args.ref_n
    l0, l1 = synthetic.rgb_disk_pair(n_ref)
    g = pk.triangle_graph()
    with threadpool_limits(limits=cores):
        eng = OracleEngine("vector", l0 - l1, n_ref, 6.0, norm_u="l12", norm_w="l1", alpha=1.0,
                           chan=graph_coef(3, g.edges, g.costs), lam_chan=pk.lambda_max_graph(g))
        what = (f"NumPy port of the reference engine (oracle/, baseline/_ref missing) at "
                f"{n_ref}^2, {cores} BLAS threads")
        _time_reference(args, eng.step, n_ref, n, world, cores, "port", what)


def _time_reference(args, step, n_ref, n, world, cores, kind, what):
    step()  # warm-up: first-touch page faults of the iterate arrays
    times = []
    t_all = time.perf_counter()
    while len(times) < max(1, args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
        if len(times) >= 2 and time.perf_counter() - t_all >= args.ref_seconds:
            break
    el = float(sum(times))
    steps = len(times)
    value = n_ref * n_ref * steps / el
    sample = (f"{steps} timed PDHG iterations (+1 warm-up) of {what}; "
              f"{el:.1f} s, {1e3 * el / steps:.0f} ms/iteration")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": 1, "ms_per_step": 1e3 * el / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference rgb_disk_pair generator (deterministic)",
        "config": {"workload": f"BASELINE configs[4] vector-OMT 3-channel, {n_ref}^2 on the "
                               f"host (our arm: n={n} global over {world} GPU(s)); one "
                               f"reference step = one PDHG iteration",
                   "n": n, "sample_n": n_ref, "same_config": n_ref == n, "k": K_CH, "ell": ELL,
                   "norms": "l12/l1", "tau": 6.0, "alpha": 1.0,
                   "steps_requested": args.steps, "warmup_requested": args.warmup},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1712_10279_b200 as pk
    from paper_1712_10279_b200 import distributed as D
    from paper_1712_10279_b200 import synthetic

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    multi = world > 1 or args.dist
    if multi:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = global_n(args.n, world)
    b = D.slab_bounds(n, world)
    r0, r1 = b[rank], b[rank + 1]
    ips = args.iters_per_step
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=1.0, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=10 ** 9, check_every=ips)
    graph = pk.triangle_graph()
    l0, l1 = synthetic.rgb_disk_rows(n, r0, r1)
    stream = torch.cuda.Stream()
    uid = D.share_unique_id(dist, rank) if multi else None
    eng = D.make_vector_slab_engine(n, graph, cfg, nranks=world, rank=rank, unique_id=uid,
                                    precision=args.precision, device=local,
                                    stream=stream.cuda_stream)
    m0, m1 = eng.set_marginals(l0, l1)
    info = eng.info()

    # warm-up: W check periods through the run loop (graph capture, clocks)
    eng.run(1e-300, 1e-300, args.warmup * ips, ips)
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.timing(1)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start.record(stream)
        # K check periods = K*ips iterations of the reference run loop
        # (S/solver.py:303-315), checks included, on the device
        hist, it_done, _, _ = eng.run(1e-300, 1e-300, args.steps * ips, ips)
        stop.record(stream)
        torch.cuda.synchronize()
    assert it_done == args.steps * ips
    last = (hist[-1].primal, hist[-1].dual, hist[-1].gap_ratio)
    ms = start.elapsed_time(stop)
    plain_ms, plain_iters = eng.timing(0)
    sweep_ms = plain_ms / max(plain_iters, 1)
    if not sweep_ms > 0:  # no plain iterations timed: fall back to the whole step
        sweep_ms = ms / max(args.steps * ips, 1)
    t = torch.tensor([ms, sweep_ms], device="cuda")
    if multi:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, sweep_ms = float(t[0]), float(t[1])
    cells = float(n) * n
    value = cells * ips * args.steps / (ms * 1e-3)
    local_cells = float(r1 - r0) * n
    balg = bytes_per_cell(args.precision) * local_cells
    peak, peak_src = peaks()
    achieved = balg / (sweep_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "sweep_traffic.json")) as f:
            tr = json.load(f)
        key = f"{args.precision}_{r1 - r0}x{n}"
        traffic = tr.get(key)
    except Exception:
        pass
    eng.close()

    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(args, n, r0, r1, world, rank, local, uid_fn=lambda: (
            D.share_unique_id(dist, rank) if multi else None), multi=multi)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.ref_n, args.cpu_seconds)
    secondary = None
    mroof = None
    ns4096 = None
    if rank == 0 and world == 1 and not args.no_secondary:
        secondary = secondary_configs(args, local)
        mroof = matrix_roofline(args, local)
        ns4096 = north_star_4096(args, local)
    if rank == 0:
        state_gb = info["state_bytes"] * 2 / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic: reference rgb_disk_pair generator (deterministic), zero init",
            "config": {
                "workload": "BASELINE configs[4]: vector-OMT 3-channel RGB disks, row-slab "
                            "sharded, ~8192^2 cells per GPU (weak scaling)",
                "n": n, "cells": int(cells), "k": K_CH, "ell": ELL, "norms": "l12/l1",
                "tau": 6.0, "alpha": 1.0, "iterations_per_step": ips, "check_every": ips,
                "parallelism": f"row-slab x{world}" if world > 1 else "single GPU",
                "l2": f"no flush needed: per-GPU iterate pair {state_gb:.1f} GB >> 126 MB L2",
                "tile": [info["tile_cols"], info["tile_rows"]],
                "regs": [info["regs_plain"], info["regs_check"]],
                "tma_stages": info["tma_stages"], "smem_per_cta": info["smem_bytes"],
                "final_primal": last[0], "final_gap": last[2]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("sweep_tma_kernel (TMA-streamed fused PDHG iteration)"
                                    if info["tma_stages"] else
                                    "sweep_kernel (register-streamed fused PDHG iteration)"),
                         "iterations_per_launch": 1,
                         "bytes_per_launch": balg, "avg_launch_ms": sweep_ms,
                         # whole-step compulsory bandwidth (checks included)
                         "step_frac": value / world * bytes_per_cell(args.precision) / 1e9 / peak,
                         "effective_gbs_per_iteration": value / world
                                                        * bytes_per_cell(args.precision) / 1e9,
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "secondary": secondary,
            "matrix_roofline": mroof,
            "north_star_4096": ns4096,
            # sweeps + one reduction per check + the initial and final evaluate/reduce
            "gpu_launches": args.steps * ips + args.steps + 3,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if multi:
        dist.barrier()
        dist.destroy_process_group()


def secondary_configs(args, device):
    """BASELINE configs[0..3] (the parity configurations) timed on the GPU
    through the engine (device time, CUDA events) next to the reference itself
    (baseline/_ref otflux, solve_* for a bounded number of iterations; the
    NumPy port when it is not installed) on the box's host cores.  Reported
    beside the headline, not as it."""
    import torch
    from threadpoolctl import threadpool_limits

    import paper_1712_10279_b200 as pk
    from oracle.pdhg import OracleEngine
    from paper_1712_10279_b200 import synthetic
    from paper_1712_10279_b200.solver import build_engine

    tri = pk.triangle_graph()
    cases = [
        ("C1 vector 3ch 64^2 x2000 (exact count)", "vector", 64,
         lambda: synthetic.rgb_disk_pair(64), tri, None,
         pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1"), 2000, 2000, 200),
        # tau = 3 = default_tau(256), the pinned C2 (tests/golden/c2_index.json):
        # the reference's termination rule (S/solver.py:294-337) ends it at
        # max_iters = 400 000 without meeting the tolerances
        ("C2 vector 3ch 256^2 to the reference's termination (tau=3, tol_gap 1e-3, tol_feas "
         "1e-5, max_iters 400000: not converged, like the reference)", "vector", 256,
         lambda: synthetic.rgb_disk_pair(256), tri, None,
         pk.SolverConfig(tau=3.0, norm_u="l12", norm_w="l1"), 400_000, 400_000, 20),
        ("C3 matrix 2x2 Hermitian 128^2 l1nuc/l1nuc x300", "matrix", 128,
         lambda: synthetic.blob_pair_k2(128), None, pk.lindblad_pair_k2(),
         pk.SolverConfig(tau=30.0, norm_u="l1nuc", norm_w="l1nuc"), 300, 300, 5),
        ("C4 matrix 3x3 DTI 256^2 l2/l1 x500", "matrix", 256,
         lambda: synthetic.matrix_blob_fixtures(256)[:2], None, pk.default_lindblad3(),
         pk.SolverConfig(tau=30.0, norm_u="l2", norm_w="l1"), 500, 500, 10),
    ]
    out = []
    for name, kind, n, gen, graph, lind, cfg0, iters, max_iters, cpu_iters in cases:
        l0, l1 = gen()
        tol = dict(tol_gap=cfg0.tol_gap, tol_feas=cfg0.tol_feas) if "convergence" in name else \
            dict(tol_gap=1e-300, tol_feas=1e-300)
        cfg = pk.SolverConfig(tau=cfg0.tau, norm_u=cfg0.norm_u, norm_w=cfg0.norm_w, alpha=1.0,
                              max_iters=max_iters, check_every=100, **tol)
        complex_path = kind == "matrix" and (cfg.norm_u.value == "l1nuc" or np.any(np.imag(l0)))
        stream = torch.cuda.Stream()
        eng = build_engine(kind, n, cfg, graph=graph, lindblad=lind, complex_path=complex_path,
                           device=device, stream=stream.cuda_stream)
        eng.set_marginals(l0, l1)
        # warm-up (lazy module load, CUDA-graph capture of the check period),
        # then the timed solve from the reference's zero initial state
        eng.run(1e-300, 1e-300, min(max_iters, 200), cfg.check_every)
        eng.zero_state()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        hist, it, conv, wall = eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
        b.record(stream)
        torch.cuda.synchronize()
        gms = a.elapsed_time(b)
        eng.close()
        # CPU: the reference itself (baseline/_ref otflux, its public solve_*
        # entry point for a bounded number of iterations, one check at the
        # end) when installed, else the NumPy port of its engine
        refmod = _import_reference()
        with threadpool_limits(limits=os.cpu_count() or 1):
            if refmod is not None:
                otflux = refmod[0]
                rcfg = otflux.SolverConfig(tau=cfg.tau, norm_u=cfg.norm_u.value,
                                           norm_w=cfg.norm_w.value, alpha=1.0, tol_gap=1e-300,
                                           tol_feas=1e-300, max_iters=cpu_iters,
                                           check_every=cpu_iters)
                if kind == "vector":
                    args_ref = (otflux.VectorDensity(l0), otflux.VectorDensity(l1),
                                otflux.triangle_graph())
                    fn = otflux.solve_vector
                else:
                    args_ref = (otflux.MatrixDensity(l0), otflux.MatrixDensity(l1),
                                otflux.LindbladSet(np.asarray(lind.matrices)))
                    fn = otflux.solve_matrix
                t0 = time.perf_counter()
                rrep, _ = fn(*args_ref, cfg=rcfg)
                cs = time.perf_counter() - t0
                assert rrep.iterations == cpu_iters
                cpu_kind = "reference"
            else:
                if kind == "vector":
                    ref = OracleEngine("vector", l0 - l1, n, cfg.tau, norm_u=cfg.norm_u.value,
                                       norm_w=cfg.norm_w.value, chan=graph.coefficients(),
                                       lam_chan=pk.lambda_max_graph(graph))
                else:
                    mats = lind.matrices
                    diff = l0 - l1
                    dt = np.complex128 if complex_path else np.float64
                    ref = OracleEngine("matrix", diff if complex_path else np.ascontiguousarray(diff.real),
                                       n, cfg.tau, norm_u=cfg.norm_u.value, norm_w=cfg.norm_w.value,
                                       chan=mats if complex_path else np.ascontiguousarray(np.real(mats)),
                                       lam_chan=pk.lambda_max_L(lind), dtype=dt)
                ref.step()
                t0 = time.perf_counter()
                for _ in range(cpu_iters):
                    ref.step()
                cs = time.perf_counter() - t0
                cpu_kind = "port"
        gpu_rate = n * n * it / (gms * 1e-3)
        cpu_rate = n * n * cpu_iters / cs
        row = dict(config=name, n=n, iterations=it, converged=conv,
                   final_primal=hist[-1].primal, gpu_seconds=gms * 1e-3,
                   gpu_cell_updates_per_s=gpu_rate, cpu_cell_updates_per_s=cpu_rate,
                   cpu_sample_iterations=cpu_iters, cpu_kind=cpu_kind,
                   speedup=gpu_rate / cpu_rate)
        if n == 256 and kind == "vector":
            # the whole reference run, timed once in the build container
            # (tools/make_c2_golden.py; the box cannot run 6 000 s per bench)
            meta = json.load(open(os.path.join(ROOT, "tests", "golden", "c2_index.json")))
            c2 = meta["C2_vec256_tau3"]
            row.update(reference_seconds_full_run=c2["reference_seconds"],
                       reference_iterations=c2["iterations"],
                       reference_converged=c2["converged"],
                       reference_transport_value=c2["transport_value"],
                       same_outcome=(it == c2["iterations"] and conv == c2["converged"]),
                       reference_basis="otflux solve_vector, whole 400000-iteration run, "
                                       "build container (8 vCPU), tools/make_c2_golden.py")
        out.append(row)
    return out


def matrix_roofline(args, device):
    """The matrix payloads (BASELINE C4 / C3 families) at 2048^2, where HBM --
    not launch latency -- bounds them: sweep time from the engine's events and
    the compulsory-bytes roofline fraction, fp64."""
    import torch

    import paper_1712_10279_b200 as pk
    from paper_1712_10279_b200 import synthetic
    from paper_1712_10279_b200.solver import build_engine

    peak, _ = peaks()
    out = []
    n = 2048
    cases = [("C4 family: 3x3 real-symmetric DTI, l2/l1, 2 Lindblad", synthetic.matrix_blob_fixtures,
              pk.default_lindblad3(), ("l2", "l1"), False, 7 * 6 + 2 * 2 * 3),
             ("C3 family: 2x2 complex Hermitian, l1nuc/l1nuc, 2 Lindblad", synthetic.blob_pair_k2,
              pk.lindblad_pair_k2(), ("l1nuc", "l1nuc"), True, (7 + 2 * 2) * 4),
             # the heaviest payloads (3x3 complex Hermitian: 2 + 2 eigensolves per cell)
             ("3x3 complex Hermitian, l1nuc/l1nuc, 2 Lindblad", synthetic.matrix_blob_fixtures,
              pk.default_lindblad3(), ("l1nuc", "l1nuc"), True, (7 + 2 * 2) * 9),
             ("3x3 complex Hermitian, l2/l1, 2 Lindblad", synthetic.matrix_blob_fixtures,
              pk.default_lindblad3(), ("l2", "l1"), True, (7 + 2 * 2) * 9)]
    for name, gen, lind, norms, cplx, words in cases:
        l0, l1 = gen(n)[:2]
        cfg = pk.SolverConfig(tau=30.0, norm_u=norms[0], norm_w=norms[1])
        s = torch.cuda.Stream()
        eng = build_engine("matrix", n, cfg, lindblad=lind, complex_path=cplx, device=device,
                           stream=s.cuda_stream)
        eng.set_marginals(l0, l1)
        eng.run(1e-300, 1e-300, 200, 100)
        eng.timing(1)
        eng.run(1e-300, 1e-300, 400, 100)
        ms, iters = eng.timing(0)
        eng.close()
        per = ms / iters * 1e-3
        balg = words * 8.0 * n * n
        out.append(dict(config=name, n=n, ms_per_iteration=per * 1e3,
                        cell_updates_per_s=n * n / per, bytes_per_cell=words * 8,
                        achieved_gbs=balg / per / 1e9, frac=balg / per / 1e9 / peak))
    return out


def north_star_4096(args, device):
    """BASELINE north_star target: the fused iteration on a 4096^2 3-channel
    vector grid on one GPU, fp64 and fp32, as a fraction of HBM bandwidth
    (sweep time from the engine's events over 500 iterations)."""
    import torch

    import paper_1712_10279_b200 as pk
    from paper_1712_10279_b200 import synthetic
    from paper_1712_10279_b200.solver import build_engine

    peak, _ = peaks()
    n = 4096
    l0, l1 = synthetic.rgb_disk_pair(n)
    out = {}
    for prec in ("f64", "f32"):
        cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1")
        s = torch.cuda.Stream()
        eng = build_engine("vector", n, cfg, graph=pk.triangle_graph(), precision=prec,
                           device=device, stream=s.cuda_stream)
        eng.set_marginals(l0, l1)
        eng.run(1e-300, 1e-300, 300, 100)
        eng.timing(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        eng.run(1e-300, 1e-300, 500, 100)
        b.record(s)
        torch.cuda.synchronize()
        ms, iters = eng.timing(0)
        eng.close()
        per = ms / iters * 1e-3
        balg = bytes_per_cell(prec) * n * n
        out[prec] = dict(sweep_ms=per * 1e3, frac=balg / per / 1e9 / peak,
                         cell_updates_per_s=n * n * 500 / (a.elapsed_time(b) * 1e-3),
                         target_frac=0.70)
    return out


def measure_e2e(args, n, r0, r1, world, rank, local, uid_fn, multi=False):
    """End to end through the public API: host marginals in, host state out."""
    import torch

    import paper_1712_10279_b200 as pk
    from paper_1712_10279_b200 import distributed as D
    from paper_1712_10279_b200 import synthetic

    M = args.e2e_iters
    cfg = pk.SolverConfig(tau=6.0, norm_u="l12", norm_w="l1", alpha=1.0, tol_gap=1e-300,
                          tol_feas=1e-300, max_iters=M, check_every=100)
    graph = pk.triangle_graph()
    l0, l1 = synthetic.rgb_disk_rows(n, r0, r1)
    if not multi:
        a, b = pk.VectorDensity(l0), pk.VectorDensity(l1)

        def call():
            return pk.solve_vector(a, b, graph, cfg=cfg, precision=args.precision, device=local)
    else:
        # one communicator per process, reused by every solve (set up once,
        # like the process group)
        comm = D.SlabCommunicator(uid_fn(), world, rank, local)

        def call():
            return D.solve_vector_rows(l0, l1, graph, n, cfg, nranks=world, rank=rank,
                                       precision=args.precision, device=local, comm=comm)
    call()  # warm-up (allocations, graph capture)
    times = []
    for _ in range(args.e2e_steps):
        if multi:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        rep, st = call()
        times.append(time.perf_counter() - t0)
    t = torch.tensor([float(np.mean(times))], device="cuda")
    if multi:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        comm.close()  # every rank, same point
    sec = float(t[0])
    cells = float(n) * n
    rows_cells = float(r1 - r0) * n
    breakdown = None
    if not multi:
        # one instrumented solve through the engine API (not part of the timed steps)
        from paper_1712_10279_b200.solver import build_engine

        tb = [time.perf_counter()]
        eng = build_engine("vector", n, cfg, graph=graph, precision=args.precision, device=local)
        tb.append(time.perf_counter())
        eng.set_marginals(l0, l1)
        tb.append(time.perf_counter())
        join = eng.prefault_async()  # as solve_vector does (solver._solve)
        eng.run(cfg.tol_gap, cfg.tol_feas, cfg.max_iters, cfg.check_every)
        out = join()
        tb.append(time.perf_counter())
        eng.get_state(out)
        tb.append(time.perf_counter())
        eng.close()
        tb.append(time.perf_counter())
        breakdown = dict(zip(["create", "upload", "run", "download", "destroy"],
                             [round(b - a, 4) for a, b in zip(tb, tb[1:])]))
    return {"value": cells * M / sec, "unit": UNIT, "breakdown_s": breakdown,
            "h2d_bytes_per_step": int(2 * rows_cells * K_CH * 8),
            "d2h_bytes_per_step": int(rows_cells * (2 * K_CH + ELL + K_CH) * 8),
            "iterations_per_step": M, "seconds_per_step": sec,
            "api": "paper_1712_10279_b200.solve_vector (host numpy in/out)" if not multi else
                   "paper_1712_10279_b200.distributed.solve_vector_rows"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

"""bench.py's multi-rank code path on one GPU: launched by torchrun (as the
driver launches N > 1) with --dist, it initialises the NCCL process group,
broadcasts the engine's NCCL unique id with torch.distributed, builds the row
slab engine through distributed.make_vector_slab_engine, times with a barrier
and a MAX all-reduce, and measures e2e through distributed.solve_vector_rows
with a SlabCommunicator -- everything an N-GPU run executes except the
exchange between two devices (covered by the NCCL-loopback slab tests)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_multi_rank_path_world1():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", "29537", "bench.py", "--dist",
           "--side", "1024", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-secondary",
           "--e2e-iters", "200", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 1e9
    assert d["e2e"]["api"] == "paper_1712_10279_b200.distributed.solve_vector_rows"
    assert d["e2e"]["value"] > 1e8
    assert 0.3 < d["roofline"]["frac"] < 1.05

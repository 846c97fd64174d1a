"""bench.py's multi-rank path (the driver's torchrun launch) on a one-GPU
box: two ranks over gloo, both on cuda:0 (FMM_BENCH_BACKEND /
FMM_BENCH_SAME_DEVICE are test-only switches; the driver's runs use NCCL
with one GPU per rank).  Rank 0 alone prints one JSON line with the
max-over-ranks step time and n_gpus = 2; the partitioned evaluation keeps
the single-GPU pair count."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_gloo():
    env = dict(os.environ, FMM_BENCH_BACKEND="gloo", FMM_BENCH_SAME_DEVICE="1", FMM_BENCH_CLOCK_Q="none")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "1", "--config", "C1", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["value"] > 0
    assert d["p2p_pairs"] > 0 and d["e2e"]["value"] > 0
    assert d["accuracy"]["force_err"] < 1e-3  # rank 0 holds the gathered result


def test_bench_two_ranks_sharded_gloo():
    env = dict(os.environ, FMM_BENCH_BACKEND="gloo", FMM_BENCH_SAME_DEVICE="1", FMM_BENCH_CLOCK_Q="none")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "1", "--config", "C1", "--no-cpu-baseline", "--sharded"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "sharded" in d["config"]["parallelism"]


def test_bench_two_ranks_weak_gloo():
    """--weak: the configuration's N per rank (2 x 10,000 bodies in all)."""
    env = dict(os.environ, FMM_BENCH_BACKEND="gloo", FMM_BENCH_SAME_DEVICE="1", FMM_BENCH_CLOCK_Q="none")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "1", "--config", "C1", "--no-cpu-baseline", "--weak"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["config"]["n"] == 20000
    assert d["value"] > 0 and d["accuracy"]["force_err"] < 1e-3

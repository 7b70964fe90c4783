"""The multi-rank bench path in real processes (2 ranks sharing one GPU, gloo
for the host collectives): the peer-memory exchange's CUDA IPC mapping and its
cross-process flag protocol, validated against NCCL-free host collectives, and
the sharded result against the unsharded kernels (bench.py --check)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("p2p,fused", [("1", "1"), ("1", "0"), ("0", "0")])
def test_two_process_sharded_bench_check(cuda_ok, p2p, fused):
    """p2p=1 fused=1: scan -> max over peer memory -> attend fused
    (alaya_sharded_step); fused=0: staged alaya_exch collectives; p2p=0: the
    torch.distributed collectives, which on one shared GPU are gloo's (NCCL
    needs one GPU per rank), and the JSON line must say so."""
    env = dict(os.environ, ALAYA_BENCH_SHARE_GPU="1", ALAYA_P2P=p2p, ALAYA_FUSED_SHARD=fused)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + 2 * int(p2p) + int(fused)), "bench.py",
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--layers", "2", "--ctx", "8192",
           "--batch", "2", "--check", "--no-e2e", "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["sharded_check"]["ok"], d["sharded_check"]
    want = {("1", "1"): "p2p-fused", ("1", "0"): "p2p", ("0", "0"): "gloo"}[(p2p, fused)]
    assert d["config"]["collectives"] == want


@pytest.mark.parametrize("world", [2, 4])
def test_strong_scaling_1m_sharded_check(cuda_ok, world):
    """Config 5 shape: one 1M-token context (B=1), strong scaling (each rank
    holds 1M/N tokens of the SAME session), fused peer path, vs unsharded."""
    env = dict(os.environ, ALAYA_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(29640 + world), "bench.py",
           "--gpus", str(world), "--steps", "1", "--warmup", "3", "--layers", "1", "--ctx", "1048576",
           "--batch", "1", "--check", "--no-e2e", "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["scaling"] == "strong" and d["config"]["batch"] == 1
    assert d["config"]["tokens_per_gpu"] == 1048576 // world
    assert d["sharded_check"]["ok"], d["sharded_check"]
    assert d["config"]["collectives"] == "p2p-fused"

"""The bench's N>1 harness (torchrun, one process per rank, barrier +
max-over-ranks timing, rank 0 prints one JSON line) with two ranks sharing
this GPU through the host-exchange collectives (GSGP_BENCH_HOST_EXCHANGE=1):
the same code path the driver's multi-GPU run takes, minus the NCCL
transport itself (one GPU here).  Also the reference arm under torchrun:
rank 0 prints, the other ranks exit 0 without work."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(*args, env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", *args]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]      # rank 0 only
    return json.loads(lines[0])


def test_bench_two_ranks_host_exchange():
    d = _torchrun("--gpus", "2", "--config", "c2", "--steps", "5", "--warmup", "3", "--no-cpu-baseline",
                  "--no-secondary", env_extra={"GSGP_BENCH_HOST_EXCHANGE": "1"})
    assert d["n_gpus"] == 2 and d["steps"] == 5 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["parallelism"].startswith("case-shard x2")
    assert d["gpu_launches"] > 0 and d["roofline"]["frac"] > 0


def test_reference_arm_under_torchrun_prints_once():
    d = _torchrun("--impl", "reference", "--gpus", "2", "--config", "c1", "--steps", "3", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] in ("reference", "port")

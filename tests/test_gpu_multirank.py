"""The multi-rank bench path (what the driver's scaling run launches), on one
GPU: two torchrun ranks share cuda:0 with gloo as the control plane
(BENCH_DIST_BACKEND=gloo); rank 0 alone prints one JSON line with the
whole-job value, max-over-ranks timing and n_gpus = 2."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("extra", [[], ["--workload", "c5", "--set", "num_nodes=200000"],
                                   ["--set", "gids_shared_cache=true", "--set", "cache_lines=20000"]],
                         ids=["replicas", "sharded", "owner_cache"])
def test_two_rank_bench_prints_one_line(extra):
    env = {**os.environ, "BENCH_DIST_BACKEND": "gloo", "PYTHONPATH": str(ROOT)}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", "c1"] + extra
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["parallelism"] == "dp2"

"""bench.py's driver contract, checked on the CPU: the reference arm (the
oracle port on the host cores) prints one JSON line with the keys the driver
reads, and the workload table names every BASELINE.json config shape."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_prints_one_contract_line():
    env = {**os.environ, "PYTHONPATH": str(ROOT)}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--workload", "c1", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_workloads_cover_the_baseline_configs():
    sys.path.insert(0, str(ROOT))
    import bench
    names = " ".join(bench.WORKLOAD_NAMES.values())
    for shape in ("100K nodes", "1M nodes", "10M nodes", "111,059,956 nodes", "100M nodes"):
        assert shape in names, shape
    assert set(bench.WORKLOADS) == set(bench.WORKLOAD_NAMES) == set(bench.L2_NOTE) == \
        set(bench.DEFAULT_POLICY)

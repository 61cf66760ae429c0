"""Host-side profile of Dataloader.next_batch (cProfile) at a bench workload.

    python tools/profile_host.py [c1|c2|...] [steps]

Prints the top functions by self time and by cumulative time; the device work
is asynchronous, so this shows where the e2e pass spends host time when the
device pipeline is faster than the host (C1).
"""
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_16384_b200 import Dataloader, make_config  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
cfg = make_config({**bench.WORKLOADS[wl], "gids_policy": bench.DEFAULT_POLICY[wl]})
dl = Dataloader(cfg)
for _ in range(20):
    dl.next_batch()
torch.cuda.synchronize()
calls = {"sample": 0}
_launch = dl._launch_sample


def _counted():
    calls["sample"] += 1
    return _launch()


dl._launch_sample = _counted
tr0 = len(dl._trace) if dl._trace is not None else 0
t0 = time.perf_counter()
for _ in range(steps):
    dl.next_batch()
torch.cuda.synchronize()
print(f"{wl}: {(time.perf_counter() - t0) / steps * 1e3:.3f} ms per next_batch (no profiler), "
      f"{calls['sample']} sample launches, {len(dl._pending)} pending, {len(dl._spec)} speculated")
if dl._trace is not None:  # GIDS_TRACE_HOST=1: run_ahead / out block / serve+speculate+precount /
    # counts wait / serve alone / speculate alone
    import numpy as np
    tr = np.array(dl._trace[tr0:]) * 1e3
    print("trace ms median:", np.round(np.median(tr, axis=0), 4), "p90:",
          np.round(np.percentile(tr, 90, axis=0), 4))
pr = cProfile.Profile()
pr.enable()
for _ in range(steps):
    dl.next_batch()
torch.cuda.synchronize()
pr.disable()
for key in ("tottime", "cumulative"):
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats(key).print_stats(30)
    print(s.getvalue())
dl.close()

"""Inclusive host time per call of the functions on Dataloader.next_batch's
path (perf_counter wrappers, ~0.3 us each; no profiler), at a bench workload.

    python tools/host_breakdown.py [c1|c2|...] [steps]
"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2306_16384_b200 import Dataloader, _native, make_config  # noqa: E402
from paper_2306_16384_b200 import loader as L  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
acc = collections.defaultdict(lambda: [0, 0])
samples = collections.defaultdict(list)


def wrap(owner, name, label=None):
    f = getattr(owner, name)
    key = label or f"{getattr(owner, '__name__', type(owner).__name__)}.{name}"

    def w(*a, **k):
        t = time.perf_counter_ns()
        try:
            return f(*a, **k)
        finally:
            e = acc[key]
            e[0] += 1
            d = time.perf_counter_ns() - t
            e[1] += d
            samples[key].append(d)
    setattr(owner, name, w)


for n in ("next_batch", "run_ahead", "_sample_one", "_launch_sample", "_speculate", "_resolve",
          "_out_block", "_account", "_storage_at_least"):
    wrap(L.Dataloader, n)
for n in ("sample", "sample_export_async", "sample_async", "contribution_async", "window_push",
          "window_pop", "serve", "serve_shift", "serve_counts", "wait_served"):
    wrap(_native.Handle, n)
wrap(L._Slots, "take")
wrap(L, "check_seeds", "check_seeds")
wrap(L, "pcg_words", "pcg_words")
wrap(L, "MiniBatch", "MiniBatch()")
wrap(L._Queued, "resolve")
wrap(torch.cuda.Event, "record", "Event.record")
wrap(torch.cuda.Stream, "wait_event", "Stream.wait_event")
wrap(torch.cuda, "current_stream", "torch.cuda.current_stream")
wrap(torch.cuda.Event, "synchronize", "Event.synchronize")
wrap(torch.cuda, "Event", "Event()")

ready = collections.Counter()
_so = L.Dataloader._sample_one


def _sample_one_probe(self):
    if self._spec:
        ready["spec sampled ready at admission"] += bool(self._spec[0].event.query())
        ready["spec admissions"] += 1
    return _so(self)


L.Dataloader._sample_one = _sample_one_probe
_rs = L._Queued.resolve


def _resolve_probe(self, *a):
    if self.batch is None:
        ready["contribution ready at resolve"] += bool(self.event.query())
        ready["resolves"] += 1
    return _rs(self, *a)


L._Queued.resolve = _resolve_probe
cfg = make_config({**bench.WORKLOADS[wl], "gids_policy": bench.DEFAULT_POLICY[wl]})
dl = Dataloader(cfg)
for n in ("push_iteration", "pop_iteration"):
    wrap(type(dl.window), n)
for _ in range(40):
    dl.next_batch()
torch.cuda.synchronize()
acc.clear()
samples.clear()
ready.clear()
ms0 = torch.cuda.memory_stats()
t0 = time.perf_counter()
for _ in range(steps):
    dl.next_batch()
torch.cuda.synchronize()
el = (time.perf_counter() - t0) / steps * 1e6
print(f"{wl}: {el:.1f} us per next_batch (with wrappers)")
ms1 = torch.cuda.memory_stats()
print("allocator:", {k: ms1.get(k, 0) - ms0.get(k, 0) for k in
                     ("num_device_alloc", "num_device_free", "num_alloc_retries",
                      "num_sync_all_streams", "allocation.all.allocated")})
for k, (c, ns) in sorted(acc.items(), key=lambda x: -x[1][1]):
    sm = sorted(samples[k])
    print(f"  {k:40s} calls/batch {c / steps:5.2f}  us/call {ns / c / 1e3:7.2f}  "
          f"us/batch {ns / steps / 1e3:7.2f}  median {sm[len(sm) // 2] / 1e3:7.2f}  "
          f"p90 {sm[int(len(sm) * 0.9)] / 1e3:7.2f}")
print("event readiness:", dict(ready))
torch.cuda.synchronize()
for label, shape in (("out block", (dl._unique_cap, dl.features.dim)), ("4 MB", (1024, 1024))):
    ts = []
    for _ in range(50):
        t = time.perf_counter_ns()
        b = dl._empty_on(dl._gat, shape, torch.float32)
        ts.append(time.perf_counter_ns() - t)
        del b
    ts.sort()
    print(f"_empty_on({label}) idle: median {ts[25] / 1e3:.2f} us")
dl.close()

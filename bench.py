"""bench.py -- GIDS sampling + tiered feature gather on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gids|reference]
                  [--workload c4|c1|c2|c2p|c3|c5|c5v] [--policy exact|setassoc]

Default workload: C4, BASELINE.json configs[3] (the north-star config).

A step is one ``Dataloader.next_batch()``: sample a minibatch (CSC walk in
HBM), lookahead-window update, cache policy, and the tier-chain gather of
every unique node's feature row into a (U, dim) fp32 tensor on the GPU.
Prints ONE JSON line (rank 0).  Under torchrun each rank serves its own
batch subsequence (data-parallel, no data-path collective, weak scaling).

--impl reference times the reference algorithm on the host cores: the CPU
oracle (oracle/, a C restatement pinned to the reference's own outputs) in
one process per core, each serving its own batch stream.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "sampled+gathered minibatches/sec"
WORKLOADS = {
    # BASELINE.json configs[1]: IGB-small shape, 10% cache + 10% constant CPU buffer
    "c2": dict(num_nodes=1_000_000, avg_degree=12.0, degree_model="uniform", feature_dim=1024,
               fanouts=[10, 15], batch_size=1024, cache_lines=100_000, buffer_fraction=0.10,
               window_depth=8, consume_rate=0.0, seed=42),
    # configs[0]: 100K nodes, everything fits the GPU cache
    # (one permutation epoch is only 97 batches here, so seeds are drawn uniformly)
    "c1": dict(num_nodes=100_000, avg_degree=12.0, degree_model="uniform", feature_dim=1024,
               fanouts=[10, 15], batch_size=1024, cache_lines=100_000, buffer_fraction=0.0,
               window_depth=8, consume_rate=0.0, seed=42, seed_mode="uniform",
               iterations=20_000),
    # configs[2]: IGB-medium shape; 2,097,152 lines (8 GiB of
    # 4 KiB pages), 10% buffer = 1M rows, misses served by the storage tier
    "c3": dict(num_nodes=10_000_000, avg_degree=12.0, degree_model="uniform", feature_dim=1024,
               fanouts=[10, 15], batch_size=1024, cache_lines=2_097_152, buffer_fraction=0.10,
               window_depth=8, consume_rate=0.0, seed=42, gids_generator="device"),
    # C2 with the reference's powerlaw degree model (the locality variant)
    "c2p": dict(num_nodes=1_000_000, avg_degree=12.0, degree_model="powerlaw",
                feature_dim=1024, fanouts=[10, 15], batch_size=1024, cache_lines=100_000,
                buffer_fraction=0.10, window_depth=8, consume_rate=0.0, seed=42),
    # configs[3]: ogbn-papers100M shape, 1 GPU; SURVEY.md s8 C4:
    # 2,097,152 cache lines (8 GiB of 4 KiB pages), 10% constant CPU buffer
    "c4": dict(num_nodes=111_059_956, avg_degree=1_615_685_872 / 111_059_956,
               degree_model="uniform", feature_dim=128, fanouts=[15, 10, 5], batch_size=4096,
               cache_lines=2_097_152, buffer_fraction=0.10, window_depth=8, consume_rate=0.0,
               seed=42, gids_generator="device"),
    # configs[4]: IGB-large shape, 409.6 GB table sharded over the
    # ranks' HBM, remote rows read over NVLink; needs >= 3 GPUs
    "c5": dict(num_nodes=100_000_000, avg_degree=1_223_571_364 / 100_000_000,
               degree_model="uniform", feature_dim=1024, fanouts=[10, 15], batch_size=1024,
               cache_lines=0, buffer_fraction=0.0, window_depth=8, consume_rate=0.0, seed=42,
               gids_generator="device", gids_sharded_table=True),
    # C5's graph (100M nodes, 1.22B edges) on ONE GPU: the sharded-table path
    # with 8 virtual shards in this GPU's HBM, rows cut to 128-d (51.2 GB) so
    # the table fits -- a proxy for one rank of C5, not C5
    "c5v": dict(num_nodes=100_000_000, avg_degree=1_223_571_364 / 100_000_000,
                degree_model="uniform", feature_dim=128, fanouts=[10, 15], batch_size=1024,
                cache_lines=0, buffer_fraction=0.0, window_depth=8, consume_rate=0.0, seed=42,
                gids_generator="device", gids_sharded_table=True, gids_virtual_shards=8),
}
DEFAULT_POLICY = {"c1": "exact", "c2": "exact", "c2p": "exact", "c3": "exact",
                  "c4": "exact", "c5": "exact", "c5v": "exact"}
WORKLOAD_NAMES = {
    "c2": "IGB-small-shaped 1M nodes / 12M edges (uniform), 1024-d fp32, fanout [10,15], "
          "batch 1024, cache 100K lines (10%) + 10% constant CPU buffer, W=8",
    "c1": "synthetic 100K nodes / 1.2M edges (uniform), 1024-d fp32, fanout [10,15], "
          "batch 1024, all rows fit the GPU cache, W=8",
    "c3": "IGB-medium-shaped 10M nodes / 120M edges (uniform), 1024-d fp32, fanout [10,15], "
          "batch 1024, cache 2,097,152 lines + 10% constant CPU buffer, W=8",
    "c2p": "IGB-small-shaped 1M nodes / 12M edges (powerlaw), 1024-d fp32, fanout [10,15], "
           "batch 1024, cache 100K lines (10%) + 10% constant CPU buffer, W=8",
    "c4": "ogbn-papers100M-shaped 111,059,956 nodes / 1,615,685,872 edges (uniform), 128-d "
          "fp32, fanout [15,10,5], batch 4096, cache 2,097,152 lines + 10% constant CPU "
          "buffer, W=8, 1 GPU",
    "c5v": "C5 graph (100M nodes / 1,223,571,364 edges) on one GPU: 8 virtual HBM shards, "
           "128-d rows (51.2 GB), fanout [10,15], batch 1024 -- a one-rank proxy of C5",
    "c5": "IGB-large-shaped 100M nodes / 1,223,571,364 edges (uniform), 1024-d fp32 "
          "(409.6 GB) sharded over the ranks' HBM, NVLink peer loads, fanout [10,15], "
          "batch 1024 per GPU",
}
L2_NOTE = {"c1": "inputs larger than L2 (410 MB HBM cache, 282 MB gathered per step)",
           "c2": "inputs larger than L2 (4.1 GB host table, 410 MB HBM cache)",
           "c3": "inputs larger than L2 (41 GB host table, 8.6 GB HBM cache)",
           "c2p": "inputs larger than L2 (4.1 GB host table, 410 MB HBM cache)",
           "c4": "inputs larger than L2 (56.9 GB host table, 1.07 GB HBM cache, 7.4 GB graph)",
           "c5": "inputs larger than L2 (409.6 GB table in HBM shards, 5.7 GB graph)",
           "c5v": "inputs larger than L2 (51.2 GB table in HBM shards, 5.7 GB graph)"}


def bench_config(workload: str, policy: str) -> dict:
    """`config` of the JSON line -- identical in both arms (the driver compares them)."""
    return {"workload": WORKLOAD_NAMES[workload], "policy": policy, "l2": L2_NOTE[workload]}


def load_peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def bind_to_gpu_numa(dev: int) -> dict:
    """Pin this rank's threads to the CPUs of its GPU's NUMA node before any
    host allocation, so the pinned tiers (first-touched by the allocating
    thread) sit on the socket whose root complex the GPU hangs off and the
    host-link reads do not cross the inter-socket link.  Best effort."""
    import torch
    try:
        p = torch.cuda.get_device_properties(dev)
        bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        base = Path("/sys/bus/pci/devices") / bdf
        node = int((base / "numa_node").read_text())
        cpus = set()
        for part in (base / "local_cpulist").read_text().strip().split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0) or cpus
        if cpus and len(cpus) < os.cpu_count():
            os.sched_setaffinity(0, cpus)
        return {"pci": bdf, "numa_node": node, "cpus": len(os.sched_getaffinity(0))}
    except Exception as e:  # no sysfs / single-socket box: nothing to do
        return {"skipped": repr(e)[:80]}


def load_traffic() -> dict:
    """dram read+write bytes per launch of each workload's dominant kernel,
    from one committed `ncu --set full` capture (profiles/ncu_traffic.json)."""
    try:
        return json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
    except Exception:
        return {}


class _ClockSampler:
    """SM clock and throttle reasons sampled in-process through NVML every
    250 ms while the timed region runs (nvidia-smi as a polling subprocess
    takes driver locks often enough to disturb the e2e pass)."""

    NAMES = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
             "sw_power_cap": 0x4}

    def __init__(self, dev: int):
        import threading
        self.sm, self.smax, self.reasons, self.err = [], [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        except Exception as e:  # no NVML: report it, keep timing
            self._nv, self.err = None, repr(e)[:120]
            return
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.smax.append(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.NAMES.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception as e:
                self.err = repr(e)[:120]
            self._stop.wait(0.25)

    def stop(self) -> dict:
        if self._nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"]}
        self._stop.set()
        self._t.join()
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None,
                "sm_max_mhz": max(self.smax) if self.smax else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "NVML in-process, 250 ms"}


def host_link_peak_gbs(dev: int) -> float:
    """Pinned host -> HBM copy bandwidth (the storage / constant-buffer tier link)."""
    import torch
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(4):
        d.copy_(h, non_blocking=True)
    e.record()
    torch.cuda.synchronize(dev)
    bw = 4 * n / (s.elapsed_time(e) * 1e-3) / 1e9
    del h, d
    return bw


def oracle_inputs(cfg, graph=None, table=None, buffer_nodes=None, stream_seed=None) -> dict:
    """Inputs of the CPU oracle loader for ``cfg``: graph / rows / pinned set are
    reused when given; the batch and RNG streams derive from ``stream_seed``
    (default cfg.seed) exactly as Dataloader derives them."""
    from _setup import resolve
    from paper_2306_16384_b200.loader import _seed_stream
    from paper_2306_16384_b200.sampling import pcg_words
    if graph is None and cfg.gids_generator == "device":
        graph, buffer_nodes = host_device_shape(cfg)
    elif graph is None:
        r = resolve(cfg, with_table=table is None)
        graph, buffer_nodes = r["graph"], r["buffer_nodes"]
        table = r["table"] if table is None else table
    ss = np.random.SeedSequence(cfg.seed if stream_seed is None else stream_seed).spawn(6)
    evict_seed = int(ss[4].generate_state(1)[0])
    from paper_2306_16384_b200.storage_model import required_accesses
    return dict(graph=graph, table=table, buffer_nodes=buffer_nodes,
                batches=_seed_stream(cfg, graph.num_nodes, ss[5], ss[3]),
                sampler_words=pcg_words(np.random.default_rng(ss[2])),
                evict_words=pcg_words(np.random.default_rng(evict_seed)), evict_seed=evict_seed,
                base_threshold=required_accesses(cfg.ssd_spec(), cfg.target_fraction))


def host_device_shape(cfg):
    """Graph and pinned set of a gids_generator='device' config built on the host
    cores by the oracle's restatements (the same generator definition and the
    float64-identical reverse PageRank), for the CPU legs."""
    from oracle import oracle as O
    from paper_2306_16384_b200.csc import GraphCsc
    threads = len(os.sched_getaffinity(0))
    graph_ss = np.random.SeedSequence(cfg.seed).spawn(6)[0]
    n, e = cfg.num_nodes, int(round(cfg.num_nodes * cfg.avg_degree))
    ip, ix = O.generate_uniform(n, e, int(graph_ss.generate_state(1)[0]), threads=threads)
    g = GraphCsc(num_nodes=n, num_edges=e, indptr=ip, indices=ix)
    row_bytes = cfg.feature_dim * 4
    k = cfg.resolved_buffer_bytes(n, row_bytes) // row_bytes
    if k <= 0:
        return g, np.empty(0, np.int64)
    scores, _, _ = O.reverse_pagerank(ip, ix, threads=threads)
    # top_k_nodes (cpu_buffer.py:102-109): descending score, ties to the lower id
    return g, np.argsort(-scores, kind="stable")[:k].astype(np.int64)


def oracle_loader(cfg, r, buffer_rows=None):
    from oracle import oracle as O
    return O.OracleLoader(r["graph"].indptr, r["graph"].indices, r["table"], r["buffer_nodes"],
                          r["batches"], cfg.fanouts, r["sampler_words"], r["evict_words"],
                          cfg.resolved_cache_lines(), cfg.window_depth, r["base_threshold"],
                          policy=cfg.gids_policy, evict_key=r["evict_seed"], keep_rows=False,
                          buffer_rows=buffer_rows)


def cpu_baseline_sample(cfg, dl, seconds: float = 12.0) -> dict:
    """The oracle loader (C restatement of the reference path), 1 host thread,
    on the same workload and graph: batches served in ~``seconds``."""
    r = oracle_inputs(cfg, dl.graph, dl.features.table, dl.buffer.node_ids)
    ld = oracle_loader(cfg, r, buffer_rows=dl.buffer.rows)
    ld.next_batch()  # warm
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < seconds:
        ld.next_batch()
        n += 1
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "minibatches/s", "cores": 1, "kind": "port",
            "sample": f"{n} consecutive batches after 1 warm batch, {dt:.1f}s, "
                      f"policy={cfg.gids_policy}, same graph and rows as the GPU run"}


def _gc_probe(stop=None):
    """Durations (ms) of the Python cyclic collector's passes: a list filled
    by a gc callback until _gc_probe(stop=that list) removes it."""
    import gc
    if stop is not None:
        for cb in list(gc.callbacks):
            if getattr(cb, "_gids_probe", None) is stop:
                gc.callbacks.remove(cb)
        return stop
    out, t = [], [0.0]

    def cb(phase, info):
        if phase == "start":
            t[0] = time.perf_counter()
        else:
            out.append((time.perf_counter() - t[0]) * 1e3)
    cb._gids_probe = out
    gc.callbacks.append(cb)
    return out


def _timeline(dl):
    """GIDS_TRACE_HOST=1: (decisions done, rows done) per batch of the last
    timed steps, ms after the first batch's decisions (device clock)."""
    tl = getattr(dl, "_timeline", None)
    if not tl:
        return None
    tl = tl[-12:]
    base = tl[0][0]
    return [[round(base.elapsed_time(d), 3), round(base.elapsed_time(g), 3)] for d, g in tl]


def decision_kernel(cfg, h, ctl_ms, gat_ms, tiers, steps):
    """The cache-decision stream's kernel when the exact (reference) policy
    runs it: k_exact_par, the reference's sequential CacheState.access over a
    batch decided by one CTA -- latency-bound on one SM (no bandwidth or
    tensor roofline applies), so it is reported by its own unit costs next
    to the gather's roofline."""
    if cfg.gids_policy != "exact" or not ctl_ms:
        return None
    st = h.exact_par_stats()
    accesses = float(tiers[0] + tiers[1] + tiers[2]) / steps  # (bypasses are among 1, 2)
    return {"kernel": "k_exact_par" if st["batches"] else "k_exact_seq",
            "bound": "latency (one SM: the reference policy's sequential eviction chain)",
            "ms_per_batch": ctl_ms, "hidden_under_gather": ctl_ms <= gat_ms,
            "ns_per_access": ctl_ms * 1e6 / accesses if accesses else None,
            "rounds_per_batch": st["rounds"] / st["batches"] if st["batches"] else None,
            "note": "step is bound by this stream when ms_per_batch > the gather's; "
                    "profiles/r02_exact_par_*.txt"}


_SHARED: dict = {}


def _ref_worker(proc, steps, budget_s, q):
    cfg, base = _SHARED["cfg"], _SHARED["base"]
    r = oracle_inputs(cfg, base["graph"], base["table"], base["buffer_nodes"],
                      stream_seed=cfg.seed + proc)
    ld = oracle_loader(cfg, r, buffer_rows=base["buffer_rows"])
    times = []
    t_start = time.perf_counter()
    for i in range(steps):
        t0 = time.perf_counter()
        ld.next_batch()
        times.append(time.perf_counter() - t0)
        if i >= 1 and time.perf_counter() - t_start > budget_s:
            break  # bounded sample: the run must end within a few minutes
    q.put(times)


def run_reference(args, cfg_dict) -> None:
    """--impl reference: the oracle port of the reference path on every host core.

    Setup (graph, rows, constant-buffer choice) is built once and shared by
    fork; each of P processes then serves its own batch stream (seed 42+p).
    A step is one batch per process; value = sum over processes of
    timed batches / their time."""
    import multiprocessing as mp

    from oracle import oracle as O
    from paper_2306_16384_b200 import make_config
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = make_config(cfg_dict)
    procs = len(os.sched_getaffinity(0))
    t_setup = time.perf_counter()
    base = oracle_inputs(cfg, table=np.zeros((1, 1), np.float32))
    g = base["graph"]
    feat_seed = int(np.random.SeedSequence(cfg.seed).spawn(6)[1].generate_state(1)[0])
    base["table"] = O.feature_table(feat_seed, g.num_nodes, cfg.feature_dim, threads=procs)
    base["buffer_rows"] = np.ascontiguousarray(base["table"][base["buffer_nodes"]])
    setup_s = time.perf_counter() - t_setup
    _SHARED.update(cfg=cfg, base=base)
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    total = args.warmup + args.steps
    budget_s = 150.0
    ps = [ctx.Process(target=_ref_worker, args=(p, total, budget_s, q)) for p in range(procs)]
    for p in ps:
        p.start()
    results = [q.get() for _ in ps]
    for p in ps:
        p.join()
    # per process: timed batches after the warm-up ones (at least one timed)
    timed = [t[min(args.warmup, len(t) - 1):] for t in results]
    rates = [len(t) / sum(t) for t in timed]
    value = float(sum(rates))
    step_ms = float(np.mean([np.mean(t) for t in timed]) * 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "minibatches/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": bench_config(args.workload, cfg.gids_policy),
            "cpu_baseline": {"value": value, "unit": "minibatches/s", "cores": procs,
                             "kind": "port",
                             "sample": f"{procs} processes x {min(len(t) for t in timed)}-"
                                       f"{max(len(t) for t in timed)} timed batches each "
                                       f"(+{args.warmup} warm, {budget_s:.0f}s cap), streams "
                                       f"seeded {cfg.seed}+p; setup {setup_s:.0f}s"},
            "e2e": {"value": value, "unit": "minibatches/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="gids", choices=["gids", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--policy", default=None, choices=["exact", "setassoc"],
                    help="cache policy (default: exact at c1/c2, setassoc at c4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--set", action="append", default=[], metavar="KEY=VALUE",
                    help="override a PipelineConfig key of the workload (experiments)")
    args = ap.parse_args()
    # the driver's --warmup is honoured as given (both arms); the default of
    # 10 matches the paper's GPU-cache warm-up
    args.policy = args.policy or DEFAULT_POLICY[args.workload]
    cfg_dict = {**WORKLOADS[args.workload], "gids_policy": args.policy}
    for kv in args.set:
        k, v = kv.split("=", 1)
        try:
            cfg_dict[k] = json.loads(v)
        except json.JSONDecodeError:
            cfg_dict[k] = v

    if args.impl == "reference":
        run_reference(args, cfg_dict)
        return

    import torch
    import torch.distributed as dist

    from paper_2306_16384_b200 import Dataloader, make_config

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if cfg_dict.get("gids_sharded_table"):
        per_gpu = 1 if cfg_dict.get("gids_virtual_shards") else world
        shard_gb = cfg_dict["num_nodes"] * cfg_dict["feature_dim"] * 4 / per_gpu / 1e9
        if shard_gb > 150:  # HBM left for the graph and workspaces on a 180 GB B200
            if rank == 0:
                print(json.dumps({"metric": METRIC, "workload": WORKLOAD_NAMES[args.workload],
                                  "n_gpus": world, "unavailable": f"the sharded table needs "
                                  f"{shard_gb:.0f} GB of HBM per GPU at {world} GPU(s); C5's "
                                  f"409.6 GB needs >= 3 GPUs"}), flush=True)
            return
    # BENCH_DIST_BACKEND=gloo lets several ranks share one GPU (a plumbing test
    # of the multi-rank path on a single-GPU box; NCCL refuses duplicate GPUs)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if backend == "gloo":
        local = local % torch.cuda.device_count()
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    numa = bind_to_gpu_numa(local) if os.environ.get("BENCH_NUMA_BIND", "1") == "1" else None
    cfg = make_config({**cfg_dict, "gids_device": local, "gids_dp_rank": rank,
                       "gids_dp_world": world})
    t_setup = time.perf_counter()
    dl = Dataloader(cfg)
    setup_s = time.perf_counter() - t_setup
    link_peak = host_link_peak_gbs(local)
    h = dl._h

    for _ in range(args.warmup):
        dl.next_batch()
    torch.cuda.synchronize(local)
    if world > 1:
        dist.barrier()

    # pass 1 (e2e): K steps through the public call, no per-phase events
    steady_profile = os.environ.get("BENCH_PROFILE_STEADY") == "1"
    if steady_profile:  # `ncu --profile-from-start off` captures pass 1 only (warm cache)
        torch.cuda.profiler.start()
    launches0 = h.launch_count()
    clk = _ClockSampler(local)
    rows_host = rows_hbm = sampled = 0
    tiers = np.zeros(4, np.int64)
    shard_rows = np.zeros(2, np.int64)  # sharded table: local, remote
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(local)
    t0 = time.perf_counter()
    start.record()
    call_ms = []  # host time per next_batch call (diagnostic: outliers in the e2e pass)
    gc_ms = _gc_probe()  # Python collector pauses inside the timed steps (diagnostic)
    tr0 = len(dl._trace) if dl._trace is not None else 0
    for _ in range(args.steps):
        th = time.perf_counter()
        mb, rows, st = dl.next_batch()
        call_ms.append((time.perf_counter() - th) * 1e3)
        sampled += st.sampled_nodes
        tiers += (st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses)
        if dl.sharded is not None:
            shard_rows += dl.shard_counts()
    end.record()
    torch.cuda.synchronize(local)
    wall = time.perf_counter() - t0
    _gc_probe(stop=gc_ms)
    trace1 = dl._trace[tr0:] if dl._trace is not None else None
    timeline1 = _timeline(dl)  # (pass 1's last batches)
    if steady_profile:
        torch.cuda.profiler.stop()
    clocks = clk.stop()
    ms = start.elapsed_time(end)
    launches = h.launch_count() - launches0

    # pass 2 (device pipeline): the next K steps with per-phase CUDA events on
    # each launching stream
    if world > 1:
        dist.barrier()
    h.set_profiling(True)
    for _ in range(args.steps):
        dl.next_batch()
    torch.cuda.synchronize(local)
    phases = h.phase_times()
    h.set_profiling(False)
    red_dev = local if backend == "nccl" else "cpu"
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms_max = float(t.item())

    row_bytes = cfg.feature_dim * 4
    host_rows = int(tiers[1] + tiers[2])
    # value: K steps through next_batch timed on the device (CUDA events on the
    # caller's stream, which waits for every batch's gather); e2e: the same K
    # steps on the host wall clock (seed batches in, tier counts read back per
    # step, rows complete) -- max over ranks for both
    t = torch.tensor([wall * 1e3], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    wall_max_ms = float(t.item())
    value = world * args.steps / (ms_max / 1e3)
    e2e_value = world * args.steps / (wall_max_ms / 1e3)
    # device pipeline: sampling (sampling stream), decisions (control stream)
    # and the gather (gather stream) overlap, so a step costs the slowest of
    # the three per-phase sums
    nb = max(1.0, phases["batches"])
    smp_ms = phases["sample_ms"] / nb
    ctl_ms = phases["cache_ms"] / nb
    gat_ms = (phases["gather_hits_ms"] + phases["gather_host_ms"]) / nb
    dev_ms = max(smp_ms, ctl_ms, gat_ms)
    t = torch.tensor([dev_ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    pipeline_bound = world / (float(t.item()) / 1e3)
    gather_gbs = sampled * row_bytes / (ms / 1e3) / 1e9
    # dominant kernel: the host-tier gather (zero-copy reads over the host link)
    host_bytes_per_launch = host_rows * row_bytes / args.steps
    host_ms = phases["gather_host_ms"] / max(1.0, phases["batches"])
    achieved_link = host_bytes_per_launch / (host_ms / 1e3) / 1e9 if host_ms else None
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    hit_ms = phases["gather_hits_ms"] / max(1.0, phases["batches"])
    hit_bytes = 2 * tiers[0] * row_bytes / args.steps  # read line + write row
    # tier-weighted roofline of the whole step: slower of host link and HBM
    hbm_bytes_step = (2 * tiers[0] + host_rows + host_rows) * row_bytes / args.steps
    t_roof = max(host_rows * row_bytes / args.steps / (link_peak * 1e9),
                 hbm_bytes_step / (hbm_peak * 1e9) if hbm_peak else 0.0)
    step_s = ms_max / 1e3 / args.steps
    traffic = load_traffic().get(args.workload)
    if dl.sharded is None and host_ms >= hit_ms:
        roofline = {"bound": "host_link", "kernel": "k_gather_host",
                    "achieved": achieved_link, "peak": link_peak, "unit": "GB/s",
                    "frac": achieved_link / link_peak if achieved_link else None,
                    "traffic": traffic.get("link_bytes_per_launch") if traffic else None,
                    "traffic_kind": "pcie__read_bytes per launch (the host link)",
                    "hbm_traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                    "traffic_source": traffic["source"] if traffic else None,
                    "algorithmic_bytes_per_launch": host_bytes_per_launch,
                    "peak_source": "pinned H2D cudaMemcpy measured in this run "
                                   "(MEASURED_PEAKS.json has no host-link entry); GPU-initiated "
                                   "reads top out at 51.4 GB/s on this link "
                                   "(profiles/r01_hostread_microbench_*.txt)",
                    "hbm_kernel": {"kernel": "k_gather_hits",
                                   "achieved": hit_bytes / (hit_ms / 1e3) / 1e9 if hit_ms else None,
                                   "peak": hbm_peak, "unit": "GB/s"}}
    elif dl.sharded is None:
        # everything (or nearly) is a cache hit: the dominant gather is HBM -> HBM
        hit_gbs = hit_bytes / (hit_ms / 1e3) / 1e9 if hit_ms else None
        roofline = {"bound": "hbm", "kernel": "k_gather_hits", "achieved": hit_gbs,
                    "peak": hbm_peak, "unit": "GB/s",
                    "frac": hit_gbs / hbm_peak if hit_gbs and hbm_peak else None,
                    "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                    "algorithmic_bytes_per_launch": hit_bytes,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)"}
    elif cfg.gids_virtual_shards:
        # all shards in this GPU's HBM: the sharded gather is an HBM copy
        byt = 2 * sampled * row_bytes / args.steps
        gbs = byt / (gat_ms / 1e3) / 1e9 if gat_ms else None
        roofline = {"bound": "hbm", "kernel": "k_gather_shards", "achieved": gbs,
                    "peak": hbm_peak, "unit": "GB/s",
                    "frac": gbs / hbm_peak if gbs and hbm_peak else None, "traffic": None,
                    "algorithmic_bytes_per_launch": byt,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)",
                    "note": "virtual shards: local HBM stands in for the peers' HBM"}
    else:
        # C5: rows come from the owners' HBM; the remote share crosses NVLink
        nvl_peak = peaks.get("nvlink_gbs") or 770.0
        remote_bytes = shard_rows[1] * row_bytes / args.steps
        gat_s = gat_ms / 1e3
        t_roof = max(remote_bytes / (nvl_peak * 1e9),
                     (sampled * 2 * row_bytes / args.steps) / (hbm_peak * 1e9) if hbm_peak else 0)
        roofline = {"bound": "nvlink", "kernel": "k_gather_shards",
                    "achieved": remote_bytes / gat_s / 1e9 if gat_s else None, "peak": nvl_peak,
                    "unit": "GB/s",
                    "frac": remote_bytes / gat_s / 1e9 / nvl_peak if gat_s else None,
                    "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                    "algorithmic_bytes_per_launch": remote_bytes,
                    "peak_source": "MEASURED_PEAKS.json nvlink_gbs" if peaks.get("nvlink_gbs")
                                   else "B200_PROFILING.md: measured peer copy 770 GB/s per "
                                        "direction on this pool (900 nominal)",
                    "rows_local_per_step": float(shard_rows[0]) / args.steps,
                    "rows_remote_per_step": float(shard_rows[1]) / args.steps}
    line = {
        "metric": METRIC, "value": value, "unit": "minibatches/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (reference generate_synthetic graph + synthetic_feature_rows table)",
        "config": bench_config(args.workload, args.policy),
        "parallelism": f"dp{world}", "global_batch": cfg.batch_size * world,
        "gather_gbps": gather_gbs,
        "tiers_per_step": {"sampled": sampled / args.steps,
                           "cache_hits": float(tiers[0]) / args.steps,
                           "cpu_buffer": float(tiers[1]) / args.steps,
                           "storage": float(tiers[2]) / args.steps,
                           "bypasses": float(tiers[3]) / args.steps},
        "phase_ms_per_step": {k: v / max(1.0, phases["batches"]) for k, v in phases.items()
                              if k != "batches"},
        "tier_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof / step_s,
                          "host_link_peak_gbs": link_peak, "hbm_peak_gbs": hbm_peak},
        "roofline": roofline,
        "step_bound": ("sampling stream" if smp_ms >= max(ctl_ms, gat_ms) else
                       "control stream (cache policy)" if ctl_ms >= gat_ms else
                       "gather stream (" + roofline["bound"] + ")"),
        "value_definition": "K steps through Dataloader.next_batch timed with CUDA events on "
                            "the caller's stream (it waits for each batch's gather), after W "
                            "warm-up steps; world x K / max over ranks",
        "device_pipeline_bound": {
            "value": pipeline_bound, "unit": "minibatches/s",
            "ms_per_step": {"sampling": smp_ms, "decisions": ctl_ms, "gather": gat_ms},
            "definition": "1 / max(per-step sampling, decision and gather stream time), "
                          "per-phase CUDA events in a second pass of K steps: the rate if "
                          "the three streams overlapped perfectly and the host cost nothing"},
        "link_ceiling": {
            "value": 1.0 / t_roof if t_roof else None, "unit": "minibatches/s",
            "vs_cpu_baseline": None,
            "note": "tier-weighted roofline rate 1/t_roof: no loader on this host link can "
                    "exceed it; divided by the reference arm's rate it bounds the ratio "
                    "the driver can measure"},
        "e2e": {"value": e2e_value, "unit": "minibatches/s", "ms_per_step": wall_max_ms / args.steps,
                "h2d_bytes_per_step": int(cfg.batch_size * 8 + host_bytes_per_launch),
                "d2h_bytes_per_step": 256,
                "note": "timed through Dataloader.next_batch (the public API): host seed "
                        "batches in, host-tier rows over the link, per-step stats read back"},
        "gpu_launches": launches, "clocks": clocks,
        "exact_par": h.exact_par_stats() if cfg.gids_policy == "exact" else None,
        "decision_kernel": decision_kernel(cfg, h, ctl_ms, gat_ms, tiers, args.steps),
        "storage_file": dl.storage_stats(),
        "numa": numa,
        "e2e_host_trace_slowest_s": (sorted(trace1, key=sum)[-3:] if trace1 else None),
        "e2e_timeline_ms": timeline1,
        "gc_pauses_ms": {"count": len(gc_ms), "max": max(gc_ms) if gc_ms else 0.0,
                         "total": sum(gc_ms)},
        "e2e_host_ms_per_call": {"min": float(np.min(call_ms)), "median": float(np.median(call_ms)),
                                 "p90": float(np.percentile(call_ms, 90)),
                                 "max": float(np.max(call_ms)),
                                 "first5": [round(x, 2) for x in call_ms[:5]]},
        "setup_s": setup_s, "wall_s": wall,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and dl.sharded is None:
        line["cpu_baseline"] = cpu_baseline_sample(cfg, dl, 12.0)
        if t_roof and line["cpu_baseline"]["value"]:
            line["link_ceiling"]["vs_cpu_baseline"] = (1.0 / t_roof) / line["cpu_baseline"]["value"]
    elif rank == 0 and dl.sharded is not None:
        line["cpu_baseline"] = {"value": None, "skipped": "the sharded-table mode has no host "
                                "tiers; its CPU counterpart is the replica loader (c2, c4 lines)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    dl.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

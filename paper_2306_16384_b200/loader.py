"""GIDS Dataloader on the B200: the reference serving loop driving CUDA kernels.

``Dataloader(cfg)`` / ``next_batch()`` / iteration / ``run()`` keep the
reference API (dataloader.py:95-389): the same setup derivation from
``cfg.seed`` (SeedSequence spawn order, dataloader.py:102-147), the same
run-ahead accumulator and lookahead ring (:184-228), the same per-iteration
accounting and CSV (:43-74,301-337).  What changes is where the work runs:

* graph, cache lines, per-node metadata: HBM (libgids handle)
* sampling, window_update, the cache policy, the tier chain and the gather:
  CUDA kernels (csrc/) behind the C ABI (include/gids.h)
* constant CPU buffer and storage tier: pinned host memory read zero-copy
  by the gather kernel

``next_batch`` returns ``(MiniBatch, rows, IterationStats)`` with the batch's
layers / unique nodes and the gathered ``(U, dim)`` fp32 rows as CUDA
tensors; the rows are ordered like ``unique_nodes`` (ascending), exactly as
the reference orders its numpy result.
"""
from __future__ import annotations

import functools
import itertools
import math
import os
import time
from collections import deque
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _native, host_tier
from .csc import (HEADER_BYTES, FeatureStore, GraphCsc, generate_synthetic, load_features,
                  load_graph, pinned_feature_table, write_synthetic_features)
from .feature_cache import GpuCacheView, WindowBuffer
from .hot_buffer import build_constant_buffer, reverse_pagerank_device, top_k_nodes_device
from .sampling import MiniBatch, Sampler, batch_iterator, check_seeds, pcg_words
from .shared_cache import OwnerShardedCache
from .sharded_table import ShardedTable
from .settings import ConfigError, InfeasibleError, PipelineConfig
from .storage_model import exact, fetch_total_us, required_accesses

EMA_EPSILON = 1e-3

CSV_HEADER = ("iteration,sampled_nodes,cache_hits,cpu_buffer_hits,ssd_accesses,"
              "bypasses,redirect_fraction,fetch_time_us,effective_bandwidth_gbps,"
              "cumulative_time_us")


@dataclass(frozen=True)
class IterationStats:
    iteration: int
    sampled_nodes: int
    cache_hits: int
    cpu_buffer_hits: int
    ssd_accesses: int
    bypasses: int
    redirect_fraction: float
    fetch_time_us: float
    effective_bandwidth_bytes_per_s: float
    cumulative_time_us: float

    def csv_row(self) -> str:
        return ",".join([
            str(self.iteration), str(self.sampled_nodes), str(self.cache_hits),
            str(self.cpu_buffer_hits), str(self.ssd_accesses), str(self.bypasses),
            f"{self.redirect_fraction:.6f}", f"{self.fetch_time_us:.3f}",
            f"{self.effective_bandwidth_bytes_per_s / 1e9:.6f}",
            f"{self.cumulative_time_us:.3f}"])


def stats_csv(stats: list[IterationStats]) -> str:
    return "\n".join([CSV_HEADER, *(s.csv_row() for s in stats)]) + "\n"


@dataclass(frozen=True)
class RunSummary:
    iterations_run: int
    sampled_total: int
    cache_hit_ratio: float
    redirect_fraction: float
    mean_bandwidth_bytes_per_s: float
    total_fetch_us: float
    total_train_us: float
    total_time_us: float


def _empty_on(device: int, torch_dev, stream, shape, dtype):
    """torch.empty from `stream`'s allocator pool: the block is written on
    that stream, so a freed block is reused there only after every stream
    recorded on it passed its last use (allocating from the caller's pool
    instead would let the sampler / gather overwrite a block the caller's
    queued kernels still read).  Raw stream switches: torch.cuda.stream()
    costs ~20 us of device-index lookups per use."""
    import torch
    dev0 = torch._C._cuda_getDevice()
    prev = torch._C._cuda_getCurrentStream(device)
    torch._C._cuda_setStream(stream_id=stream.stream_id, device_index=stream.device_index,
                             device_type=stream.device_type)  # (makes `device` current)
    try:
        return torch.empty(shape, dtype=dtype, device=torch_dev)
    finally:
        torch._C._cuda_setStream(stream_id=prev[0], device_index=prev[1], device_type=prev[2])
        if dev0 != device:
            torch._C._cuda_setDevice(dev0)


class _Slots:
    """Equal blocks handed out K at a time from one allocation: each is a
    view, and the allocation returns to torch's pool (after the streams
    recorded on it) when the last of its views is gone."""

    __slots__ = ("_alloc", "_k", "_big", "_next")

    def __init__(self, alloc, k: int):
        self._alloc, self._k, self._big, self._next = alloc, k, None, k

    def take(self):
        if self._next == self._k:
            self._big, self._next = self._alloc(), 0
        v = self._big[self._next]
        self._next += 1
        return v


class _Queued:
    """A sampled batch whose outputs may still be in flight on the control
    stream; ``resolve()`` waits for them (normally long finished) and fixes
    the sizes, the run-ahead contribution and the host Generator's offset."""

    __slots__ = ("seeds", "block", "ecap", "sizes", "sizes_ptr", "event", "batch",
                 "storage_accesses", "error", "counted_at")

    def __init__(self, seeds, block, ecap, sizes, sizes_ptr, event):
        # block: int64 [2 ecap edges | unique nodes] (workspace bounds);
        # sizes: its pinned sizes row (numpy view) at host address sizes_ptr
        self.seeds, self.block, self.ecap, self.sizes, self.sizes_ptr, self.event = \
            seeds, block, ecap, sizes, sizes_ptr, event
        self.batch = None
        self.storage_accesses = None
        self.error = None
        self.counted_at = -1  # serves before its contribution was counted (-1: not yet)

    @property
    def unique_ptr(self) -> int:
        return self.block.data_ptr() + 16 * self.ecap

    def resolve(self, n_layers: int, rng) -> None:
        if self.batch is not None:
            return
        self.event.synchronize()
        sz = self.sizes.tolist()
        lens, n_unique, draws, contrib, overflow = (sz[:n_layers], sz[n_layers],
                                                    sz[n_layers + 1], sz[n_layers + 2],
                                                    sz[n_layers + 3])
        if overflow:
            raise _native.GidsError("sampler workspace bound exceeded")
        layers, off, b = [], 0, self.block
        for ln in lens:
            layers.append(b[2 * off:2 * (off + ln)].view(ln, 2))
            off += ln
        if draws:
            rng.bit_generator.advance(draws)
        self.batch = MiniBatch(seeds=self.seeds, layers=layers,
                               unique_nodes=b[2 * self.ecap:2 * self.ecap + n_unique])
        self.storage_accesses = contrib


def _seed_stream(cfg: PipelineConfig, n: int, work_ss, shuffle_ss):
    """Host seed supply (dataloader.py:163-180), then the data-parallel slice."""
    if cfg.seed_mode == "permutation":
        count = n if cfg.seed_count is None else min(cfg.seed_count, n)
        it = batch_iterator(np.arange(n, dtype=np.int64)[:count], cfg.batch_size,
                            shuffle=cfg.shuffle, rng=np.random.default_rng(shuffle_ss))
    else:
        rng = np.random.default_rng(work_ss)
        count = ((cfg.warmup + cfg.iterations) * cfg.batch_size if cfg.seed_count is None
                 else cfg.seed_count)
        if cfg.seed_mode == "uniform":
            seeds = rng.integers(0, n, size=count)
        else:  # zipf over ids: low ids are hot
            p = np.arange(1, n + 1, dtype=np.float64) ** (-cfg.zipf_a)
            p /= p.sum()
            seeds = rng.choice(n, size=count, p=p)
        it = batch_iterator(seeds, cfg.batch_size, shuffle=False)
    if cfg.gids_dp_world == 1:
        return it
    return (b for i, b in enumerate(it) if i % cfg.gids_dp_world == cfg.gids_dp_rank)


class Dataloader:
    """GIDS dataloader: sampling + tiered feature gather on one B200."""

    def __init__(self, cfg: PipelineConfig):
        if not cfg.gids:
            raise ConfigError("gids=False selects the reference CPU simulator; this package "
                              "implements the GIDS GPU path only")
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("the GIDS dataloader needs a CUDA device (none visible)")
        _native.lib()  # fail loudly when the CUDA library is missing
        self.cfg = cfg
        self.spec = cfg.ssd_spec()
        self.device = cfg.gids_device
        self._torch_dev = torch.device("cuda", self.device)
        torch.cuda.set_device(self.device)

        graph_ss, feat_ss, sampler_ss, shuffle_ss, evict_ss, work_ss = \
            np.random.SeedSequence(cfg.seed).spawn(6)
        self.sharded = None
        self._storage_file = None
        self._file_offset = self._file_page = None
        dev_graph = self._build_graph_and_features(int(graph_ss.generate_state(1)[0]),
                                                   int(feat_ss.generate_state(1)[0]))
        row_bytes = self.features.row_bytes
        if row_bytes > self.spec.page_bytes:
            raise InfeasibleError(f"feature row ({row_bytes} B) exceeds one cache line / page "
                                  f"({self.spec.page_bytes} B)")
        self._build_constant_buffer(dev_graph, row_bytes)

        evict_seed = int(evict_ss.generate_state(1)[0])
        shared = cfg.gids_shared_cache
        # owner-sharded cache: each owner's eviction stream is its own jump of
        # the eviction generator (the replicas' caches all start from it)
        ev_words = pcg_words(np.random.Generator(np.random.PCG64(evict_seed).jumped(
            cfg.gids_dp_rank)) if shared else np.random.default_rng(evict_seed))
        self._h = _native.Handle(
            num_nodes=self.graph.num_nodes, num_edges=self.graph.num_edges,
            feature_dim=self.features.dim, device=self.device,
            cache_lines=0 if self.sharded else cfg.resolved_cache_lines(),
            policy="exact" if self.sharded else cfg.gids_policy, ways=32,
            evict_key=evict_seed, window_depth=cfg.window_depth, fanouts=cfg.fanouts,
            max_seeds=cfg.batch_size,
            eviction_words=ev_words)
        self._h.load_graph_device(*dev_graph)
        del dev_graph
        if self.sharded is not None:
            self._h.set_sharded_table(self.sharded.ptrs, self.sharded.rank)
        elif self._storage_file is not None:
            off = HEADER_BYTES if cfg.graph_path is not None else cfg.gids_storage_offset
            self._h.set_storage_file(self._storage_file, off, self.spec.page_bytes,
                                     io_threads=cfg.gids_io_threads, direct=cfg.gids_io_direct)
            self._file_offset, self._file_page = off, self.spec.page_bytes
        else:
            pinned = self.features.pinned
            self._h.set_backing(pinned if isinstance(pinned, torch.Tensor) else self.features.table,
                                self.graph.num_nodes)
        if self.buffer.pinned is not None:
            self._h.set_constant_buffer(self.buffer.device_ids, self.buffer.pinned)
        else:
            self._h.set_constant_buffer(self.buffer.node_ids, self.buffer.rows)
        # streams: cache decisions (ctl) and row movement (gather), plus sampling
        # and run-ahead admissions below;
        # the decisions of batch b+1 overlap the host-link gather of batch b
        # stream priority: the host link is the bottleneck resource, so by
        # default the gather's blocks are dispatched first when SM slots free
        # up (GIDS_PRIORITY=ctl flips it, for experiments)
        gather_first = os.environ.get("GIDS_PRIORITY", "gather") != "ctl"
        self._ctl = torch.cuda.Stream(self.device, priority=0 if gather_first else -1)
        self._gat = torch.cuda.Stream(self.device, priority=-1 if gather_first else 0)
        # run-ahead contributions (a read of the cache's residency at admission)
        # go on a third stream ordered only after the previous batch's
        # decisions and the batch's own sampling, so the host resolving them
        # never waits behind the speculative sampling queued on ctl; the next
        # decisions wait for them in turn
        self._cnt = torch.cuda.Stream(self.device)
        # sampling has its own stream too: it reads only the graph and the
        # sampler's stream state, so batch b+k is sampled while batch b's
        # decisions run on ctl (the decisions need a batch only after the
        # host resolved it, i.e. after its sampling finished)
        self._smp = torch.cuda.Stream(self.device, priority=0 if gather_first else -1)
        self.cache = GpuCacheView(self._h, self.spec.page_bytes)
        self.window = WindowBuffer(cfg.window_depth, self._h, self._ctl.cuda_stream)
        self.window.defer = True  # (folded into the next serve: gids_serve_shift)
        self.shared = None
        if shared:
            # the handle's window counters serve the owner role (owned parts of
            # every rank's batches); the run-ahead ring stays unbound
            self.window = WindowBuffer(0)
            self.shared = OwnerShardedCache(self._h, cfg.gids_dp_rank, cfg.gids_dp_world,
                                            cfg.window_depth, self.device)
            self._sent = 0
        self._sampler = Sampler(self._h, self.graph.num_nodes, cfg.fanouts)

        self.base_threshold = required_accesses(self.spec, cfg.target_fraction)
        self.redirect_ema = 0.0
        if cfg.gids_dp_world > 1:
            self._sampler_rng = np.random.Generator(
                np.random.PCG64(sampler_ss).jumped(cfg.gids_dp_rank))
        else:
            self._sampler_rng = np.random.default_rng(sampler_ss)
        self._batches = _seed_stream(cfg, self.graph.num_nodes, work_ss, shuffle_ss)
        self._seeds_trusted = True  # (int64 ids in [0, N) by construction)
        self._exhausted = False
        self._seeds_done = False
        self._pending: deque[_Queued] = deque()
        # resolution runs oldest first, so the resolved entries are a prefix
        self._n_resolved = 0
        self._spec: deque[_Queued] = deque()  # sampled ahead, not yet admitted
        self._spec_depth = cfg.gids_speculate
        self._resolved_storage = 0  # sum of resolved contributions of pending batches
        self._ringed = 0
        self._rng_on_device = False
        self._edge_cap, self._unique_cap = self._h.sample_capacity()
        # per-batch blocks come K at a time from one allocation (a torch
        # allocation costs ~15 us of host time in the serving loop): output
        # rows from the gather stream's pool, sampled edges + unique nodes
        # from the sampling stream's
        row_block = self._unique_cap * self.features.dim * 4
        k_out = max(1, min(4, (2 << 30) // max(1, row_block)))
        # (functools.partial over plain values: no reference back to the
        # loader, which must die -- and unmap its host tiers -- when dropped)
        self._out_slots = _Slots(functools.partial(
            _empty_on, self.device, self._torch_dev, self._gat,
            (k_out, self._unique_cap, self.features.dim), torch.float32), k_out)
        smp_block = (2 * self._edge_cap + self._unique_cap) * 8
        k_smp = max(1, min(8, (256 << 20) // max(1, smp_block)))
        self._smp_slots = _Slots(functools.partial(
            _empty_on, self.device, self._torch_dev, self._smp,
            (k_smp, 2 * self._edge_cap + self._unique_cap), torch.int64), k_smp)
        # pre-warm the gather pool with the blocks a pipelined caller keeps
        # live (its batch, the one being gathered, the next one, and one freed
        # but not yet retired)
        warm = [self._out_slots._alloc() for _ in range(2 if k_out > 1 else 4)]
        # ... and the sampling pool with the groups a steady run-ahead window
        # keeps live (a cudaMalloc inside the loop stalled a C4 step by 40-90 ms)
        warm += [self._smp_slots._alloc() for _ in
                 range(-(-(cfg.window_depth + cfg.gids_speculate + 8) // k_smp))]
        del warm
        ring = cfg.runahead_cap + cfg.gids_speculate + 4
        self._sizes = torch.zeros((ring, len(cfg.fanouts) + 5), dtype=torch.int64,
                                  pin_memory=True)
        self._sizes_np = self._sizes.numpy()
        self._sizes_ptr = self._sizes.data_ptr()
        self._seed_stage = torch.empty((ring, cfg.batch_size), dtype=torch.int64,
                                       pin_memory=True).numpy()
        self._cur_streams: dict = {}  # raw caller stream -> torch Stream (record_stream)
        self._sizes_next = 0

        self._iteration = 0
        self._serves = 0  # serves launched (contributions are counted between two)
        # host-time trace of next_batch (diagnostics): run-ahead, output
        # allocation, serve launch, wait for the decisions -- seconds per call
        self._trace = [] if os.environ.get("GIDS_TRACE_HOST") == "1" else None
        self._timeline = []  # with _trace: per batch (decided, gathered) CUDA events
        self._clock_us = Fraction(0)
        self._fetch_us_total = Fraction(0)
        self._train_us_total = Fraction(0)
        self._row_frac = Fraction(row_bytes)
        self._cpu_bytes_per_s = exact(cfg.cpu_gbps) * 10**9
        self._cpu_us_per_row = self._row_frac * 1_000_000 / self._cpu_bytes_per_s
        self._row_us_bytes = self._row_frac * 1_000_000
        self._train_us_per_node = (Fraction(1_000_000) / exact(cfg.consume_rate)
                                   if cfg.consume_rate > 0 else 0)
        self.last_counts = None

    def _build_graph_and_features(self, graph_seed: int, feat_seed: int):
        """Graph (dataloader.py:105-117) and the storage tier: files, the
        reference's generator or the GPU generator; pinned host rows, the
        .gfea file itself, or HBM shards.  Returns the graph in HBM."""
        cfg = self.cfg
        import torch
        self._shared = []  # node-shared host regions (host_tier.py)
        if cfg.graph_path is not None:
            self.graph = load_graph(cfg.graph_path)
            host = load_features(cfg.features_path, mmap=True)
            if host.num_nodes != self.graph.num_nodes:
                raise ConfigError("feature table and graph disagree on node count")
            self._storage_file = str(cfg.features_path) if cfg.gids_storage == "file" else None
            # file tier: the rows stay in the file (memory-mapped for the host API)
            if self._storage_file:
                self.features = host
            elif self._shared_host():
                tok = self._host_token = host_tier.job_token()

                def fill(view):
                    for r in range(0, host.num_nodes, 1 << 18):
                        view[r:r + (1 << 18)] = host.table[r:r + (1 << 18)]
                self._shared.append(host_tier.SharedRegion(
                    f"gids-{tok}-table", (host.num_nodes, host.dim), np.float32,
                    self._host_creator, fill))
                self.features = FeatureStore(num_nodes=host.num_nodes, dim=host.dim,
                                             table=self._shared[-1].array)
            else:
                self.features = self._pin_table(host)
            return self._upload_graph(self.graph)
        if cfg.gids_generator == "device":
            # counter-based uniform generator in HBM (csrc/graph_setup.cu)
            n, e = cfg.num_nodes, int(round(cfg.num_nodes * cfg.avg_degree))
            dev_graph = _native.generate_uniform_graph(self.device, n, e, graph_seed)
            self.graph = GraphCsc(num_nodes=n, num_edges=e,
                                  indptr=dev_graph[0].cpu().numpy().view(np.uint64),
                                  indices=dev_graph[1].cpu().numpy().astype(np.uint64))
        else:
            self.graph = generate_synthetic(cfg.num_nodes, cfg.avg_degree, cfg.degree_model,
                                            seed=graph_seed, exponent=cfg.degree_exponent)
            dev_graph = self._upload_graph(self.graph)
        if cfg.gids_sharded_table:
            # C5: the table lives in the ranks' HBM (sharded_table.py)
            virtual = cfg.gids_virtual_shards > 0
            g = cfg.gids_virtual_shards if virtual else cfg.gids_dp_world
            self.sharded = ShardedTable(cfg.num_nodes, cfg.feature_dim, feat_seed, self.device,
                                        0 if virtual else cfg.gids_dp_rank, g, virtual=virtual)
            self.features = FeatureStore(num_nodes=cfg.num_nodes, dim=cfg.feature_dim,
                                         table=None, seed=feat_seed)
        elif cfg.gids_storage == "file":
            # the synthetic table written once to a .gfea file, then served
            # from the file (csrc/storage_file.cu)
            write_synthetic_features(cfg.gids_storage_path, cfg.num_nodes, cfg.feature_dim,
                                     feat_seed, self.device, offset=cfg.gids_storage_offset)
            table = np.memmap(cfg.gids_storage_path, dtype=np.float32, mode="r",
                              offset=cfg.gids_storage_offset,
                              shape=(cfg.num_nodes, cfg.feature_dim))
            self.features = FeatureStore(num_nodes=cfg.num_nodes, dim=cfg.feature_dim,
                                         table=table, seed=feat_seed)
            self._storage_file = str(cfg.gids_storage_path)
        elif self._shared_host():
            tok = self._host_token = host_tier.job_token()
            n, dim = cfg.num_nodes, cfg.feature_dim
            st = _native.stream_ptr(self.device)

            def fill(view):  # the GPU writes the reference's rows into the mapping
                for r0 in range(0, n, 1 << 20):
                    k = min(1 << 20, n - r0)
                    _native.synthesize_rows(self.device, feat_seed, r0, k, dim,
                                            view[r0:r0 + k].ctypes.data, st)
                torch.cuda.synchronize(self.device)
            self._shared.append(host_tier.SharedRegion(
                f"gids-{tok}-table", (n, dim), np.float32, self._host_creator, fill))
            self.features = FeatureStore(num_nodes=n, dim=dim, table=self._shared[-1].array,
                                         seed=feat_seed)
        else:
            self.features = pinned_feature_table(cfg.num_nodes, cfg.feature_dim, feat_seed,
                                                 self.device)
        return dev_graph

    def _shared_host(self) -> bool:
        """One node-shared host tier (host_tier.py) instead of a private copy."""
        c = self.cfg
        return (c.gids_shared_host and c.gids_dp_world > 1 and host_tier._dist() is not None
                and not c.gids_sharded_table and c.gids_storage == "pinned")

    @property
    def _host_creator(self) -> bool:
        return host_tier.local_rank(self.cfg.gids_dp_rank) == 0

    def _build_constant_buffer(self, dev_graph, row_bytes: int) -> None:
        """ConstantBuffer (dataloader.py:125-135): reverse PageRank + top-k on
        the GPU, float64-identical to cpu_buffer.py:26-109, so the pinned set
        is the reference's."""
        budget = self.cfg.resolved_buffer_bytes(self.graph.num_nodes, row_bytes)
        if budget // row_bytes > 0:
            self.pagerank, dev_scores = reverse_pagerank_device(self.device, *dev_graph)
            chosen = top_k_nodes_device(dev_scores, budget // row_bytes)
            del dev_scores
            pin = True
            if self._shared:  # the buffer's GPU copy joins the node-shared host tier
                def pin(shape, fill):
                    self._shared.append(host_tier.SharedRegion(
                        f"gids-{self._host_token}-buffer", shape, np.float32,
                        self._host_creator, fill))
                    return self._shared[-1].array
            self.buffer = build_constant_buffer(self.pagerank.scores, self.features, budget,
                                                pinned=chosen, pin_memory=pin)
        else:
            self.pagerank = None
            self.buffer = build_constant_buffer(np.empty(0), self.features, 0,
                                                pinned=np.empty(0, dtype=np.int64))
        self._pinned_mask = np.zeros(self.graph.num_nodes, dtype=bool)
        self._pinned_mask[self.buffer.node_ids] = True

    def _empty_on(self, stream, shape, dtype):
        return _empty_on(self.device, self._torch_dev, stream, shape, dtype)

    def _out_block(self):
        """Output rows of one batch: a block of the workspace bound (a view of
        the first U rows is returned), so torch's caching allocator keeps
        cycling the same pre-warmed allocations (exact-size requests, U
        varies, made it cudaMalloc fresh segments, stalling next_batch by
        10-90 ms)."""
        return self._out_slots.take()

    def _upload_graph(self, g: GraphCsc):
        """Host GraphCsc -> (indptr int64, indices int32) CUDA tensors."""
        import torch
        if g.num_nodes >= 1 << 31:
            raise ValueError("the CUDA path stores node ids as int32 (num_nodes < 2^31)")
        ip = torch.from_numpy(np.array(g.indptr, dtype=np.uint64).view(np.int64)).to(
            self._torch_dev)
        ix = torch.from_numpy(np.asarray(g.indices).astype(np.int32)).to(self._torch_dev)
        return ip, ix

    def _pin_table(self, host: FeatureStore) -> FeatureStore:
        import torch
        buf = torch.empty((host.num_nodes, host.dim), dtype=torch.float32, pin_memory=True)
        view = buf.numpy()
        step = 1 << 18
        for r in range(0, host.num_nodes, step):
            view[r:r + step] = host.table[r:r + step]
        return FeatureStore(num_nodes=host.num_nodes, dim=host.dim, table=view, pinned=buf)

    def gids_init(self, offset: int | None = None, cacheline_bytes: int | None = None,
                  num_elements: int | None = None, n_ssd: int | None = None,
                  path: str | None = None) -> dict:
        """The GIDS init call: lays out the backing store
        before the first batch.

        path: serve the storage tier from this file -- fp32 rows of ``dim``
        elements from byte ``offset`` (24 = the .gfea header, graph.py:304-309;
        0 = a raw row dump), read in pages of ``cacheline_bytes`` through the
        page-coalescing accumulator (csrc/storage_file.cu); without a path an
        existing file tier is re-laid-out with the given offset / page.
        num_elements: N * dim, checked against the graph and the table.
        n_ssd: devices the storage tier stripes over -- the accumulator's
        saturation threshold (storage.py:92-104) and the fetch clock scale
        with it (SsdSpec.n_ssd).  Arguments left None keep the current value.
        Returns the resolved layout."""
        import dataclasses
        if self._iteration > 0 or self._pending or self._spec:
            raise ConfigError("gids_init configures the backing store before the first batch")
        n, dim, rb = self.graph.num_nodes, self.features.dim, self.features.row_bytes
        if num_elements is not None and num_elements != n * dim:
            raise ConfigError(f"gids_init num_elements={num_elements} disagrees with the "
                              f"loader ({n * dim} = {n} nodes x {dim})")
        if offset is None:  # keep the current layout (the .gfea header for a new file)
            offset = self._file_offset if self._storage_file is not None else HEADER_BYTES
        if offset < 0:
            raise ConfigError("gids_init offset must be non-negative")
        if n_ssd is not None:
            if n_ssd < 1:
                raise ConfigError("gids_init n_ssd must be >= 1")
            self.spec = dataclasses.replace(self.spec, n_ssd=int(n_ssd))
            self.base_threshold = required_accesses(self.spec, self.cfg.target_fraction)
        page = int(cacheline_bytes) if cacheline_bytes is not None else self.spec.page_bytes
        if rb > page:
            raise InfeasibleError(f"feature row ({rb} B) exceeds one cache line / page "
                                  f"({page} B)")
        if path is not None or (self._storage_file is not None and
                                (offset != self._file_offset or page != self._file_page)):
            if self.sharded is not None:
                raise ConfigError("the HBM-sharded table has no backing file")
            target = str(path) if path is not None else self._storage_file
            if os.path.getsize(target) < offset + n * rb:
                raise ConfigError(f"{target}: shorter than offset + {n} rows x {rb} B")
            self._h.set_storage_file(target, offset, page, io_threads=self.cfg.gids_io_threads,
                                     direct=self.cfg.gids_io_direct)
            table = np.memmap(target, dtype=np.float32, mode="r", offset=offset, shape=(n, dim))
            self.features = FeatureStore(num_nodes=n, dim=dim, table=table,
                                         seed=self.features.seed)
            self._storage_file, self._file_offset, self._file_page = target, offset, page
        return {"offset": self._file_offset if self._storage_file else offset,
                "cacheline_bytes": self._file_page if self._storage_file else page,
                "num_elements": n * dim, "n_ssd": self.spec.n_ssd, "row_bytes": rb,
                "storage": "file" if self._storage_file else
                           ("hbm-sharded" if self.sharded else "pinned"),
                "path": self._storage_file, "base_threshold": self.base_threshold}

    # -- run-ahead accumulator (dataloader.py:184-228)
    def effective_threshold(self) -> int:
        return math.ceil(self.base_threshold / max(EMA_EPSILON, 1.0 - self.redirect_ema))

    @property
    def _pending_storage(self) -> int:
        """Sum of the pending batches' contributions (resolves them all)."""
        for q in itertools.islice(self._pending, self._n_resolved, None):
            self._resolve(q)
        return self._resolved_storage

    def _resolve(self, q: _Queued) -> None:
        if q.batch is None:
            q.resolve(len(self.cfg.fanouts), self._sampler_rng)
            self._resolved_storage += q.storage_accesses
            self._n_resolved += 1

    def _storage_at_least(self, bound: int) -> bool:
        """pending_storage >= bound, resolving (oldest first) only as needed."""
        if self._resolved_storage >= bound:
            return True
        for q in itertools.islice(self._pending, self._n_resolved, None):
            if q.batch is None:
                self._resolve(q)
                if self._resolved_storage >= bound:
                    return True
        return False

    def _launch_sample(self):
        """Sample the next seed batch on the control stream (outputs exported
        asynchronously); None when the seeds are exhausted.  A seed error is
        carried in the entry and raised when the batch is admitted, where the
        reference would raise it."""
        import torch
        try:
            seeds = next(self._batches)
        except StopIteration:
            self._seeds_done = True
            return None
        try:  # (_seed_stream draws ids in [0, N): checked once, at construction)
            seeds = seeds if self._seeds_trusted else check_seeds(seeds, self.graph.num_nodes)
        except ValueError as e:
            q = _Queued(seeds, None, 0, None, 0, None)
            q.error = e
            return q
        st = self._smp.cuda_stream
        words = None if self._rng_on_device else pcg_words(self._sampler_rng)
        self._rng_on_device = True
        # one block for the batch's edges and unique nodes (views of it, made
        # when the batch resolves); its seeds and sizes in pinned ring rows (a
        # row is reused only after its batch resolved, i.e. its stream work ran)
        block = self._smp_slots.take()
        i = self._sizes_next
        self._sizes_next = (i + 1) % self._sizes_np.shape[0]
        ptr = self._sizes_ptr + i * self._sizes_np.strides[0]
        staged = self._seed_stage[i, :len(seeds)]
        staged[:] = seeds
        b0 = block.data_ptr()
        self._h.sample_async(staged, words, st, b0, b0 + 16 * self._edge_cap, ptr)
        sampled = torch.cuda.Event()
        sampled.record(self._smp)
        return _Queued(seeds, block, self._edge_cap, self._sizes_np[i], ptr, sampled)

    def _sample_one(self) -> bool:
        """One batch joins the run-ahead queue (dataloader.py:194-205): the next
        speculatively sampled batch, else a fresh one.  Its contribution is
        counted now, against the cache as the reference would see it."""
        import torch
        q = self._spec.popleft() if self._spec else self._launch_sample()
        if q is None:
            self._exhausted = True
            return False
        if q.error is not None:
            raise q.error
        if q.counted_at != self._serves:  # (else counted already, against this same cache)
            self._count(q)
        self._pending.append(q)
        return True

    def _count(self, q: _Queued) -> None:
        """q's run-ahead contribution against the cache as the last serve left
        it (the control stream's decisions), on the count stream."""
        import torch
        L = len(self.cfg.fanouts)
        row = q.sizes_ptr
        cnt = self._cnt
        cnt.wait_event(q.event)  # the batch's sampling and size export
        # (the handle orders the count after the last serve's decisions and the
        # next serve after the count, on the device)
        q.block.record_stream(cnt)
        self._h.contribution_async(q.unique_ptr, row + 8 * L, row + 8 * (L + 2),
                                   cnt.cuda_stream)
        q.event = torch.cuda.Event()
        q.event.record(cnt)
        q.counted_at = self._serves

    def _precount(self) -> None:
        """Count the batch the next call admits now: the cache stays as this
        serve leaves it until the next serve, so the count is the one its
        admission would make -- and the host does not wait for it there (a
        serve in between, i.e. a call admitting nothing, makes it recount)."""
        if self._spec and self._spec[0].error is None and \
                self._spec[0].counted_at != self._serves:
            self._count(self._spec[0])

    def _speculate(self) -> None:
        """Sample up to gids_speculate batches beyond the run-ahead queue, so
        the sampling of the batch the next call admits runs while this batch
        is gathered (the sampled content is fixed by the seed order and the
        sampler stream, so it does not depend on when it is drawn)."""
        while len(self._spec) < self._spec_depth and not self._seeds_done:
            q = self._launch_sample()
            if q is None:
                break
            self._spec.append(q)
            if q.error is not None:
                break

    def run_ahead(self) -> None:
        want = self.cfg.window_depth + 1
        while not self._exhausted:
            short_window = len(self._pending) < want
            # need_threshold = pending_storage < effective_threshold(); only
            # resolved as far as the comparison requires
            if not short_window and self._storage_at_least(self.effective_threshold()):
                break
            if len(self._pending) >= self.cfg.runahead_cap:
                break
            if not short_window and not self._storage_at_least(1):
                break
            self._sample_one()
        while self._ringed < min(self.window.depth, len(self._pending)):
            q = self._pending[self._ringed]
            self._resolve(q)
            self.window.push_iteration(q.batch.unique_nodes, trusted=True)
            self._ringed += 1

    # -- serving (dataloader.py:232-299)
    def next_batch(self):
        if self.shared is not None:
            return self._next_batch_shared()
        import torch
        tr = self._trace
        if tr is not None:
            t0 = time.perf_counter()
        self.run_ahead()
        if not self._pending:
            raise StopIteration
        inflight = self._pending_storage
        entry = self._pending.popleft()
        self._n_resolved -= 1
        self._resolved_storage -= entry.storage_accesses
        if self._ringed > 0:
            self.window.pop_iteration()
            self._ringed -= 1
        self.run_ahead()
        if tr is not None:
            t1 = time.perf_counter()

        batch = entry.batch
        unique = batch.unique_nodes
        n = unique.numel()
        rows = self._out_block()[:n]
        unique.record_stream(self._gat)
        unique.record_stream(self._ctl)
        if tr is not None:
            t2 = time.perf_counter()
        pop, push = self.window.take_shift()
        self._h.serve_shift(unique, self._iteration, rows, self._ctl.cuda_stream,
                            self._gat.cuda_stream, pop, push)
        self._serves += 1
        if tr is not None:  # device timeline per batch: decisions done, rows done
            t2s = time.perf_counter()
            decided = torch.cuda.Event(enable_timing=True)
            decided.record(self._ctl)
            gathered = torch.cuda.Event(enable_timing=True)
            gathered.record(self._gat)
            self._timeline.append((decided, gathered))
        # the next batches' sampling is launched before the host waits for
        # the decisions' counts, so the sampling stream stays busy while the
        # host accounts and returns (the sampled content is fixed by the seed
        # order and the sampler stream, not by when it is drawn)
        self._speculate()
        if tr is not None:
            t2p = time.perf_counter()
        self._precount()
        if tr is not None:
            t3 = time.perf_counter()
        c = self._h.serve_counts()  # waits for the decisions only, not the gather
        if tr is not None:
            # run-ahead, output block, serve + speculate + precount, counts wait;
            # then the serve / speculate parts of the third
            tr.append((t1 - t0, t2 - t1, t3 - t2, time.perf_counter() - t3, t2s - t2,
                       t2p - t2s))
        self.last_counts = c
        # hand the batch to the caller's stream without blocking the host
        sid = torch._C._cuda_getCurrentStream(self.device)
        cur = self._cur_streams.get(sid)
        if cur is None:
            cur = self._cur_streams.setdefault(sid, torch.cuda.Stream(
                stream_id=sid[0], device_index=sid[1], device_type=sid[2]))
        self._h.wait_served(cur.cuda_stream)
        rows.record_stream(cur)
        unique.record_stream(cur)  # (the layers share unique's allocation)
        if self.cfg.verify_gather:
            self._verify(unique, rows)
        stats = self._account(c.sampled, c.cache_hits, c.cpu_buffer_hits, c.storage,
                              c.bypasses, inflight)
        self._iteration += 1
        return batch, rows, stats

    def _next_batch_shared(self):
        """One global step of the owner-sharded cache (shared_cache.py): this
        rank's batch, decided by the owners of its nodes, gathered from the
        owners' lines and this rank's host tiers.  Collective over the ranks."""
        import torch
        sh = self.shared
        G, r = sh.G, self.cfg.gids_dp_rank
        st = _native.stream_ptr(self.device)
        self.run_ahead()
        if not self._pending:
            raise StopIteration
        # the owners need this rank's batches up to `ahead` steps on (window)
        while self._sent <= self._iteration + sh.ahead and \
                self._sent - self._iteration < len(self._pending):
            q = self._pending[self._sent - self._iteration]
            self._resolve(q)
            sh.send_lists(self._sent * G + r, q.batch.unique_nodes, st)
            self._sent += 1
        inflight = self._pending_storage
        entry = self._pending.popleft()
        self._n_resolved -= 1
        self._resolved_storage -= entry.storage_accesses
        self.run_ahead()
        batch = entry.batch
        unique = batch.unique_nodes
        n = unique.numel()
        # the owner decisions change residency the admissions' counts read
        torch.cuda.current_stream(self.device).wait_stream(self._cnt)
        dec, tiers = sh.serve_step(self._iteration, unique, st)
        rows = self._out_block()[:n]
        sh.gather(unique, dec, rows, st)
        if self.cfg.verify_gather:
            self._verify(unique, rows)
        hits, buf, ssd, byp = (int(v) for v in tiers)
        self.last_counts = None
        stats = self._account(n, hits, buf, ssd, byp, inflight)
        self._iteration += 1
        return batch, rows, stats

    def _verify(self, unique, rows) -> None:
        if self.features.seed is not None:
            bad = _native.verify_rows(self.device, self.features.seed, unique, rows,
                                      self._gat.cuda_stream)
        else:
            expect = self.features.rows(unique.cpu().numpy())
            bad = int((rows.cpu().numpy() != expect).any(axis=1).sum())
        if bad:
            raise AssertionError("gathered rows diverge from the feature table")

    def _account(self, sampled, hits, buf_hits, ssd, bypasses, inflight) -> IterationStats:
        # exact rationals as the reference (dataloader.py:301-337); the per-row
        # and per-node constants are folded once (rational arithmetic is exact,
        # so the values are unchanged) and zero terms skip the Fraction work
        fetch_us = 0
        if ssd > 0:
            joint = max(inflight, ssd)
            fetch_us = fetch_total_us(self.spec, joint) * Fraction(ssd, joint)
        if buf_hits:
            fetch_us = fetch_us + buf_hits * self._cpu_us_per_row
        train_us = sampled * self._train_us_per_node if self._train_us_per_node else 0
        step = fetch_us if fetch_us >= train_us else train_us
        if step:
            self._clock_us += step
        if fetch_us:
            self._fetch_us_total += fetch_us
        if train_us:
            self._train_us_total += train_us
        redirect = (hits + buf_hits) / sampled if sampled else 0.0
        a = self.cfg.redirect_ema_alpha
        self.redirect_ema = a * redirect + (1.0 - a) * self.redirect_ema
        if fetch_us > 0:
            bw = float(sampled * self._row_us_bytes / fetch_us)
        else:
            bw = float("inf") if sampled else 0.0
        return IterationStats(iteration=self._iteration, sampled_nodes=sampled, cache_hits=hits,
                              cpu_buffer_hits=buf_hits, ssd_accesses=ssd, bypasses=bypasses,
                              redirect_fraction=redirect, fetch_time_us=float(fetch_us),
                              effective_bandwidth_bytes_per_s=bw,
                              cumulative_time_us=float(self._clock_us))

    def __iter__(self):
        return self

    def __next__(self):
        return self.next_batch()

    def storage_stats(self) -> dict | None:
        """File tier: cumulative pages / bytes read, read calls, host I/O ms."""
        return self._h.storage_file_stats() if self._storage_file is not None else None

    def shard_counts(self) -> tuple[int, int]:
        """Sharded-table mode: rows of the last batch read from this rank's
        shard (HBM) and from peers (NVLink)."""
        return self._h.shard_counts()

    def close(self) -> None:
        import torch
        torch.cuda.synchronize(self.device)
        if getattr(self, "shared", None) is not None:
            import torch.distributed as dist
            if self.cfg.gids_dp_world > 1 and dist.is_available() and dist.is_initialized():
                dist.barrier()  # no peer may still be reading or writing this rank's lines
            self.shared.close()
            self.shared = None
        self._h.close()
        if self.sharded is not None:
            import torch.distributed as dist
            if self.cfg.gids_dp_world > 1 and dist.is_available() and dist.is_initialized():
                dist.barrier()  # no peer may still be reading this rank's shard
            self.sharded.close()
        for r in getattr(self, "_shared", []):  # this rank's mapping of the node's host tier
            r.close()
        self._shared = []


def run(dl: Dataloader, iterations: int | None = None, warmup: int | None = None):
    """Warm-up then measured iterations; stops early when seeds run out."""
    iterations = dl.cfg.iterations if iterations is None else iterations
    warmup = dl.cfg.warmup if warmup is None else warmup
    for _ in range(warmup):
        try:
            dl.next_batch()
        except StopIteration:
            break
    c0, f0, t0 = dl._clock_us, dl._fetch_us_total, dl._train_us_total
    measured: list[IterationStats] = []
    for _ in range(iterations):
        try:
            measured.append(dl.next_batch()[2])
        except StopIteration:
            break
    sampled = sum(s.sampled_nodes for s in measured)
    hits = sum(s.cache_hits for s in measured)
    redirected = hits + sum(s.cpu_buffer_hits for s in measured)
    fetch = dl._fetch_us_total - f0
    rb = dl.features.row_bytes
    return measured, RunSummary(
        iterations_run=len(measured), sampled_total=sampled,
        cache_hit_ratio=hits / sampled if sampled else 0.0,
        redirect_fraction=redirected / sampled if sampled else 0.0,
        mean_bandwidth_bytes_per_s=float(sampled * rb * 1_000_000 / fetch) if fetch > 0 else 0.0,
        total_fetch_us=float(fetch), total_train_us=float(dl._train_us_total - t0),
        total_time_us=float(dl._clock_us - c0))

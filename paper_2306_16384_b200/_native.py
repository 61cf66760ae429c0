"""ctypes binding of libgids.so (include/gids.h).

The CUDA library is the only compute path: if it is missing this module
raises ImportError with the build command instead of falling back to any
CPU implementation.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libgids.so"
if os.environ.get("GIDS_LIB"):  # an alternative build of the same ABI (experiments)
    LIB_PATH = Path(os.environ["GIDS_LIB"]).resolve()
ABI_VERSION = 1
MAX_LAYERS = 8

OK, E_INVALID, E_CUDA, E_CAPACITY, E_STATE = 0, -1, -2, -3, -4
POLICY_EXACT, POLICY_SETASSOC = 0, 1
KIND_HIT, KIND_MISS, KIND_BYPASS = 0, 1, 2


class GidsConfig(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("num_edges", C.c_int64),
                ("feature_dim", C.c_int32), ("device", C.c_int32),
                ("cache_lines", C.c_int64), ("policy", C.c_int32), ("ways", C.c_int32),
                ("evict_key", C.c_uint64), ("window_depth", C.c_int32),
                ("n_layers", C.c_int32), ("fanouts", C.c_int32 * MAX_LAYERS),
                ("max_seeds", C.c_int64)]


class TierCounts(C.Structure):
    _fields_ = [(k, C.c_int64) for k in
                ("sampled", "cache_hits", "cpu_buffer_hits", "storage", "bypasses")]


class CacheCounters(C.Structure):
    _fields_ = [(k, C.c_int64) for k in
                ("hits", "misses", "bypasses", "evictions", "total_increments",
                 "total_decrements", "safe_count", "filled")]


class GidsError(RuntimeError):
    """A CUDA-side failure of the GIDS library."""


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"GIDS CUDA library not built ({LIB_PATH}); run "
            "`python -c 'import __graft_entry__ as g; g.build()'` or "
            "`make -C paper_2306_16384_b200/csrc`")
    L = C.CDLL(str(LIB_PATH))
    vp, i64, u64, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32
    sig = {
        "gids_abi_version": ([], C.c_int),
        "gids_last_error": ([], C.c_char_p),
        "gids_create": ([C.POINTER(GidsConfig), vp, C.POINTER(vp)], C.c_int),
        "gids_destroy": ([vp], C.c_int),
        "gids_load_graph": ([vp, vp, vp], C.c_int),
        "gids_set_backing": ([vp, vp, i64], C.c_int),
        "gids_set_constant_buffer": ([vp, vp, i64, vp], C.c_int),
        "gids_sample": ([vp, vp, i64, vp, vp], C.c_int),
        "gids_sample_frontier": ([vp, vp, i64, vp, vp], C.c_int),
        "gids_owner_split": ([vp, vp, i64, i32, vp, vp, vp, vp], C.c_int),
        "gids_shared_marks": ([vp, vp, vp, i64, i32, i32, vp, vp], C.c_int),
        "gids_shared_final": ([vp, vp, vp, vp, i64, i32, vp, vp], C.c_int),
        "gids_shared_unsplit": ([vp, vp, vp, i64, vp, vp], C.c_int),
        "gids_shared_tiers": ([vp, vp, vp, i64, vp, vp], C.c_int),
        "gids_shared_gather": ([vp, vp, vp, i64, i32, vp, vp, i32, vp], C.c_int),
        "gids_cache_rows_ptr": ([vp], vp),
        "gids_sample_sizes": ([vp, vp, vp, vp, vp], C.c_int),
        "gids_sample_export": ([vp, vp, vp, vp], C.c_int),
        "gids_sample_export_async": ([vp, vp, vp, vp, vp], C.c_int),
        "gids_sample_capacity": ([vp, vp, vp], C.c_int),
        "gids_sample_async": ([vp, vp, i64, vp, vp, vp, vp, vp], C.c_int),
        "gids_sampler_rng": ([vp, vp], C.c_int),
        "gids_window_push": ([vp, vp, i64, vp], C.c_int),
        "gids_window_pop": ([vp, vp, i64, vp], C.c_int),
        "gids_serve": ([vp, vp, i64, u64, vp, vp, vp], C.c_int),
        "gids_serve_counts": ([vp, C.POINTER(TierCounts)], C.c_int),
        "gids_wait_served": ([vp, vp], C.c_int),
        "gids_serve_shift": ([vp, vp, i64, u64, vp, vp, vp, vp, i64, vp, i64], C.c_int),
        "gids_serve_decisions": ([vp, vp, vp, vp], C.c_int),
        "gids_cache_stats": ([vp, C.POINTER(CacheCounters)], C.c_int),
        "gids_cache_rng": ([vp, vp], C.c_int),
        "gids_cache_lines": ([vp, vp, vp], C.c_int),
        "gids_cache_capacity": ([vp], i64),
        "gids_synthesize_rows": ([i32, u64, i64, i64, i32, vp, vp], C.c_int),
        "gids_verify_rows": ([i32, u64, vp, i64, i32, vp, vp, vp], C.c_int),
        "gids_launch_count": ([vp], i64),
        "gids_serve_graph_replays": ([vp], i64),
        "gids_exact_par_batches": ([vp], i64),
        "gids_exact_par_stats": ([vp, vp], C.c_int),
        "gids_generate_uniform_graph": ([i32, i64, i64, u64, vp, vp, vp], C.c_int),
        "gids_reverse_pagerank": ([i32, i64, i64, vp, vp, C.c_double, C.c_double, i32, vp, vp,
                                   vp, vp], C.c_int),
        "gids_load_graph_device": ([vp, vp, vp], C.c_int),
        "gids_contribution_async": ([vp, vp, vp, vp, vp], C.c_int),
        "gids_host_register": ([vp, i64], C.c_int),
        "gids_host_unregister": ([vp], C.c_int),
        "gids_cache_window_update": ([vp, vp, i64, vp, vp], C.c_int),
        "gids_cache_access": ([vp, vp, i64, vp, vp, vp, vp], C.c_int),
        "gids_cache_reuse": ([vp, vp], C.c_int),
        "gids_set_storage_file": ([vp, C.c_char_p, i64, i32, i64, i32, i32], C.c_int),
        "gids_storage_file_stats": ([vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64),
                                     C.POINTER(C.c_double), C.POINTER(i32)], C.c_int),
        "gids_device_alloc": ([i32, i64, C.POINTER(vp)], C.c_int),
        "gids_device_free": ([i32, vp], C.c_int),
        "gids_ipc_handle": ([i32, vp, vp], C.c_int),
        "gids_ipc_open": ([i32, vp, C.POINTER(vp)], C.c_int),
        "gids_ipc_close": ([i32, vp], C.c_int),
        "gids_set_sharded_table": ([vp, vp, i32, i32], C.c_int),
        "gids_shard_counts": ([vp, C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "gids_synthesize_rows_strided": ([i32, u64, i64, i64, i64, i32, vp, vp], C.c_int),
        "gids_set_profiling": ([vp, C.c_int], C.c_int),
        "gids_phase_times": ([vp, vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.gids_abi_version() != ABI_VERSION:
        raise ImportError("libgids.so ABI version mismatch; rebuild it")
    _lib = L
    return L


def exported_symbols() -> list[str]:
    """Every entry point include/gids.h declares (checked by the CPU tests)."""
    return ["gids_abi_version", "gids_last_error", "gids_create", "gids_destroy",
            "gids_load_graph", "gids_set_backing", "gids_set_constant_buffer", "gids_sample", "gids_sample_frontier",
            "gids_sample_sizes", "gids_sample_export", "gids_sample_export_async",
            "gids_sample_capacity", "gids_sampler_rng", "gids_window_push", "gids_window_pop",
            "gids_serve", "gids_serve_counts", "gids_serve_decisions", "gids_cache_stats",
            "gids_cache_rng", "gids_cache_lines", "gids_cache_capacity",
            "gids_synthesize_rows", "gids_verify_rows", "gids_set_profiling",
            "gids_phase_times", "gids_launch_count", "gids_generate_uniform_graph",
            "gids_reverse_pagerank", "gids_load_graph_device", "gids_device_alloc",
            "gids_device_free", "gids_ipc_handle",
            "gids_ipc_open", "gids_ipc_close", "gids_set_sharded_table", "gids_shard_counts",
            "gids_synthesize_rows_strided", "gids_set_storage_file", "gids_storage_file_stats",
            "gids_cache_window_update", "gids_cache_access", "gids_cache_reuse",
            "gids_contribution_async", "gids_host_register", "gids_host_unregister",
            "gids_exact_par_batches", "gids_exact_par_stats", "gids_owner_split",
            "gids_shared_marks", "gids_shared_final", "gids_shared_unsplit", "gids_shared_tiers",
            "gids_shared_gather", "gids_cache_rows_ptr", "gids_wait_served",
            "gids_serve_shift", "gids_serve_graph_replays", "gids_sample_async"]


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = lib().gids_last_error().decode(errors="replace")
    if rc == E_INVALID:
        raise ValueError(msg)
    if rc == E_STATE:
        from .feature_cache import CacheProtocolError
        raise CacheProtocolError(msg)
    raise GidsError(f"{what}: {msg}" if what else msg)


def _p(a) -> int:
    """Raw address of a numpy array, a torch tensor, or an address already."""
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def stream_ptr(device: int = 0) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


class Handle:
    """One gids_handle: device-resident graph, cache and workspaces."""

    def __init__(self, *, num_nodes, num_edges, feature_dim, device, cache_lines, policy,
                 ways, evict_key, window_depth, fanouts, max_seeds, eviction_words):
        L = lib()
        fans = [int(f) for f in fanouts]
        if not 1 <= len(fans) <= MAX_LAYERS:
            raise ValueError(f"the CUDA sampler supports 1..{MAX_LAYERS} layers")
        cfg = GidsConfig()
        cfg.num_nodes, cfg.num_edges, cfg.feature_dim = num_nodes, num_edges, feature_dim
        cfg.device, cfg.cache_lines = device, cache_lines
        cfg.policy = POLICY_SETASSOC if policy == "setassoc" else POLICY_EXACT
        cfg.ways, cfg.evict_key, cfg.window_depth = ways, evict_key, window_depth
        cfg.n_layers = len(fans)
        for i, f in enumerate(fans):
            cfg.fanouts[i] = f
        cfg.max_seeds = max_seeds
        self.cfg = cfg
        self.device = device
        self.n_layers = len(fans)
        self.dim = feature_dim
        words = np.ascontiguousarray(eviction_words, dtype=np.uint64)
        h = C.c_void_p()
        check(L.gids_create(C.byref(cfg), words.ctypes.data, C.byref(h)), "gids_create")
        self.h = h
        self._keep = []  # host arrays the library reads zero-copy

    def close(self) -> None:
        if getattr(self, "h", None):
            lib().gids_destroy(self.h)
            self.h = None
            self._keep = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- setup
    def load_graph(self, indptr: np.ndarray, indices: np.ndarray) -> None:
        ip = np.ascontiguousarray(indptr, dtype=np.uint64)
        ix = np.ascontiguousarray(indices, dtype=np.uint64)
        check(lib().gids_load_graph(self.h, ip.ctypes.data, ix.ctypes.data), "load_graph")

    def load_graph_device(self, indptr, indices) -> None:
        """indptr int64[N+1] / indices int32[E] CUDA tensors (copied into the handle)."""
        check(lib().gids_load_graph_device(self.h, _p(indptr), _p(indices)), "load_graph_device")

    def set_sharded_table(self, shard_ptrs, my_shard: int) -> None:
        ptrs = np.ascontiguousarray(shard_ptrs, dtype=np.uint64)
        check(lib().gids_set_sharded_table(self.h, ptrs.ctypes.data, len(ptrs), my_shard),
              "set_sharded_table")

    def shard_counts(self) -> tuple[int, int]:
        a, b = C.c_int64(), C.c_int64()
        check(lib().gids_shard_counts(self.h, C.byref(a), C.byref(b)), "shard_counts")
        return a.value, b.value

    def set_storage_file(self, path: str, offset: int, page_bytes: int, max_pages: int = 0,
                         io_threads: int = 8, direct: bool = False) -> None:
        check(lib().gids_set_storage_file(self.h, str(path).encode(), offset, page_bytes,
                                          max_pages, io_threads, 1 if direct else 0),
              "set_storage_file")

    def storage_file_stats(self) -> dict:
        p, b, r, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        ms = C.c_double()
        check(lib().gids_storage_file_stats(self.h, C.byref(p), C.byref(b), C.byref(r),
                                            C.byref(ms), C.byref(d)), "storage_file_stats")
        return {"pages": p.value, "bytes": b.value, "runs": r.value, "io_ms": ms.value,
                "direct": bool(d.value)}

    def set_backing(self, table, n_rows: int) -> None:
        self._keep.append(table)
        check(lib().gids_set_backing(self.h, _p(table), n_rows), "set_backing")

    def set_constant_buffer(self, node_ids: np.ndarray, rows) -> None:
        ids = np.ascontiguousarray(node_ids, dtype=np.int64)
        if len(ids):
            self._keep.append(rows)
        check(lib().gids_set_constant_buffer(self.h, ids.ctypes.data, len(ids),
                                             _p(rows) if len(ids) else None),
              "set_constant_buffer")

    # -- sampling
    def sample(self, seeds: np.ndarray, words, stream: int) -> None:
        """words: the Generator's 6-word state to (re)seed the device stream, or
        None to continue the device-resident stream."""
        s = np.ascontiguousarray(seeds, dtype=np.int64)
        w = None if words is None else np.ascontiguousarray(words, dtype=np.uint64)
        check(lib().gids_sample(self.h, s.ctypes.data, len(s),
                                None if w is None else w.ctypes.data, stream), "sample")

    def sample_async(self, seeds: np.ndarray, words, stream: int, edges_ptr: int,
                     unique_ptr: int, sizes_ptr: int) -> None:
        """sample() then sample_export_async() in one call; seeds: contiguous
        int64 (pinned: the copy does not stall the host)."""
        check(lib().gids_sample_async(self.h, seeds.ctypes.data, len(seeds),
                                      None if words is None else words.ctypes.data, stream,
                                      edges_ptr, unique_ptr, sizes_ptr), "sample_async")

    def sample_frontier(self, frontier: np.ndarray, words, stream: int) -> None:
        """One layer over an explicit frontier, in order, repeats included."""
        f = np.ascontiguousarray(frontier, dtype=np.int64)
        w = None if words is None else np.ascontiguousarray(words, dtype=np.uint64)
        check(lib().gids_sample_frontier(self.h, f.ctypes.data, len(f),
                                         None if w is None else w.ctypes.data, stream),
              "sample_frontier")

    def sample_export_async(self, edges, unique, sizes_host, stream: int) -> None:
        check(lib().gids_sample_export_async(self.h, _p(edges), _p(unique), _p(sizes_host),
                                             stream), "sample_export_async")

    def contribution_async(self, unique, n_ptr: int, out_ptr: int, stream: int) -> None:
        check(lib().gids_contribution_async(self.h, _p(unique), n_ptr, out_ptr, stream),
              "contribution_async")

    def sample_capacity(self) -> tuple[int, int]:
        e, u = C.c_int64(), C.c_int64()
        check(lib().gids_sample_capacity(self.h, C.byref(e), C.byref(u)), "sample_capacity")
        return e.value, u.value

    def sampler_rng(self) -> np.ndarray:
        w = np.zeros(6, np.uint64)
        check(lib().gids_sampler_rng(self.h, w.ctypes.data), "sampler_rng")
        return w

    def sample_sizes(self):
        lens = np.zeros(self.n_layers, np.int64)
        nu, dr, co = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().gids_sample_sizes(self.h, lens.ctypes.data, C.byref(nu), C.byref(dr),
                                      C.byref(co)), "sample_sizes")
        return lens, nu.value, dr.value, co.value

    def sample_export(self, edges, unique, stream: int) -> None:
        check(lib().gids_sample_export(self.h, _p(edges) if edges is not None else None,
                                       _p(unique) if unique is not None else None, stream),
              "sample_export")

    # -- window and serving
    def window_push(self, nodes, stream: int) -> None:
        check(lib().gids_window_push(self.h, _p(nodes), nodes.numel(), stream), "window_push")

    def window_pop(self, nodes, stream: int) -> None:
        check(lib().gids_window_pop(self.h, _p(nodes), nodes.numel(), stream), "window_pop")

    def serve(self, unique, epoch: int, out, stream: int, gather_stream: int | None = None) -> None:
        check(lib().gids_serve(self.h, _p(unique), unique.numel(), epoch, _p(out), stream,
                               gather_stream), "serve")

    def serve_shift(self, unique, epoch: int, out, stream: int, gather_stream: int | None,
                    pop, push) -> None:
        """window_pop(pop); window_push(push); serve(...) -- one call (None: no list)."""
        check(lib().gids_serve_shift(
            self.h, _p(unique), unique.numel(), epoch, _p(out), stream, gather_stream,
            None if pop is None else _p(pop), 0 if pop is None else pop.numel(),
            None if push is None else _p(push), 0 if push is None else push.numel()),
            "serve_shift")

    def wait_served(self, stream: int) -> None:
        """`stream` waits (device-side) for the last serve's decisions and gather."""
        check(lib().gids_wait_served(self.h, stream), "wait_served")

    def serve_counts(self) -> TierCounts:
        t = TierCounts()
        check(lib().gids_serve_counts(self.h, C.byref(t)), "serve_counts")
        return t

    def serve_decisions(self, kind, line, stream: int) -> None:
        check(lib().gids_serve_decisions(self.h, _p(kind), _p(line), stream), "serve_decisions")

    def cache_window_update(self, nodes, counts, stream: int) -> None:
        check(lib().gids_cache_window_update(self.h, _p(nodes), nodes.numel(),
                                             _p(counts) if counts is not None else None, stream),
              "cache_window_update")

    def cache_access(self, nodes, kind, line, victim, stream: int) -> None:
        check(lib().gids_cache_access(self.h, _p(nodes), nodes.numel(), _p(kind), _p(line),
                                      _p(victim) if victim is not None else None, stream),
              "cache_access")

    # -- owner-sharded cache (csrc/shared_cache.cu)
    def owner_split(self, unique, G: int, out, perm, stream: int) -> np.ndarray:
        counts = np.zeros(G, np.int64)
        check(lib().gids_owner_split(self.h, _p(unique), unique.numel(), G, _p(out), _p(perm),
                                     counts.ctypes.data, stream), "owner_split")
        return counts

    def shared_marks(self, kind, line, batch: int, step0: int, flags, stream: int) -> None:
        check(lib().gids_shared_marks(self.h, _p(kind), _p(line), kind.numel(), batch, step0,
                                      _p(flags), stream), "shared_marks")

    def shared_final(self, kind, line, flags, batch: int, packed, stream: int) -> None:
        check(lib().gids_shared_final(self.h, _p(kind), _p(line), _p(flags), kind.numel(), batch,
                                      _p(packed), stream), "shared_final")

    def shared_unsplit(self, packed, perm, dec, stream: int) -> None:
        check(lib().gids_shared_unsplit(self.h, _p(packed), _p(perm), packed.numel(), _p(dec),
                                        stream), "shared_unsplit")

    def shared_tiers(self, unique, dec, stream: int) -> np.ndarray:
        out = np.zeros(4, np.int64)
        check(lib().gids_shared_tiers(self.h, _p(unique), _p(dec), unique.numel(),
                                      out.ctypes.data, stream), "shared_tiers")
        return out

    def shared_gather(self, unique, dec, owner_rows, out, phase: int, stream: int) -> None:
        rows = np.ascontiguousarray(owner_rows, dtype=np.uint64)
        check(lib().gids_shared_gather(self.h, _p(unique), _p(dec), unique.numel(), len(rows),
                                       rows.ctypes.data, _p(out), phase, stream), "shared_gather")

    def cache_rows_ptr(self) -> int:
        return int(lib().gids_cache_rows_ptr(self.h) or 0)

    def cache_reuse(self, num_nodes: int) -> np.ndarray:
        out = np.zeros(num_nodes, np.uint32)
        check(lib().gids_cache_reuse(self.h, out.ctypes.data), "cache_reuse")
        return out

    def cache_stats(self) -> CacheCounters:
        c = CacheCounters()
        check(lib().gids_cache_stats(self.h, C.byref(c)), "cache_stats")
        return c

    def cache_rng(self) -> np.ndarray:
        w = np.zeros(6, np.uint64)
        check(lib().gids_cache_rng(self.h, w.ctypes.data), "cache_rng")
        return w

    def cache_lines(self):
        n = self.capacity()
        node = np.zeros(max(n, 1), np.int64)
        st = np.zeros(max(n, 1), np.int8)
        check(lib().gids_cache_lines(self.h, node.ctypes.data, st.ctypes.data), "cache_lines")
        return node[:n], st[:n]

    def capacity(self) -> int:
        return int(lib().gids_cache_capacity(self.h))

    def set_profiling(self, on: bool) -> None:
        check(lib().gids_set_profiling(self.h, 1 if on else 0), "set_profiling")

    def phase_times(self) -> dict:
        out = np.zeros(5, np.float64)
        check(lib().gids_phase_times(self.h, out.ctypes.data), "phase_times")
        return dict(zip(("sample_ms", "cache_ms", "gather_hits_ms", "gather_host_ms",
                         "batches"), out.tolist()))

    def launch_count(self) -> int:
        return int(lib().gids_launch_count(self.h))

    def graphs_replayed(self) -> int:
        """Serves replayed as CUDA graphs (evidence counter)."""
        return int(lib().gids_serve_graph_replays(self.h))

    def exact_par_batches(self) -> int:
        return int(lib().gids_exact_par_batches(self.h))

    def exact_par_stats(self) -> dict:
        out = np.zeros(16, np.int64)
        check(lib().gids_exact_par_stats(self.h, out.ctypes.data), "exact_par_stats")
        d = dict(zip(("rounds", "ended_rejection", "ended_change_list", "ended_lost_line",
                      "cyc_draws", "cyc_tables", "cyc_first_select", "cyc_sort",
                      "cyc_masks", "cyc_resolve", "cyc_lost_lines", "fixpoint_passes",
                      "cyc_verify", "cyc_commit", "cyc_ring", "cyc_spare"),
                     out.tolist()), batches=self.exact_par_batches())
        # (the per-phase cycle counters are compiled in only with -DGIDS_XP_PROF=1)
        d["cycle_counters"] = any(v for k, v in d.items() if k.startswith("cyc_"))
        return d


def synthesize_rows(device: int, seed: int, row0: int, n: int, dim: int, dst, stream: int) -> None:
    check(lib().gids_synthesize_rows(device, seed & ((1 << 64) - 1), row0, n, dim, _p(dst),
                                     stream), "synthesize_rows")


def verify_rows(device: int, seed: int, nodes, rows, stream: int) -> int:
    bad = C.c_int64()
    check(lib().gids_verify_rows(device, seed & ((1 << 64) - 1), _p(nodes), nodes.numel(),
                                 rows.shape[1], _p(rows), C.byref(bad), stream), "verify_rows")
    return bad.value


def generate_uniform_graph(device: int, num_nodes: int, num_edges: int, seed: int):
    """GPU uniform generator (csrc/graph_setup.cu): (indptr int64, indices int32) on cuda."""
    import torch
    dev = torch.device("cuda", device)
    indptr = torch.empty(num_nodes + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(max(num_edges, 1), dtype=torch.int32, device=dev)
    check(lib().gids_generate_uniform_graph(device, num_nodes, num_edges,
                                            seed & ((1 << 64) - 1), _p(indptr), _p(indices),
                                            stream_ptr(device)), "generate_uniform_graph")
    return indptr, indices[:num_edges]


def reverse_pagerank(device: int, indptr, indices, damping: float = 0.85, tol: float = 1e-8,
                     max_iter: int = 200):
    """cpu_buffer.py:26-74 on the GPU over a device CSC: (scores f64 cuda, converged, iters)."""
    import torch
    n = indptr.numel() - 1
    scores = torch.empty(n, dtype=torch.float64, device=indptr.device)
    it, conv = C.c_int32(), C.c_int32()
    check(lib().gids_reverse_pagerank(device, n, indices.numel(), _p(indptr),
                                      _p(indices) if indices.numel() else None, float(damping),
                                      float(tol), int(max_iter), _p(scores), C.byref(it),
                                      C.byref(conv), stream_ptr(device)), "reverse_pagerank")
    return scores, bool(conv.value), int(it.value)


def device_alloc(device: int, nbytes: int) -> int:
    ptr = C.c_void_p()
    check(lib().gids_device_alloc(device, nbytes, C.byref(ptr)), "device_alloc")
    return int(ptr.value)


def device_free(device: int, ptr: int) -> None:
    check(lib().gids_device_free(device, C.c_void_p(ptr)), "device_free")


def ipc_handle(device: int, ptr: int) -> bytes:
    """64-byte CUDA IPC handle of a gids_device_alloc allocation."""
    buf = (C.c_uint8 * 64)()
    check(lib().gids_ipc_handle(device, C.c_void_p(ptr), buf), "ipc_handle")
    return bytes(buf)


def ipc_open(device: int, handle: bytes) -> int:
    if len(handle) != 64:
        raise ValueError("CUDA IPC handles are 64 bytes")
    buf = (C.c_uint8 * 64).from_buffer_copy(handle)
    ptr = C.c_void_p()
    check(lib().gids_ipc_open(device, buf, C.byref(ptr)), "ipc_open")
    return int(ptr.value)


def ipc_close(device: int, ptr: int) -> None:
    check(lib().gids_ipc_close(device, C.c_void_p(ptr)), "ipc_close")


def synthesize_rows_strided(device: int, seed: int, row0: int, stride: int, n: int, dim: int,
                            dst, stream: int) -> None:
    """dst: a tensor or a raw device address."""
    check(lib().gids_synthesize_rows_strided(device, seed & ((1 << 64) - 1), row0, stride, n,
                                             dim, dst if isinstance(dst, int) else _p(dst),
                                             stream), "synthesize_rows_strided")


class HugePageHost:
    """Host memory on transparent 2 MiB pages, page-locked and mapped for
    zero-copy reads (gids_host_register).  ``array(shape, dtype)`` views it."""

    def __init__(self, nbytes: int):
        import mmap
        align = 2 << 20
        self._map = mmap.mmap(-1, nbytes + align)
        base = np.frombuffer(self._map, dtype=np.uint8)
        addr = base.ctypes.data
        self._off = (-addr) % align
        self.nbytes = nbytes
        try:
            self._map.madvise(mmap.MADV_HUGEPAGE, self._off, nbytes - nbytes % align or nbytes)
        except (AttributeError, OSError, ValueError):
            pass  # THP unavailable: still correct, just 4 KiB pages
        self._view = base[self._off:self._off + nbytes]
        self._view[::4096] = 0  # fault the pages in (huge where the kernel allows)
        self.ptr = self._view.ctypes.data
        check(lib().gids_host_register(C.c_void_p(self.ptr), nbytes), "host_register")

    def array(self, shape, dtype) -> np.ndarray:
        return self._view.view(dtype).reshape(shape)

    def close(self) -> None:
        if getattr(self, "ptr", None):
            lib().gids_host_unregister(C.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SharedHost:
    """A POSIX shared-memory region (/dev/shm/<name>) mapped into this process
    and page-locked + mapped for zero-copy GPU reads (gids_host_register):
    the node's one host tier, shared by every local rank instead of one
    private pinned copy per rank.  ``create`` makes (and sizes) it; the other
    ranks attach.  ``unlink`` drops the name once every rank has attached
    (the mappings stay valid until closed)."""

    def __init__(self, name: str, nbytes: int, create: bool, register: bool = True):
        import mmap
        import os
        self.name, self.nbytes = name, int(nbytes)
        self.path = "/dev/shm/" + name
        flags = os.O_RDWR | (os.O_CREAT | os.O_EXCL if create else 0)
        fd = os.open(self.path, flags, 0o600)
        try:
            if create:
                os.ftruncate(fd, self.nbytes)
            elif os.fstat(fd).st_size != self.nbytes:
                raise RuntimeError(f"{self.path}: size {os.fstat(fd).st_size} != {self.nbytes}")
            self._map = mmap.mmap(fd, self.nbytes, mmap.MAP_SHARED,
                                  mmap.PROT_READ | mmap.PROT_WRITE)
        finally:
            os.close(fd)
        self._view = np.frombuffer(self._map, dtype=np.uint8)
        self.ptr = self._view.ctypes.data
        self._registered = False
        if register:
            check(lib().gids_host_register(C.c_void_p(self.ptr), self.nbytes), "host_register")
            self._registered = True

    def array(self, shape, dtype) -> np.ndarray:
        return self._view.view(dtype).reshape(shape)

    def unlink(self) -> None:
        import os
        try:
            os.unlink(self.path)
        except FileNotFoundError:
            pass

    def close(self) -> None:
        if getattr(self, "_registered", False):
            lib().gids_host_unregister(C.c_void_p(self.ptr))
            self._registered = False
        if getattr(self, "_map", None) is not None:
            self._view = None
            try:
                self._map.close()
            except BufferError:  # a numpy view is still alive; the GC unmaps it
                pass
            self._map = None

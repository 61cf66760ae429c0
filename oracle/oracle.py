"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg import this module; the product package never does.  The oracle is
pinned against golden fixtures produced by the reference itself
(``tests/golden/make_golden.py``; checked in ``tests/test_oracle.py``).

``OracleLoader`` restates the reference's serving loop
(``dataloader.py:184-299``: run-ahead accumulator, lookahead ring,
window_update, per-node tier chain, gather) on top of the C kernels in
``gids_oracle.c``.  Setup (graph, features, constant-buffer choice, seed
batches, RNG states) is passed in, so the same inputs drive the oracle and
the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import math
import subprocess
from collections import deque
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libgids_oracle.so"

K_HIT, K_MISS, K_BYPASS = 0, 1, 2
POLICY = {"exact": 0, "setassoc": 1}

_lib = None
_P = np.ctypeslib.ndpointer


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        u64p, i64p, f64p = C.POINTER(C.c_uint64), C.POINTER(C.c_int64), C.POINTER(C.c_double)
        vp = C.c_void_p
        L.or_pcg_raw.argtypes = [vp, vp, C.c_int64]
        L.or_pcg_doubles.argtypes = [vp, vp, C.c_int64]
        L.or_pcg_bounded.argtypes = [vp, vp, vp, C.c_int64]
        L.or_pcg_advance.argtypes = [vp, C.c_uint64, C.c_uint64]
        L.or_sample_subgraph.argtypes = [vp, vp, C.c_int64, vp, C.c_int64, vp, C.c_int,
                                         vp, vp, C.c_int64, vp, vp, vp, vp]
        L.or_sample_subgraph.restype = C.c_int
        L.or_cache_new.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int, vp, C.c_uint64]
        L.or_cache_new.restype = vp
        L.or_cache_free.argtypes = [vp]
        L.or_cache_window_update.argtypes = [vp, vp, C.c_int64, vp, vp, C.c_int, vp]
        L.or_cache_access_batch.argtypes = [vp, vp, C.c_int64, C.c_uint64, vp, vp]
        L.or_cache_stats.argtypes = [vp, vp]
        L.or_cache_rng.argtypes = [vp, vp]
        L.or_cache_lines.argtypes = [vp]
        L.or_cache_lines.restype = C.c_int64
        L.or_contribution.argtypes = [vp, vp, C.c_int64, vp]
        L.or_contribution.restype = C.c_int64
        L.or_cache_lines_snapshot.argtypes = [vp, vp, vp]
        L.or_gather.argtypes = [vp, C.c_int64, vp, vp, vp, vp, vp, vp, vp, C.c_int64, vp]
        L.or_feature_rows.argtypes = [C.c_uint64, vp, C.c_int64, C.c_int64, vp]
        L.or_feature_table.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, vp, C.c_int]
        L.or_generate_uniform.argtypes = [C.c_int64, C.c_int64, C.c_uint64, vp, vp, C.c_int]
        L.or_generate_uniform.restype = C.c_int
        L.or_pairwise_sum.argtypes = [vp, C.c_int64]
        L.or_pairwise_sum.restype = C.c_double
        L.or_reverse_pagerank.argtypes = [vp, vp, C.c_int64, C.c_double, C.c_double, C.c_int,
                                          vp, vp, vp, C.c_int]
        L.or_reverse_pagerank.restype = C.c_int
        _lib = L
        del u64p, i64p, f64p
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# --------------------------------------------------------------------- PCG64
def words_of(bitgen) -> np.ndarray:
    """numpy PCG64 state -> the 6-word ABI [s_hi, s_lo, inc_hi, inc_lo, has32, u32]."""
    st = bitgen.state
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m, st["has_uint32"], st["uinteger"]],
                    dtype=np.uint64)


def pcg_raw(words: np.ndarray, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().or_pcg_raw(_ptr(words), _ptr(out), n)
    return out


def pcg_doubles(words: np.ndarray, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().or_pcg_doubles(_ptr(words), _ptr(out), n)
    return out


def pcg_bounded(words: np.ndarray, ns) -> np.ndarray:
    ns = np.ascontiguousarray(ns, dtype=np.uint64)
    out = np.empty(len(ns), np.uint64)
    lib().or_pcg_bounded(_ptr(words), _ptr(ns), _ptr(out), len(ns))
    return out


def pcg_advance(words: np.ndarray, delta: int) -> None:
    lib().or_pcg_advance(_ptr(words), (delta >> 64) & ((1 << 64) - 1), delta & ((1 << 64) - 1))


# ------------------------------------------------------------------- sampler
def edge_capacity(num_nodes: int, n_seeds: int, fanouts) -> int:
    cap, front = 0, min(n_seeds, num_nodes)
    for f in fanouts:
        e = front * int(f)
        cap += e
        front = min(num_nodes, e)
    return cap


def sample_subgraph(indptr: np.ndarray, indices: np.ndarray, seeds, fanouts,
                    words: np.ndarray):
    """Restated sample_subgraph (sampler.py:87-112). ``words`` advances in place.

    Returns (layers: list[(E_l,2) int64], unique_nodes, draws)."""
    indptr = np.ascontiguousarray(indptr, dtype=np.uint64)
    indices = np.ascontiguousarray(indices, dtype=np.uint64)
    seeds = np.ascontiguousarray(seeds, dtype=np.int64)
    fans = np.ascontiguousarray(fanouts, dtype=np.int64)
    n = len(indptr) - 1
    cap = max(1, edge_capacity(n, len(seeds), fans))
    edges = np.empty((cap, 2), np.int64)
    lens = np.zeros(len(fans), np.int64)
    uniq = np.empty(len(seeds) + 2 * cap, np.int64)
    nu = np.zeros(1, np.int64)
    draws = np.zeros(1, np.int64)
    rc = lib().or_sample_subgraph(_ptr(indptr), _ptr(indices), n, _ptr(seeds), len(seeds),
                                  _ptr(fans), len(fans), _ptr(words), _ptr(edges), cap,
                                  _ptr(lens), _ptr(uniq), _ptr(nu), _ptr(draws))
    if rc != 0:
        raise RuntimeError("oracle sampler: edge capacity exceeded")
    layers, off = [], 0
    for ln in lens.tolist():
        layers.append(edges[off:off + ln].copy())
        off += ln
    return layers, uniq[:nu[0]].copy(), int(draws[0])


# --------------------------------------------------------------------- cache
class OracleCache:
    """CacheState restatement (cache.py:94-218) or the set-associative policy."""

    def __init__(self, num_nodes: int, lines: int, policy: str = "exact", ways: int = 32,
                 rng_words: np.ndarray | None = None, evict_key: int = 0):
        self._words = (np.zeros(6, np.uint64) if rng_words is None
                       else np.ascontiguousarray(rng_words, dtype=np.uint64).copy())
        self.h = lib().or_cache_new(num_nodes, lines, POLICY[policy], ways,
                                    _ptr(self._words), evict_key)
        self.lines = lib().or_cache_lines(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_cache_free(self.h)
            self.h = None

    def window_update(self, current: np.ndarray, future_lists) -> np.ndarray:
        cur = np.ascontiguousarray(current, dtype=np.int64)
        fl = [np.asarray(f, dtype=np.int64) for f in future_lists]
        fut = np.ascontiguousarray(np.concatenate(fl) if fl else np.empty(0, np.int64))
        off = np.zeros(len(fl) + 1, np.int64)
        off[1:] = np.cumsum([len(f) for f in fl]) if fl else []
        counts = np.zeros(len(cur), np.int64)
        lib().or_cache_window_update(self.h, _ptr(cur), len(cur), _ptr(fut), _ptr(off),
                                     len(fl), _ptr(counts))
        return counts

    def access_batch(self, nodes: np.ndarray, epoch: int = 0):
        nodes = np.ascontiguousarray(nodes, dtype=np.int64)
        kind = np.empty(len(nodes), np.int8)
        slot = np.empty(len(nodes), np.int64)
        lib().or_cache_access_batch(self.h, _ptr(nodes), len(nodes), epoch, _ptr(kind), _ptr(slot))
        return kind, slot

    def stats(self) -> dict:
        out = np.zeros(8, np.int64)
        lib().or_cache_stats(self.h, _ptr(out))
        keys = ("hits", "misses", "bypasses", "evictions", "total_increments",
                "total_decrements", "safe_count", "fill")
        return dict(zip(keys, out.tolist()))

    def rng_words(self) -> np.ndarray:
        w = np.zeros(6, np.uint64)
        lib().or_cache_rng(self.h, _ptr(w))
        return w

    def contribution(self, nodes: np.ndarray, pinned_off: np.ndarray) -> int:
        nodes = np.ascontiguousarray(nodes, dtype=np.int64)
        return int(lib().or_contribution(self.h, _ptr(nodes), len(nodes), _ptr(pinned_off)))

    def lines_snapshot(self):
        node = np.empty(self.lines, np.int64)
        st = np.empty(self.lines, np.int8)
        lib().or_cache_lines_snapshot(self.h, _ptr(node), _ptr(st))
        return node, st


def gather(nodes, kind, slot, pinned_off, buffer_rows, table, cache_rows):
    nodes = np.ascontiguousarray(nodes, dtype=np.int64)
    dim = table.shape[1]
    out = np.empty((len(nodes), dim), np.float32)
    tiers = np.zeros(4, np.int64)
    buf = buffer_rows if len(buffer_rows) else np.zeros((1, dim), np.float32)
    lib().or_gather(_ptr(nodes), len(nodes), _ptr(kind), _ptr(slot), _ptr(pinned_off),
                    _ptr(buf), _ptr(table), _ptr(cache_rows), _ptr(out), dim, _ptr(tiers))
    return out, tiers


def feature_rows(seed: int, nodes, dim: int) -> np.ndarray:
    nodes = np.ascontiguousarray(nodes, dtype=np.int64)
    out = np.empty((len(nodes), dim), np.float32)
    lib().or_feature_rows(seed, _ptr(nodes), len(nodes), dim, _ptr(out))
    return out


def feature_table(seed: int, num_nodes: int, dim: int, threads: int = 1,
                  out: np.ndarray | None = None) -> np.ndarray:
    """The whole synthetic table (graph.py:256-275), computed on ``threads`` host cores."""
    if out is None:
        out = np.empty((num_nodes, dim), np.float32)
    lib().or_feature_table(seed & ((1 << 64) - 1), 0, num_nodes, dim, _ptr(out), threads)
    return out


def generate_uniform(num_nodes: int, num_edges: int, seed: int, threads: int = 1):
    """CPU restatement of the GPU uniform generator (csrc/graph_setup.cu header).
    Returns (indptr u64[N+1], indices u64[E])."""
    indptr = np.zeros(num_nodes + 1, np.uint64)
    indices = np.zeros(max(num_edges, 1), np.uint64)
    rc = lib().or_generate_uniform(num_nodes, num_edges, seed & ((1 << 64) - 1), _ptr(indptr),
                                   _ptr(indices), threads)
    if rc:
        raise ValueError("generate_uniform: a node's in-degree exceeds 1024")
    return indptr, indices[:num_edges]


def pairwise_sum(a: np.ndarray) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().or_pairwise_sum(_ptr(a), len(a)))


def reverse_pagerank(indptr, indices, damping=0.85, tol=1e-8, max_iter=200, threads=1):
    """cpu_buffer.py:26-74 (unit weights) in C: (scores, converged, iterations)."""
    ip = np.ascontiguousarray(indptr, dtype=np.uint64)
    ix = np.ascontiguousarray(indices, dtype=np.uint64)
    n = len(ip) - 1
    scores = np.zeros(n, np.float64)
    it, conv = C.c_int(), C.c_int()
    lib().or_reverse_pagerank(_ptr(ip), _ptr(ix) if len(ix) else None, n, damping, tol,
                              max_iter, _ptr(scores), C.byref(it), C.byref(conv), threads)
    return scores, bool(conv.value), it.value


def required_accesses_optane(target_fraction: float = 0.95) -> int:
    # storage.py:92-104 for the intel-optane preset (25 us + 5 us, 1.5 M IOPS)
    from fractions import Fraction
    from decimal import Decimal
    f = Fraction(Decimal(str(target_fraction)))
    return math.ceil(f / (1 - f) * Fraction(30, 1_000_000) * 1_500_000)


# -------------------------------------------------------------------- loader
class OracleLoader:
    """Restatement of Dataloader's serving loop (dataloader.py:184-299).

    Parameters are resolved values (no config parsing): graph arrays, the
    feature table, the constant-buffer node list (pin order), the seed batch
    sequence, the sampler / eviction RNG word states, and the knobs.
    """

    def __init__(self, indptr, indices, table, buffer_nodes, seed_batches, fanouts,
                 sampler_words, evict_words, cache_lines, window_depth, base_threshold,
                 policy="exact", ways=32, evict_key=0, redirect_ema_alpha=0.2,
                 runahead_cap=256, keep_rows=True, buffer_rows=None):
        self.indptr = np.ascontiguousarray(indptr, dtype=np.uint64)
        self.indices = np.ascontiguousarray(indices, dtype=np.uint64)
        self.n = len(self.indptr) - 1
        self.table = table
        self.dim = table.shape[1]
        self.buffer_nodes = np.asarray(buffer_nodes, dtype=np.int64)
        self.pinned_off = np.full(self.n, -1, np.int32)
        self.pinned_off[self.buffer_nodes] = np.arange(len(self.buffer_nodes), dtype=np.int32)
        if buffer_rows is not None:  # rows of buffer_nodes, already gathered
            self.buffer_rows = buffer_rows
        else:
            self.buffer_rows = np.ascontiguousarray(table[self.buffer_nodes]) if len(
                self.buffer_nodes) else np.zeros((0, self.dim), np.float32)
        self.batches = iter(seed_batches)
        self.fanouts = list(fanouts)
        self.words = np.ascontiguousarray(sampler_words, dtype=np.uint64).copy()
        self.cache = OracleCache(self.n, cache_lines, policy, ways, evict_words, evict_key)
        self.cache_rows = np.zeros((max(1, self.cache.lines), self.dim), np.float32)
        self.W = window_depth
        self.base_threshold = base_threshold
        self.alpha = redirect_ema_alpha
        self.cap = runahead_cap
        self.keep_rows = keep_rows
        self.ema = 0.0
        self.pending: deque = deque()
        self.pending_storage = 0
        self.window: deque = deque()
        self.ringed = 0
        self.exhausted = False
        self.epoch = 0

    def effective_threshold(self) -> int:
        return math.ceil(self.base_threshold / max(1e-3, 1.0 - self.ema))

    def _sample_one(self) -> bool:
        try:
            seeds = next(self.batches)
        except StopIteration:
            self.exhausted = True
            return False
        layers, uniq, _ = sample_subgraph(self.indptr, self.indices, seeds, self.fanouts,
                                          self.words)
        contrib = self.cache.contribution(uniq, self.pinned_off)
        self.pending.append((seeds, layers, uniq, contrib))
        self.pending_storage += contrib
        return True

    def run_ahead(self) -> None:
        want = self.W + 1
        while not self.exhausted:
            need_window = len(self.pending) < want
            need_thr = self.pending_storage < self.effective_threshold()
            if not (need_window or need_thr):
                break
            if len(self.pending) >= self.cap:
                break
            if (not need_window) and self.pending_storage == 0:
                break
            self._sample_one()
        while self.ringed < min(self.W, len(self.pending)):
            self.window.append(self.pending[self.ringed][2])
            self.ringed += 1

    def next_batch(self):
        self.run_ahead()
        if not self.pending:
            raise StopIteration
        inflight = self.pending_storage
        seeds, layers, uniq, contrib = self.pending.popleft()
        self.pending_storage -= contrib
        if self.ringed > 0:
            self.window.popleft()
            self.ringed -= 1
        self.run_ahead()
        self.cache.window_update(uniq, list(self.window))
        kind, slot = self.cache.access_batch(uniq, self.epoch)
        self.epoch += 1
        rows, tiers = gather(uniq, kind, slot, self.pinned_off, self.buffer_rows, self.table,
                             self.cache_rows)
        sampled = len(uniq)
        redirect = (tiers[0] + tiers[1]) / sampled if sampled else 0.0
        self.ema = self.alpha * redirect + (1.0 - self.alpha) * self.ema
        return {"seeds": seeds, "layers": layers, "unique": uniq,
                "rows": rows if self.keep_rows else None, "tiers": tiers,
                "inflight": inflight, "kind": kind, "slot": slot}


def shared_cache_tiers(indptr, indices, buffer_nodes, rank_batches, fanouts, rank_words,
                       evict_seed: int, lines: int, window_depth: int, steps: int):
    """Multi-rank oracle of the owner-sharded cache (shared_cache.py):
    G ranks, rank r serving global batches r, r+G, ... sampled from its own
    stream; one reference CacheState per owner (nodes v with v % G == o, its
    eviction stream PCG64(evict_seed).jumped(o)) driven by its nodes of every
    batch in global batch order, the window being its nodes of the next W
    batches (cache.py:66-218).  Returns, per global batch, (unique nodes,
    [hits, buffer, storage, bypasses])."""
    G = len(rank_batches)
    n = len(indptr) - 1
    total = steps * G + window_depth
    uniq = []
    words = [np.ascontiguousarray(w, dtype=np.uint64).copy() for w in rank_words]
    nxt = [0] * G
    for b in range(total):
        r = b % G
        seeds = rank_batches[r][nxt[r]]
        nxt[r] += 1
        _, u, _ = sample_subgraph(indptr, indices, seeds, fanouts, words[r])
        uniq.append(np.asarray(u, dtype=np.int64))
    pinned = np.zeros(n, bool)
    pinned[np.asarray(buffer_nodes, dtype=np.int64)] = True
    caches = []
    for o in range(G):
        bg = np.random.PCG64(evict_seed).jumped(o)
        st = bg.state
        m = (1 << 64) - 1
        s, inc = st["state"]["state"], st["state"]["inc"]
        w = np.array([s >> 64, s & m, inc >> 64, inc & m, st["has_uint32"], st["uinteger"]],
                     dtype=np.uint64)
        caches.append(OracleCache(n, lines, "exact", rng_words=w))
    out = []
    for b in range(steps * G):
        u = uniq[b]
        kind = np.empty(len(u), np.int8)
        for o in range(G):
            mine = (u % G) == o
            cur = u[mine]
            fut = [f[(f % G) == o] for f in uniq[b + 1:b + 1 + window_depth]]
            caches[o].window_update(cur, fut)
            k, _ = caches[o].access_batch(cur)
            kind[mine] = k
        hit = kind == 0
        out.append((u, [int(hit.sum()), int((~hit & pinned[u]).sum()),
                        int((~hit & ~pinned[u]).sum()), int((kind == 2).sum())]))
    return out

"""GPU software cache: protocol types and the lookahead window (cache.py mirror).

The cache itself lives in HBM inside the libgids handle (csrc/cache.cu); this
module keeps the reference's vocabulary around it:

* ``CacheProtocolError`` / ``LineState`` / ``AccessKind`` / ``AccessResult`` /
  ``CacheStats``  cache.py:34-63
* ``WindowBuffer``  cache.py:66-91 -- a ring of the next W batches' unique
  lists (device tensors); push/pop also move the per-node lookahead counts
  the GPU ``window_update`` reads (cache.py:190-218)
* ``GpuCacheView``  read-only CacheState-like counters of a handle
  (cache.py:104-113,182-187)
* ``CacheState`` / ``window_update``  cache.py:94-218 driven directly: the
  reference's exact policy on a libgids handle of its own (HBM), for callers
  that use the cache without the loader
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from enum import Enum, IntEnum

import numpy as np

from . import _native


class CacheProtocolError(Exception):
    """The window-buffer discipline was violated by the caller."""


class LineState(IntEnum):
    EMPTY = 0
    SAFE_TO_EVICT = 1
    IN_USE = 2


class AccessKind(Enum):
    HIT = "hit"
    MISS = "miss"
    BYPASS = "bypass"


KIND_OF_CODE = {_native.KIND_HIT: AccessKind.HIT, _native.KIND_MISS: AccessKind.MISS,
                _native.KIND_BYPASS: AccessKind.BYPASS}


@dataclass(frozen=True)
class AccessResult:
    kind: AccessKind
    slot: int | None = None
    evicted: int | None = None


@dataclass(frozen=True)
class CacheStats:
    hits: int
    misses: int
    bypasses: int
    evictions: int
    hit_ratio: float


class WindowBuffer:
    """Ring of up to ``depth`` future per-iteration unique-node lists."""

    def __init__(self, depth: int, handle: _native.Handle | None = None,
                 stream: int | None = None):
        if depth < 0:
            raise ValueError("depth must be non-negative")
        self.depth = depth
        self.lists: deque = deque()
        self._h = handle
        self._stream = stream
        # deferred device updates (the loader folds a pop + push into its
        # next serve, gids_serve_shift): ("pop" | "push", nodes) in order
        self.defer = False
        self._ops: list = []

    def _st(self) -> int:
        return self._stream if self._stream is not None else _native.stream_ptr(self._h.device)

    def __len__(self) -> int:
        return len(self.lists)

    def push_iteration(self, nodes, trusted: bool = False) -> None:
        """Append one future iteration's ascending unique list (a CUDA int64
        tensor; an unbound window also takes array-likes, as the reference's)."""
        if len(self.lists) >= self.depth:
            raise CacheProtocolError(f"window already holds {self.depth} iterations")
        if not hasattr(nodes, "numel"):
            if self._h is not None:
                raise TypeError("a handle-bound window takes CUDA int64 tensors")
            nodes = np.asarray(nodes, dtype=np.int64)
            if len(nodes) > 1 and np.any(np.diff(nodes) <= 0):
                raise CacheProtocolError("iteration list must be ascending and unique")
            self.lists.append(nodes)
            return
        if not trusted and nodes.numel() > 1 and not bool((nodes[1:] > nodes[:-1]).all()):
            raise CacheProtocolError("iteration list must be ascending and unique")
        self.lists.append(nodes)
        if self._h is not None:
            if self.defer:
                self._ops.append(("push", nodes))
            else:
                self._h.window_push(nodes, self._st())

    def pop_iteration(self):
        if not self.lists:
            raise CacheProtocolError("window is empty")
        nodes = self.lists.popleft()
        if self._h is not None:
            if self.defer:
                self._ops.append(("pop", nodes))
            else:
                self._h.window_pop(nodes, self._st())
        return nodes

    def flush(self) -> None:
        """Launch the deferred device updates, in order."""
        ops, self._ops = self._ops, []
        for op, nodes in ops:
            if op == "push":
                self._h.window_push(nodes, self._st())
            else:
                self._h.window_pop(nodes, self._st())

    def take_shift(self):
        """(pop, push) lists for gids_serve_shift when the deferred updates are
        at most one pop then at most one push; otherwise they are launched
        now and (None, None) is returned."""
        ops = self._ops
        if not ops:
            return None, None
        if len(ops) == 1:
            self._ops = []
            return (ops[0][1], None) if ops[0][0] == "pop" else (None, ops[0][1])
        if len(ops) == 2 and ops[0][0] == "pop" and ops[1][0] == "push":
            self._ops = []
            return ops[0][1], ops[1][1]
        self.flush()
        return None, None


class GpuCacheView:
    """CacheState-shaped read access to the HBM cache of a handle."""

    def __init__(self, handle: _native.Handle, page_bytes: int):
        self._h = handle
        self.capacity_lines = handle.capacity()
        self.line_bytes = page_bytes

    def _c(self):
        return self._h.cache_stats()

    hits = property(lambda self: self._c().hits)
    misses = property(lambda self: self._c().misses)
    bypasses = property(lambda self: self._c().bypasses)
    evictions = property(lambda self: self._c().evictions)
    total_increments = property(lambda self: self._c().total_increments)
    total_decrements = property(lambda self: self._c().total_decrements)

    def stats(self) -> CacheStats:
        c = self._c()
        total = c.hits + c.misses + c.bypasses
        return CacheStats(hits=c.hits, misses=c.misses, bypasses=c.bypasses,
                          evictions=c.evictions, hit_ratio=c.hits / total if total else 0.0)

    def lines(self):
        """(node per line, LineState code per line) snapshot."""
        return self._h.cache_lines()

    @property
    def resident(self) -> dict:
        node, _ = self._h.cache_lines()
        return {int(x): i for i, x in enumerate(node.tolist()) if x >= 0}

    def eviction_rng_words(self):
        return self._h.cache_rng()


NodeId = int


class CacheState(GpuCacheView):
    """CacheState (cache.py:94-187) in HBM, driven by libgids.

    The reference's policy exactly (fully associative, lowest empty line
    first, uniform eviction among SafeToEvict lines from the numpy stream of
    ``eviction_seed``, bypass when every line is InUse).  Same constructor
    plus ``num_nodes`` (per-node state is dense on the GPU) and ``device``.
    ``access(node)`` serves one node like the reference; ``access_batch``
    serves distinct nodes in order in one call (the loader's path)."""

    def __init__(self, capacity_lines: int, line_bytes: int, eviction_seed: int = 0, *,
                 num_nodes: int, device: int = 0):
        if capacity_lines < 0:
            raise ValueError("capacity_lines must be non-negative")
        if line_bytes < 1:
            raise ValueError("line_bytes must be positive")
        if num_nodes < 1:
            raise ValueError("num_nodes must be positive")
        import torch

        from .sampling import pcg_words
        self.num_nodes = num_nodes
        self._dev = torch.device("cuda", device)
        h = _native.Handle(num_nodes=num_nodes, num_edges=0, feature_dim=1, device=device,
                           cache_lines=capacity_lines, policy="exact", ways=32, evict_key=0,
                           window_depth=255, fanouts=[1], max_seeds=num_nodes,
                           eviction_words=pcg_words(np.random.default_rng(eviction_seed)))
        super().__init__(h, line_bytes)
        self._owned = h

    def _nodes(self, nodes):
        import torch
        arr = np.asarray(nodes, dtype=np.int64).reshape(-1)
        if len(arr) and (arr.min() < 0 or arr.max() >= self.num_nodes):
            bad = int(arr[(arr < 0) | (arr >= self.num_nodes)][0])
            raise ValueError(f"node {bad} out of range (num_nodes={self.num_nodes})")
        return torch.as_tensor(arr).to(self._dev)

    def access_batch(self, nodes):
        """Serve distinct nodes in order: (kind int8[n] of _native.KIND_*,
        line int32[n], -1 on bypass)."""
        import torch
        t = self._nodes(nodes)
        n = t.numel()
        if n > 1 and int(torch.unique(t).numel()) != n:
            raise ValueError("access_batch takes distinct nodes (use access() per repeat)")
        kind = torch.empty(n, dtype=torch.int8, device=self._dev)
        line = torch.empty(n, dtype=torch.int32, device=self._dev)
        st = _native.stream_ptr(self._dev.index)
        self._h.cache_access(t, kind, line, None, st)
        return kind.cpu().numpy(), line.cpu().numpy()

    def access(self, node: NodeId) -> AccessResult:
        """Serve one node; classify as hit, miss (inserted), or bypass."""
        import torch
        t = self._nodes([node])
        kind = torch.empty(1, dtype=torch.int8, device=self._dev)
        line = torch.empty(1, dtype=torch.int32, device=self._dev)
        victim = torch.empty(1, dtype=torch.int64, device=self._dev)
        self._h.cache_access(t, kind, line, victim, _native.stream_ptr(self._dev.index))
        k = KIND_OF_CODE[int(kind.item())]
        if k is AccessKind.BYPASS:
            return AccessResult(k)
        v = int(victim.item())
        return AccessResult(k, slot=int(line.item()),
                            evicted=v if (k is AccessKind.MISS and v >= 0) else None)

    @property
    def slot_node(self) -> np.ndarray:
        return self._h.cache_lines()[0]

    @property
    def line_state(self) -> np.ndarray:
        return self._h.cache_lines()[1]

    @property
    def reuse_counter(self) -> dict:
        r = self._h.cache_reuse(self.num_nodes)
        nz = np.flatnonzero(r)
        return dict(zip(nz.tolist(), r[nz].astype(np.int64).tolist()))

    def close(self) -> None:
        self._owned.close()


def window_update(cache: CacheState, window: WindowBuffer, current_batch) -> dict:
    """Fold the current batch's future occurrences into the cache metadata
    (cache.py:190-218): each node's count of window lists containing it
    raises its reuse counter and flips its resident SafeToEvict line to
    InUse, on the GPU.  Returns {node: count} for the whole batch."""
    import torch
    h = cache._h
    st = _native.stream_ptr(cache._dev.index)
    cur = cache._nodes(current_batch)
    if len(window.lists) > 255:
        raise ValueError("the GPU lookahead counts are 8-bit: at most 255 window lists")
    lists = [l if hasattr(l, "numel") else cache._nodes(l) for l in window.lists]
    for l in lists:
        h.window_push(l, st)
    counts = torch.zeros(cur.numel(), dtype=torch.int32, device=cache._dev)
    h.cache_window_update(cur, counts, st)
    for l in lists:
        h.window_pop(l, st)
    return dict(zip(cur.cpu().tolist(), counts.cpu().tolist()))

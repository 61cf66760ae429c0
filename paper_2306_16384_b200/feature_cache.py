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
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from enum import Enum, IntEnum

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

    def _st(self) -> int:
        return self._stream if self._stream is not None else _native.stream_ptr(self._h.device)

    def __len__(self) -> int:
        return len(self.lists)

    def push_iteration(self, nodes, trusted: bool = False) -> None:
        """Append one future iteration's ascending unique list (a CUDA int64 tensor)."""
        if len(self.lists) >= self.depth:
            raise CacheProtocolError(f"window already holds {self.depth} iterations")
        if not trusted and nodes.numel() > 1 and not bool((nodes[1:] > nodes[:-1]).all()):
            raise CacheProtocolError("iteration list must be ascending and unique")
        self.lists.append(nodes)
        if self._h is not None:
            self._h.window_push(nodes, self._st())

    def pop_iteration(self):
        if not self.lists:
            raise CacheProtocolError("window is empty")
        nodes = self.lists.popleft()
        if self._h is not None:
            self._h.window_pop(nodes, self._st())
        return nodes


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

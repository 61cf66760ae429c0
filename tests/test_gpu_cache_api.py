"""The cache driven directly: GPU CacheState / window_update (cache.py:94-218).

Paired traces in the style of the reference's tests/test_cache.py:34-53: the
GPU cache and the oracle cache (pinned to the reference's CacheState by the
golden runs) replay the same window updates and accesses, and every step's
result, the eviction victims, the line table, the reuse counters and the
tallies agree."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2306_16384_b200 import (AccessKind, CacheProtocolError, CacheState, WindowBuffer,
                                   window_update)
from paper_2306_16384_b200.sampling import pcg_words

pytestmark = pytest.mark.gpu
KIND = {AccessKind.HIT: O.K_HIT, AccessKind.MISS: O.K_MISS, AccessKind.BYPASS: O.K_BYPASS}


def _pair(capacity, universe, seed):
    gpu = CacheState(capacity, line_bytes=64, eviction_seed=seed, num_nodes=universe)
    ref = O.OracleCache(universe, capacity, "exact",
                        rng_words=pcg_words(np.random.default_rng(seed)))
    return gpu, ref


def _same_state(gpu, ref, universe):
    node, state = gpu.lines()
    onode, ostate = ref.lines_snapshot()
    assert np.array_equal(node, onode) and np.array_equal(state, ostate)
    s = ref.stats()
    assert (gpu.hits, gpu.misses, gpu.bypasses, gpu.evictions) == \
        (s["hits"], s["misses"], s["bypasses"], s["evictions"])
    assert (gpu.total_increments, gpu.total_decrements) == \
        (s["total_increments"], s["total_decrements"])


def _paired_trace(capacity, depth, lists, seed, universe):
    gpu, ref = _pair(capacity, universe, seed)
    for i, cur in enumerate(lists):
        future = lists[i + 1:i + 1 + depth]
        win = WindowBuffer(depth)
        for l in future:
            win.push_iteration(l)
        report = window_update(gpu, win, cur)
        counts = ref.window_update(cur, future)
        assert report == dict(zip(cur.tolist(), counts.tolist()))
        for x in cur.tolist():
            before, _ = ref.lines_snapshot()
            got = gpu.access(x)
            kind, slot = ref.access_batch(np.array([x]))
            assert KIND[got.kind] == int(kind[0])
            if got.kind is not AccessKind.BYPASS:
                assert got.slot == int(slot[0])
            if got.kind is AccessKind.MISS:
                prev = int(before[got.slot])
                assert got.evicted == (prev if prev >= 0 else None)
        _same_state(gpu, ref, universe)
    leftover = sum(gpu.reuse_counter.values())
    assert gpu.total_increments == gpu.total_decrements + leftover
    gpu.close()


def _random_trace(rng, universe, iterations, max_list):
    return [np.unique(rng.integers(0, universe, size=int(rng.integers(1, max_list + 1))))
            for _ in range(iterations)]


def test_gpu_cache_documented_scenario():
    lists = [np.array([1, 2, 3]), np.array([1, 4]), np.array([2, 5, 6]), np.array([1, 2]),
             np.array([7])]
    _paired_trace(3, 2, lists, 5, universe=16)


def test_gpu_cache_random_traces():
    rng = np.random.default_rng(12)
    for trial in range(24):
        capacity = int(rng.integers(1, 65))
        universe = int(rng.integers(8, 257))
        lists = _random_trace(rng, universe, int(rng.integers(2, 8)), int(rng.integers(4, 40)))
        _paired_trace(capacity, (0, 2, 8)[trial % 3], lists, trial, universe)


def test_gpu_cache_batch_access_equals_per_node_access():
    rng = np.random.default_rng(4)
    lists = _random_trace(rng, 200, 8, 60)
    a = CacheState(24, 64, eviction_seed=9, num_nodes=200)
    b = CacheState(24, 64, eviction_seed=9, num_nodes=200)
    for i, cur in enumerate(lists):
        win = WindowBuffer(3)
        for l in lists[i + 1:i + 4]:
            win.push_iteration(l)
        assert window_update(a, win, cur) == window_update(b, win, cur)
        kind, line = a.access_batch(cur)
        per = [b.access(int(x)) for x in cur]
        assert [KIND[r.kind] for r in per] == kind.tolist()
        assert [r.slot if r.slot is not None else -1 for r in per] == line.tolist()
    assert np.array_equal(a.lines()[0], b.lines()[0]) and a.stats() == b.stats()


def test_gpu_cache_protocol_and_validation():
    with pytest.raises(ValueError):
        CacheState(-1, 64, num_nodes=4)
    with pytest.raises(ValueError):
        CacheState(4, 0, num_nodes=4)
    c = CacheState(4, 64, num_nodes=10)
    with pytest.raises(ValueError, match="out of range"):
        c.access(10)
    with pytest.raises(ValueError, match="distinct"):
        c.access_batch([1, 1])
    w = WindowBuffer(1)
    w.push_iteration([1, 2])
    with pytest.raises(CacheProtocolError):
        w.push_iteration([3])
    with pytest.raises(CacheProtocolError):
        WindowBuffer(2).push_iteration([2, 1])
    victims = set()
    for seed in range(20):  # eviction choice is not degenerate
        c = CacheState(4, 64, eviction_seed=seed, num_nodes=128)
        for x in range(4):
            c.access(x)
        victims.add(c.access(99).evicted)
    assert len(victims) > 1

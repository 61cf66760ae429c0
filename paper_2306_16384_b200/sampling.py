"""Layered uniform neighbour sampling on the GPU (sampler.py mirror).

``sample_subgraph(g, seeds, fanouts, rng)`` keeps the reference signature,
argument meaning and errors (sampler.py:23-29,87-112) and returns the same
MiniBatch -- with ``layers`` and ``unique_nodes`` as int64 CUDA tensors.  The
draws are bit-identical to the reference's because the kernel addresses
every draw of the numpy PCG64 stream by offset (see csrc/sampler.cu), and
``rng`` is advanced by exactly the number of doubles the reference would
have consumed, so the next call continues the same stream.
"""
from __future__ import annotations

import weakref
from dataclasses import dataclass
from typing import Iterator, Sequence

import numpy as np

from . import _native
from .csc import GraphCsc

Fanouts = Sequence[int]


def check_fanouts(fanouts: Fanouts) -> list[int]:
    fans = [int(f) for f in fanouts]
    if not fans:
        raise ValueError("fanouts must be non-empty")
    if any(f < 1 for f in fans):
        raise ValueError("every fanout must be >= 1")
    return fans


def check_seeds(seeds, num_nodes: int) -> np.ndarray:
    s = np.asarray(seeds, dtype=np.int64)
    if len(s) == 0:
        raise ValueError("seeds must be non-empty")
    if s.min() < 0 or s.max() >= num_nodes:
        out = (s < 0) | (s >= num_nodes)
        raise ValueError(f"seed node {int(s[out][0])} out of range (num_nodes={num_nodes})")
    return s


@dataclass(frozen=True)
class MiniBatch:
    """One sampled minibatch (sampler.py:32-47); layers[l] is (E_l, 2) [src, dst]."""

    seeds: np.ndarray
    layers: list
    unique_nodes: object

    @property
    def num_sampled_edges(self) -> int:
        return sum(int(l.shape[0]) for l in self.layers)

    def to_numpy(self) -> "MiniBatch":
        return MiniBatch(seeds=self.seeds,
                         layers=[l.cpu().numpy() if hasattr(l, "cpu") else l for l in self.layers],
                         unique_nodes=self.unique_nodes.cpu().numpy()
                         if hasattr(self.unique_nodes, "cpu") else self.unique_nodes)


def pcg_words(rng) -> np.ndarray:
    """The 6-word ABI state of a numpy PCG64-backed Generator."""
    bg = getattr(rng, "bit_generator", rng)
    st = bg.state
    if st.get("bit_generator") != "PCG64":
        raise TypeError("the GPU sampler reproduces numpy PCG64 streams (np.random.default_rng)")
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m, st["has_uint32"], st["uinteger"]],
                    dtype=np.uint64)


class Sampler:
    """Sampling front end bound to one device handle (graph resident in HBM)."""

    def __init__(self, handle: _native.Handle, num_nodes: int, fanouts: Fanouts):
        self.h = handle
        self.num_nodes = num_nodes
        self.fanouts = check_fanouts(fanouts)

    def launch(self, seeds: np.ndarray, rng, stream: int) -> None:
        self.h.sample(seeds, pcg_words(rng), stream)

    def collect(self, seeds: np.ndarray, rng, stream: int, torch_stream=None):
        """Sizes -> tensors -> export; advances rng.  Returns (MiniBatch, contribution).

        ``torch_stream`` (the torch.cuda.Stream behind ``stream``) owns the
        output tensors when given; otherwise the current stream does."""
        import contextlib

        import torch
        lens, n_unique, draws, contrib = self.h.sample_sizes()
        dev = torch.device("cuda", self.h.device)
        total = int(lens.sum())
        ctx = torch.cuda.stream(torch_stream) if torch_stream is not None else \
            contextlib.nullcontext()
        with ctx:
            edges = torch.empty((total, 2), dtype=torch.int64, device=dev)
            unique = torch.empty(n_unique, dtype=torch.int64, device=dev)
        self.h.sample_export(edges, unique, stream)
        layers, off = [], 0
        for ln in lens.tolist():
            layers.append(edges[off:off + ln])
            off += ln
        if draws:
            rng.bit_generator.advance(draws)
        return MiniBatch(seeds=seeds, layers=layers, unique_nodes=unique), contrib

    def sample(self, seeds, rng) -> MiniBatch:
        s = check_seeds(seeds, self.num_nodes)
        st = _native.stream_ptr(self.h.device)
        self.launch(s, rng, st)
        return self.collect(s, rng, st)[0]


_HANDLES: dict = {}


def _sampler_for(g: GraphCsc, fans: list[int], n_seeds: int, device: int) -> Sampler:
    key = (id(g), tuple(fans), device)
    hit = _HANDLES.get(key)
    if hit is not None and hit[0]() is g and hit[1].h.cfg.max_seeds >= n_seeds:
        return hit[1]
    cap = 1 << max(10, (n_seeds - 1).bit_length())
    h = _native.Handle(num_nodes=g.num_nodes, num_edges=g.num_edges, feature_dim=1, device=device,
                       cache_lines=0, policy="exact", ways=32, evict_key=0, window_depth=0,
                       fanouts=fans, max_seeds=cap, eviction_words=np.zeros(6, np.uint64))
    h.load_graph(g.indptr, g.indices)
    smp = Sampler(h, g.num_nodes, fans)
    _HANDLES[key] = (weakref.ref(g, lambda _r, k=key: _HANDLES.pop(k, None)), smp)
    return smp


def sample_subgraph(g: GraphCsc, seeds, fanouts: Fanouts, rng, device: int = 0) -> MiniBatch:
    """k-hop sample from ``seeds``, one layer per fanout (sampler.py:87-112), on the GPU."""
    fans = check_fanouts(fanouts)
    s = check_seeds(seeds, g.num_nodes)
    return _sampler_for(g, fans, len(s), device).sample(s, rng)


def sample_layer(g: GraphCsc, frontier, fanout: int, rng, device: int = 0):
    """One hop (sampler.py:50-84) on the GPU: up to ``fanout`` distinct
    in-neighbours per frontier entry, (E, 2) [src, dst] grouped in frontier
    order.  The frontier is taken exactly as given -- any order, repeats
    expanded again with draws of their own -- as the reference's loop does."""
    if fanout < 1:
        raise ValueError("fanout must be >= 1")
    f = np.asarray(frontier, dtype=np.int64).reshape(-1)
    if len(f) == 0:
        import torch
        return torch.empty((0, 2), dtype=torch.int64, device=torch.device("cuda", device))
    f = check_seeds(f, g.num_nodes)
    smp = _sampler_for(g, [int(fanout)], len(f), device)
    st = _native.stream_ptr(device)
    smp.h.sample_frontier(f, pcg_words(rng), st)
    return smp.collect(f, rng, st)[0].layers[0]


def batch_iterator(seed_set, batch_size: int, shuffle: bool = False,
                   rng=None) -> Iterator[np.ndarray]:
    """Consecutive ``batch_size`` chunks of the (optionally permuted) seed set."""
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    seeds = np.asarray(seed_set, dtype=np.int64)
    if shuffle:
        if rng is None:
            raise ValueError("shuffle requires an rng")
        seeds = rng.permutation(seeds)
    return (seeds[i:i + batch_size] for i in range(0, len(seeds), batch_size))

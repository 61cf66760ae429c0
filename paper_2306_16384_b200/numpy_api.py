"""The reference's output types, exactly: numpy arrays instead of CUDA tensors.

The package returns device tensors (``MiniBatch.layers`` / ``unique_nodes``
and the gathered rows stay in HBM for the consumer, a GPU model).  Code
written against the reference that expects numpy -- its tests, CPU-side
tooling -- can use these drop-ins instead; each is the package call followed
by one device-to-host copy:

* ``Dataloader``        next_batch() -> (MiniBatch of numpy, rows np.ndarray, stats)
* ``sample_layer`` / ``sample_subgraph``   sampler.py:50-112 with numpy results
* ``CacheState``        the reference constructor (no node count; dense
                        per-node GPU state sized for ids below ``NODE_BOUND``)

tests/refshim/tierloader (the reference's own tests run against the package)
is built on this module.
"""
from __future__ import annotations

import numpy as np

from . import feature_cache as _c
from . import loader as _l
from . import sampling as _s

NODE_BOUND = 1 << 20


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def sample_layer(g, frontier, fanout, rng):
    return _np(_s.sample_layer(g, frontier, fanout, rng))


def sample_subgraph(g, seeds, fanouts, rng):
    return _s.sample_subgraph(g, seeds, fanouts, rng).to_numpy()


class CacheState(_c.CacheState):
    def __init__(self, capacity_lines, line_bytes, eviction_seed=0):
        super().__init__(capacity_lines, line_bytes, eviction_seed, num_nodes=NODE_BOUND)


class Dataloader(_l.Dataloader):
    def next_batch(self):
        mb, rows, st = super().next_batch()
        return mb.to_numpy(), rows.cpu().numpy(), st


def run(dl, iterations=None, warmup=None):
    return _l.run(dl, iterations, warmup)

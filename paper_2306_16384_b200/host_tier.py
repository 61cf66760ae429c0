"""One host tier per node, shared by the data-parallel ranks on it.

The reference holds one FeatureStore (graph.py:278-301) and one
ConstantBuffer (cpu_buffer.py:112-139).  Data-parallel replicas that each
pinned a private copy would hold G copies of the table and the buffer in
host DRAM (C4 x 8 ranks: ~8 x (57 + 5.7) GB) and pin them G times.  Here the
node's local rank 0 creates both in POSIX shared memory and fills them once;
every local rank maps the same pages and page-locks its mapping for
zero-copy reads (``_native.SharedHost``).  The names come from a token
broadcast over ``torch.distributed`` (the control plane); they are unlinked
as soon as every rank has attached, so nothing outlives the job.

Only the bytes are shared: each rank still reads its own batches' rows over
its own PCIe link, so per-rank results are exactly those of a private copy
(tests/test_host_tier.py, tests/test_gpu_shared_host.py).
"""
from __future__ import annotations

import os
import secrets
from typing import Callable

import numpy as np

from . import _native


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def local_rank(default: int) -> int:
    return int(os.environ.get("LOCAL_RANK", default))


def job_token() -> str:
    """A name shared by every rank of the job (rank 0's random token)."""
    dist = _dist()
    tok = [secrets.token_hex(6) if (dist is None or dist.get_rank() == 0) else None]
    if dist is not None:
        dist.broadcast_object_list(tok, src=0)
    return tok[0]


def _barrier() -> None:
    dist = _dist()
    if dist is not None:
        dist.barrier()


class SharedRegion:
    """``shape``/``dtype`` array in /dev/shm: created and filled by the local
    creator, attached by the other local ranks (collective: every rank calls
    it in the same order)."""

    def __init__(self, name: str, shape, dtype, creator: bool,
                 fill: Callable[[np.ndarray], None], register: bool = True):
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        self.region = None
        if creator:
            self.region = _native.SharedHost(name, max(nbytes, 1), create=True, register=register)
            fill(self.region.array(shape, dtype) if nbytes else np.empty(shape, dtype))
        _barrier()  # filled
        if not creator:
            self.region = _native.SharedHost(name, max(nbytes, 1), create=False,
                                             register=register)
        _barrier()  # everyone attached
        if creator:
            self.region.unlink()
        _barrier()  # the name is gone for every rank when this returns
        self.array = self.region.array(shape, dtype) if nbytes else np.empty(shape, dtype)

    def close(self) -> None:
        self.array = None
        if self.region is not None:
            self.region.close()
            self.region = None

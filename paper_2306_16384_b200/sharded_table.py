"""HBM-sharded feature table for data-parallel ranks.

When the feature table is larger than one GPU (C5: 100M x 1024-d fp32 =
409.6 GB over 8 x B200), each rank keeps one shard in its HBM: node v is
owned by shard ``v % G`` at row ``v // G``.  Shards are exported as CUDA IPC
handles, exchanged once through ``torch.distributed`` (the control plane),
and opened by every rank, so a rank's gather kernel reads local rows from
HBM and remote rows as peer loads over NVLink -- the data path has no
collective.  ``virtual_shards`` places all G shards on this rank's device
(one process), which runs the same kernel over local pointers; tests use it
to check the sharded gather on a single GPU.

The shard contents are the reference's synthetic rows (graph.py:256-275),
written on the device (``gids_synthesize_rows_strided``).
"""
from __future__ import annotations

from . import _native


def exchange_handles(handle: bytes, group=None) -> list[bytes]:
    """All ranks' 64-byte IPC handles, in rank order (torch.distributed)."""
    import torch.distributed as dist
    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    return [bytes(h) for h in out]


def shard_rows(num_nodes: int, shard: int, n_shards: int) -> int:
    """Rows held by ``shard``: nodes shard, shard+G, ... below num_nodes."""
    return max(0, (num_nodes - shard + n_shards - 1) // n_shards)


class ShardedTable:
    def __init__(self, num_nodes: int, dim: int, seed: int, device: int, rank: int,
                 world: int, virtual: bool = False, group=None):
        import torch
        self.num_nodes, self.dim, self.seed = num_nodes, dim, seed
        self.device, self.rank, self.world = device, rank, world
        self._opened: list[int] = []
        st = _native.stream_ptr(device)
        mine = range(world) if virtual else [rank]
        # each shard is its own device allocation (an IPC handle maps a whole
        # allocation, so it must not be a sub-block of torch's caching allocator)
        self.shards: dict[int, int] = {}
        self.local_bytes = 0
        for s in mine:
            n = shard_rows(num_nodes, s, world)
            nbytes = max(n, 1) * dim * 4
            ptr = _native.device_alloc(device, nbytes)
            self.shards[s] = ptr
            self.local_bytes += nbytes
            _native.synthesize_rows_strided(device, seed, s, world, n, dim, ptr, st)
        torch.cuda.synchronize(device)
        if virtual or world == 1:
            self.ptrs = [self.shards[s] for s in range(world)]
        else:
            handles = exchange_handles(_native.ipc_handle(device, self.shards[rank]), group)
            self.ptrs = []
            for s, hd in enumerate(handles):
                if s == rank:
                    self.ptrs.append(self.shards[rank])
                else:
                    p = _native.ipc_open(device, hd)
                    self._opened.append(p)
                    self.ptrs.append(p)

    def close(self) -> None:
        """Unmap the peers' shards and free this rank's (callers synchronise
        with their peers first: a freed shard must not be read remotely)."""
        for p in self._opened:
            try:
                _native.ipc_close(self.device, p)
            except Exception:
                pass
        self._opened = []
        for p in self.shards.values():
            try:
                _native.device_free(self.device, p)
            except Exception:
                pass
        self.shards = {}

"""Owner-sharded cache of data-parallel ranks.

Data-parallel ranks serve their own batches (rank r: global batches r, r+G,
...).  With ``gids_shared_cache`` they share one cache instead of keeping G
replicas: node v lives only in the HBM cache lines of its owner, rank v % G,
so the aggregate cache holds G times as many distinct rows.  One exchange
step per global step s (batches sG .. sG+G-1):

1. every rank groups the unique nodes of a batch by owner (``gids_owner_split``)
   and sends each owner its list -- for the window, ``ceil(W/G)`` steps
   ahead of the step that serves it;
2. each owner runs the reference policy (``window_update`` +
   ``CacheState.access``, cache.py:144-218) over the G lists of the step in
   global batch order, the window being the owned parts of the next W
   batches, and marks fresh hits / final inserters (``gids_shared_marks``,
   ``gids_shared_final``);
3. the decisions go back; each requester gathers its rows -- hits from the
   owner's lines (peer loads over NVLink through CUDA IPC pointers), the rest
   from its own host tiers -- and after a cross-rank barrier the final
   inserters write their rows into the owners' lines (peer stores).

The exchange is two ``all_to_all`` collectives of node ids / packed decisions
(``torch.distributed``: NCCL on GPUs, gloo in the CPU-side tests); rows never
cross a collective.  The multi-rank oracle is one reference CacheState per
owner over its nodes of every batch in global batch order
(tests/test_gpu_shared_cache.py).
"""
from __future__ import annotations

import math

import numpy as np

from . import _native


def _dist():
    import torch.distributed as dist
    return dist


class OwnerShardedCache:
    """The exchange protocol of one rank (owner and requester roles)."""

    def __init__(self, handle: _native.Handle, rank: int, world: int, window_depth: int,
                 device: int, group=None):
        import torch
        self.h, self.rank, self.G, self.W = handle, rank, world, window_depth
        self.dev = torch.device("cuda", device)
        self.group = group
        self.ahead = max(1, math.ceil(window_depth / world)) if window_depth else 0
        self._owned: dict[int, object] = {}   # global batch -> owned node list (device)
        self._split: dict[int, tuple] = {}    # own global batch -> (perm, counts)
        self._wpushed: list[int] = []         # batches whose owned lists are in the window
        self.debug = None                     # tests: {batch: (owned nodes, kinds, lines)}
        dist = _dist()
        backend = dist.get_backend(group) if dist.is_initialized() else "gloo"
        self._xdev = self.dev if backend == "nccl" else torch.device("cpu")
        # owners' cache rows: this rank's own, the peers' opened from CUDA IPC handles
        mine = handle.cache_rows_ptr()
        self._opened: list[int] = []
        if world == 1:
            self.rows = [mine]
        else:
            out: list = [None] * world
            dist.all_gather_object(out, _native.ipc_handle(device, mine), group=group)
            self.rows = []
            for o, hd in enumerate(out):
                if o == rank:
                    self.rows.append(mine)
                else:
                    p = _native.ipc_open(device, bytes(hd))
                    self._opened.append(p)
                    self.rows.append(p)

    # -- exchange helpers
    def _a2a(self, chunks: list, dtype):
        """all_to_all of variable-size int64 device tensors (chunk o to rank o);
        returns the received chunks (from rank o at index o) on the device."""
        import torch
        G = self.G
        if G == 1:
            return [chunks[0]]
        dist = _dist()
        sizes = torch.tensor([c.numel() for c in chunks], dtype=torch.int64, device=self._xdev)
        rsizes = torch.empty(G, dtype=torch.int64, device=self._xdev)
        dist.all_to_all_single(rsizes, sizes, group=self.group)
        send = torch.cat(chunks).to(self._xdev) if sum(c.numel() for c in chunks) else \
            torch.empty(0, dtype=dtype, device=self._xdev)
        rs = rsizes.tolist()
        recv = torch.empty(sum(rs), dtype=dtype, device=self._xdev)
        dist.all_to_all_single(recv, send, output_split_sizes=rs,
                               input_split_sizes=sizes.tolist(), group=self.group)
        recv = recv.to(self.dev)
        return list(torch.split(recv, rs))

    def send_lists(self, batch_id: int, unique, stream: int) -> None:
        """Step 1 for one of this rank's batches (global id batch_id): its
        nodes grouped by owner go to their owners (collective)."""
        import torch
        n = unique.numel()
        grouped = torch.empty(n, dtype=torch.int64, device=self.dev)
        perm = torch.empty(n, dtype=torch.int32, device=self.dev)
        counts = self.h.owner_split(unique, self.G, grouped, perm, stream)
        torch.cuda.current_stream(self.dev).synchronize()
        self._split[batch_id] = (perm, counts)
        parts = list(torch.split(grouped, counts.tolist()))
        recv = self._a2a(parts, torch.int64)
        step = batch_id // self.G
        for src, lst in enumerate(recv):
            self._owned[step * self.G + src] = lst.contiguous()

    def serve_step(self, step: int, unique, stream: int):
        """Steps 2-3 for global step `step` (collective); returns this rank's
        decisions (packed int64 per unique node, unique order) and its batch's
        tier counts [hits, buffer, storage, bypasses]."""
        import torch
        G, h = self.G, self.h
        st = stream
        step0 = step * G
        dec_parts = []
        per = []
        for b in range(step0, step0 + G):
            # the window: owned parts of batches b+1 .. b+W (cache.py:66-91)
            while self._wpushed and self._wpushed[0] <= b:
                h.window_pop(self._owned[self._wpushed.pop(0)], st)
            nxt = self._wpushed[-1] + 1 if self._wpushed else b + 1
            for f in range(nxt, b + self.W + 1):
                if f in self._owned:
                    h.window_push(self._owned[f], st)
                    self._wpushed.append(f)
            cur = self._owned[b]
            n = cur.numel()
            kind = torch.empty(n, dtype=torch.int8, device=self.dev)
            line = torch.empty(n, dtype=torch.int32, device=self.dev)
            flags = torch.empty(n, dtype=torch.uint8, device=self.dev)
            if n:
                h.cache_window_update(cur, None, st)
                h.cache_access(cur, kind, line, None, st)
                h.shared_marks(kind, line, b, step0, flags, st)
            per.append((b, kind, line, flags))
            if self.debug is not None:
                self.debug[b] = (cur.cpu().numpy(), kind.cpu().numpy(), line.cpu().numpy())
        for b, kind, line, flags in per:
            packed = torch.empty(kind.numel(), dtype=torch.int64, device=self.dev)
            if kind.numel():
                h.shared_final(kind, line, flags, b, packed, st)
            dec_parts.append(packed)
        torch.cuda.current_stream(self.dev).synchronize()
        for b in range(step0, step0 + G):  # (the window keeps the lists it still needs)
            if b not in self._wpushed:
                self._owned.pop(b, None)
        recv = self._a2a(dec_parts, torch.int64)  # from owner o: my batch's owned part
        mine = step0 + self.rank
        perm, counts = self._split.pop(mine)
        packed = torch.cat(recv) if recv else torch.empty(0, dtype=torch.int64, device=self.dev)
        dec = torch.empty(unique.numel(), dtype=torch.int64, device=self.dev)
        h.shared_unsplit(packed, perm, dec, st)
        tiers = h.shared_tiers(unique, dec, st)
        return dec, tiers

    def gather(self, unique, dec, out, stream: int) -> None:
        """Step 3's row movement (collective: two barriers)."""
        import torch
        dist = _dist()
        self.h.shared_gather(unique, dec, self.rows, out, 0, stream)
        torch.cuda.current_stream(self.dev).synchronize()
        if self.G > 1:
            dist.barrier(group=self.group)  # every hit of the step read before any insert
        self.h.shared_gather(unique, dec, self.rows, out, 1, stream)
        torch.cuda.current_stream(self.dev).synchronize()
        if self.G > 1:
            dist.barrier(group=self.group)  # inserts landed before the next step's reads

    def close(self) -> None:
        for p in self._opened:
            try:
                _native.ipc_close(self.dev.index, p)
            except Exception:
                pass
        self._opened = []


def decode(dec: np.ndarray):
    """(kind, line, flags) arrays from packed decisions."""
    d = np.asarray(dec, dtype=np.int64)
    return ((d >> 32) & 0xff).astype(np.int8), (d & 0xffffffff).astype(np.int64), \
        ((d >> 40) & 0xff).astype(np.uint8)

"""One host tier per node shared by the data-parallel ranks (host_tier.py).

CPU (gloo, world_size 2, two processes): both ranks agree on the job token,
local rank 0 creates and fills the region, rank 1 maps the same pages (a
write by one rank is seen by the other: one copy, not two), the name is
unlinked once both attached, and a second region gets a distinct name.
(The GPU side -- both ranks page-locking the mapping and serving identical
rows and tiers from it -- is tests/test_gpu_shared_host.py.)"""
from __future__ import annotations

import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2306_16384_b200 import host_tier
    os.environ["LOCAL_RANK"] = str(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    tok = host_tier.job_token()
    creator = host_tier.local_rank(rank) == 0

    def fill(v):
        v[:] = np.arange(v.size, dtype=np.float32).reshape(v.shape)
    a = host_tier.SharedRegion(f"gids-{tok}-t", (1000, 16), np.float32, creator, fill,
                               register=False)
    ok_fill = bool((a.array.reshape(-1) == np.arange(16000, dtype=np.float32)).all())
    unlinked = not os.path.exists(f"/dev/shm/gids-{tok}-t")
    dist.barrier()
    if rank == 1:
        a.array[3, 5] = -7.0  # one copy: rank 0 must see it
    dist.barrier()
    seen = float(a.array[3, 5])
    b = host_tier.SharedRegion(f"gids-{tok}-b", (10, 4), np.float32, creator,
                               lambda v: v.fill(2.0), register=False)
    ok_b = bool((b.array == 2.0).all())
    dist.barrier()
    a.close()
    b.close()
    q.put((rank, tok, ok_fill, unlinked, seen, ok_b))
    dist.destroy_process_group()


def test_shared_region_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = {r: rest for r, *rest in (q.get(timeout=120) for _ in ps)}
    for p in ps:
        p.join(timeout=60)
    assert got[0][0] == got[1][0]  # same token
    for r in range(2):
        tok, ok_fill, unlinked, seen, ok_b = got[r]
        assert ok_fill and unlinked and ok_b
        assert seen == -7.0

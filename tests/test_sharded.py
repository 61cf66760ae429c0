"""HBM-sharded feature table.

CPU: the owner rule covers every node exactly once, and the IPC-handle
exchange over torch.distributed (gloo, world_size 2) delivers every rank's
handle in rank order.  GPU: the sharded gather (own shard over HBM, the
others through peer pointers) returns the reference's rows bit for bit --
single process with virtual shards, and two processes on one device whose
shards are opened from real CUDA IPC handles."""
from __future__ import annotations

import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2306_16384_b200.sharded_table import exchange_handles, shard_rows


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("n,g", [(1, 1), (10, 3), (100_003, 8), (7, 8)])
def test_owner_rule_covers_every_node_once(n, g):
    rows = [shard_rows(n, s, g) for s in range(g)]
    assert sum(rows) == n
    seen = np.zeros(n, np.int64)
    for s in range(g):
        ids = s + g * np.arange(rows[s])
        seen[ids] += 1
    assert (seen == 1).all()


def _exchange_worker(rank, world, port, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    mine = bytes([rank]) * 64
    q.put((rank, exchange_handles(mine)))
    dist.destroy_process_group()


def test_ipc_handle_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        assert got[r] == [bytes([0]) * 64, bytes([1]) * 64]


def _cfg(**kw):
    from paper_2306_16384_b200 import make_config
    base = dict(num_nodes=60_000, avg_degree=12.0, degree_model="uniform", feature_dim=64,
                fanouts=[10, 15], batch_size=256, cache_lines=0, buffer_fraction=0.0,
                window_depth=4, consume_rate=0.0, seed=11, gids_generator="device",
                gids_sharded_table=True)
    base.update(kw)
    return make_config(base)


@pytest.mark.gpu
def test_gpu_virtual_shards_match_reference_rows():
    from paper_2306_16384_b200 import Dataloader
    g = 3
    dl = Dataloader(_cfg(gids_virtual_shards=g, verify_gather=True))
    ref = Dataloader(_cfg(gids_sharded_table=False, cache_lines=1000))  # same sampling
    seed = dl.features.seed
    for _ in range(5):
        mb, rows, st = dl.next_batch()
        rmb, _, _ = ref.next_batch()
        u = mb.unique_nodes.cpu().numpy()
        assert np.array_equal(u, rmb.unique_nodes.cpu().numpy())
        assert np.array_equal(rows.cpu().numpy(), O.feature_rows(seed, u, 64))
        assert (st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses) == \
            (len(u), 0, 0, 0)
        local, remote = dl.shard_counts()
        assert local == int((u % g == 0).sum()) and local + remote == len(u)
    dl.close()
    ref.close()


def _ipc_worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        from paper_2306_16384_b200 import Dataloader
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        dl = Dataloader(_cfg(gids_dp_rank=rank, gids_dp_world=world, gids_device=0))
        seed = dl.features.seed
        out = []
        for _ in range(3):
            mb, rows, st = dl.next_batch()
            u = mb.unique_nodes.cpu().numpy()
            ok = np.array_equal(rows.cpu().numpy(), O.feature_rows(seed, u, 64))
            local, remote = dl.shard_counts()
            out.append((bool(ok), local == int((u % world == rank).sum()), local + remote == len(u),
                        remote > 0))
        dist.barrier()  # peers keep their shards alive until everyone has read
        dl.close()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, None, repr(e)))


@pytest.mark.gpu
def test_gpu_two_process_ipc_shards_on_one_device():
    """Two ranks on cuda:0, each owning half the table; each rank's remote
    rows are read through a CUDA IPC mapping of the other's shard."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, out, err in res:
        assert err is None, (rank, err)
        assert all(all(t) for t in out), (rank, out)

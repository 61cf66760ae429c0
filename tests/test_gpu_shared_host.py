"""Two data-parallel ranks on one GPU (gloo control plane) serving from ONE
node-shared host tier (host_tier.py): each rank's batches -- unique nodes,
tier counts and gathered rows -- equal those of the same rank served from a
private pinned copy, and the table / constant-buffer rows are one mapping
created by local rank 0 (the reference has one FeatureStore,
graph.py:278-301)."""
from __future__ import annotations

import hashlib
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = dict(num_nodes=60_000, avg_degree=10.0, degree_model="uniform", feature_dim=64,
           page_bytes=4096, fanouts=[5, 5], batch_size=256, cache_lines=2_000,
           window_depth=4, buffer_fraction=0.1, consume_rate=0.0, seed=5,
           gids_generator="device", gids_dp_world=2)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(cfg, batches=4):
    from paper_2306_16384_b200 import Dataloader
    dl = Dataloader(cfg)
    out = []
    for _ in range(batches):
        mb, rows, st = dl.next_batch()
        out.append((hashlib.sha256(mb.unique_nodes.cpu().numpy().tobytes()).hexdigest(),
                    [st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses],
                    hashlib.sha256(rows.cpu().numpy().tobytes()).hexdigest()))
    shared = len(dl._shared)
    dl.close()
    return out, shared


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2306_16384_b200 import make_config
    os.environ["LOCAL_RANK"] = str(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    shared, n_regions = _run(make_config({**CFG, "gids_dp_rank": rank}))
    dist.barrier()
    private, n_priv = _run(make_config({**CFG, "gids_dp_rank": rank,
                                        "gids_shared_host": False}))
    q.put((rank, shared, private, n_regions, n_priv))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_share_one_host_tier():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = {r: rest for r, *rest in (q.get(timeout=600) for _ in ps)}
    for p in ps:
        p.join(timeout=120)
    for r in range(2):
        shared, private, n_regions, n_priv = got[r]
        assert n_regions == 2 and n_priv == 0  # table + buffer mapped from the node's tier
        assert shared == private, r
    assert got[0][0] != got[1][0]  # the ranks serve different batches

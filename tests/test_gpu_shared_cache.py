"""Owner-sharded cache of data-parallel ranks (SURVEY.md section 8(e) exchange
step; shared_cache.py, csrc/shared_cache.cu).  Two and three ranks on one GPU
(gloo control plane, CUDA IPC between the processes): node v is cached only
by rank v % G, which decides both ranks' accesses of it with the reference policy in
global batch order.  Per global batch, the unique nodes and the tier counts
equal the multi-rank oracle -- one reference CacheState per owner
(oracle.shared_cache_tiers) -- and every gathered row, whether peer-loaded
from the other rank's lines, read from this rank's lines, or from the host
tiers, equals the feature table (verify_gather + sha)."""
from __future__ import annotations

import hashlib
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = dict(num_nodes=30_000, avg_degree=8.0, degree_model="uniform", feature_dim=32,
           page_bytes=4096, fanouts=[5, 5], batch_size=128, cache_lines=1_500,
           window_depth=3, buffer_fraction=0.05, consume_rate=0.0, seed=9,
           gids_policy="exact", gids_shared_cache=True, gids_dp_world=2, verify_gather=True)
STEPS = 10


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2306_16384_b200 import Dataloader, make_config
    os.environ["LOCAL_RANK"] = str(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        dl = Dataloader(make_config({**CFG, "gids_dp_rank": rank, "gids_dp_world": world}))
        out = []
        for _ in range(STEPS):
            mb, rows, st = dl.next_batch()
            out.append((mb.unique_nodes.cpu().numpy(),
                        [st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses],
                        hashlib.sha256(rows.cpu().numpy().tobytes()).hexdigest()))
        lines = dl.cache.lines()[0]
        dl.close()
        q.put((rank, out, lines, None))
    except Exception as e:  # surface the child's error in the parent
        import traceback
        q.put((rank, None, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_share_one_owner_sharded_cache_match_oracle(world):
    from _setup import resolve
    from oracle import oracle as O
    from paper_2306_16384_b200 import make_config
    from paper_2306_16384_b200.loader import _seed_stream
    from paper_2306_16384_b200.sampling import pcg_words
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = {r: rest for r, *rest in (q.get(timeout=600) for _ in ps)}
    for p in ps:
        p.join(timeout=120)
    for r in range(world):
        assert got[r][2] is None, got[r][2]

    base = make_config({**CFG, "gids_shared_cache": False, "gids_dp_world": 1})
    r0 = resolve(base)
    batches, words = [], []
    for rank in range(world):
        cfg = make_config({**CFG, "gids_dp_rank": rank, "gids_dp_world": world})
        ss = np.random.SeedSequence(cfg.seed).spawn(6)
        words.append(pcg_words(np.random.Generator(np.random.PCG64(ss[2]).jumped(rank))))
        batches.append(list(_seed_stream(cfg, cfg.num_nodes, ss[5], ss[3])))
    want = O.shared_cache_tiers(r0["graph"].indptr, r0["graph"].indices, r0["buffer_nodes"],
                                batches, base.fanouts, words, r0["evict_seed"],
                                base.resolved_cache_lines(), base.window_depth, STEPS)
    table = r0["table"]
    hits = 0
    for s in range(STEPS):
        for rank in range(world):
            u, tiers, rows_sha = got[rank][0][s]
            wu, wt = want[s * world + rank]
            assert np.array_equal(u, wu), (s, rank)
            assert tiers == wt, (s, rank, tiers, wt)
            assert rows_sha == hashlib.sha256(table[u].tobytes()).hexdigest(), (s, rank)
            hits += tiers[0]
    assert hits > 0  # some rows came from the owners' lines
    # each owner's lines hold only its own nodes
    for rank in range(world):
        lines = got[rank][1]
        held = lines[lines >= 0]
        assert len(held) and np.all(held % world == rank)

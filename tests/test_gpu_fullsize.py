"""BASELINE.json's papers100M shape (C4, the north-star config) at full size on
the GPU, bit for bit against the oracle.

* properties: 1.6B-edge graph from the device generator, reverse PageRank
  converged, a constant buffer of exactly 10% of the nodes, ascending unique
  nodes, tier identities, and every gathered row re-derived on the device
  from the feature formula (verify_gather);
* the reference's own cache policy (CacheState, cache.py:144-180) at the
  headline size -- 2,097,152 lines, every storage miss an eviction once the
  cache is full -- against the oracle's sequential CacheState: per batch the
  seeds, every sampled layer, the unique nodes, tier counts and gathered rows;
  at the end the whole line table (node + LineState per line), the cache
  counters and the eviction PCG64 state;
* the set-associative policy on the same graph, same per-batch checks and
  final line table.
The oracle side rebuilds the graph and the pinned set on the host cores with
its own restatements (generator, float64 reverse PageRank), so setup is
checked too.  Several minutes of host work (C4 graph + PageRank in C)."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c4_host():
    import bench
    from paper_2306_16384_b200 import make_config
    cfg = make_config({**bench.WORKLOADS["c4"], "gids_policy": "exact"})
    return bench.host_device_shape(cfg)


def _compare(policy: str, batches: int, host) -> None:
    import bench
    from paper_2306_16384_b200 import Dataloader, make_config
    g, buf = host
    cfg = make_config({**bench.WORKLOADS["c4"], "gids_policy": policy})
    assert cfg.resolved_cache_lines() == 2_097_152
    dl = Dataloader(cfg)
    try:
        assert (dl.graph.num_nodes, dl.graph.num_edges) == (111_059_956, 1_615_685_872)
        assert np.array_equal(dl.graph.indptr, g.indptr)
        assert np.array_equal(dl.graph.indices, g.indices)
        assert np.array_equal(dl.buffer.node_ids, buf)
        r = bench.oracle_inputs(cfg, g, dl.features.table, buf)
        ld = bench.oracle_loader(cfg, r, buffer_rows=dl.buffer.rows)
        ld.keep_rows = True
        for b in range(batches):
            o = ld.next_batch()
            mb, rows, st = dl.next_batch()
            assert np.array_equal(np.asarray(mb.seeds), o["seeds"]), (policy, b)
            assert len(mb.layers) == len(o["layers"]) == 3
            for li, (a, e) in enumerate(zip(mb.layers, o["layers"])):
                assert np.array_equal(a.cpu().numpy(), e), (policy, b, li)
            assert np.array_equal(mb.unique_nodes.cpu().numpy(), o["unique"]), (policy, b)
            got = [st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses]
            assert got == o["tiers"].tolist(), (policy, b, got, o["tiers"].tolist())
            assert np.array_equal(rows.cpu().numpy(), o["rows"]), (policy, b)
        node, state = dl.cache.lines()
        onode, ostate = ld.cache.lines_snapshot()
        assert np.array_equal(node, onode), policy
        assert np.array_equal(state, ostate), policy
        os_ = ld.cache.stats()
        c = dl.cache
        assert [c.hits, c.misses, c.bypasses, c.evictions] == \
            [os_["hits"], os_["misses"], os_["bypasses"], os_["evictions"]], policy
        if policy == "exact":
            assert os_["evictions"] > 1_000_000  # the cache filled and kept evicting
            assert dl.cache.eviction_rng_words().tolist() == ld.cache.rng_words().tolist()
            assert dl._h.exact_par_batches() > 0  # the CTA-parallel policy decided them
    finally:
        dl.close()


def test_gpu_c4_fullsize_properties():
    import bench
    from paper_2306_16384_b200 import Dataloader, make_config
    cfg = make_config({**bench.WORKLOADS["c4"], "gids_policy": "exact", "verify_gather": True})
    dl = Dataloader(cfg)
    try:
        g = dl.graph
        assert (g.num_nodes, g.num_edges) == (111_059_956, 1_615_685_872)
        assert dl.pagerank.converged
        assert len(dl.buffer) == int(g.num_nodes * 0.10)
        for _ in range(3):
            mb, rows, st = dl.next_batch()  # verify_gather: rows re-derived on device
            u = mb.unique_nodes
            assert bool((u[1:] > u[:-1]).all())
            assert st.sampled_nodes == u.numel() == rows.shape[0]
            assert st.cache_hits + st.cpu_buffer_hits + st.ssd_accesses == st.sampled_nodes
            assert st.bypasses <= st.cpu_buffer_hits + st.ssd_accesses
            f = len(np.unique(mb.seeds))
            for l, fan in zip(mb.layers, cfg.fanouts):
                assert l.shape[0] <= f * fan
                f = len(np.unique(l[:, 0].cpu().numpy()))
    finally:
        dl.close()


def test_gpu_c4_fullsize_exact_policy_matches_oracle(c4_host):
    _compare("exact", 3, c4_host)


def test_gpu_c4_fullsize_setassoc_matches_oracle(c4_host):
    _compare("setassoc", 2, c4_host)

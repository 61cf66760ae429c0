"""Dataloader on the GPU vs the reference's golden runs (exact policy) and the
oracle (set-associative policy).  Bit-exact per batch: seeds, unique nodes,
every layer, the gathered rows, tier counts, the CSV row and cache counters."""
import numpy as np
import pytest

from _setup import config_of, fixture, resolve, sha
from oracle import oracle as O
from paper_2306_16384_b200 import Dataloader, make_config, run, stats_csv

pytestmark = pytest.mark.gpu

LOADERS = ["c09", "alltiers", "edgeless", "c1small", "c2small", "desk", "locality_w0",
           "locality_w8"]


@pytest.mark.parametrize("name", LOADERS)
def test_gpu_loader_matches_reference_run(name):
    fx = fixture(name)
    dl = Dataloader(config_of(fx))
    assert np.array_equal(dl.buffer.node_ids, fx["buffer_nodes"])
    assert dl.base_threshold == int(fx["base_threshold"])
    for b in range(int(fx["n_batches"])):
        mb, rows, st = dl.next_batch()
        assert np.array_equal(mb.seeds, fx[f"b{b}_seeds"]), b
        assert np.array_equal(mb.unique_nodes.cpu().numpy(), fx[f"b{b}_unique"]), b
        assert [sha(l.cpu().numpy().astype("<i8")) for l in mb.layers] == \
            list(fx[f"b{b}_layer_sha"]), b
        assert sha(rows.cpu().numpy()) == str(fx[f"b{b}_rows_sha"]), b
        assert [st.sampled_nodes, st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses,
                st.bypasses] == fx["tiers"][b].tolist(), b
        assert st.csv_row() == str(fx["csv"][b]), b
        c = dl.cache
        assert [c.hits, c.misses, c.bypasses, c.evictions, c.total_increments,
                c.total_decrements, len(dl._pending)] == fx["cache_stats"][b].tolist(), b
    dl.close()


def test_gpu_c09_known_answer():
    """test_acceptance.py:242-258: 1040/1351/1793/3012 and 84 evictions."""
    fx = fixture("c09")
    dl = Dataloader(config_of(fx, verify_gather=True))
    tiers = np.zeros(4, np.int64)
    for _ in range(27):
        _, _, st = dl.next_batch()
        tiers += (st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses)
    assert tiers.tolist() == [1040, 1351, 1793, 3012]
    assert dl.cache.evictions == 84


def test_gpu_edgeless_runahead_arithmetic():
    """test_dataloader.py:32-54: 855 threshold, 3 pending batches, 210 us."""
    fx = fixture("edgeless")
    dl = Dataloader(config_of(fx))
    dl.run_ahead()
    assert dl.base_threshold == 855 and len(dl._pending) == 3 and dl._pending_storage == 900
    _, _, st = dl.next_batch()
    assert st.fetch_time_us == 210.0 and st.bypasses == 300
    measured, summary = run(dl, iterations=2, warmup=0)
    assert summary.iterations_run == 2
    assert stats_csv(measured).startswith("iteration,sampled_nodes")


@pytest.mark.parametrize("name", ["alltiers", "c2small", "locality_w8"])
def test_gpu_setassoc_matches_oracle(name):
    fx = fixture(name)
    cfg = config_of(fx, gids_policy="setassoc")
    r = resolve(cfg)
    ld = O.OracleLoader(r["graph"].indptr, r["graph"].indices, r["table"], r["buffer_nodes"],
                        r["batches"], cfg.fanouts, r["sampler_words"], r["evict_words"],
                        cfg.resolved_cache_lines(), cfg.window_depth, r["base_threshold"],
                        policy="setassoc", evict_key=r["evict_seed"])
    dl = Dataloader(cfg)
    n = min(int(fx["n_batches"]), 40)
    for b in range(n):
        o = ld.next_batch()
        mb, rows, st = dl.next_batch()
        assert np.array_equal(mb.unique_nodes.cpu().numpy(), o["unique"]), b
        assert [st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses] == \
            o["tiers"].tolist(), b
        assert np.array_equal(rows.cpu().numpy(), o["rows"]), b
    os_ = ld.cache.stats()
    c = dl.cache
    assert [c.hits, c.misses, c.bypasses, c.evictions] == \
        [os_["hits"], os_["misses"], os_["bypasses"], os_["evictions"]]
    node, st = dl.cache.lines()
    onode, ost = ld.cache.lines_snapshot()
    assert np.array_equal(node, onode) and np.array_equal(st, ost)


def test_gpu_exact_cache_state_matches_oracle_after_evictions():
    fx = fixture("locality_w0")
    cfg = config_of(fx)
    r = resolve(cfg)
    ld = O.OracleLoader(r["graph"].indptr, r["graph"].indices, r["table"], r["buffer_nodes"],
                        r["batches"], cfg.fanouts, r["sampler_words"], r["evict_words"],
                        cfg.resolved_cache_lines(), cfg.window_depth, r["base_threshold"])
    dl = Dataloader(cfg)
    for _ in range(60):
        ld.next_batch()
        dl.next_batch()
    node, st = dl.cache.lines()
    onode, ost = ld.cache.lines_snapshot()
    assert np.array_equal(node, onode) and np.array_equal(st, ost)
    assert dl.cache.eviction_rng_words().tolist() == ld.cache.rng_words().tolist()


def test_gpu_c2_shape_properties():
    """C2 shape (1M nodes / 12M edges, 1024-d, 10% cache + 10% buffer, W=8) at
    full size: every gathered row re-derived on device (verify_gather), tier
    identities per batch, ascending unique nodes."""
    cfg = make_config(dict(num_nodes=1_000_000, avg_degree=12.0, degree_model="uniform",
                           feature_dim=1024, fanouts=[10, 15], batch_size=1024,
                           cache_lines=100_000, buffer_fraction=0.10, window_depth=8,
                           consume_rate=0.0, seed=42, verify_gather=True))
    dl = Dataloader(cfg)
    for _ in range(6):
        mb, rows, st = dl.next_batch()
        u = mb.unique_nodes
        assert bool((u[1:] > u[:-1]).all())
        assert st.cache_hits + st.cpu_buffer_hits + st.ssd_accesses == st.sampled_nodes
        assert rows.shape == (u.numel(), 1024)
    assert dl.cache.evictions > 0 or dl.cache.bypasses > 0
    dl.close()


@pytest.mark.parametrize("policy", ["exact", "setassoc"])
def test_gpu_c2_fullsize_matches_oracle(policy):
    """The default bench workload (BASELINE configs[1]) at full size, bit for
    bit against the oracle for 12 batches: unique nodes, every layer, tier
    counts, the CSV-relevant inflight, gathered rows, and the cache's line
    table and eviction RNG at the end.  With the set-associative policy this
    is also the concurrency check of the four streams at a size where the
    sampling of later batches overlaps the decisions (a shared scan
    workspace once corrupted both here)."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    cfg = make_config({**bench.WORKLOADS["c2"], "gids_policy": policy})
    dl = Dataloader(cfg)
    r = bench.oracle_inputs(cfg, dl.graph, dl.features.table, dl.buffer.node_ids)
    ld = bench.oracle_loader(cfg, r, buffer_rows=dl.buffer.rows)
    ld.keep_rows = True
    for b in range(12):
        o = ld.next_batch()
        mb, rows, st = dl.next_batch()
        assert np.array_equal(mb.unique_nodes.cpu().numpy(), o["unique"]), b
        for l, ol in zip(mb.layers, o["layers"]):
            assert np.array_equal(l.cpu().numpy(), ol), b
        assert [st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses] == \
            o["tiers"].tolist(), b
        assert np.array_equal(rows.cpu().numpy(), o["rows"]), b
    if policy == "exact":
        node, state = dl.cache.lines()
        onode, ostate = ld.cache.lines_snapshot()
        assert np.array_equal(node, onode) and np.array_equal(state, ostate)
        assert dl.cache.eviction_rng_words().tolist() == ld.cache.rng_words().tolist()
    dl.close()


def test_gpu_device_generator_loader_matches_oracle():
    """gids_generator='device' (the C4/C5 path at a small shape): the graph is
    built in HBM, the constant buffer chosen by the GPU reverse PageRank; the
    oracle gets the same inputs from its own CPU restatements (generator,
    float64-identical PageRank, stable top-k) and the runs agree bit for bit."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    cfg = make_config(dict(num_nodes=300_000, avg_degree=14.55, degree_model="uniform",
                           feature_dim=128, fanouts=[15, 10, 5], batch_size=512,
                           cache_lines=20_000, buffer_fraction=0.10, window_depth=8,
                           consume_rate=0.0, seed=7, gids_generator="device",
                           gids_policy="setassoc"))
    dl = Dataloader(cfg)
    g, buf = bench.host_device_shape(cfg)
    assert np.array_equal(dl.graph.indptr, g.indptr)
    assert np.array_equal(dl.graph.indices, g.indices)
    assert np.array_equal(dl.buffer.node_ids, buf)
    r = bench.oracle_inputs(cfg, g, dl.features.table, buf)
    ld = O.OracleLoader(g.indptr, g.indices, dl.features.table, buf, r["batches"], cfg.fanouts,
                        r["sampler_words"], r["evict_words"], cfg.resolved_cache_lines(),
                        cfg.window_depth, r["base_threshold"], policy="setassoc",
                        evict_key=r["evict_seed"])
    for b in range(12):
        o = ld.next_batch()
        mb, rows, st = dl.next_batch()
        assert np.array_equal(mb.unique_nodes.cpu().numpy(), o["unique"]), b
        for l, ol in zip(mb.layers, o["layers"]):
            assert np.array_equal(l.cpu().numpy(), ol), b
        assert [st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses] == \
            o["tiers"].tolist(), b
        assert np.array_equal(rows.cpu().numpy(), o["rows"]), b
    dl.close()


@pytest.mark.parametrize("policy", ["exact", "setassoc"])
def test_gpu_data_parallel_replicas_match_oracle(policy):
    """Data-parallel replicas: rank r of 3 serves global batches
    r, r+3, ... with sampler stream PCG64(sampler_ss).jumped(r) and its own
    cache; each rank's run equals the oracle fed the same slice and stream."""
    from paper_2306_16384_b200.loader import _seed_stream
    from paper_2306_16384_b200.sampling import pcg_words
    base = dict(num_nodes=20_000, avg_degree=10.0, degree_model="uniform", feature_dim=32,
                fanouts=[6, 8], batch_size=128, cache_lines=2_000, buffer_fraction=0.05,
                window_depth=4, consume_rate=0.0, seed=5, gids_policy=policy)
    r0 = resolve(make_config(base))
    for rank in range(3):
        cfg = make_config({**base, "gids_dp_rank": rank, "gids_dp_world": 3})
        ss = np.random.SeedSequence(cfg.seed).spawn(6)
        words = pcg_words(np.random.Generator(np.random.PCG64(ss[2]).jumped(rank)))
        batches = list(_seed_stream(cfg, cfg.num_nodes, ss[5], ss[3]))
        ld = O.OracleLoader(r0["graph"].indptr, r0["graph"].indices, r0["table"],
                            r0["buffer_nodes"], batches, cfg.fanouts, words, r0["evict_words"],
                            cfg.resolved_cache_lines(), cfg.window_depth, r0["base_threshold"],
                            policy=policy, evict_key=r0["evict_seed"])
        dl = Dataloader(cfg)
        for b in range(8):
            o = ld.next_batch()
            mb, rows, st = dl.next_batch()
            assert np.array_equal(mb.seeds, batches[b]), (rank, b)
            assert np.array_equal(mb.unique_nodes.cpu().numpy(), o["unique"]), (rank, b)
            assert [st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses] == \
                o["tiers"].tolist(), (rank, b)
            assert np.array_equal(rows.cpu().numpy(), o["rows"]), (rank, b)
        dl.close()


@pytest.mark.parametrize("lines,nodes,batch", [(200_000, 1_000_000, 2048),
                                               (1_000_000, 3_000_000, 4096)],
                         ids=["no-register-prefix", "global-tables"])
def test_gpu_exact_policy_large_caches_match_oracle(lines, nodes, batch):
    """The exact policy beyond its fast structures: more than 131072 lines (no
    register prefix: three-level table select) and more than fit shared memory
    (bitmaps in global memory).  Bit-exact vs the oracle once evictions run."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    cfg = make_config(dict(num_nodes=nodes, avg_degree=8.0, degree_model="uniform",
                           feature_dim=16, fanouts=[10, 10], batch_size=batch,
                           cache_lines=lines, buffer_fraction=0.02, window_depth=2,
                           consume_rate=0.0, seed=21, gids_generator="device"))
    dl = Dataloader(cfg)
    g, buf = bench.host_device_shape(cfg)
    r = bench.oracle_inputs(cfg, g, dl.features.table, buf)
    ld = O.OracleLoader(g.indptr, g.indices, dl.features.table, buf, r["batches"], cfg.fanouts,
                        r["sampler_words"], r["evict_words"], cfg.resolved_cache_lines(),
                        cfg.window_depth, r["base_threshold"])
    for b in range(10):
        o = ld.next_batch()
        mb, rows, st = dl.next_batch()
        assert [st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses] == \
            o["tiers"].tolist(), b
        assert np.array_equal(rows.cpu().numpy(), o["rows"]), b
    assert dl.cache.evictions > 0
    node, state = dl.cache.lines()
    onode, ostate = ld.cache.lines_snapshot()
    assert np.array_equal(node, onode) and np.array_equal(state, ostate)
    assert dl.cache.eviction_rng_words().tolist() == ld.cache.rng_words().tolist()
    dl.close()


@pytest.mark.parametrize("name", ["c2small", "locality_w8"])
def test_gpu_loader_direct_launches_match_reference_run(name, monkeypatch):
    """GIDS_NO_GRAPHS=1: the sampling sequence and the serve launched kernel by
    kernel instead of replayed as CUDA graphs -- the same bits."""
    monkeypatch.setenv("GIDS_NO_GRAPHS", "1")
    fx = fixture(name)
    dl = Dataloader(config_of(fx))
    try:
        for b in range(int(fx["n_batches"])):
            mb, rows, st = dl.next_batch()
            assert np.array_equal(mb.unique_nodes.cpu().numpy(), fx[f"b{b}_unique"]), b
            assert sha(rows.cpu().numpy()) == str(fx[f"b{b}_rows_sha"]), b
            assert st.csv_row() == str(fx["csv"][b]), b
        assert not dl._h.graphs_replayed()
    finally:
        dl.close()


def test_gpu_loader_serve_graphs_replayed():
    """The default path replays the serve as graphs from the third batch on."""
    fx = fixture("c2small")
    dl = Dataloader(config_of(fx))
    try:
        for b in range(int(fx["n_batches"])):
            mb, rows, st = dl.next_batch()
            assert sha(rows.cpu().numpy()) == str(fx[f"b{b}_rows_sha"]), b
        assert dl._h.graphs_replayed() == int(fx["n_batches"]) - 2  # (the first two direct)
    finally:
        dl.close()


def test_gpu_loader_is_freed_without_the_cycle_collector():
    """Dropping a loader frees it at once (its host tiers are unmapped then):
    nothing it owns refers back to it."""
    import gc
    import weakref
    gc.disable()
    try:
        dl = Dataloader(config_of(fixture("c09")))
        dl.next_batch()
        dl.close()
        ref = weakref.ref(dl)
        del dl
        assert ref() is None
    finally:
        gc.enable()

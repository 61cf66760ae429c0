"""File-backed storage tier (csrc/storage_file.cu).

The storage rows of each batch are read from the .gfea file in pages through
the page-coalescing accumulator.  Checked against the reference's golden runs
(rows, tiers, CSV -- including c09's 256-byte pages, where the 24-byte header
makes every row straddle two pages), against the oracle for the
set-associative policy, and page for page: the pages read are exactly the
distinct pages the batch's storage rows span."""
from __future__ import annotations

import numpy as np
import pytest

from _setup import config_of, fixture, resolve, sha
from oracle import oracle as O
from paper_2306_16384_b200 import (Dataloader, FeatureStore, load_features, make_config,
                                   save_features, save_graph)
from paper_2306_16384_b200.csc import HEADER_BYTES, write_synthetic_features

pytestmark = pytest.mark.gpu


def test_gpu_synthetic_gfea_file_matches_save_features(tmp_path):
    a, b = tmp_path / "gpu.gfea", tmp_path / "ref.gfea"
    write_synthetic_features(a, 1000, 24, 1234, chunk_rows=300)
    save_features(FeatureStore.synthetic(1000, 24, 1234), b)
    assert a.read_bytes() == b.read_bytes()
    assert np.array_equal(load_features(a).table, FeatureStore.synthetic(1000, 24, 1234).table)


@pytest.mark.parametrize("name", ["c09", "alltiers", "c2small", "desk"])
def test_gpu_file_tier_matches_reference_run(name, tmp_path):
    fx = fixture(name)
    cfg = config_of(fx, gids_storage="file", gids_storage_path=str(tmp_path / "t.gfea"),
                    gids_io_threads=3)
    dl = Dataloader(cfg)
    assert dl.gids_init(offset=24, cacheline_bytes=cfg.page_bytes)["storage"] == "file"
    for b in range(int(fx["n_batches"])):
        mb, rows, st = dl.next_batch()
        assert np.array_equal(mb.unique_nodes.cpu().numpy(), fx[f"b{b}_unique"]), b
        assert sha(rows.cpu().numpy()) == str(fx[f"b{b}_rows_sha"]), b
        assert st.csv_row() == str(fx["csv"][b]), b
    dl.close()


def _pages(nodes, row_bytes, page):
    b0 = HEADER_BYTES + np.asarray(nodes, np.int64) * row_bytes
    return np.unique(np.concatenate([b0 // page, (b0 + row_bytes - 1) // page]))


@pytest.mark.parametrize("policy", ["exact", "setassoc"])
def test_gpu_file_tier_pages_and_rows_match_oracle(policy, tmp_path):
    fx = fixture("alltiers")
    cfg = config_of(fx, gids_policy=policy, gids_storage="file",
                    gids_storage_path=str(tmp_path / "t.gfea"))
    r = resolve(cfg)
    ld = O.OracleLoader(r["graph"].indptr, r["graph"].indices, r["table"], r["buffer_nodes"],
                        r["batches"], cfg.fanouts, r["sampler_words"], r["evict_words"],
                        cfg.resolved_cache_lines(), cfg.window_depth, r["base_threshold"],
                        policy=policy, evict_key=r["evict_seed"])
    pinned = np.zeros(cfg.num_nodes, bool)
    pinned[r["buffer_nodes"]] = True
    dl = Dataloader(cfg)
    rb = cfg.feature_dim * 4
    expect_pages = 0
    for b in range(min(int(fx["n_batches"]), 30)):
        o = ld.next_batch()
        mb, rows, st = dl.next_batch()
        assert np.array_equal(rows.cpu().numpy(), o["rows"]), b
        storage = o["unique"][(o["kind"] != O.K_HIT) & ~pinned[o["unique"]]]
        expect_pages += len(_pages(storage, rb, cfg.page_bytes)) if len(storage) else 0
        assert dl.storage_stats()["pages"] == expect_pages, b
    dl.close()


def test_gpu_file_tier_from_graph_and_feature_files(tmp_path):
    """graph_path / features_path configs serve the given .gfea file as is."""
    from paper_2306_16384_b200 import generate_synthetic
    g = generate_synthetic(4000, 8.0, "uniform", seed=3)
    save_graph(g, tmp_path / "g.gcsc")
    table = np.random.default_rng(0).standard_normal((4000, 20)).astype(np.float32)
    save_features(FeatureStore(4000, 20, table), tmp_path / "f.gfea")
    base = dict(graph_path=str(tmp_path / "g.gcsc"), features_path=str(tmp_path / "f.gfea"),
                fanouts=[5, 5], batch_size=64, cache_lines=300, buffer_fraction=0.05,
                window_depth=2, consume_rate=0.0, seed=1, page_bytes=128)
    ref = Dataloader(make_config(base))
    dl = Dataloader(make_config({**base, "gids_storage": "file", "gids_io_direct": True}))
    for b in range(10):
        m1, r1, s1 = ref.next_batch()
        m2, r2, s2 = dl.next_batch()
        u = m2.unique_nodes.cpu().numpy()
        assert np.array_equal(u, m1.unique_nodes.cpu().numpy())
        assert np.array_equal(r2.cpu().numpy(), table[u]), b
        assert s1.csv_row() == s2.csv_row()
    dl.close()
    ref.close()


def test_gpu_file_tier_direct_io_matches_pinned_tier(tmp_path):
    """4 KiB pages with O_DIRECT (when the filesystem allows it): the same
    rows and tier counts as the pinned-host tier."""
    base = dict(num_nodes=20_000, avg_degree=10.0, degree_model="uniform", feature_dim=256,
                fanouts=[8, 8], batch_size=256, cache_lines=1_000, buffer_fraction=0.05,
                window_depth=4, consume_rate=0.0, seed=13, page_bytes=4096)
    ref = Dataloader(make_config(base))
    dl = Dataloader(make_config({**base, "gids_storage": "file", "gids_io_direct": True,
                                 "gids_storage_path": str(tmp_path / "d.gfea")}))
    for b in range(8):
        _, r1, s1 = ref.next_batch()
        _, r2, s2 = dl.next_batch()
        assert np.array_equal(r1.cpu().numpy(), r2.cpu().numpy()), b
        assert s1.csv_row() == s2.csv_row(), b
    st = dl.storage_stats()
    assert st["pages"] > 0 and st["bytes"] == st["pages"] * 4096
    dl.close()
    ref.close()


def test_gpu_gids_init_lays_out_the_backing_store(tmp_path):
    """The GIDS init call configures the store: a raw row dump
    at a 4 KiB offset, 4 KiB cache-line pages, two SSDs.  The loader then
    serves exactly what a loader configured that way from the start serves
    (rows, tiers, CSV rows -- n_ssd moves the accumulator threshold and the
    clock), and the call is refused once a batch has been served or when
    the element count disagrees."""
    from paper_2306_16384_b200 import ConfigError
    fx = fixture("alltiers")
    want = Dataloader(config_of(fx, n_ssd=2))
    dl = Dataloader(config_of(fx))
    n, dim = dl.graph.num_nodes, dl.features.dim
    raw = tmp_path / "rows.bin"
    with open(raw, "wb") as fh:
        fh.write(b"\0" * 4096)
        fh.write(np.ascontiguousarray(dl.features.table, np.float32).tobytes())
    with pytest.raises(ConfigError):
        dl.gids_init(offset=4096, num_elements=n * dim + 1, path=str(raw))
    one_ssd = dl.base_threshold
    lay = dl.gids_init(offset=4096, cacheline_bytes=4096, num_elements=n * dim, n_ssd=2,
                       path=str(raw))
    assert lay["storage"] == "file" and lay["offset"] == 4096 and lay["n_ssd"] == 2
    assert lay["base_threshold"] == want.base_threshold == 2 * one_ssd
    for b in range(6):
        mb, rows, st = dl.next_batch()
        mb2, rows2, st2 = want.next_batch()
        assert np.array_equal(mb.unique_nodes.cpu().numpy(), mb2.unique_nodes.cpu().numpy())
        assert np.array_equal(rows.cpu().numpy(), rows2.cpu().numpy()), b
        assert st.csv_row() == st2.csv_row(), b
    assert dl.storage_stats()["pages"] > 0
    with pytest.raises(ConfigError):
        dl.gids_init(offset=4096)
    dl.close()
    want.close()


@pytest.mark.parametrize("name", ["alltiers", "c2small"])
def test_gpu_page_aligned_file_layout_matches_reference_run(name, tmp_path):
    """The storage file laid out with row 0 at a page boundary
    (gids_storage_offset = page_bytes): every row is one page read instead of
    the .gfea layout's two (a 24-byte header makes each row straddle a page
    boundary); rows, tiers and CSV rows as the reference's run."""
    fx = fixture(name)
    cfg = config_of(fx, gids_storage="file", gids_storage_path=str(tmp_path / "t.bin"))
    cfg = config_of(fx, gids_storage="file", gids_storage_path=str(tmp_path / "t.bin"),
                    gids_storage_offset=cfg.page_bytes)
    dl = Dataloader(cfg)
    assert dl.gids_init(cacheline_bytes=cfg.page_bytes)["offset"] == cfg.page_bytes
    storage_rows = 0
    for b in range(int(fx["n_batches"])):
        mb, rows, st = dl.next_batch()
        assert np.array_equal(mb.unique_nodes.cpu().numpy(), fx[f"b{b}_unique"]), b
        assert sha(rows.cpu().numpy()) == str(fx[f"b{b}_rows_sha"]), b
        assert st.csv_row() == str(fx["csv"][b]), b
        storage_rows += st.ssd_accesses
    if cfg.feature_dim * 4 == cfg.page_bytes:  # a row is exactly one page
        assert dl.storage_stats()["pages"] == storage_rows
    dl.close()

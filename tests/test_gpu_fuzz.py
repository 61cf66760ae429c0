"""Randomised differential test: many small configurations (both policies,
fanouts below and above a warp, window depths 0..W, empty / tiny / large
caches, constant buffers on and off, row widths that are not multiples of 16
bytes, seed modes) served by the GPU and by the oracle, batch for batch."""
from __future__ import annotations

import numpy as np
import pytest

from _setup import resolve
from oracle import oracle as O
from paper_2306_16384_b200 import Dataloader, make_config

pytestmark = pytest.mark.gpu


def _random_cfg(rng) -> dict:
    n = int(rng.integers(200, 20_000))
    return dict(
        num_nodes=n, avg_degree=float(rng.choice([0.5, 3.0, 8.0, 20.0])),
        degree_model=str(rng.choice(["uniform", "powerlaw"])),
        feature_dim=int(rng.choice([1, 3, 16, 33, 64])),
        fanouts=[int(x) for x in rng.choice([1, 4, 10, 33, 50], size=int(rng.integers(1, 4)))],
        batch_size=int(rng.choice([1, 7, 64, 256])),
        cache_lines=int(rng.choice([0, 1, 5, 100, n // 4, 2 * n])),
        buffer_fraction=float(rng.choice([0.0, 0.02, 0.2])),
        window_depth=int(rng.choice([0, 1, 4, 8])),
        seed_mode=str(rng.choice(["permutation", "uniform", "zipf"])),
        zipf_a=1.3, consume_rate=0.0, page_bytes=4096, iterations=30, warmup=0,
        seed=int(rng.integers(0, 1 << 30)),
        gids_policy=str(rng.choice(["exact", "setassoc"])))


@pytest.mark.parametrize("trial", range(40))
def test_gpu_random_configs_match_oracle(trial, tmp_path):
    rng = np.random.default_rng(1000 + trial)
    raw = _random_cfg(rng)
    if rng.random() < 0.25:  # the storage tier served from the .gfea file
        raw.update(gids_storage="file", gids_storage_path=str(tmp_path / "t.gfea"),
                   page_bytes=int(rng.choice([256, 4096])),
                   feature_dim=int(rng.choice([1, 3, 16, 33, 64])))
    cfg = make_config(raw)
    r = resolve(cfg)
    ld = O.OracleLoader(r["graph"].indptr, r["graph"].indices, r["table"], r["buffer_nodes"],
                        r["batches"], cfg.fanouts, r["sampler_words"], r["evict_words"],
                        cfg.resolved_cache_lines(), cfg.window_depth, r["base_threshold"],
                        policy=cfg.gids_policy, evict_key=r["evict_seed"])
    dl = Dataloader(cfg)
    for b in range(12):
        try:
            o = ld.next_batch()
        except StopIteration:
            with pytest.raises(StopIteration):
                dl.next_batch()
            break
        mb, rows, st = dl.next_batch()
        assert np.array_equal(mb.unique_nodes.cpu().numpy(), o["unique"]), (trial, b)
        for l, ol in zip(mb.layers, o["layers"]):
            assert np.array_equal(l.cpu().numpy(), ol), (trial, b)
        assert [st.cache_hits, st.cpu_buffer_hits, st.ssd_accesses, st.bypasses] == \
            o["tiers"].tolist(), (trial, b)
        assert np.array_equal(rows.cpu().numpy(), o["rows"]), (trial, b)
    dl.close()

"""Resolve a reference-style config into the concrete inputs both the CUDA
path and the CPU oracle consume (graph, rows, pinned set, seed batches, RNG
states).  Uses only the package's host-side setup code."""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

from paper_2306_16384_b200.csc import generate_synthetic, synthetic_feature_rows
from paper_2306_16384_b200.hot_buffer import build_constant_buffer, reverse_pagerank
from paper_2306_16384_b200.csc import FeatureStore
from paper_2306_16384_b200.loader import _seed_stream
from paper_2306_16384_b200.sampling import pcg_words
from paper_2306_16384_b200.settings import make_config
from paper_2306_16384_b200.storage_model import required_accesses

GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fixture(name: str):
    return np.load(GOLDEN / f"loader_{name}.npz", allow_pickle=False)


def config_of(fx, **extra):
    raw = json.loads(str(fx["config"]))
    return make_config({**raw, **extra})


def resolve(cfg, with_table: bool = True) -> dict:
    graph_ss, feat_ss, sampler_ss, shuffle_ss, evict_ss, work_ss = \
        np.random.SeedSequence(cfg.seed).spawn(6)
    g = generate_synthetic(cfg.num_nodes, cfg.avg_degree, cfg.degree_model,
                           seed=int(graph_ss.generate_state(1)[0]), exponent=cfg.degree_exponent)
    feat_seed = int(feat_ss.generate_state(1)[0])
    table = synthetic_feature_rows(feat_seed, np.arange(g.num_nodes), cfg.feature_dim) \
        if with_table else None
    row_bytes = cfg.feature_dim * 4
    budget = cfg.resolved_buffer_bytes(g.num_nodes, row_bytes)
    if budget // row_bytes > 0:
        fs = FeatureStore(g.num_nodes, cfg.feature_dim,
                          table if table is not None else np.zeros((g.num_nodes, 1), np.float32))
        buf = build_constant_buffer(reverse_pagerank(g).scores, fs, budget).node_ids
    else:
        buf = np.empty(0, np.int64)
    evict_seed = int(evict_ss.generate_state(1)[0])
    return dict(graph=g, table=table, feat_seed=feat_seed, buffer_nodes=buf,
                batches=list(_seed_stream(cfg, g.num_nodes, work_ss, shuffle_ss)),
                sampler_words=pcg_words(np.random.default_rng(sampler_ss)),
                evict_words=pcg_words(np.random.default_rng(evict_seed)), evict_seed=evict_seed,
                base_threshold=required_accesses(cfg.ssd_spec(), cfg.target_fraction))

"""Generate golden fixtures by running the REFERENCE implementation.

Run here (the reference tree exists only in the build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``tierloader`` from ``/root/reference/pkg/src`` (read-only) and
writes small ``.npz`` files next to this script.  Those files are what the
oracle and the CUDA path are pinned against; nothing at test time reads the
reference tree.

Fixtures
--------
rng.npz       numpy PCG64 streams: raw next64 outputs, random() doubles,
              integers(n) sequences (buffered-uint32 Lemire), advance() and
              jumped() states.  Pins the RNG the sampler (sampler.py:75) and the
              eviction draw (cache.py:165) consume.
sample_layer.npz  sample_layer (sampler.py:50-84) over frontiers the loader
              never produces: repeated and unsorted entries, each expanded
              with draws of its own, fanout above and below 32.
sample.npz    sample_subgraph (sampler.py:87-112) on tree / star / hub /
              uniform / powerlaw / parallel-edge / edgeless graphs: every
              layer, unique_nodes and the generator state afterwards.
loader_*.npz  Dataloader.next_batch (dataloader.py:232-299) runs: per batch
              seeds, unique nodes, sha256 of each layer and of the gathered
              rows, tier counts, the CSV row, and cache statistics; plus the
              graph / constant-buffer identity so setup is pinned as well.
"""
from __future__ import annotations

import dataclasses
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from tierloader.config import make_config, load_config  # noqa: E402
from tierloader.dataloader import Dataloader  # noqa: E402
from tierloader.graph import build_csc, generate_synthetic  # noqa: E402
from tierloader.sampler import sample_layer, sample_subgraph  # noqa: E402

OUT = Path(__file__).resolve().parent
U64 = (1 << 64) - 1


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def split128(x: int) -> tuple[int, int]:
    return (x >> 64) & U64, x & U64


def state_words(bg) -> list[int]:
    st = bg.state
    s_hi, s_lo = split128(st["state"]["state"])
    i_hi, i_lo = split128(st["state"]["inc"])
    return [s_hi, s_lo, i_hi, i_lo, int(st["has_uint32"]), int(st["uinteger"])]


# ---------------------------------------------------------------------------
def make_rng() -> None:
    seeds = [0, 1, 42, 12345, 2**32 - 1]
    rec: dict[str, np.ndarray] = {}
    init, raw, dbl = [], [], []
    for s in seeds:
        bg = np.random.PCG64(s)
        init.append(state_words(bg))
        raw.append(np.random.PCG64(s).random_raw(64))
        dbl.append(np.random.Generator(np.random.PCG64(s)).random(64))
    rec["seeds"] = np.array(seeds, dtype=np.uint64)
    rec["init"] = np.array(init, dtype=np.uint64)
    rec["raw"] = np.array(raw, dtype=np.uint64)
    rec["dbl"] = np.array(dbl, dtype=np.float64)

    ns = [1, 2, 3, 7, 100, 1000, 65537, 2**31 - 1, 2**32 - 5]
    ints, after = [], []
    for n in ns:
        g = np.random.default_rng(7)
        ints.append([int(g.integers(n)) for _ in range(101)])
        after.append(state_words(g.bit_generator))
    rec["int_n"] = np.array(ns, dtype=np.uint64)
    rec["int_draws"] = np.array(ints, dtype=np.uint64)
    rec["int_after"] = np.array(after, dtype=np.uint64)

    # mixed-n sequence exactly as CacheState would issue it (shrinking safe counts)
    g = np.random.default_rng(99)
    mixed_n = np.array([5, 1, 1, 4, 3, 1000, 1, 2, 2**20, 17] * 10, dtype=np.uint64)
    rec["mixed_n"] = mixed_n
    rec["mixed_draws"] = np.array([int(g.integers(int(n))) for n in mixed_n], dtype=np.uint64)
    rec["mixed_after"] = np.array(state_words(g.bit_generator), dtype=np.uint64)

    ks = [0, 1, 2, 3, 63, 64, 1000, 123456789, 2**40 + 17]
    adv = []
    for k in ks:
        bg = np.random.PCG64(42)
        bg.advance(k)
        adv.append(state_words(bg))
    rec["adv_k"] = np.array(ks, dtype=np.uint64)
    rec["adv_state"] = np.array(adv, dtype=np.uint64)
    jmp = []
    for j in [1, 2, 5]:
        jmp.append(state_words(np.random.PCG64(42).jumped(j)))
    rec["jumped"] = np.array(jmp, dtype=np.uint64)
    np.savez_compressed(OUT / "rng.npz", **rec)


# ---------------------------------------------------------------------------
def graphs() -> dict:
    tree = build_csc([(1, 0), (2, 0), (3, 0), (4, 1), (5, 1), (6, 2), (7, 2),
                      (8, 3), (9, 3)], num_nodes=10)
    star = build_csc([(i, 0) for i in range(1, 301)], num_nodes=301)
    hub_edges = [(i, 0) for i in range(1, 600)] + [(0, i) for i in range(1, 600, 3)] \
        + [(i + 1, i) for i in range(1, 599)]
    hub = build_csc(hub_edges, num_nodes=600)
    par = build_csc([(1, 0)] * 5 + [(2, 0)] * 3 + [(3, 1), (3, 1), (0, 1), (2, 3)],
                    num_nodes=4)
    return {
        "tree": tree, "star": star, "hub": hub, "parallel": par,
        "edgeless": build_csc([], num_nodes=50),
        "uniform": generate_synthetic(3000, 12.0, "uniform", seed=5),
        "powerlaw": generate_synthetic(4000, 10.0, "powerlaw", seed=6),
    }


def make_sample() -> None:
    gs = graphs()
    cases = [
        ("tree", [0], [3, 3], 0),
        ("tree", [0, 1, 2], [1, 2], 1),
        ("star", [0], [25], 2),
        ("star", [0, 5], [40], 3),           # fanout > 32
        ("star", [0], [300], 4),             # deg == fanout: whole slice
        ("hub", [0, 1, 2, 3], [7, 3, 2], 5),
        ("hub", list(range(0, 600, 7)), [33, 5], 6),
        ("parallel", [0, 1, 3], [2, 2], 7),
        ("edgeless", [3, 9, 3], [2, 2], 8),
        ("uniform", None, [10, 15], 9),
        ("uniform", None, [15, 10, 5], 10),
        ("powerlaw", None, [10, 15], 11),
        ("powerlaw", None, [5, 5, 5], 12),
        ("powerlaw", None, [1], 13),
    ]
    rec: dict[str, np.ndarray] = {}
    meta = []
    for gname, g in gs.items():
        rec[f"g_{gname}_indptr"] = g.indptr.astype(np.uint64)
        rec[f"g_{gname}_indices"] = g.indices.astype(np.uint64)
    for ci, (gname, seeds, fans, rs) in enumerate(cases):
        g = gs[gname]
        if seeds is None:
            seeds = np.random.default_rng(100 + ci).integers(0, g.num_nodes, 256)
        seeds = np.asarray(seeds, dtype=np.int64)
        rng = np.random.default_rng(rs)
        st0 = state_words(rng.bit_generator)
        mb = sample_subgraph(g, seeds, fans, rng)
        rec[f"c{ci}_seeds"] = seeds
        rec[f"c{ci}_fanouts"] = np.array(fans, dtype=np.int64)
        rec[f"c{ci}_state0"] = np.array(st0, dtype=np.uint64)
        rec[f"c{ci}_state1"] = np.array(state_words(rng.bit_generator), dtype=np.uint64)
        for li, layer in enumerate(mb.layers):
            rec[f"c{ci}_layer{li}"] = layer.astype(np.int64)
        rec[f"c{ci}_unique"] = mb.unique_nodes.astype(np.int64)
        meta.append({"case": ci, "graph": gname, "n_layers": len(mb.layers)})
    rec["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "sample.npz", **rec)


# ---------------------------------------------------------------------------
LOADER_CONFIGS = {
    # c09 acceptance config (test_acceptance.py:242-247): all four tiers + evictions
    "c09": dict(num_nodes=5000, avg_degree=8.0, degree_model="powerlaw",
                feature_dim=64, page_bytes=256, fanouts=[4, 4], batch_size=64,
                seed_mode="zipf", zipf_a=1.5, cache_lines=48, window_depth=4,
                buffer_fraction=0.05, iterations=25, warmup=2, consume_rate=0.0,
                seed=3),
    # ALL_TIERS (test_dataloader.py:120-124)
    "alltiers": dict(num_nodes=5000, avg_degree=8.0, degree_model="powerlaw",
                     feature_dim=64, page_bytes=256, fanouts=[4, 4], batch_size=64,
                     seed_mode="zipf", zipf_a=1.5, cache_lines=256, window_depth=4,
                     buffer_fraction=0.05, iterations=30, warmup=3,
                     consume_rate=0.0, seed=3),
    # EDGELESS (test_dataloader.py:19-25)
    "edgeless": dict(num_nodes=2000, avg_degree=0.0, degree_model="uniform",
                     feature_dim=16, fanouts=[2], batch_size=300,
                     seed_mode="permutation", shuffle=False,
                     cache_lines=0, window_depth=0, buffer_fraction=0.0,
                     ssd_preset="intel-optane", target_fraction=0.95,
                     iterations=3, warmup=0, consume_rate=0.0, seed=11),
    # C1 shape at reduced size: uniform, every row fits the cache (no evictions)
    "c1small": dict(num_nodes=20000, avg_degree=12.0, degree_model="uniform",
                    feature_dim=1024, fanouts=[10, 15], batch_size=256,
                    cache_lines=20000, window_depth=8, buffer_fraction=0.0,
                    iterations=8, warmup=0, consume_rate=0.0, seed=42),
    # C2 shape at reduced size: 10% cache + 10% constant CPU buffer, W=8
    "c2small": dict(num_nodes=20000, avg_degree=12.0, degree_model="uniform",
                    feature_dim=1024, fanouts=[10, 15], batch_size=256,
                    cache_lines=2000, window_depth=8, buffer_fraction=0.10,
                    iterations=12, warmup=0, consume_rate=2.9e7, seed=42),
    # desk.yaml (the reference's demo config), default consume rate
    "desk": "desk.yaml",
    # locality.yaml at W=0 and W=8 (test_acceptance c05 hit ratios)
    "locality_w0": ("locality.yaml", {"window_depth": 0}),
    "locality_w8": ("locality.yaml", {"window_depth": 8}),
}


def _cfg(spec):
    cfgdir = REF.parent / "configs"
    if isinstance(spec, dict):
        return make_config(spec), spec
    if isinstance(spec, str):
        cfg = load_config(cfgdir / spec)
    else:
        name, over = spec
        cfg = load_config(cfgdir / name, over)
    # record the resolved keys (the YAML files themselves are not copied)
    raw = {k: (list(v) if isinstance(v, tuple) else v)
           for k, v in dataclasses.asdict(cfg).items()}
    return cfg, raw


def make_loader(name: str, spec, n_batches: int | None = None, keep_rows: bool = False) -> None:
    cfg, raw = _cfg(spec)
    dl = Dataloader(cfg)
    n = n_batches if n_batches is not None else cfg.warmup + cfg.iterations
    rec: dict[str, np.ndarray] = {}
    rec["graph_indptr_sha"] = np.array(sha(dl.graph.indptr.astype("<u8")))
    rec["graph_indices_sha"] = np.array(sha(dl.graph.indices.astype("<u8")))
    rec["num_edges"] = np.array(dl.graph.num_edges)
    rec["buffer_nodes"] = dl.buffer.node_ids.astype(np.int64)
    rec["table_sha"] = np.array(sha(dl.features.table))
    rec["base_threshold"] = np.array(dl.base_threshold)
    csv, tiers, cstats = [], [], []
    for b in range(n):
        try:
            mb, rows, st = dl.next_batch()
        except StopIteration:
            break
        rec[f"b{b}_seeds"] = mb.seeds.astype(np.int64)
        rec[f"b{b}_unique"] = mb.unique_nodes.astype(np.int64)
        rec[f"b{b}_layer_sha"] = np.array([sha(l.astype("<i8")) for l in mb.layers])
        rec[f"b{b}_layer_len"] = np.array([len(l) for l in mb.layers], dtype=np.int64)
        rec[f"b{b}_rows_sha"] = np.array(sha(rows.astype("<f4")))
        if keep_rows:
            rec[f"b{b}_layers"] = np.concatenate([l.reshape(-1) for l in mb.layers]) \
                if mb.layers else np.empty(0, np.int64)
        csv.append(st.csv_row())
        tiers.append([st.sampled_nodes, st.cache_hits, st.cpu_buffer_hits,
                      st.ssd_accesses, st.bypasses])
        c = dl.cache
        cstats.append([c.hits, c.misses, c.bypasses, c.evictions,
                       c.total_increments, c.total_decrements, len(dl._pending)])
    rec["n_batches"] = np.array(len(csv))
    rec["csv"] = np.array(csv)
    rec["tiers"] = np.array(tiers, dtype=np.int64)
    rec["cache_stats"] = np.array(cstats, dtype=np.int64)
    rec["config"] = np.array(json.dumps(raw))
    np.savez_compressed(OUT / f"loader_{name}.npz", **rec)
    print(name, "batches", len(csv), "tiers", np.array(tiers).sum(0).tolist(),
          "evictions", dl.cache.evictions)


def make_sample_layer() -> None:
    gs = graphs()
    r = np.random.default_rng(31)
    cases = [
        ("star", np.zeros(5000, np.int64), 3, 2024),          # one node, 5000 times
        ("star", np.array([0, 7, 0, 0, 300, 0]), 40, 7),        # fanout > 32, repeats
        ("hub", r.integers(0, 600, 3000), 5, 8),                # unsorted, repeats
        ("uniform", r.permutation(3000)[:700].repeat(2), 10, 9),
        ("powerlaw", r.integers(0, 4000, 5000), 17, 10),
        ("edgeless", np.array([4, 4, 1]), 2, 11),
    ]
    rec: dict[str, np.ndarray] = {}  # (graphs: the same g_* arrays as sample.npz)
    meta = []
    for ci, (gname, front, fan, rs) in enumerate(cases):
        rng = np.random.default_rng(rs)
        rec[f"c{ci}_frontier"] = np.asarray(front, np.int64)
        rec[f"c{ci}_state0"] = np.array(state_words(rng.bit_generator), dtype=np.uint64)
        rec[f"c{ci}_edges"] = sample_layer(gs[gname], front, fan, rng).astype(np.int64)
        rec[f"c{ci}_state1"] = np.array(state_words(rng.bit_generator), dtype=np.uint64)
        meta.append({"case": ci, "graph": gname, "fanout": fan})
    rec["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "sample_layer.npz", **rec)


def main() -> None:
    if sys.argv[1:] == ["sample_layer"]:  # regenerate that file only
        make_sample_layer()
        return
    make_rng()
    make_sample_layer()
    make_sample()
    for name, spec in LOADER_CONFIGS.items():
        keep = name in ("c09", "alltiers", "edgeless")
        nb = None
        if name == "desk":
            nb = 20
        make_loader(name, spec, n_batches=nb, keep_rows=keep)


if __name__ == "__main__":
    main()

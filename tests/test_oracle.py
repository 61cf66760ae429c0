"""Pin the CPU oracle to the reference: every golden fixture (made by running
the reference, tests/golden/make_golden.py) must be reproduced exactly."""
import json

import numpy as np
import pytest

from _setup import GOLDEN, config_of, fixture, resolve, sha
from oracle import oracle as O

pytestmark = pytest.mark.filterwarnings("ignore::DeprecationWarning")


@pytest.fixture(scope="module")
def rng_fx():
    return np.load(GOLDEN / "rng.npz")


def test_pcg64_raw_and_doubles(rng_fx):
    for i in range(len(rng_fx["seeds"])):
        w = rng_fx["init"][i].copy()
        assert np.array_equal(O.pcg_raw(w, 64), rng_fx["raw"][i])
        w = rng_fx["init"][i].copy()
        assert np.array_equal(O.pcg_doubles(w, 64), rng_fx["dbl"][i])


def test_pcg64_bounded_lemire_buffered(rng_fx):
    base = O.words_of(np.random.default_rng(7).bit_generator)
    for n, draws, after in zip(rng_fx["int_n"], rng_fx["int_draws"], rng_fx["int_after"]):
        w = base.copy()
        got = O.pcg_bounded(w, np.full(101, n, np.uint64))
        assert np.array_equal(got, draws), int(n)
        assert np.array_equal(w, after), int(n)
    w = O.words_of(np.random.default_rng(99).bit_generator)
    assert np.array_equal(O.pcg_bounded(w, rng_fx["mixed_n"]), rng_fx["mixed_draws"])
    assert np.array_equal(w, rng_fx["mixed_after"])


def test_pcg64_advance_and_jumped(rng_fx):
    base = O.words_of(np.random.PCG64(42))
    for k, st in zip(rng_fx["adv_k"], rng_fx["adv_state"]):
        w = base.copy()
        O.pcg_advance(w, int(k))
        assert np.array_equal(w, st), int(k)
    for j, st in zip([1, 2, 5], rng_fx["jumped"]):
        w = base.copy()
        O.pcg_advance(w, j * 0x9E3779B97F4A7C15F39CC0605CEDC835)
        assert np.array_equal(w[:4], st[:4])


def sample_cases():
    fx = np.load(GOLDEN / "sample.npz")
    meta = json.loads(str(fx["meta"]))
    return fx, meta


@pytest.mark.parametrize("case", range(14))
def test_oracle_sampler_matches_reference(case):
    fx, meta = sample_cases()
    m = meta[case]
    g = m["graph"]
    indptr, indices = fx[f"g_{g}_indptr"], fx[f"g_{g}_indices"]
    w = fx[f"c{case}_state0"].copy()
    layers, uniq, draws = O.sample_subgraph(indptr, indices, fx[f"c{case}_seeds"],
                                            fx[f"c{case}_fanouts"], w)
    assert len(layers) == m["n_layers"]
    for li, layer in enumerate(layers):
        assert np.array_equal(layer, fx[f"c{case}_layer{li}"]), li
    assert np.array_equal(uniq, fx[f"c{case}_unique"])
    assert np.array_equal(w[:4], fx[f"c{case}_state1"][:4])


LOADERS = ["c09", "alltiers", "edgeless", "c1small", "c2small", "desk", "locality_w0",
           "locality_w8"]


def run_oracle_loader(name, policy="exact"):
    fx = fixture(name)
    cfg = config_of(fx)
    r = resolve(cfg)
    assert sha(r["graph"].indptr.astype("<u8")) == str(fx["graph_indptr_sha"])
    assert sha(r["graph"].indices.astype("<u8")) == str(fx["graph_indices_sha"])
    assert np.array_equal(r["buffer_nodes"], fx["buffer_nodes"])
    assert r["base_threshold"] == int(fx["base_threshold"])
    ld = O.OracleLoader(r["graph"].indptr, r["graph"].indices, r["table"], r["buffer_nodes"],
                        r["batches"], cfg.fanouts, r["sampler_words"], r["evict_words"],
                        cfg.resolved_cache_lines(), cfg.window_depth, r["base_threshold"],
                        policy=policy, evict_key=r["evict_seed"],
                        redirect_ema_alpha=cfg.redirect_ema_alpha, runahead_cap=cfg.runahead_cap)
    return fx, cfg, r, ld


@pytest.mark.parametrize("name", LOADERS)
def test_oracle_loader_matches_reference(name):
    fx, cfg, r, ld = run_oracle_loader(name)
    assert sha(r["table"]) == str(fx["table_sha"])
    for b in range(int(fx["n_batches"])):
        out = ld.next_batch()
        assert np.array_equal(out["seeds"], fx[f"b{b}_seeds"]), b
        assert np.array_equal(out["unique"], fx[f"b{b}_unique"]), b
        assert [sha(l.astype("<i8")) for l in out["layers"]] == list(fx[f"b{b}_layer_sha"]), b
        assert sha(out["rows"]) == str(fx[f"b{b}_rows_sha"]), b
        t = out["tiers"]
        assert [len(out["unique"]), t[0], t[1], t[2], t[3]] == fx["tiers"][b].tolist(), b
        st = ld.cache.stats()
        expect = fx["cache_stats"][b].tolist()
        assert [st["hits"], st["misses"], st["bypasses"], st["evictions"],
                st["total_increments"], st["total_decrements"], len(ld.pending)] == expect, b


def naive_setassoc(nodes_per_batch, future, lines, key, ways=32):
    """Pure-Python statement of the set-associative policy."""
    from oracle.oracle import OracleCache  # noqa: F401  (policy contract reference only)
    M = (1 << 64) - 1

    def mix(z):
        z = (z + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    sets = lines // ways
    tag = [[-1] * ways for _ in range(sets)]
    safe = [[False] * ways for _ in range(sets)]
    where, counter = {}, {}
    log = []
    for epoch, (cur, fut) in enumerate(zip(nodes_per_batch, future)):
        futs = [set(f.tolist()) for f in fut]
        for x in cur.tolist():
            c = sum(1 for f in futs if x in f)
            if c:
                before = counter.get(x, 0)
                counter[x] = before + c
                if before == 0 and x in where:
                    s, w = where[x]
                    safe[s][w] = False
        for x in cur.tolist():
            c = counter.get(x, 0)
            if c > 0:
                c -= 1
                counter[x] = c
            s = (mix(x) * sets) >> 64
            if x in where:
                _, w = where[x]
                if c == 0:
                    safe[s][w] = True
                log.append(("hit", s * ways + w))
                continue
            w = next((i for i in range(ways) if tag[s][i] < 0), None)
            if w is None:
                cand = [i for i in range(ways) if safe[s][i]]
                if not cand:
                    log.append(("bypass", -1))
                    continue
                h = mix(key ^ mix((epoch * 0xD1B54A32D192ED03 + x) & M))
                w = cand[((h >> 32) * len(cand)) >> 32]
                del where[tag[s][w]]
            tag[s][w] = x
            where[x] = (s, w)
            safe[s][w] = c == 0
            log.append(("miss", s * ways + w))
    return log


def test_oracle_setassoc_matches_naive_statement():
    rng = np.random.default_rng(5)
    n_nodes, lines, W = 3000, 256, 3
    batches = [np.unique(rng.integers(0, n_nodes, 400)) for _ in range(12)]
    fut = [batches[i + 1:i + 1 + W] for i in range(len(batches))]
    expect = naive_setassoc(batches, fut, lines, key=1234)
    c = O.OracleCache(n_nodes, lines, "setassoc", 32, None, 1234)
    got = []
    names = {0: "hit", 1: "miss", 2: "bypass"}
    for e, (cur, f) in enumerate(zip(batches, fut)):
        c.window_update(cur, f)
        kind, slot = c.access_batch(cur, e)
        got += [(names[int(k)], int(s)) for k, s in zip(kind, slot)]
    assert got == expect
    assert c.stats()["evictions"] > 0

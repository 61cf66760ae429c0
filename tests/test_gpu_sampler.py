"""CUDA sampler (csrc/sampler.cu) vs the reference's golden samples and the oracle.

Bit-exact: layers (src, dst) in frontier order, unique_nodes, and the numpy
Generator state after the call (the host advances by the draws the kernel
reports)."""
import json

import numpy as np
import pytest

from _setup import GOLDEN
from oracle import oracle as O
from paper_2306_16384_b200 import GraphCsc, build_csc, generate_synthetic, sample_subgraph
from paper_2306_16384_b200.sampling import pcg_words

pytestmark = pytest.mark.gpu


def gen_from_words(w) -> np.random.Generator:
    bg = np.random.PCG64()
    bg.state = {"bit_generator": "PCG64",
                "state": {"state": (int(w[0]) << 64) | int(w[1]),
                          "inc": (int(w[2]) << 64) | int(w[3])},
                "has_uint32": int(w[4]), "uinteger": int(w[5])}
    return np.random.Generator(bg)


def host(mb):
    return [l.cpu().numpy() for l in mb.layers], mb.unique_nodes.cpu().numpy()


@pytest.mark.parametrize("case", range(14))
def test_gpu_sampler_matches_reference_fixture(case):
    fx = np.load(GOLDEN / "sample.npz")
    m = json.loads(str(fx["meta"]))[case]
    ip, ix = fx[f"g_{m['graph']}_indptr"], fx[f"g_{m['graph']}_indices"]
    g = GraphCsc(num_nodes=len(ip) - 1, num_edges=len(ix), indptr=ip, indices=ix)
    rng = gen_from_words(fx[f"c{case}_state0"])
    mb = sample_subgraph(g, fx[f"c{case}_seeds"], fx[f"c{case}_fanouts"], rng)
    layers, uniq = host(mb)
    assert len(layers) == m["n_layers"]
    for li, layer in enumerate(layers):
        assert np.array_equal(layer, fx[f"c{case}_layer{li}"]), li
    assert np.array_equal(uniq, fx[f"c{case}_unique"])
    assert np.array_equal(pcg_words(rng)[:4], fx[f"c{case}_state1"][:4])


def compare_with_oracle(g, seeds, fanouts, seed=0):
    rng = np.random.default_rng(seed)
    w = pcg_words(rng)
    o_layers, o_uniq, o_draws = O.sample_subgraph(g.indptr, g.indices, seeds, fanouts, w.copy())
    mb = sample_subgraph(g, seeds, fanouts, rng)
    layers, uniq = host(mb)
    for a, b in zip(layers, o_layers):
        assert np.array_equal(a, b)
    assert np.array_equal(uniq, o_uniq)
    ref = np.random.default_rng(seed)
    ref.bit_generator.advance(o_draws)
    assert pcg_words(rng).tolist() == pcg_words(ref).tolist()
    return mb


@pytest.mark.parametrize("model,fans", [("uniform", [15, 10, 5]), ("uniform", [10, 15]),
                                        ("powerlaw", [10, 15]), ("powerlaw", [40, 3])])
def test_gpu_sampler_matches_oracle_midsize(model, fans):
    g = generate_synthetic(60_000, 14.5, model, seed=17)
    seeds = np.random.default_rng(3).integers(0, g.num_nodes, 2048)
    mb = compare_with_oracle(g, seeds, fans, seed=11)
    assert mb.num_sampled_edges > 0


def test_gpu_sampler_sequence_continues_the_stream():
    g = generate_synthetic(20_000, 12.0, "uniform", seed=2)
    rng = np.random.default_rng(5)
    w = pcg_words(rng)
    for b in range(5):
        seeds = np.arange(b * 500, b * 500 + 500)
        o_layers, o_uniq, _ = O.sample_subgraph(g.indptr, g.indices, seeds, [10, 15], w)
        layers, uniq = host(sample_subgraph(g, seeds, [10, 15], rng))
        assert np.array_equal(uniq, o_uniq)
        assert all(np.array_equal(a, c) for a, c in zip(layers, o_layers))
        assert pcg_words(rng)[:4].tolist() == w[:4].tolist()


def test_gpu_sampler_edge_cases():
    # isolated seed, duplicate seeds, empty later layers
    g = build_csc([], num_nodes=4)
    mb = sample_subgraph(g, [2, 2], [3, 3], np.random.default_rng(0))
    assert mb.unique_nodes.cpu().tolist() == [2]
    assert [tuple(l.shape) for l in mb.layers] == [(0, 2), (0, 2)]
    with pytest.raises(ValueError, match="seeds must be non-empty"):
        sample_subgraph(g, [], [1], np.random.default_rng(0))
    with pytest.raises(ValueError, match=r"seed node 9 out of range \(num_nodes=4\)"):
        sample_subgraph(g, [1, 9], [1], np.random.default_rng(0))
    with pytest.raises(ValueError, match="every fanout must be >= 1"):
        sample_subgraph(g, [1], [0], np.random.default_rng(0))


def test_gpu_sampler_large_properties():
    """Full-size property check (papers100M-like degree, 4096 seeds, [15,10,5]):
    bit-exact against the oracle, plus sortedness and endpoint ranges."""
    n = 2_000_000
    rng = np.random.default_rng(1)
    deg = rng.poisson(14.5, n).astype(np.uint64)
    indptr = np.zeros(n + 1, np.uint64)
    np.cumsum(deg, out=indptr[1:])
    e = int(indptr[-1])
    indices = rng.integers(0, n, e).astype(np.uint64)
    for_sort = np.repeat(np.arange(n), deg.astype(np.int64))
    order = np.lexsort((indices, for_sort))
    indices = indices[order]
    g = GraphCsc(num_nodes=n, num_edges=e, indptr=indptr, indices=indices)
    seeds = rng.integers(0, n, 4096)
    mb = compare_with_oracle(g, seeds, [15, 10, 5], seed=4)
    layers, uniq = host(mb)
    assert np.all(np.diff(uniq) > 0)
    for layer in layers:
        src, dst = layer[:, 0], layer[:, 1]
        lo, hi = indptr[dst].astype(np.int64), indptr[dst + 1].astype(np.int64)
        assert np.all(hi > lo)
        assert np.all((src >= 0) & (src < n))


@pytest.mark.parametrize("case", range(6))
def test_gpu_sample_layer_matches_reference_fixture(case):
    """sample_layer over frontiers taken as given (sampler.py:59-84): repeats
    expanded again with their own draws, unsorted order kept, fanout above
    and below 32 -- bit-exact edges and Generator state vs the reference."""
    from paper_2306_16384_b200 import sample_layer
    fx = np.load(GOLDEN / "sample_layer.npz")
    gx = np.load(GOLDEN / "sample.npz")
    m = json.loads(str(fx["meta"]))[case]
    ip, ix = gx[f"g_{m['graph']}_indptr"], gx[f"g_{m['graph']}_indices"]
    g = GraphCsc(num_nodes=len(ip) - 1, num_edges=len(ix), indptr=ip, indices=ix)
    rng = gen_from_words(fx[f"c{case}_state0"])
    edges = sample_layer(g, fx[f"c{case}_frontier"], m["fanout"], rng).cpu().numpy()
    assert np.array_equal(edges, fx[f"c{case}_edges"])
    assert np.array_equal(pcg_words(rng)[:4], fx[f"c{case}_state1"][:4])


def test_gpu_sample_layer_inclusion_frequency():
    """The reference's Monte-Carlo check (pkg/tests/test_sampler.py:64-75):
    100,000 copies of a star's centre, 3 of 5 leaves each: every leaf is
    drawn with probability 3/5."""
    from paper_2306_16384_b200 import sample_layer
    g = build_csc([(i, 0) for i in range(1, 6)], num_nodes=6)
    trials = 100_000
    edges = sample_layer(g, np.zeros(trials, np.int64), 3,
                         np.random.default_rng(2024)).cpu().numpy()
    assert edges.shape == (3 * trials, 2)
    freq = np.bincount(edges[:, 0], minlength=6)[1:] / trials
    assert np.all(np.abs(freq - 0.6) <= 0.01)
    per = edges[:, 0].reshape(trials, 3)
    assert np.all((per[:, 0] != per[:, 1]) & (per[:, 1] != per[:, 2]) & (per[:, 0] != per[:, 2]))

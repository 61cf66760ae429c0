"""Setup-time graph work: the uniform generator and reverse PageRank.

CPU tests pin the C oracle to (a) the numpy statement of the generator
(tests/graphgen_ref.py) and (b) the reference's reverse_pagerank
(cpu_buffer.py:26-74, restated bit-exactly in hot_buffer.py and pinned by the
golden buffer sets) and numpy's own pairwise sum.  GPU tests hold the CUDA
kernels (csrc/graph_setup.cu) to the same outputs, bit for bit."""
from __future__ import annotations

import numpy as np
import pytest

import graphgen_ref as G
from oracle import oracle as O
from paper_2306_16384_b200.csc import GraphCsc, generate_synthetic
from paper_2306_16384_b200.hot_buffer import reverse_pagerank

GEN_CASES = [(1, 0, 3), (50, 1000, 7), (97, 400, 1), (2000, 24000, 42), (5000, 60000, 9)]


@pytest.mark.parametrize("n,e,seed", GEN_CASES)
def test_oracle_generator_matches_numpy_statement(n, e, seed):
    ip, ix = O.generate_uniform(n, e, seed, threads=3)
    rp, rx = G.generate_uniform(n, e, seed)
    assert np.array_equal(ip, rp) and np.array_equal(ix, rx)
    g = GraphCsc(num_nodes=n, num_edges=e, indptr=ip, indices=ix)
    for v in range(n):  # ascending and distinct within every destination
        seg = ix[int(ip[v]):int(ip[v + 1])]
        assert np.all(seg[1:] > seg[:-1])
    assert g.num_edges == e


def test_generator_degree_distribution_is_uniform_binomial():
    n, e = 20000, 240000
    ip, _ = O.generate_uniform(n, e, 5, threads=4)
    deg = np.diff(ip.astype(np.int64))
    assert abs(deg.mean() - 12.0) < 1e-9
    assert abs(deg.var() - 12.0) < 0.6  # Poisson(12)-like, as for uniform endpoints


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 100, 128, 129, 1000, 8193, 100003, 1 << 20])
def test_pairwise_sum_matches_numpy(n):
    a = np.random.default_rng(n).random(n) * 1e-3
    assert O.pairwise_sum(a) == float(np.sum(a))


def _graphs():
    yield "powerlaw", generate_synthetic(3000, 6.0, "powerlaw", seed=11)
    yield "uniform", generate_synthetic(4000, 9.0, "uniform", seed=12)
    ip, ix = O.generate_uniform(6000, 30000, 13)
    yield "gpu-generator", GraphCsc(num_nodes=6000, num_edges=30000, indptr=ip, indices=ix)


@pytest.mark.parametrize("name,g", list(_graphs()), ids=lambda x: x if isinstance(x, str) else "")
def test_oracle_pagerank_matches_reference_bitwise(name, g):
    ref = reverse_pagerank(g)
    s, conv, it = O.reverse_pagerank(g.indptr, g.indices, threads=4)
    assert (conv, it) == (ref.converged, ref.iterations)
    assert np.array_equal(s, ref.scores), name
    # short runs too (max_iter hit, not converged)
    ref3 = reverse_pagerank(g, max_iter=3)
    s3, c3, i3 = O.reverse_pagerank(g.indptr, g.indices, max_iter=3)
    assert (c3, i3) == (ref3.converged, 3) and np.array_equal(s3, ref3.scores)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("n,e,seed", GEN_CASES + [(200000, 2909800, 77)])
def test_gpu_generator_matches_oracle(n, e, seed):
    from paper_2306_16384_b200 import _native
    ip, ix = _native.generate_uniform_graph(0, n, e, seed)
    rp, rx = O.generate_uniform(n, e, seed, threads=8)
    assert np.array_equal(ip.cpu().numpy().astype(np.uint64), rp)
    assert np.array_equal(ix.cpu().numpy().astype(np.uint64), rx)


@pytest.mark.gpu
@pytest.mark.parametrize("name,g", list(_graphs()), ids=lambda x: x if isinstance(x, str) else "")
def test_gpu_pagerank_matches_reference_bitwise(name, g):
    import torch

    from paper_2306_16384_b200 import _native
    ip = torch.from_numpy(g.indptr.astype(np.int64)).cuda()
    ix = torch.from_numpy(g.indices.astype(np.int32)).cuda()
    ref = reverse_pagerank(g)
    s, conv, it = _native.reverse_pagerank(0, ip, ix)
    assert (conv, it) == (ref.converged, ref.iterations)
    assert np.array_equal(s.cpu().numpy(), ref.scores), name
    ref3 = reverse_pagerank(g, max_iter=3)
    s3, c3, i3 = _native.reverse_pagerank(0, ip, ix, max_iter=3)
    assert (c3, i3) == (False, 3) and np.array_equal(s3.cpu().numpy(), ref3.scores)


@pytest.mark.gpu
def test_gpu_pagerank_large_generated_graph_matches_oracle():
    from paper_2306_16384_b200 import _native
    n, e = 300000, 4365000
    ip, ix = _native.generate_uniform_graph(0, n, e, 3)
    s, conv, it = _native.reverse_pagerank(0, ip, ix)
    rp, rx = O.generate_uniform(n, e, 3, threads=8)
    rs, rconv, rit = O.reverse_pagerank(rp, rx, threads=8)
    assert (conv, it) == (rconv, rit)
    assert np.array_equal(s.cpu().numpy(), rs)

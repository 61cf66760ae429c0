"""Pure-numpy statement of the GPU uniform graph generator (TEST INFRASTRUCTURE).

The definition lives in the header of paper_2306_16384_b200/csrc/graph_setup.cu;
this file restates it independently of the C oracle so that both the oracle
(oracle/gids_oracle.c ``or_generate_uniform``) and the CUDA kernels are held
to it.  Small graphs only (per-node Python loop)."""
from __future__ import annotations

import numpy as np

U = np.uint64
GOLD, C1, C2 = U(0x9E3779B97F4A7C15), U(0xBF58476D1CE4E5B9), U(0x94D049BB133111EB)
DST_SALT, SRC_SALT = 0x243F6A8885A308D3, 0x13198A2E03707344
MASK = (1 << 64) - 1


def mix64(z):
    z = np.asarray(z, dtype=U) + GOLD
    z = (z ^ (z >> U(30))) * C1
    z = (z ^ (z >> U(27))) * C2
    return z ^ (z >> U(31))


def hi64(x, n: int):
    """floor(x * n / 2^64) without 128-bit integers (n < 2^31)."""
    x = np.asarray(x, dtype=U)
    return ((x >> U(32)) * U(n) + (((x & U(0xFFFFFFFF)) * U(n)) >> U(32))) >> U(32)


def generate_uniform(n: int, e: int, seed: int):
    with np.errstate(over="ignore"):
        s_dst = mix64(U(seed ^ DST_SALT))
        s_src = mix64(U(seed ^ SRC_SALT))
        dst = hi64(mix64(s_dst + np.arange(e, dtype=U)), n).astype(np.int64)
        deg = np.bincount(dst, minlength=n)
        indptr = np.zeros(n + 1, np.uint64)
        np.cumsum(deg, out=indptr[1:])
        indices = np.zeros(e, np.uint64)
        for v in np.flatnonzero(deg):
            d = int(deg[v])
            zv = mix64(s_src ^ U(v))
            seg = hi64(mix64(zv + np.arange(d, dtype=U)), n)
            a = 1
            while True:
                seg = np.sort(seg)
                rep = np.flatnonzero(seg[1:] == seg[:-1]) + 1
                if len(rep) == 0:
                    break
                seg[rep] = hi64(mix64(zv + U(a << 32) + rep.astype(U)), n)
                a += 1
            indices[int(indptr[v]):int(indptr[v]) + d] = seg
    return indptr, indices

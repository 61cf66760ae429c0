import numpy as np

from paper_2306_16384_b200 import sampling as _s
from paper_2306_16384_b200.sampling import Fanouts, MiniBatch, batch_iterator  # noqa: F401


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def sample_layer(g, frontier, fanout, rng):
    return _np(_s.sample_layer(g, frontier, fanout, rng))


def sample_subgraph(g, seeds, fanouts, rng):
    return _s.sample_subgraph(g, seeds, fanouts, rng).to_numpy()

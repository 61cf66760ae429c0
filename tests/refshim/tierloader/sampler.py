from paper_2306_16384_b200.numpy_api import sample_layer, sample_subgraph  # noqa: F401
from paper_2306_16384_b200.sampling import Fanouts, MiniBatch, batch_iterator  # noqa: F401

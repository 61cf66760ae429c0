from paper_2306_16384_b200 import feature_cache as _c
from paper_2306_16384_b200.feature_cache import (AccessKind, AccessResult,  # noqa: F401
                                                 CacheProtocolError, CacheStats, LineState,
                                                 WindowBuffer, window_update)


class CacheState(_c.CacheState):
    """The reference constructor (no node-count argument): per-node state is
    dense on the GPU, sized for the node ids the reference tests use."""

    def __init__(self, capacity_lines, line_bytes, eviction_seed=0):
        super().__init__(capacity_lines, line_bytes, eviction_seed, num_nodes=1 << 20)

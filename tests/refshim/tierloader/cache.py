from paper_2306_16384_b200.feature_cache import (AccessKind, AccessResult,  # noqa: F401
                                                 CacheProtocolError, CacheStats, LineState,
                                                 WindowBuffer, window_update)
from paper_2306_16384_b200.numpy_api import CacheState  # noqa: F401

"""paper_2306_16384_b200 -- the GIDS dataloader hot path, B200-native.

Drop-in for the reference ``tierloader`` serving path (Dataloader /
next_batch, sample_subgraph, the window-buffered cache, constant CPU buffer
and storage tier) with the work done by hand-written sm_100a CUDA kernels in
``libgids.so`` (C ABI: include/gids.h).  Public names follow the reference's
``tierloader/__init__.py``.
"""
from .csc import (BadMagicError, FeatureStore, FileFormatError, GraphCsc, TruncatedFileError,
                  VersionMismatchError, build_csc, generate_synthetic, load_features, load_graph,
                  neighbors, pinned_feature_table, save_features, save_graph,
                  synthetic_feature_rows)
from .feature_cache import (AccessKind, AccessResult, CacheProtocolError, CacheState,
                            CacheStats, GpuCacheView, LineState, WindowBuffer, window_update)
from .hot_buffer import (ConstantBuffer, PageRankResult, build_constant_buffer,
                         reverse_pagerank, top_k_nodes)
from .loader import CSV_HEADER, Dataloader, IterationStats, RunSummary, run, stats_csv
from .sampling import (Fanouts, MiniBatch, batch_iterator, check_fanouts, sample_layer,
                       sample_subgraph)
from .settings import ConfigError, InfeasibleError, PipelineConfig, load_config, make_config
from .storage_model import (PRESETS, FetchTiming, SsdSpec, achieved_fraction, fetch_total_us,
                            preset, required_accesses, simulate_fetch)

__version__ = "0.1.0"

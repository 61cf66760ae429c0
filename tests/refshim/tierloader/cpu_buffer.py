from paper_2306_16384_b200.hot_buffer import *  # noqa: F401,F403
from paper_2306_16384_b200.hot_buffer import (ConstantBuffer, PageRankResult,  # noqa: F401
                                              build_constant_buffer, reverse_pagerank,
                                              top_k_nodes)

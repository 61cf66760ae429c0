from paper_2306_16384_b200.csc import *  # noqa: F401,F403
from paper_2306_16384_b200.csc import (BadMagicError, FeatureStore, FileFormatError,  # noqa: F401
                                       GraphCsc, TruncatedFileError, VersionMismatchError,
                                       build_csc, generate_synthetic, load_features, load_graph,
                                       neighbors, save_features, save_graph,
                                       synthetic_feature_rows)

from paper_2306_16384_b200.loader import CSV_HEADER, IterationStats, RunSummary, stats_csv  # noqa: F401
from paper_2306_16384_b200.numpy_api import Dataloader, run  # noqa: F401

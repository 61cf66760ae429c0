from paper_2306_16384_b200 import loader as _l
from paper_2306_16384_b200.loader import (CSV_HEADER, IterationStats, RunSummary,  # noqa: F401
                                          stats_csv)


class Dataloader(_l.Dataloader):
    """next_batch hands back numpy (MiniBatch, rows, stats) as the reference."""

    def next_batch(self):
        mb, rows, st = super().next_batch()
        return mb.to_numpy(), rows.cpu().numpy(), st


def run(dl, iterations=None, warmup=None):
    return _l.run(dl, iterations, warmup)

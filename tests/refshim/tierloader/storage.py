from paper_2306_16384_b200.storage_model import *  # noqa: F401,F403
from paper_2306_16384_b200.storage_model import (PRESETS, FetchTiming, SsdSpec,  # noqa: F401
                                                 achieved_fraction, fetch_total_us, preset,
                                                 required_accesses, simulate_fetch)
from paper_2306_16384_b200.storage_model import exact as _frac  # noqa: F401

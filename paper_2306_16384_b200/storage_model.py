"""Storage-tier sizing and the virtual fetch clock kept for IterationStats.

The B200 path measures real time, but ``Dataloader.next_batch`` must still
report the reference's per-iteration accounting byte-for-byte (CSV columns
``fetch_time_us`` / ``effective_bandwidth_gbps`` / ``cumulative_time_us``,
dataloader.py:301-337).  Those use the three-phase SSD envelope of
``storage.py``; this module restates the parts the loader needs:

* ``SsdSpec`` / ``PRESETS`` / ``preset``   storage.py:33-89
* ``required_accesses``                    storage.py:92-104 (the accumulator's
                                           base threshold; 855 for Optane @ 0.95)
* ``achieved_fraction``                    storage.py:107-114
* ``fetch_total_us``                       storage.py:177-188 (closed form)
* ``FetchTiming`` / ``simulate_fetch``     storage.py:117-174 -- the phase breakdown
                                           of one fetch.  The reference replays it
                                           as a discrete-event loop over n_ssd
                                           round-robin servers; with balanced dealing
                                           the last completion is ceil(n/n_ssd)
                                           quanta past t_init, so it is computed in
                                           closed form (same exact rationals)

All arithmetic is exact (``fractions.Fraction``), floats read at their
shortest decimal repr, as the reference does.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from decimal import Decimal
from fractions import Fraction


def exact(x) -> Fraction:
    """Rational value of x; floats are taken at their shortest decimal repr."""
    if isinstance(x, Fraction):
        return x
    if isinstance(x, int):
        return Fraction(x)
    return Fraction(Decimal(repr(float(x))))


@dataclass(frozen=True)
class SsdSpec:
    iop_peak: float
    n_ssd: int = 1
    t_init: float = 25e-6
    t_term: float = 5e-6
    page_bytes: int = 4096

    def __post_init__(self):
        checks = ((self.iop_peak > 0, "iop_peak must be positive"),
                  (self.n_ssd >= 1, "n_ssd must be >= 1"),
                  (self.t_init >= 0 and self.t_term >= 0, "phase durations must be non-negative"),
                  (self.page_bytes >= 1, "page_bytes must be positive"))
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    @property
    def peak_bandwidth(self) -> float:
        return self.iop_peak * self.n_ssd * self.page_bytes


# launch+setup 25 us and termination 5 us; the 980 Pro also pays its 324 us
# read latency up front (storage.py:62-76).  The phase lengths are formed as
# microseconds * 1e-6 exactly like the reference, because the exact clock
# reads the resulting doubles (2.4999999999999998e-05, not 25e-6).
_SETUP_US, _TERM_US = 25.0, 5.0
PRESETS: dict[str, SsdSpec] = {
    "intel-optane": SsdSpec(iop_peak=1.5e6, t_init=_SETUP_US * 1e-6, t_term=_TERM_US * 1e-6),
    "samsung-980pro": SsdSpec(iop_peak=7.0e5, t_init=(_SETUP_US + 324.0) * 1e-6,
                              t_term=_TERM_US * 1e-6),
}


def preset(name: str, n_ssd: int = 1) -> SsdSpec:
    if name not in PRESETS:
        raise ValueError(f"unknown preset {name!r} (have: {', '.join(sorted(PRESETS))})")
    base = PRESETS[name]
    if n_ssd == base.n_ssd:
        return base
    return SsdSpec(iop_peak=base.iop_peak, n_ssd=n_ssd, t_init=base.t_init, t_term=base.t_term,
                   page_bytes=base.page_bytes)


def required_accesses(spec: SsdSpec, target_fraction: float) -> int:
    """Concurrent accesses for T_s / (T_i + T_s + T_t) >= f, per device, times n_ssd."""
    f = exact(target_fraction)
    if not 0 < f < 1:
        raise ValueError("target_fraction must be strictly between 0 and 1")
    overhead = exact(spec.t_init) + exact(spec.t_term)
    return spec.n_ssd * math.ceil(f / (1 - f) * overhead * exact(spec.iop_peak))


def achieved_fraction(spec: SsdSpec, n_access: int) -> float:
    if n_access < 0:
        raise ValueError("n_access must be non-negative")
    if n_access == 0:
        return 0.0
    steady = Fraction(n_access) / (exact(spec.iop_peak) * spec.n_ssd)
    return float(steady / (exact(spec.t_init) + steady + exact(spec.t_term)))


def fetch_total_us(spec: SsdSpec, n_access: int) -> Fraction:
    """Envelope of one fetch of n accesses dealt round-robin over n_ssd devices."""
    total = (exact(spec.t_init) + exact(spec.t_term)) * 1_000_000
    if n_access > 0:
        per_device = math.ceil(Fraction(n_access, spec.n_ssd))
        total += Fraction(1_000_000) / exact(spec.iop_peak) * per_device
    return total


@dataclass(frozen=True)
class FetchTiming:
    """Phase breakdown of one fetch (seconds); achieved_iops over all devices."""

    n_access: int
    t_init: float
    t_steady: float
    t_term: float
    achieved_iops: float
    achieved_fraction: float

    @property
    def total(self) -> float:
        return self.t_init + self.t_steady + self.t_term


def simulate_fetch(spec: SsdSpec, n_access: int) -> FetchTiming:
    """One batched fetch of n accesses: t_init, then every device retires one
    access per 1/iop_peak s (the fullest of the round-robin loads sets the
    steady phase), then t_term."""
    if n_access < 0:
        raise ValueError("n_access must be non-negative")
    init_us = exact(spec.t_init) * 1_000_000
    term_us = exact(spec.t_term) * 1_000_000
    steady_us = Fraction(1_000_000) / exact(spec.iop_peak) * math.ceil(
        Fraction(n_access, spec.n_ssd)) if n_access > 0 else Fraction(0)
    total_us = init_us + steady_us + term_us
    rate = Fraction(n_access) * 1_000_000 / total_us if total_us else Fraction(0)
    return FetchTiming(n_access=n_access, t_init=float(init_us) / 1e6,
                       t_steady=float(steady_us) / 1e6, t_term=float(term_us) / 1e6,
                       achieved_iops=float(rate),
                       achieved_fraction=float(rate / (exact(spec.iop_peak) * spec.n_ssd)))

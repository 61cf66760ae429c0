"""PipelineConfig: the reference's flat run configuration plus the GIDS flag.

Mirrors ``config.py`` of the reference (``PipelineConfig`` config.py:26-104,
``make_config`` :160-169, ``load_config`` :172-182, ``validate_config``
:185-215): same keys, defaults, YAML coercion rules and error messages, so
an existing YAML file drives this package unchanged.  Added keys (all
prefixed ``gids``) select the B200 path:

* ``gids``            the GIDS flag; this package only
                      implements the GPU path, so False is rejected.
* ``gids_policy``     "exact"  = the reference CacheState policy, bit-exact;
                      "setassoc" = 32-way set-associative HBM cache
                      (DESIGN.md section 4), fully parallel per set.
* ``gids_device``     CUDA ordinal.
* ``gids_dp_rank`` / ``gids_dp_world``  data-parallel batch sharding: rank r
                      serves global batches r, r+W, ... with its own sampler
                      stream PCG64(sampler_ss).jumped(r).
* ``gids_generator``  "reference" = the reference's numpy generator
                      (graph.py:112-207, bit-identical graphs); "device" =
                      the counter-based uniform generator in HBM
                      (csrc/graph_setup.cu), for the 100M-node shapes the
                      numpy generator cannot build (degree_model uniform only).
* ``gids_sharded_table``  C5: the synthetic feature table lives in the HBM of
                      the data-parallel ranks, node v in shard v % G, read by
                      peer loads over NVLink (sharded_table.py); no host tiers.
* ``gids_virtual_shards`` G > 0 keeps all G shards on this process's GPU
                      (single-GPU runs of the sharded path).
* ``gids_storage``    "pinned" = the storage tier in page-locked host memory
                      read zero-copy; "file" = the .gfea file itself, read in
                      pages of ``page_bytes`` after the 24-byte header through
                      the page-coalescing accumulator (csrc/storage_file.cu).
                      A synthetic config writes its table to
                      ``gids_storage_path`` first.
* ``gids_storage_offset`` byte offset of row 0 in a synthetic config's storage
                      file (24: the .gfea layout; a page multiple aligns every
                      row to pages -- the GIDS init call's offset).
* ``gids_io_threads`` / ``gids_io_direct``  pread threads / O_DIRECT for "file".
* ``gids_shared_host`` with several data-parallel ranks (torch.distributed
                      initialised), the ranks of a node share ONE host tier:
                      the pinned storage table and the constant buffer's rows
                      live in POSIX shared memory created by local rank 0 and
                      mapped + page-locked by every rank (host_tier.py),
                      instead of a private copy per rank.
* ``gids_shared_cache`` with several data-parallel ranks, one owner-sharded
                      cache instead of G replicas: node v is cached only by rank
                      v % G, which decides every rank's accesses of it with the
                      reference policy in global batch order; hits are peer
                      loads (shared_cache.py; exact policy).
* ``gids_speculate``  batches sampled ahead of the run-ahead queue (their
                      contributions are still counted when they join it, so
                      results are unchanged; 0 disables).
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from typing import Any

import yaml

from .storage_model import PRESETS, SsdSpec, preset


class ConfigError(Exception):
    """The configuration file or override set is not usable."""


class InfeasibleError(ConfigError):
    """The configuration is well-formed but no pipeline can satisfy it."""


@dataclass(frozen=True)
class PipelineConfig:
    # where the graph and rows come from (files, or synthetic when null)
    graph_path: str | None = None
    features_path: str | None = None
    num_nodes: int = 100_000
    avg_degree: float = 15.0
    degree_model: str = "powerlaw"
    degree_exponent: float = 2.0
    feature_dim: int = 1024
    # sampling
    fanouts: tuple[int, ...] = (5, 5, 5)
    batch_size: int = 4096
    seed_mode: str = "permutation"
    seed_count: int | None = None
    zipf_a: float = 1.2
    shuffle: bool = True
    # storage tier model
    ssd_preset: str | None = "intel-optane"
    iop_peak: float | None = None
    n_ssd: int = 1
    t_init_us: float | None = None
    t_term_us: float | None = None
    page_bytes: int = 4096
    target_fraction: float = 0.95
    # cache and constant CPU buffer
    cache_mb: float = 8192.0
    cache_lines: int | None = None
    window_depth: int = 8
    buffer_fraction: float = 0.10
    buffer_bytes: int | None = None
    cpu_gbps: float = 25.0
    # run shape
    consume_rate: float = 2.9e7
    iterations: int = 100
    warmup: int = 10
    seed: int = 42
    redirect_ema_alpha: float = 0.2
    runahead_cap: int = 256
    verify_gather: bool = False
    # GIDS extension (this package)
    gids: bool = True
    gids_policy: str = "exact"
    gids_device: int = 0
    gids_dp_rank: int = 0
    gids_dp_world: int = 1
    gids_generator: str = "reference"
    gids_sharded_table: bool = False
    gids_virtual_shards: int = 0
    gids_storage: str = "pinned"
    gids_storage_path: str | None = None
    gids_storage_offset: int = 24
    gids_io_threads: int = 8
    gids_io_direct: bool = False
    gids_speculate: int = 2
    gids_shared_host: bool = True
    gids_shared_cache: bool = False

    def ssd_spec(self) -> SsdSpec:
        if self.ssd_preset is None:
            if self.iop_peak is None:
                raise ConfigError("custom SSD spec requires iop_peak")
            spec = SsdSpec(iop_peak=self.iop_peak, n_ssd=self.n_ssd, page_bytes=self.page_bytes)
        elif self.ssd_preset in PRESETS:
            spec = preset(self.ssd_preset, n_ssd=self.n_ssd)
        else:
            raise ConfigError(f"unknown ssd_preset {self.ssd_preset!r} "
                              f"(have: {', '.join(sorted(PRESETS))})")
        patch: dict[str, Any] = {"page_bytes": self.page_bytes}
        if self.iop_peak is not None:
            patch["iop_peak"] = self.iop_peak
        if self.t_init_us is not None:
            patch["t_init"] = self.t_init_us * 1e-6
        if self.t_term_us is not None:
            patch["t_term"] = self.t_term_us * 1e-6
        try:
            return dataclasses.replace(spec, **patch)
        except ValueError as e:
            raise ConfigError(str(e)) from e

    def resolved_cache_lines(self) -> int:
        if self.cache_lines is None:
            return int(self.cache_mb * 2**20) // self.page_bytes
        if self.cache_lines < 0:
            raise ConfigError("cache_lines must be non-negative")
        return self.cache_lines

    def resolved_buffer_bytes(self, num_nodes: int, row_bytes: int) -> int:
        if self.buffer_bytes is not None:
            if self.buffer_bytes < 0:
                raise ConfigError("buffer_bytes must be non-negative")
            return self.buffer_bytes
        if not 0.0 <= self.buffer_fraction <= 1.0:
            raise ConfigError("buffer_fraction must be within [0, 1]")
        return int(num_nodes * self.buffer_fraction) * row_bytes


_SPEC = {f.name: f.type for f in dataclasses.fields(PipelineConfig)}


def _as_type(key: str, value: Any) -> Any:
    """Coerce one raw value to the field's declared type (YAML 1.1 leaves
    unsigned scientific notation such as ``2.9e7`` as a string)."""
    if key == "fanouts":
        if isinstance(value, (list, tuple)) and value:
            return tuple(int(v) for v in value)
        raise ConfigError(f"{key} must be a non-empty list")
    declared = _SPEC[key]
    optional = declared.endswith(" | None")
    kind = declared[:-len(" | None")] if optional else declared
    if value is None:
        if optional:
            return None
        raise ConfigError(f"{key} must not be null")
    bad = ConfigError(f"{key} expects {kind}, got {value!r}")
    if kind == "bool":
        if isinstance(value, bool):
            return value
        raise bad
    if isinstance(value, bool):
        raise bad
    if kind == "str":
        if isinstance(value, str):
            return value
        raise bad
    try:
        number = float(value)
    except (TypeError, ValueError):
        raise bad from None
    if kind == "int":
        if not number.is_integer():
            raise bad
        return int(number)
    return number


def make_config(overrides: dict[str, Any]) -> PipelineConfig:
    clean = {}
    for key, value in overrides.items():
        if key not in _SPEC:
            raise ConfigError(f"unknown config key {key!r}")
        clean[key] = _as_type(key, value)
    cfg = PipelineConfig(**clean)
    validate_config(cfg)
    return cfg


def load_config(path, overrides: dict[str, Any] | None = None) -> PipelineConfig:
    with open(path) as fh:
        raw = yaml.safe_load(fh)
    raw = {} if raw is None else raw
    if not isinstance(raw, dict):
        raise ConfigError("config file must contain a single mapping")
    raw.update(overrides or {})
    return make_config(raw)


_RULES = [
    (lambda c: 0.0 < c.target_fraction < 1.0,
     "target_fraction must be strictly between 0 and 1"),
    (lambda c: c.batch_size >= 1, "batch_size must be >= 1"),
    (lambda c: bool(c.fanouts) and min(c.fanouts) >= 1,
     "fanouts must be non-empty with every entry >= 1"),
    (lambda c: c.window_depth >= 0, "window_depth must be non-negative"),
    (lambda c: c.iterations >= 1, "iterations must be >= 1"),
    (lambda c: c.warmup >= 0, "warmup must be non-negative"),
    (lambda c: c.seed_mode in ("permutation", "uniform", "zipf"),
     lambda c: f"unknown seed_mode {c.seed_mode!r}"),
    (lambda c: c.seed_mode != "zipf" or c.zipf_a > 1.0, "zipf_a must be > 1"),
    (lambda c: c.degree_model in ("uniform", "powerlaw"),
     lambda c: f"unknown degree_model {c.degree_model!r}"),
    (lambda c: c.degree_model != "powerlaw" or c.degree_exponent > 1.0,
     "degree_exponent must be > 1"),
    (lambda c: c.consume_rate >= 0, "consume_rate must be non-negative (0 = unbounded)"),
    (lambda c: c.cpu_gbps > 0, "cpu_gbps must be positive"),
    (lambda c: c.runahead_cap >= 1, "runahead_cap must be >= 1"),
    (lambda c: 0 <= c.redirect_ema_alpha <= 1, "redirect_ema_alpha must be within [0, 1]"),
    (lambda c: (c.graph_path is None) == (c.features_path is None),
     "graph_path and features_path must be given together"),
    # GIDS extension
    (lambda c: c.gids_policy in ("exact", "setassoc"),
     lambda c: f"unknown gids_policy {c.gids_policy!r}"),
    (lambda c: 0 <= c.gids_dp_rank < c.gids_dp_world,
     "gids_dp_rank must be within [0, gids_dp_world)"),
    (lambda c: c.window_depth <= 255, "window_depth above 255 is not supported by the GPU window"),
    (lambda c: c.gids_generator in ("reference", "device"),
     lambda c: f"unknown gids_generator {c.gids_generator!r}"),
    (lambda c: c.gids_generator != "device" or c.degree_model == "uniform",
     "gids_generator 'device' builds uniform graphs only"),
    (lambda c: not c.gids_sharded_table or c.graph_path is None,
     "gids_sharded_table shards the synthetic feature table (no features_path)"),
    (lambda c: not c.gids_sharded_table or (c.buffer_fraction == 0.0 and not c.buffer_bytes),
     "gids_sharded_table keeps every row in HBM: buffer_fraction must be 0"),
    (lambda c: c.gids_virtual_shards >= 0, "gids_virtual_shards must be non-negative"),
    (lambda c: c.gids_storage in ("pinned", "file"),
     lambda c: f"unknown gids_storage {c.gids_storage!r}"),
    (lambda c: c.gids_storage != "file" or c.graph_path is not None
     or c.gids_storage_path is not None,
     "gids_storage 'file' needs features_path or gids_storage_path"),
    (lambda c: c.gids_storage != "file" or not c.gids_sharded_table,
     "gids_storage 'file' and gids_sharded_table are exclusive"),
    (lambda c: c.gids_io_threads >= 1, "gids_io_threads must be >= 1"),
    (lambda c: c.gids_storage_offset >= 24, "gids_storage_offset must be >= 24 (the header)"),
    (lambda c: c.gids_speculate >= 0, "gids_speculate must be non-negative"),
    (lambda c: c.gids_virtual_shards == 0 or c.gids_dp_world == 1,
     "gids_virtual_shards is for single-process runs (gids_dp_world 1)"),
    (lambda c: not c.gids_shared_cache or (c.gids_policy == "exact" and not c.gids_sharded_table
                                           and c.gids_storage == "pinned"),
     "gids_shared_cache runs the exact policy over a pinned host tier"),
]


def validate_config(cfg: PipelineConfig) -> None:
    for ok, msg in _RULES:
        if not ok(cfg):
            raise ConfigError(msg(cfg) if callable(msg) else msg)

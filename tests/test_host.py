"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
host-side setup (config, storage sizing, synthetic graph, hot-node choice,
seed streams) and the data-parallel batch split."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from _setup import config_of, fixture, sha
from paper_2306_16384_b200 import (ConfigError, PipelineConfig, fetch_total_us, make_config,
                                   preset, required_accesses)
from paper_2306_16384_b200 import _native
from paper_2306_16384_b200.loader import _seed_stream

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "gids.h").read_text()
    return sorted(set(re.findall(r"GIDS_API\s+[\w\s\*]+?\b(gids_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_native.exported_symbols()) == syms
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (gids_\w+)", out))
    assert set(syms) <= exported
    assert lib.gids_abi_version() == _native.ABI_VERSION


def test_library_targets_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_defaults_and_errors():
    c = PipelineConfig()
    assert c.gids and c.gids_policy == "exact"
    with pytest.raises(ConfigError, match="unknown config key 'bogus'"):
        make_config({"bogus": 1})
    assert make_config({"consume_rate": "2.9e7"}).consume_rate == 2.9e7
    with pytest.raises(ConfigError, match="batch_size expects int"):
        make_config({"batch_size": 1.5})
    with pytest.raises(ConfigError, match="unknown gids_policy"):
        make_config({"gids_policy": "lru"})
    assert make_config({"cache_mb": 1.0, "page_bytes": 4096}).resolved_cache_lines() == 256


def test_storage_sizing_known_answers():
    assert required_accesses(preset("intel-optane"), 0.95) == 855
    for k in (2, 3, 8):
        assert required_accesses(preset("intel-optane", n_ssd=k), 0.95) == k * 855
    # 900 accesses in flight: 25 + 900/1.5 + 5 = 630 us (test_dataloader.py:45-54)
    assert float(fetch_total_us(preset("intel-optane"), 900) / 3) == 210.0


@pytest.mark.parametrize("name", ["c09", "c2small", "desk"])
def test_setup_reproduces_reference_graph_and_buffer(name):
    from _setup import resolve
    fx = fixture(name)
    r = resolve(config_of(fx), with_table=False)
    assert sha(r["graph"].indptr.astype("<u8")) == str(fx["graph_indptr_sha"])
    assert sha(r["graph"].indices.astype("<u8")) == str(fx["graph_indices_sha"])
    assert np.array_equal(r["buffer_nodes"], fx["buffer_nodes"])
    for b, seeds in enumerate(r["batches"][:int(fx["n_batches"])]):
        assert np.array_equal(seeds, fx[f"b{b}_seeds"]), b


def test_data_parallel_split_partitions_the_batch_sequence():
    cfg = make_config(dict(num_nodes=5000, batch_size=64, seed=3))
    ss = np.random.SeedSequence(cfg.seed).spawn(6)
    full = list(_seed_stream(cfg, 5000, ss[5], ss[3]))
    parts = []
    for r in range(3):
        c = make_config(dict(num_nodes=5000, batch_size=64, seed=3, gids_dp_rank=r,
                             gids_dp_world=3))
        parts.append(list(_seed_stream(c, 5000, ss[5], ss[3])))
    for r, part in enumerate(parts):
        assert all(np.array_equal(a, b) for a, b in zip(part, full[r::3]))
    assert sum(len(p) for p in parts) == len(full)


def test_window_deferred_shift_folds_one_pop_then_one_push():
    """WindowBuffer in the loader's deferred mode: one pop then one push are
    handed to the serve (gids_serve_shift); any other sequence is launched in
    order (a recording stand-in for the handle)."""
    from paper_2306_16384_b200.feature_cache import WindowBuffer

    class _H:
        def __init__(self):
            self.ops = []

        def window_push(self, nodes, st):
            self.ops.append(("push", nodes))

        def window_pop(self, nodes, st):
            self.ops.append(("pop", nodes))

    class _T(list):  # a tensor stand-in: numel() and identity
        def numel(self):
            return len(self)

    h = _H()
    w = WindowBuffer(4, h, stream=0)
    w.defer = True
    a, b, c = _T([1, 2]), _T([3]), _T([4, 5])
    w.push_iteration(a, trusted=True)
    w.push_iteration(b, trusted=True)
    assert w.take_shift() == (None, None) and h.ops == [("push", a), ("push", b)]
    h.ops.clear()
    assert w.pop_iteration() is a
    w.push_iteration(c, trusted=True)
    pop, push = w.take_shift()
    assert pop is a and push is c and h.ops == []
    assert w.pop_iteration() is b
    assert w.take_shift() == (b, None) and h.ops == []
    assert list(w.lists) == [c]


def test_slots_hand_out_views_k_at_a_time():
    """Per-batch blocks come K at a time from one allocation."""
    import numpy as np

    from paper_2306_16384_b200.loader import _Slots
    allocs = []

    def alloc():
        allocs.append(np.zeros((3, 4)))
        return allocs[-1]

    s = _Slots(alloc, 3)
    views = [s.take() for _ in range(7)]
    assert len(allocs) == 3
    assert all(v.base is allocs[i // 3] for i, v in enumerate(views))

"""The C ABI from plain C (examples/gids_minimal.c): compiles and links
against include/gids.h + libgids.so on the CPU; runs on the GPU."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2306_16384_b200"


def _build(out: Path) -> None:
    cmd = ["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", str(ROOT / "include"),
           "-I", "/usr/local/cuda/include", str(ROOT / "examples" / "gids_minimal.c"),
           "-L", str(PKG), "-lgids", "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{PKG}", "-o", str(out)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_c_example_compiles_and_links(tmp_path):
    _build(tmp_path / "gids_minimal")
    assert (tmp_path / "gids_minimal").exists()


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    exe = tmp_path / "gids_minimal"
    _build(exe)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("unique=")

"""Run the reference's own test files (pkg/tests/*.py) against the GPU package.

  python tools/run_reference_tests.py --stage   # here: copy the reference tests
                                               # into oracle/_ref/reftests/ (git-ignored,
                                               # travels to the GPU box with the snapshot)
  python tools/run_reference_tests.py [-k EXPR] # on a GPU box: run them

The tests import ``tierloader``; tests/refshim/tierloader aliases it to
paper_2306_16384_b200 (numpy outputs, the reference's CacheState constructor),
so the files run unchanged.  Prints one line per test file (passed / failed /
errors) and the failing test ids, and writes the junit XML next to the tests."""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import xml.etree.ElementTree as ET
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
STAGE = ROOT / "oracle" / "_ref" / "reftests"
SRC = Path("/root/reference/pkg/tests")


def stage() -> None:
    if not SRC.is_dir():
        print(f"no reference tests at {SRC}; nothing staged")
        return
    STAGE.mkdir(parents=True, exist_ok=True)
    for p in sorted(SRC.glob("*.py")):
        shutil.copy2(p, STAGE / p.name)
    cfg = SRC.parent / "configs"  # the acceptance tests read ../configs/*.yaml
    if cfg.is_dir():
        shutil.copytree(cfg, STAGE.parent / "configs", dirs_exist_ok=True)
    print(f"staged {len(list(STAGE.glob('*.py')))} files into {STAGE}")


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", action="store_true")
    ap.add_argument("-k", default=None)
    ap.add_argument("--xml", default=str(STAGE / "junit.xml"))
    a = ap.parse_args()
    if a.stage:
        stage()
        return 0
    if not STAGE.is_dir():
        print("reference tests not staged (run --stage where /root/reference exists)")
        return 2
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "refshim"), str(ROOT),
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", str(STAGE), "-q", "-p", "no:cacheprovider",
           "--rootdir", str(STAGE), f"--junitxml={a.xml}", "--timeout=1200"]
    if a.k:
        cmd += ["-k", a.k]
    r = subprocess.run(cmd, cwd=STAGE, env=env, capture_output=True, text=True)
    per = defaultdict(lambda: [0, 0, 0])
    failed = []
    if Path(a.xml).exists():
        for tc in ET.parse(a.xml).getroot().iter("testcase"):
            f = (tc.get("classname") or "").split(".")[0] or tc.get("file", "?")
            bad = tc.find("failure") is not None or tc.find("error") is not None
            skip = tc.find("skipped") is not None
            per[f][1 if bad else (2 if skip else 0)] += 1
            if bad:
                el = tc.find("failure") if tc.find("failure") is not None else tc.find("error")
                msg = (el.get("message") or "").splitlines()[0][:160] if el is not None else ""
                failed.append(f"{f}::{tc.get('name')}  {msg}")
    print("reference test file          passed  failed  skipped")
    for f in sorted(per):
        p, b, s = per[f]
        print(f"{f:28s} {p:6d} {b:7d} {s:8d}")
    tot = [sum(v[i] for v in per.values()) for i in range(3)]
    print(f"{'TOTAL':28s} {tot[0]:6d} {tot[1]:7d} {tot[2]:8d}")
    for line in failed:
        print("FAIL", line)
    print("\n".join(r.stdout.strip().splitlines()[-3:]))
    if r.returncode not in (0, 1):
        print(r.stderr[-3000:])
    return 0


if __name__ == "__main__":
    sys.exit(main())

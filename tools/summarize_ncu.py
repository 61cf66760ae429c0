"""Summaries of ncu captures for profiles/ (run here, reads gpurun_out/)."""
import csv
import collections
import subprocess
import sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "pcie__read_bytes.sum.per_second",
        "pcie__write_bytes.sum.per_second", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum"]


def full_summary(rep: Path) -> str:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append(f"kernel: {r[h.index('Kernel Name')]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"  {k:60s} {r[i]:>18s} {u[i]}")
    stall = subprocess.run(["ncu", "-i", str(rep), "--page", "details", "--csv", "--section",
                            "WarpStateStats"], capture_output=True, text=True).stdout
    out.append("warp state (details page, WarpStateStats):")
    for line in stall.splitlines()[1:]:
        f = list(csv.reader([line]))[0]
        if len(f) > 14:
            out.append(f"  {f[-3]:50s} {f[-1]:>12s} {f[-2]}")
    return "\n".join(out) + "\n"


def launch_summary(path: Path) -> str:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = ["kernel,launches,total_ms,share_pct,avg_us"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k},{n},{v / 1e6:.3f},{v / tot * 100:.2f},{v / n / 1e3:.1f}")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    kind, src, dst = sys.argv[1], Path(sys.argv[2]), Path(sys.argv[3])
    dst.write_text(full_summary(src) if kind == "full" else launch_summary(src))
    print(dst.read_text()[:3000])

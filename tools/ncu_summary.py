"""One-launch ncu capture (.ncu-rep) -> the metric summary kept under profiles/:
    python tools/ncu_summary.py report.ncu-rep out.txt"""
import csv, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "pcie__read_bytes.sum",
           "pcie__read_bytes.sum.per_second", "pcie__write_bytes.sum.per_second",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
name = vals[hdr.index("Kernel Name")]
lines = [f"kernel: {name}"]
for m in metrics:
    if m in hdr:
        i = hdr.index(m)
        lines.append(f"  {m:60s} {vals[i]:>22s} {units[i]}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

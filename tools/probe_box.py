"""One-off probe of the GPU box: host RAM, cores, host-link bandwidth (pinned H2D DMA,
zero-copy reads through a torch view of pinned memory)."""
import os, subprocess, time, json
import torch
out = {}
out["cpu_count"] = os.cpu_count()
out["sched_affinity"] = len(os.sched_getaffinity(0))
with open("/proc/meminfo") as f:
    out["meminfo"] = [l.strip() for l in f.readlines()[:3]]
with open("/proc/cpuinfo") as f:
    out["cpu_model"] = next(l.split(":")[1].strip() for l in f if l.startswith("model name"))
out["nvsmi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,memory.total,pcie.link.gen.max,pcie.link.width.max,clocks.max.sm", "--format=csv"], capture_output=True, text=True).stdout
out["df"] = subprocess.run(["df", "-h", "/tmp", "/dev/shm", "."], capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
for gb in (1, 4):
    n = gb << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); 
    for _ in range(5): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    out[f"h2d_{gb}GB_GBs"] = 5 * n / (s.elapsed_time(e) * 1e-3) / 1e9
    s.record();
    for _ in range(5): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    out[f"d2h_{gb}GB_GBs"] = 5 * n / (s.elapsed_time(e) * 1e-3) / 1e9
    del h, d
# big pinned alloc test
t0 = time.time()
try:
    big = torch.empty(64 << 30, dtype=torch.uint8, pin_memory=True)
    out["pin64GB_s"] = time.time() - t0
    del big
except Exception as ex:
    out["pin64GB_err"] = str(ex)[:200]
print(json.dumps(out, indent=1))

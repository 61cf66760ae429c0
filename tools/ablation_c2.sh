#!/usr/bin/env bash
# Paper-style ablations on B200 at C2: window buffering
# depth and constant-CPU-buffer size vs cache hit ratio, host traffic and rate.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() {  # name, extra args
  timeout 900 python bench.py --no-cpu-baseline --steps 50 "${@:2}" > gpurun_out/abl_$1.json 2>&1
  python - "$1" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/abl_{sys.argv[1]}.json").read().strip().splitlines()[-1])
t = d["tiers_per_step"]
print(json.dumps({"case": sys.argv[1], "e2e": round(d["e2e"]["value"], 1),
                  "hit_ratio": round(t["cache_hits"] / t["sampled"], 4),
                  "buffer_ratio": round(t["cpu_buffer"] / t["sampled"], 4),
                  "storage_ratio": round(t["storage"] / t["sampled"], 4),
                  "host_gbs": round(d["roofline"]["achieved"], 1)}))
PY
}
for w in 0 4 8; do run w$w --set window_depth=$w; done
for b in 0.0 0.1 0.2; do run buf$b --set buffer_fraction=$b; done

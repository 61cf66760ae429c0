cd $GRAFT_REPO_ROOT
for i in 1 2 3 4 5 6 7 8; do timeout 300 python tools/_dbg_shared2.py 2 2>&1 | grep -E "^mode"; done
timeout 900 python -m pytest tests/test_gpu_exact_par.py tests/test_gpu_fuzz.py tests/test_gpu_shared_cache.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_exact.json 2> gpurun_out/c4_exact.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/c4_exact.json").read().strip().splitlines()[-1])
print(d["value"], d["phase_ms_per_step"])
P

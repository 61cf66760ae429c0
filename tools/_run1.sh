cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_exact_par.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -1
timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_exact.json 2> gpurun_out/c4_exact.err
python - <<'P'
import json
d=json.loads(open("gpurun_out/c4_exact.json").read().strip().splitlines()[-1])
print(d["value"], d["phase_ms_per_step"]); x=d["exact_par"]
print({k:(round(v/x["rounds"]) if k.startswith("cyc") else v) for k,v in x.items()})
P

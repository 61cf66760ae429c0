cd $GRAFT_REPO_ROOT
for v in "" "GIDS_PRIORITY=ctl"; do
env $v GIDS_TRACE_HOST=1 timeout 600 python bench.py --workload c3 --policy exact --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c3_tl.json 2>&1
python - <<'P'
import json
d=json.loads(open("gpurun_out/c3_tl.json").read().strip().splitlines()[-1])
print(d["value"], d["phase_ms_per_step"]); print(d["e2e_timeline_ms"])
P
done
GIDS_TRACE_HOST=1 timeout 600 python bench.py --workload c3 --policy setassoc --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c3_tl.json 2>&1
python - <<'P'
import json
d=json.loads(open("gpurun_out/c3_tl.json").read().strip().splitlines()[-1])
print(d["value"], d["phase_ms_per_step"]); print(d["e2e_timeline_ms"])
P
timeout 600 python -m pytest tests/test_gpu_cache_api.py tests/test_gpu_loader.py -q -x 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x 2>&1 | tail -5

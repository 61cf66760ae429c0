cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_loader.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2 3 4 5; do
GIDS_TRACE_HOST=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b27_$i.json 2>&1
python - gpurun_out/b27_$i.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['e2e']['value'],1), d['e2e_host_ms_per_call'], [[round(x*1e3,2) for x in t] for t in d['e2e_host_trace_slowest_s']])
PY
done

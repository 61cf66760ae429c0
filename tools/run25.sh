cd $GRAFT_REPO_ROOT
for i in 1 2 3 4; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b25_$i.json 2>&1
python - gpurun_out/b25_$i.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['e2e']['value'],1), d['e2e_host_ms_per_call'])
PY
done

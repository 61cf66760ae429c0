cd $GRAFT_REPO_ROOT
for w in 4 8 16 32; do
  GIDS_GATHER_WPS=$w timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b6_$w.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/b6_$w.json').read().strip().splitlines()[-1]); print('wps=$w', round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})
"
done
GIDS_GATHER_WPS=8 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --policy setassoc > gpurun_out/b6_sa8.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b6_sa8.json').read().strip().splitlines()[-1]); print('sa wps=8', round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})
"

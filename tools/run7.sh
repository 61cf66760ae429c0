cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for w in 1 2 4; do
  GIDS_GATHER_WPS=$w timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b7_$w.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/b7_$w.json').read().strip().splitlines()[-1]); print('wps=$w', round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})
" || tail -5 gpurun_out/b7_$w.json
done
GIDS_GATHER_WPS=2 timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --policy setassoc > gpurun_out/b7_sa.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b7_sa.json').read().strip().splitlines()[-1]); print('sa wps=2', round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})
"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_exact_seq" -s 25 -c 1 -o gpurun_out/prof_exact_ss python bench.py --steps 25 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_e2.log 2>&1; tail -2 gpurun_out/ncu_e2.log

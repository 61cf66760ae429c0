cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b10_c2.json 2>&1; tail -c 400 gpurun_out/b10_c2.json
python - <<'PY'
import json
d=json.loads(open('gpurun_out/b10_c2.json').read().strip().splitlines()[-1]); print('c2', round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, d['roofline']['achieved'])
PY
for w in 2 4; do
GIDS_GATHER_WPS=$w timeout 1500 python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b10_c4_$w.json 2>&1
python - <<PY
import json
d=json.loads(open('gpurun_out/b10_c4_$w.json').read().strip().splitlines()[-1]); print('c4 wps=$w', round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, d['roofline']['achieved'], d['roofline']['hbm_kernel'])
PY
done

cd $GRAFT_REPO_ROOT
for pol in exact setassoc; do
GIDS_TRACE_HOST=1 timeout 600 python bench.py --workload c1 --policy $pol > gpurun_out/b28_$pol.json 2>&1
python - gpurun_out/b28_$pol.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['e2e']['value'],1), d['tiers_per_step'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, d['e2e_host_ms_per_call'], [[round(x*1e3,2) for x in t] for t in d['e2e_host_trace_slowest_s']], d['roofline']['hbm_kernel'], d.get('cpu_baseline'))
PY
done

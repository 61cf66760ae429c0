cd $GRAFT_REPO_ROOT
summ() { python - "$1" "$2" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],1), round(d['e2e']['value'],1), d['tiers_per_step'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, round(d['roofline']['achieved'],2), d.get('cpu_baseline'), d['setup_s'], flush=True)
PY
}
timeout 1500 python bench.py --workload c3 --steps 30 --warmup 10 > gpurun_out/b33_c3.json 2>&1; summ gpurun_out/b33_c3.json c3; tail -2 gpurun_out/b33_c3.json | cut -c1-300
timeout 900 python bench.py --workload c2p > gpurun_out/b33_c2p.json 2>&1; summ gpurun_out/b33_c2p.json c2p

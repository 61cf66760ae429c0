cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
summ() { python - "$1" "$2" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, d['e2e_host_ms_per_call']['median'], flush=True)
PY
}
for sp in 0 2; do
timeout 600 python bench.py --workload c1 --warmup 40 --steps 100 --no-cpu-baseline --set gids_speculate=$sp > gpurun_out/t_c1.json 2>&1; summ gpurun_out/t_c1.json "c1 exact spec=$sp"
timeout 600 python bench.py --workload c1 --policy setassoc --warmup 40 --steps 100 --no-cpu-baseline --set gids_speculate=$sp > gpurun_out/t_c1.json 2>&1; summ gpurun_out/t_c1.json "c1 setassoc spec=$sp"
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t_c2.json 2>&1; summ gpurun_out/t_c2.json "c2 exact spec=2"

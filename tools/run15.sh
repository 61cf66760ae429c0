cd $GRAFT_REPO_ROOT
summ() { python - "$1" "$2" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, round(d['roofline']['achieved'],2), flush=True)
PY
}
for pr in gather ctl; do
GIDS_PRIORITY=$pr timeout 600 python bench.py --steps 80 --warmup 5 --no-cpu-baseline > gpurun_out/b15.json 2>&1; summ gpurun_out/b15.json "c2 prio=$pr"
done
for pr in gather ctl; do
GIDS_PRIORITY=$pr timeout 1500 python bench.py --workload c4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b15_c4_$pr.json 2>&1; summ gpurun_out/b15_c4_$pr.json "c4 prio=$pr"
done
GIDS_GATHER_WPS=8 GIDS_GATHER_UNROLL=4 timeout 1500 python bench.py --workload c4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b15_c4_84.json 2>&1; summ gpurun_out/b15_c4_84.json "c4 prio=gather wps8 u4"

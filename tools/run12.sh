cd $GRAFT_REPO_ROOT
summ() { python - "$1" "$2" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, round(d['roofline']['achieved'],2), flush=True)
PY
}
for rep in 1 2; do
for cfg in "1 1" "1 2" "2 1" "1 4" "2 2" "2 4" "4 1" "4 2"; do set -- $cfg
GIDS_GATHER_WPS=$1 GIDS_GATHER_UNROLL=$2 timeout 600 python bench.py --steps 80 --warmup 5 --no-cpu-baseline > gpurun_out/b12.json 2>&1; summ gpurun_out/b12.json "c2 wps=$1 u=$2"
done; done

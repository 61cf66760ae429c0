cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
summ() { python - "$1" "$2" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, round(d['roofline']['achieved'],2))
PY
}
for u in 8 4; do
GIDS_GATHER_UNROLL=$u timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b11_c2_$u.json 2>&1; summ gpurun_out/b11_c2_$u.json "c2 u=$u"
done
for w in 2 4; do for u in 8 4; do
GIDS_GATHER_UNROLL=$u GIDS_GATHER_WPS=$w timeout 1500 python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b11_c4_${w}_$u.json 2>&1; summ gpurun_out/b11_c4_${w}_$u.json "c4 wps=$w u=$u"
done; done

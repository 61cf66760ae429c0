cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for b in 1 2 3 4; do for u in 4 8; do
GIDS_HIT_BPS=$b GIDS_HIT_UNROLL=$u timeout 600 python bench.py --workload c1 --steps 200 --warmup 40 --no-cpu-baseline > gpurun_out/c1_hit_${b}_${u}.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/c1_hit_${b}_${u}.json'));print('bps $b unroll $u', round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,4) for k,v in d['phase_ms_per_step'].items()}, round(d['roofline']['achieved'],1))"
done; done

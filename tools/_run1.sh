cd $GRAFT_REPO_ROOT
for cfg in "4 4" "8 4" "4 8" "8 8" "16 4" "2 8"; do set -- $cfg
GIDS_SHARD_BPS=$1 GIDS_SHARD_U=$2 timeout 600 python bench.py --workload c5v --steps 30 --warmup 10 --no-cpu-baseline > gpurun_out/c5v.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/c5v.json').read().strip().splitlines()[-1]); print('bps $1 u $2', round(d['value']), d['roofline']['achieved'], d['phase_ms_per_step'])"
done

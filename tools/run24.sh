cd $GRAFT_REPO_ROOT
summ() { python - "$1" "$2" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, round(d['roofline']['achieved'],2), d['clocks'], flush=True)
PY
}
for i in 1 2 3; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b24_$i.json 2>&1; summ gpurun_out/b24_$i.json "c2 default run $i"
done
timeout 600 python bench.py --no-cpu-baseline --set gids_sharded_table=true --set gids_virtual_shards=4 --set buffer_fraction=0.0 --set cache_lines=0 > gpurun_out/b24_vs.json 2>&1; tail -c 2500 gpurun_out/b24_vs.json

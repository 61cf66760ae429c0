cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_storage_file.py -q -x 2>&1 | grep -E "assert|Error|passed|failed" | head -10
for t in 128 256; do
timeout 900 python bench.py --workload c2 --steps 8 --warmup 3 --no-cpu-baseline --set gids_storage=file --set gids_storage_path=/tmp/c2.gfea --set gids_io_direct=true --set gids_storage_offset=4096 --set gids_io_threads=$t > gpurun_out/c2f_$t.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/c2f_$t.json').read().strip().splitlines()[-1]); print('c2 file threads $t', d['value'], d['storage_file'])" 2>&1 | tail -1
rm -f /tmp/c2.gfea
done

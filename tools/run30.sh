cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_storage_file.py -m gpu -q -x 2>&1 | tail -15
summ() { python - "$1" "$2" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, d.get('storage_file'), flush=True)
PY
}
timeout 900 python bench.py --no-cpu-baseline --set gids_storage=file --set gids_storage_path=/dev/shm/c2.gfea --set gids_io_threads=16 > gpurun_out/b30_shm.json 2>&1; summ gpurun_out/b30_shm.json "c2 file /dev/shm 16thr"; tail -3 gpurun_out/b30_shm.json | cut -c1-300
rm -f /dev/shm/c2.gfea
timeout 900 python bench.py --no-cpu-baseline --set gids_storage=file --set gids_storage_path=/tmp/c2.gfea --set gids_io_threads=16 --set gids_io_direct=true > gpurun_out/b30_direct.json 2>&1; summ gpurun_out/b30_direct.json "c2 file /tmp O_DIRECT 16thr"
rm -f /tmp/c2.gfea

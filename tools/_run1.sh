cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_loader.py tests/test_gpu_exact_par.py -q -x 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --workload c1 --steps 200 --warmup 40 --no-cpu-baseline > gpurun_out/c1.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/c1.json').read().strip().splitlines()[-1]); print('c1', d['value'], d['e2e']['value'], d['phase_ms_per_step'], d['e2e_host_ms_per_call']['median'])"; done

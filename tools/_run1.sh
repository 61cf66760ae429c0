cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 1500 python -m pytest tests/test_gpu_exact_par.py tests/test_gpu_fuzz.py tests/test_gpu_loader.py -q -x 2>&1 | tail -3
timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4_prof.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/bench_c4_prof.json'));print(round(d['value'],2), round(d['e2e']['value'],2), d['decision_kernel']['ms_per_batch'], d['decision_kernel']['rounds_per_batch'], d['e2e_host_ms_per_call']['max'])"
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3

cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 1500 python -m pytest tests/test_gpu_loader.py tests/test_gpu_multirank.py tests/test_gpu_shared_cache.py tests/test_gpu_storage_file.py tests/test_gpu_cache_api.py -q -x 2>&1 | tail -3
timeout 600 python tools/host_breakdown.py c1 400 2>&1 | tail -34 | head -12
for i in 1 2 3; do
timeout 600 python bench.py --workload c1 --steps 100 --warmup 40 --no-cpu-baseline > gpurun_out/bench_c1_nw$i.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/bench_c1_nw$i.json'));print(round(d['value'],1), round(d['e2e']['value'],1), d['tier_roofline']['frac'], d['e2e_host_ms_per_call']['median'])"
done

cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 1200 python -m pytest tests/test_gpu_loader.py tests/test_gpu_sampler.py tests/test_gpu_multirank.py tests/test_gpu_shared_cache.py -x -q 2>&1 | tail -3
timeout 600 python tools/host_breakdown.py c1 400 2>&1 | tail -28
for i in 1 2; do
timeout 600 python bench.py --workload c1 --steps 200 --warmup 40 --no-cpu-baseline > gpurun_out/bench_c1_slots$i.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/bench_c1_slots$i.json'));print(round(d['value'],1), round(d['e2e']['value'],1), d['tier_roofline']['frac'], d['e2e_host_ms_per_call']['median'])"
done

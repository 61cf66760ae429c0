cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 1200 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_loader.py tests/test_gpu_cache_api.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -4
timeout 600 python tools/host_breakdown.py c1 400 2>&1 | tail -24
timeout 600 python bench.py --workload c1 --steps 100 --warmup 40 --no-cpu-baseline > gpurun_out/bench_c1_shift.json 2>&1; tail -c 300 gpurun_out/bench_c1_shift.json

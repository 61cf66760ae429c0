cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 900 python -m pytest tests/test_gpu_loader.py tests/test_gpu_multirank.py tests/test_gpu_shared_cache.py -x -q 2>&1 | tail -5
GIDS_SERVE_TIMING=1 timeout 600 python tools/host_breakdown.py c1 400 2>&1 | tail -30
timeout 600 python bench.py --workload c1 --steps 100 --warmup 40 --no-cpu-baseline > gpurun_out/bench_c1_alloc.json 2>&1; tail -c 300 gpurun_out/bench_c1_alloc.json

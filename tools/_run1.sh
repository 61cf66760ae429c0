cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python tools/host_breakdown.py c1 400 2>&1 | tail -24
timeout 600 python bench.py --workload c1 --steps 100 --warmup 40 --no-cpu-baseline > gpurun_out/bench_c1_graph.json 2>&1; tail -c 300 gpurun_out/bench_c1_graph.json
timeout 600 python bench.py --workload c2 --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2_graph.json 2>&1; tail -c 300 gpurun_out/bench_c2_graph.json

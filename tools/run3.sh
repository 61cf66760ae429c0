cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_exact3.json 2> gpurun_out/bench_exact3.err; tail -c 2500 gpurun_out/bench_exact3.json; tail -3 gpurun_out/bench_exact3.err
timeout 600 python bench.py --steps 50 --warmup 5 --policy setassoc --no-cpu-baseline > gpurun_out/bench_sa3.json 2>&1; tail -c 1200 gpurun_out/bench_sa3.json

cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b9_c2.json 2>&1; tail -c 600 gpurun_out/b9_c2.json
timeout 1500 python bench.py --workload c4 --steps 20 --warmup 5 > gpurun_out/b9_c4.json 2>&1; tail -c 3000 gpurun_out/b9_c4.json

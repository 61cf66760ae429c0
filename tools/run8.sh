cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 300 python tools/probe_box.py > gpurun_out/probe.json 2>&1; cat gpurun_out/probe.json | head -40
lscpu | head -20
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/b8.json 2>&1; tail -c 1500 gpurun_out/b8.json

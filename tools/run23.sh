cd $GRAFT_REPO_ROOT
nproc; free -g | head -2
timeout 900 python bench.py --impl reference --steps 10 --warmup 2 > gpurun_out/ref_c2.json 2>&1; tail -c 1200 gpurun_out/ref_c2.json
timeout 2400 python bench.py --impl reference --workload c4 --steps 3 --warmup 1 > gpurun_out/ref_c4.json 2>&1; tail -c 1500 gpurun_out/ref_c4.json
free -g | head -2

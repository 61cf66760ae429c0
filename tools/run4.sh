cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_exact4.json 2> gpurun_out/bench_exact4.err; tail -c 2500 gpurun_out/bench_exact4.json; tail -3 gpurun_out/bench_exact4.err
timeout 600 python bench.py --steps 50 --warmup 5 --policy setassoc --no-cpu-baseline > gpurun_out/bench_sa4.json 2>&1; tail -c 1500 gpurun_out/bench_sa4.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gather_host" -s 6 -c 1 -o gpurun_out/prof_gather_r01 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_g.log 2>&1; tail -2 gpurun_out/ncu_g.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_exact_seq" -s 6 -c 1 -o gpurun_out/prof_exact_r01 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_e.log 2>&1; tail -2 gpurun_out/ncu_e.log

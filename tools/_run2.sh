cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exact_par -s 5 -c 1 -o gpurun_out/prof_c4_exact_par2 python bench.py --workload c4 --policy exact --steps 2 --warmup 4 --no-cpu-baseline > gpurun_out/ncu_xp.log 2>&1
tail -2 gpurun_out/ncu_xp.log

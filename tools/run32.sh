cd $GRAFT_REPO_ROOT
export BENCH_PROFILE_STEADY=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches_steady.csv python bench.py --steps 20 --warmup 30 --no-cpu-baseline > gpurun_out/c2_steady.log 2>&1; tail -c 300 gpurun_out/c2_steady.log
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches_steady.csv python bench.py --workload c4 --steps 10 --warmup 10 --no-cpu-baseline > gpurun_out/c4_steady.log 2>&1; tail -c 300 gpurun_out/c4_steady.log

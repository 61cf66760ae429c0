cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
GIDS_NO_GRAPHS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_hits -s 60 -c 1 \
    -o gpurun_out/prof_c1_gather_hits python bench.py --workload c1 --steps 5 --warmup 40 \
    --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1
tail -3 gpurun_out/ncu_c1.log
ls -la gpurun_out/*.ncu-rep
timeout 1500 python tools/run_reference_tests.py > gpurun_out/reftests.txt 2>&1; tail -5 gpurun_out/reftests.txt

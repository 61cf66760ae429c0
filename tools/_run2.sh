cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --impl reference --workload c4 --policy exact --steps 3 --warmup 2 > gpurun_out/ref_c4_exact.json 2> gpurun_out/ref_c4_exact.err
tail -c 1500 gpurun_out/ref_c4_exact.json

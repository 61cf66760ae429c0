set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_exact.json 2> gpurun_out/bench_exact.err; tail -c 3000 gpurun_out/bench_exact.json
timeout 600 python bench.py --steps 50 --warmup 5 --policy setassoc --no-cpu-baseline > gpurun_out/bench_sa.json 2> gpurun_out/bench_sa.err; tail -c 3000 gpurun_out/bench_sa.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.json 2>&1; tail -c 1500 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather_host|k_exact_seq|k_sample_layer" -s 12 -c 6 -o gpurun_out/prof_r01 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -5 gpurun_out/ncu_full.log; ls -la gpurun_out/

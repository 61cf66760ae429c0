cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_sharded.py -m gpu -q -x 2>&1 | tail -30
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather_host" -s 6 -c 1 -o gpurun_out/prof_c2_gather_host python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c2_ncu.log 2>&1; tail -1 gpurun_out/c2_ncu.log
KS='regex:k_sample_layer|k_seed_mark|k_bm_|k_td_|k_rng|k_contribution|k_copy_edges|k_widen|k_window|k_sa_|k_tier_count|k_gather|k_i32|k_i64|DeviceSelect|k_post|k_exact'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k "$KS" -c 3000 --csv --log-file gpurun_out/c2_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c2_ncu1.log 2>&1; tail -1 gpurun_out/c2_ncu1.log | cut -c1-100

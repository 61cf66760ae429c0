cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_exact_par.py -q 2>&1 | tail -1; done
GIDS_SERVE_TIMING=1 GIDS_TRACE_HOST=1 timeout 600 python tools/profile_host.py c1 300 > gpurun_out/host_profile_c1.txt 2>&1; grep -E "per next_batch|trace ms|serve host" gpurun_out/host_profile_c1.txt

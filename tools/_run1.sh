cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_shared_cache.py -q 2>&1 | tail -2
timeout 1500 python tools/run_reference_tests.py > gpurun_out/reftests.txt 2>&1; head -14 gpurun_out/reftests.txt

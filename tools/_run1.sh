cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 1500 python -m pytest tests/test_gpu_loader.py tests/test_gpu_cache_api.py tests/test_gpu_shared_cache.py tests/test_gpu_storage_file.py tests/test_c_example.py -q -x 2>&1 | tail -2
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1

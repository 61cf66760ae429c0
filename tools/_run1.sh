cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 1200 python -m pytest tests/test_gpu_loader.py -q -x 2>&1 | tail -4

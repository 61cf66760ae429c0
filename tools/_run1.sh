cd $GRAFT_REPO_ROOT
for i in 1 2 3 4 5; do timeout 900 python -m pytest tests/test_gpu_loader.py -q -x -k matches_reference_run 2>&1 | grep -E "^E  |passed|failed|^FAILED" | head -4; done

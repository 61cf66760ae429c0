cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
GIDS_FULLSIZE=1 timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -x -k oracle 2>&1 | tail -4

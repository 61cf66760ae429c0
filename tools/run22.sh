cd $GRAFT_REPO_ROOT
timeout 600 tools/hostread_bench 4096 8 0.05 0 1
timeout 600 tools/hostread_bench 512 8 0.05 0 1

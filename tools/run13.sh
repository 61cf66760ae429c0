cd $GRAFT_REPO_ROOT
timeout 300 tools/hostread_bench 512 8 0.05
timeout 300 tools/hostread_bench 4096 8 0.05

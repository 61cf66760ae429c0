cd $GRAFT_REPO_ROOT
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag; grep -i huge /proc/meminfo
timeout 600 tools/hostread_bench 512 57 0.027 0 1
timeout 600 tools/hostread_bench 512 57 0.027 1 1
timeout 300 tools/hostread_bench 4096 57 0.002 0 1
grep -i AnonHuge /proc/meminfo

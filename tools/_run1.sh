cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
echo "exit=${PIPESTATUS[0]}"
dmesg 2>/dev/null | grep -i "out of memory" | tail -2

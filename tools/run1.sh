set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "sampler" 2>&1 | tail -30
timeout 900 python -m pytest tests -m gpu -q -k "loader" 2>&1 | tail -40
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 5 2>&1 | tail -5

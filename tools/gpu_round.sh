#!/usr/bin/env bash
# One GPU pass over everything a round is judged on (run under gpurun):
#   tools/gpu_round.sh [quick]
# GPU tests + smoke, the default bench line (C4, exact policy) and the
# reference arm at the same config, steady-state ncu launch list and full
# captures of the two dominant kernels (host-tier gather, exact policy).
# Outputs land in gpurun_out/ (copy what is kept into profiles/).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
set -x
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -2
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2>&1; tail -c 600 gpurun_out/bench_c4.json
[ "$1" = quick ] && exit 0
timeout 1500 python bench.py --impl reference --steps 3 --warmup 2 > gpurun_out/bench_ref_c4.json 2>&1
timeout 600 python bench.py --workload c1 --steps 100 --warmup 40 > gpurun_out/bench_c1.json 2>&1
timeout 600 python bench.py --workload c2 --steps 50 --warmup 10 > gpurun_out/bench_c2.json 2>&1
export BENCH_PROFILE_STEADY=1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/c4_launches_steady.csv python bench.py --steps 6 --warmup 6 \
    --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/c1_launches_steady.csv python bench.py --workload c1 --steps 20 \
    --warmup 40 --no-cpu-baseline > /dev/null 2>&1
unset BENCH_PROFILE_STEADY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_hits -s 60 -c 1 \
    -o gpurun_out/prof_c1_gather_hits python bench.py --workload c1 --steps 5 --warmup 40 \
    --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_gather_host -s 12 -c 1 \
    -o gpurun_out/prof_c4_gather_host python bench.py --steps 5 --warmup 10 \
    --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_exact_par -s 6 -c 1 \
    -o gpurun_out/prof_c4_exact_par python bench.py --steps 2 --warmup 4 \
    --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out

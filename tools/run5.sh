cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_exact5.json 2> gpurun_out/bench_exact5.err; python -c "
import json
for f in ['gpurun_out/bench_exact5.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['phase_ms_per_step'], d['tier_roofline'])
"; tail -3 gpurun_out/bench_exact5.err
timeout 600 python bench.py --steps 50 --warmup 5 --policy setassoc --no-cpu-baseline > gpurun_out/bench_sa5.json 2>&1; python -c "
import json
for f in ['gpurun_out/bench_sa5.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['phase_ms_per_step'], d['tier_roofline'])
"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gather_host" -s 3 -c 1 -o gpurun_out/prof_gather_r01 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_g.log 2>&1; tail -2 gpurun_out/ncu_g.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_exact_seq" -s 3 -c 1 -o gpurun_out/prof_exact_r01 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_e.log 2>&1; tail -2 gpurun_out/ncu_e.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches_r01.csv

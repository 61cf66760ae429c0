cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for i in 1 2 3 4; do
timeout 1200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4_trace$i.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/bench_c4_trace$i.json'));print(d['e2e_host_ms_per_call'], d['gc_pauses_ms'])"
done

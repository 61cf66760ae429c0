cd $GRAFT_REPO_ROOT
summ() { python - "$1" "$2" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['phase_ms_per_step'].items()}, round(d['roofline']['achieved'],2), d['tiers_per_step'], flush=True)
PY
}
timeout 600 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_prod|k_ldg" --csv --log-file gpurun_out/mb_ncu.csv tools/hostread_bench 512 57 0.027 0 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/mb_ncu.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]; h=rows[hi]
for r in rows[hi+1:]:
    if len(r)>h.index('Metric Value'): print(r[h.index('ID')], r[h.index('Kernel Name')][:40], r[h.index('Metric Name')], r[h.index('Metric Value')])
PY
timeout 1500 python bench.py --workload c4 --steps 30 --warmup 5 --no-cpu-baseline --set buffer_fraction=0.0 > gpurun_out/b18a.json 2>&1; summ gpurun_out/b18a.json "c4 nobuf"
timeout 1500 python bench.py --workload c4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b18b.json 2>&1; summ gpurun_out/b18b.json "c4 (rebuilt: wps2 u2)"

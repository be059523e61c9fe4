timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_dyn.csv python bench.py --steps 2 --warmup 1 --workload c4_sort --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_dyn.csv')) if len(r)>10 and r[0].isdigit()]
seen={}
for r in rows:
    n=r[4].split('(')[0][-40:]
    seen.setdefault(n,[]).append(float(r[-1])/1e3)
for n,v in seen.items(): print(f"{n:42s} n={len(v):3d} first {v[0]:9.1f} us  min {min(v):9.1f}")
PY

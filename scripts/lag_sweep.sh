#!/bin/bash
# headline step time against the shading lag K (tiles); default K = 1.5 x resident CTAs
for lag in ${LAGS:-592 740 888 1036 1184}; do
  r=$(VR_LAG=$lag timeout 300 python bench.py --steps ${STEPS:-60} --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "lag $lag $r" | tee -a gpurun_out/lag.log
done

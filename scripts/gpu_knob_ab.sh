#!/bin/bash
# A/B of environment knobs: KNOBS="A=1;B=2 C=3" (sets separated by ';'), WORKLOADS="c4_sort ..."
mkdir -p gpurun_out
IFS=';' read -ra SETS <<< "${KNOBS:-X=0}"
for set in "${SETS[@]}"; do
  echo "== $set"
  for wl in ${WORKLOADS:-c4_sort c4_hash}; do
    env $set python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-others --workload $wl 2>gpurun_out/knob_err.log | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('   $wl', round(d['ms_per_step'],4), d.get('stage_ms'), 'frac', round(d.get('stage_roofline',{}).get('frac',0),3))"
    grep vrgeom gpurun_out/knob_err.log | head -1
  done
done

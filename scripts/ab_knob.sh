#!/bin/bash
# A/B of one debug knob (csrc/vr_common.cuh DebugKnobs) over the dynamic-batch rows of the bench.
# usage: KNOB=VR_DYN3_TILE_SHIFT VALUES="0 3 4 5" bash scripts/ab_knob.sh
mkdir -p gpurun_out
for rep in 1 2; do
for v in $VALUES; do
  env $KNOB=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$KNOB=$v', ' '.join('%s %.4f/%.4f' % (k, v['ms_per_step'], (v.get('stage_ms') or {}).get('dedup', 0)) for k, v in d['others'].items() if isinstance(v, dict) and 'ms_per_step' in v and k != 'c1_sort'))
" | tee -a gpurun_out/ab_knob.log
done
done

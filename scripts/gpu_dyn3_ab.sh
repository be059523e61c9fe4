#!/bin/bash
# A/B of the dyn3 knobs on the shuffled mesh (gpurun): prints ms per step and the kernel split
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dyn3.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
run() {
  echo "== $*"
  for wl in ${WORKLOADS:-c4_sort c4_hash c3_dyn_sort}; do
    env "$@" python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-others --workload $wl 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('   $wl', round(d['ms_per_step'],4), d.get('stage_ms'), 'frac', round(d.get('stage_roofline',{}).get('frac',0),3))"
  done
}
run VR_L2_HINTS=1 VR_DYN3_PREFETCH=1
run VR_L2_HINTS=0 VR_DYN3_PREFETCH=1
run VR_L2_HINTS=1 VR_DYN3_PREFETCH=0
run VR_L2_HINTS=0 VR_DYN3_PREFETCH=0

#!/bin/bash
# A/B on one box: every variants/*.so is copied over the in-tree library; prints the dynamic-batch rows of the bench.
mkdir -p gpurun_out
LIB=paper_1805_08893_b200/libvrgeom.so
cp $LIB /tmp/keep.so
for rep in 1 2; do
for v in variants/*.so; do
  cp $v $LIB
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', ' '.join('%s %.4f/%.4f' % (k, v['ms_per_step'], (v.get('stage_ms') or {}).get('dedup', 0)) for k, v in d['others'].items() if isinstance(v, dict) and 'ms_per_step' in v and k != 'c1_sort'))
" | tee -a gpurun_out/ab_dyn3.log
done
done
cp /tmp/keep.so $LIB

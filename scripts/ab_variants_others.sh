#!/bin/bash
# A/B of whole libraries over the dynamic-batch rows of the bench: every variants/*.so in turn.
LIB=paper_1805_08893_b200/libvrgeom.so
cp $LIB /tmp/keep.so
for rep in 1 2; do
for v in variants/*.so; do
  cp $v $LIB
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', ' '.join('%s %.4f' % (k, v['ms_per_step']) for k, v in d['others'].items() if isinstance(v, dict) and 'ms_per_step' in v and k != 'c1_sort'))
"
done
done
cp /tmp/keep.so $LIB

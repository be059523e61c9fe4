#!/bin/bash
# A/B of whole libraries: every variants/*.so is copied over the in-tree library in turn; headline workload only.
LIB=paper_1805_08893_b200/libvrgeom.so
cp $LIB /tmp/keep.so
for rep in 1 2; do
for v in variants/*.so; do
  cp $v $LIB
  timeout 200 python bench.py --no-others --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['sustained']['ms_per_step'], d['roofline']['frac'])"
done
done
cp /tmp/keep.so $LIB

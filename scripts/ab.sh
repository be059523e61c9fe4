#!/bin/bash
# A/B on one box: every variants/*.so is copied over the in-tree library and timed on the headline workload.
mkdir -p gpurun_out
LIB=paper_1805_08893_b200/libvrgeom.so
cp $LIB /tmp/keep.so
for rep in 1 2; do
for v in variants/*.so; do
  cp $v $LIB
  r=$(timeout 300 python bench.py --steps ${STEPS:-60} --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])")
  echo "$v $r" | tee -a gpurun_out/ab.log
done
done
cp /tmp/keep.so $LIB

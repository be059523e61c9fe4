#!/bin/bash
# ncu on the three-kernel sort/hash/phash path: launch list + one full capture per dyn3 kernel, per workload.
mkdir -p gpurun_out
for wl in ${WORKLOADS:-c4_sort c4_hash}; do
  B="python bench.py --steps 2 --warmup 1 --workload $wl --no-others --no-cpu-baseline"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$wl.csv $B > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dyn3 -s ${SKIP:-4} -c ${COUNT:-4} -f -o gpurun_out/prof_$wl $B > gpurun_out/prof_$wl.log 2>&1
done
ls -la gpurun_out

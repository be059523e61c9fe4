#!/bin/bash
# ncu evidence for the bench workload: launch list + full capture of the two main kernels.
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS}"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/launches.log 2>&1
for k in ${KERNELS:-warp_tpb finalize}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-3} -c 1 -f -o gpurun_out/prof_$k $B > gpurun_out/prof_$k.log 2>&1
done
ls -la gpurun_out

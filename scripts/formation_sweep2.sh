#!/bin/bash
# kernel times (ncu launch list) of the window walk against its run length (start primitives per thread)
for wl in c4_sort c3_dyn_sort; do
for run in ${RUNS:-10 14 18 22 30 46}; do
  VR_GREEDY_RUN_S=$run timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:greedy_next -c 1 --csv --log-file /tmp/g.csv python bench.py --steps 2 --warmup 1 --workload $wl --no-others --no-cpu-baseline > /dev/null 2>&1
  echo "$wl run $run: $(tail -1 /tmp/g.csv | awk -F'\",\"' '{print $NF}')"
done; done

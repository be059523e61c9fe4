for wl in c4_sort c3_dyn_sort; do
for kv in "VR_GREEDY_RUN=64" "VR_GREEDY_RUN=32" "VR_GREEDY_RUN=16" "VR_GREEDY_RUN=8" "VR_LINK_TILE=2048" "VR_LINK_TILE=3072" "VR_LINK_TILE=6144"; do
  r=$(env $kv python bench.py --steps 10 --workload $wl --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['batch_formation_ms'])")
  echo "$wl $kv formation_ms $r"
done; done

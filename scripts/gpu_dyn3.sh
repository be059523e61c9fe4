#!/bin/bash
# dyn3 parity tests + the bench's per-strategy block (gpurun)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dyn3.py tests/test_gpu_parity.py tests/test_gpu_draws.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dyn3.log 2>&1
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/bench_dyn3.log') if l.startswith('{')][-1])
print('headline', round(d['ms_per_step'],4), d['roofline']['frac'])
for k,v in d['others'].items():
    if isinstance(v,dict) and "ms_per_step" in v:
        print(f"{k:20s} {v['ms_per_step']:.4f} ms  frac {v.get('stage_roofline',{}).get('frac',0):.3f}  {v.get('stage_ms')}")
PY
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/bench_dyn3.log') if l.startswith('{')][-1])
print(json.dumps(d['others'].get('shader_load'), indent=0)[:1500])
print(json.dumps(d['others'].get('clients'), indent=0)[:1500])
print('e2e', d['e2e']['value'], d['e2e']['ms_per_step'])
PY
tail -3 gpurun_out/bench_dyn3.log | cut -c1-600

#!/bin/bash
# A/B timing of env-var variants on the 1M-tet scene (config 5)
for v in "$@"; do
  env $v timeout 900 python bench.py --scene H --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/abh.log 2>&1
  tail -1 gpurun_out/abh.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_frame']; print('$v', round(d['value'],2), {n: k[n] for n in k if k[n] > 1})" || tail -5 gpurun_out/abh.log
done

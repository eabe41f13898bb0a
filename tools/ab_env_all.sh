#!/bin/bash
# A/B timing of env-var variants of the default bench workload, every kernel's ms/frame:
#   tools/ab_env_all.sh "SS_X=0" "SS_LIB_OVERRIDE=build_var/x.so" ...
for v in "$@"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_frame']; print('$v', round(d['value'],1), round(sum(k.values()),2), {n: round(k[n],3) for n in k})" || tail -5 gpurun_out/ab.log
done

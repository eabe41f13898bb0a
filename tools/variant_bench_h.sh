#!/bin/bash
# A/B of library variants on the 1M-tet snake (bench --scene H)
for lib in "$@"; do
  SS_LIB_OVERRIDE=$lib timeout 600 python bench.py --scene H --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/vbh.log 2>&1
  tail -1 gpurun_out/vbh.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_frame']; print('$lib', round(d['value'],2), {n: k[n] for n in k if k[n] > 1})"
done

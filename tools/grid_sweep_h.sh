#!/bin/bash
# A/B of the grid caps on the 1M-tet scene: args "stream,eval,reduce"
for cfg in "$@"; do
  IFS=, read sb eb rb <<< "$cfg"
  SS_STREAM_BLOCKS=$sb SS_EVAL_BLOCKS=$eb SS_REDUCE_BLOCKS=$rb timeout 600 python bench.py --scene H --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gsh.log 2>&1
  tail -1 gpurun_out/gsh.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_frame']; print('$cfg', round(d['value'],2), {n: k[n] for n in k if k[n] > 1})"
done

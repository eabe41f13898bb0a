#!/bin/bash
# cluster (1, 32 envs) and streaming (1024 envs) throughput per library variant
for lib in "$@"; do
  for cfg in "1 cluster" "32 cluster" "1024 streaming"; do
    set -- $cfg
    SS_LIB_OVERRIDE=$lib timeout 300 python bench.py --envs $1 --solver $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/vc.log 2>&1
    v=$(tail -1 gpurun_out/vc.log | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))" 2>/dev/null)
    echo "$lib envs=$1 $2 $v"
  done
done

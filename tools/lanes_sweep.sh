#!/bin/bash
# Concurrent-lane sweep (SS_LANES) on the default 1024-env workload, alternating.
for rep in 1 2; do
  for l in ${LANES:-2 3 4}; do
    SS_LANES=$l timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ls.log 2>&1
    tail -1 gpurun_out/ls.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lanes $l', round(d['value'],1), d['clocks']['sm_mhz'], d['config']['solver'])"
  done
done

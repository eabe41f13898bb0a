#!/bin/bash
# Concurrent-lane sweep (SS_LANES) on small batches (ENVS, default 128 256 512), alternating.
for n in ${ENVS:-128 256 512}; do
  for rep in 1 2; do
    for l in ${LANES:-1 2 3 4}; do
      SS_LANES=$l timeout 600 python bench.py --envs $n --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/lsm.log 2>&1
      tail -1 gpurun_out/lsm.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('envs $n lanes $l', round(d['value'],1), d['clocks']['sm_mhz'], d['config']['solver'])"
    done
  done
done

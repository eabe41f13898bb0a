#!/bin/bash
# k_apply_rows / k_newton_final grid sweep (SS_REDUCE_BLOCKS), alternating
for rep in 1 2; do
  for b in 296 592 888 1184; do
    SS_REDUCE_BLOCKS=$b timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rs.log 2>&1
    tail -1 gpurun_out/rs.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_frame']; print('reduce blocks $b', round(d['value'],1), k['k_apply_rows'], k['k_newton_final'], d['clocks']['sm_mhz'])"
  done
done

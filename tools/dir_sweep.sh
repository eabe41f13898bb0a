#!/bin/bash
# k_pcr_dir grid sweep (SS_DIR_BLOCKS; default = occupancy x SMs), alternating
for rep in 1 2; do
  for b in 296 444 592 888; do
    SS_DIR_BLOCKS=$b timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ds.log 2>&1
    tail -1 gpurun_out/ds.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_frame']; print('dir blocks $b', round(d['value'],1), k['k_pcr_dir'], d['clocks']['sm_mhz'])"
  done
done

#!/bin/bash
# snake-steps/s of the streaming and cluster solvers vs batch size (sets the
# solver="auto" threshold in ss_create)
for e in ${@:-1 2 4 8 16 32 64 128 256}; do
  for s in streaming cluster; do
    timeout 300 python bench.py --envs $e --steps 10 --warmup 3 --no-cpu-baseline --profile-frames 1 --solver $s > gpurun_out/xo.log 2>&1
    v=$(tail -1 gpurun_out/xo.log | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))" 2>/dev/null)
    echo "envs=$e solver=$s value=$v"
  done
done

#!/bin/bash
# A/B timing of library variants: tools/variant_bench.sh lib1.so lib2.so ...
# (each run: bench.py default workload, kernel ms/frame summary)
for lib in "$@"; do
  SS_LIB_OVERRIDE=$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/vb.log 2>&1
  tail -1 gpurun_out/vb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_frame']; print('$lib', round(d['value'],1), {n: k[n] for n in k if k[n] > 1})"
done

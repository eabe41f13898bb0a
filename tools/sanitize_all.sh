#!/bin/bash
# compute-sanitizer over the tools/sanitize.py workloads; one log per tool x
# workload under gpurun_out/sanitize/ (summaries copied to profiles/)
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for tool in memcheck racecheck synccheck initcheck; do
  for w in cluster streaming fused builder; do
    [ "$tool" = "initcheck" ] && [ "$w" = "cluster" ] && continue
    timeout 900 $CS --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize.py $w > gpurun_out/sanitize/${tool}_${w}.log 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize/${tool}_${w}.log | tail -1)"
  done
done

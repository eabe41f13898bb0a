#!/bin/bash
# A/B of env-var variants, full bench JSON kept: tools/ab_save.sh tag "ENV=.." "ENV=.." [-- bench args]
tag=$1; shift
vars=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do vars+=("$1"); shift; done
[ "$1" == "--" ] && shift
args="$@"; [ -z "$args" ] && args="--steps 5 --warmup 3 --no-cpu-baseline"
for v in "${vars[@]}"; do
  env $v timeout 600 python bench.py $args > gpurun_out/ab_${tag}.log 2>&1
  line=$(grep '^{' gpurun_out/ab_${tag}.log | tail -1)
  echo "$v $line" >> gpurun_out/ab_${tag}.jsonl
  echo "$line" | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_frame']; print('$v', round(d['value'],1), 'clk', d.get('clocks',{}).get('sm_mhz'), 'dom', d['roofline'].get('kernel'), round(d['roofline']['frac'],3), {n: k[n] for n in k if k[n] > 1})" || tail -5 gpurun_out/ab_${tag}.log
done

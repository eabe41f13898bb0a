#!/bin/bash
# Every bench configuration on one box (one JSON summary line each).
summ() { python -c "import json,sys; l=[x for x in sys.stdin if x.startswith('{')]; d=json.loads(l[-1]); print('$1', round(d.get('value',0),2), d.get('unit'), 'e2e', round(d.get('e2e',{}).get('value',0),2), 'frac', d.get('roofline',{}).get('frac'), 'clk', d.get('clocks',{}).get('sm_mhz'))"; }
timeout 900 python bench.py 2>&1 | summ "S1024"
timeout 900 python bench.py --total-envs 65536 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | summ "S65536"
timeout 900 python bench.py --envs 256 --no-cpu-baseline 2>&1 | summ "S256"
timeout 900 python bench.py --envs 128 --no-cpu-baseline 2>&1 | summ "S128"
timeout 900 python bench.py --envs 1 --no-cpu-baseline 2>&1 | summ "S1"
timeout 900 python bench.py --scene H --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | summ "H"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | summ "reference"
timeout 900 python tools/sweep_bench.py 2>&1 | tail -2

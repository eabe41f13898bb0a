#!/bin/bash
# J^T gather split sweep (SS_GATHER_SPLIT): coupled Table II scenes and the
# 1M-tet snake (one env each), then parity of the streaming tests at split 4.
for s in 1 2 4 8; do
  echo "== split $s"
  SS_GATHER_SPLIT=$s timeout 600 python tools/table2.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['snakes'], d['total_ms'])"
  SS_GATHER_SPLIT=$s timeout 600 python bench.py --scene H --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('H', round(d['value'],2), d['kernels_ms_per_frame']['k_gather'])"
done

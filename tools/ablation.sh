#!/bin/bash
# N1: layer latency with and without Expert-Centric Scheduling on B200.
cd "$(dirname "$0")/.."
for c in ${CONFIGS:-C3a C3b C4pp C4}; do
  for ek in auto token warp; do
    timeout 900 python bench.py --config $c --expert-kernel $ek --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$c', '$ek', round(l['ms_per_step'],3), 'ms', l.get('stage_ms',''))"
  done
done

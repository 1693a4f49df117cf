#!/bin/bash
# N1 (PAPER Table 4) on this B200: layer latency of the full layer and of
# each ablation -- w/o Shared Dense MLP (d_ff = 0), w/o Cartesian Product Router (dense
# gate projection + top-K over N), w/o Expert-Centric Scheduling (token-centric executor)
# -- plus the full layer on the one-pass ROWS executor and the expert-major plan.
cd "$(dirname "$0")/.."
for c in ${CONFIGS:-C3a C4}; do
  for v in "full:" "no_mlp:--no-shared-mlp" "no_cpr:--router dense" "no_ecs:--expert-kernel token" \
           "rows_grouped:--v-layout rows" "rows_expert_major:--expert-kernel warp"; do
    name=${v%%:*}; flags=${v#*:}
    timeout 1200 python bench.py --config $c $flags --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$c', '$name', round(l['ms_per_step'],3), 'ms', l.get('config',{}).get('ablation',''), l.get('workspace_bytes',''), {k: round(v,3) for k,v in l.get('stage_ms',{}).items()})"
  done
done

#!/bin/bash
# bench.py stage times under env settings: SWEEP="A=1 B=2;A=3" CONFIG=C3a bash tools/sweep_env.sh
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
IFS=';' read -ra SETS <<< "${SWEEP:-X=0}"
for cfg in "${SETS[@]}"; do
  env $cfg timeout 600 python bench.py --config ${CONFIG:-C3a} --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e $ARGS > /tmp/b.log 2>&1
  echo "== $cfg: $(tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: round(v,3) for k,v in d.get('stage_ms',{}).items()})" 2>&1 | tail -1)"
done

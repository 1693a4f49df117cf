#!/bin/bash
# ncu captures: launch list of one bench step + full set of one kernel ($1 regex)
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CFG=${CONFIG:-C3a}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}.csv \
  python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s ${SKIP:-1} -c 1 -o gpurun_out/prof_$1_${CFG} \
  python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$1.log 2>&1
tail -3 gpurun_out/ncu_$1.log

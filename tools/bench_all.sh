#!/bin/bash
# one bench line per workload into gpurun_out/${TAG}/bench_<config>.json (C3a with the CPU
# oracle baseline, the others without), then the launch lists of C3a and C4
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
OUT=gpurun_out/${TAG:-v}
mkdir -p $OUT
for c in ${CONFIGS:-C3a C1 C2 C3b C4 C4p C4pp C5 C5s}; do
  extra="--no-cpu-baseline"; [ "$c" = "C3a" ] && extra=""
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 $extra > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "$c rc=$? $(tail -1 $OUT/bench_$c.json | cut -c1-120)"
done

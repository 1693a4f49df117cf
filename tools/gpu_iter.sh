#!/bin/bash
# one iteration on the GPU box: build, a filtered parity run, then bench lines for $CONFIGS
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${TESTS:+-k "$TESTS"} > gpurun_out/pytest_iter.log 2>&1
  echo "pytest rc=$?"; tail -5 gpurun_out/pytest_iter.log
fi
for c in ${CONFIGS:-C3a}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; python tools/summ.py gpurun_out/bench_$c.json
done

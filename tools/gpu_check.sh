#!/bin/bash
# GPU pass: build, parity tests (optionally filtered by $1), smoke, short bench.
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --config ${CONFIG:-C3a} --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench.log | cut -c1-1500
fi
if [ -n "$REF" ]; then
timeout 900 python bench.py --impl reference --config ${CONFIG:-C3a} --steps 3 --warmup 1 --ref-seconds 20 > gpurun_out/bench_ref.log 2>&1
tail -1 gpurun_out/bench_ref.log | cut -c1-800
fi

cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/ev
# the driver's commands on this tree
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev/pytest_gpu.log; tail -2 gpurun_out/ev/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; tail -1 gpurun_out/ev/smoke.log
timeout 900 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; python tools/summ.py gpurun_out/ev/bench.json
timeout 900 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/ev/bench_reference.json 2>&1; tail -1 gpurun_out/ev/bench_reference.json | cut -c1-200
# launch list of the same bench command (ncu, serialised, cold): per-kernel share of the step
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_C3a.csv python bench.py --gpus 1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu launches rc=$?"
# ablations (PAPER Table 4) on this tree
CONFIGS="C3a C4" bash tools/ablation.sh > gpurun_out/ev/ablation.log 2>&1; cat gpurun_out/ev/ablation.log | cut -c1-160

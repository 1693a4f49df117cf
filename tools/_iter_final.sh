# the round's closing evidence on the current tree: the driver's commands, every workload's
# bench line, the launch list of the default bench, fresh ncu captures of the dominant kernel
# (C3a pass V) and of the N4 fused GEMM (C5s)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
O=gpurun_out/final; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --gpus 1 --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; python tools/summ.py $O/bench.json
timeout 900 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > $O/bench_reference.json 2>&1; tail -1 $O/bench_reference.json | cut -c1-160
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3a.csv python bench.py --gpus 1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu launches rc=$?"
TAG=final/all bash tools/bench_all.sh
KERN=expert_vslice_kernel CONFIG=C3a TAG=_final bash tools/ncu_full.sh
KERN=gemm_i8_topk_kernel CONFIG=C5s TAG=_final bash tools/ncu_full.sh
mv gpurun_out/full_*_final* $O/ 2>/dev/null; ls $O

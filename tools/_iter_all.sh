cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/all
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k c2_sweep > gpurun_out/all/pytest_c2.log 2>&1; echo "c2 pytest rc=$?"; tail -1 gpurun_out/all/pytest_c2.log
timeout 900 python tools/c2_sweep.py > gpurun_out/all/c2_sweep.jsonl 2> gpurun_out/all/c2_sweep.err; echo "c2 sweep rc=$?"; wc -l gpurun_out/all/c2_sweep.jsonl
TAG=all STEPS=10 bash tools/bench_all.sh
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/all/bench_reference.json 2>&1; tail -1 gpurun_out/all/bench_reference.json | cut -c1-300

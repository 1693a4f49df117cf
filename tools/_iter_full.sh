cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_C3a.json 2> gpurun_out/bench_C3a.err; python tools/summ.py gpurun_out/bench_C3a.json
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5.json 2>&1; python tools/summ.py gpurun_out/bench_C5.json
python -m paper_2602_05711_b200.build --measure > /dev/null
for pad in 0 4096 14336; do OMNIMOE_LIB=$PWD/paper_2602_05711_b200/libomnimoe_measure.so OMNIMOE_WS_PAD_COUNTERS=$pad timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_pad$pad.json 2>&1; echo "pad $pad"; python tools/summ.py gpurun_out/bench_C5_pad$pad.json; done

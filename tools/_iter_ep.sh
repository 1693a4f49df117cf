cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_ep.py -m gpu -q -x --durations=6 > gpurun_out/pytest_ep.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/pytest_ep.log
mkdir -p gpurun_out/ep
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 2 --backend gloo --cpu-seconds 10 > gpurun_out/ep/bench_C5_gloo2.json 2> gpurun_out/ep/bench_C5_gloo2.err; echo "C5 gloo2 rc=$?"; tail -1 gpurun_out/ep/bench_C5_gloo2.json | cut -c1-1500; tail -3 gpurun_out/ep/bench_C5_gloo2.err

cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
python -m paper_2602_05711_b200.build --measure > /dev/null 2>&1
export OMNIMOE_LIB=$PWD/paper_2602_05711_b200/libomnimoe_measure.so
OMNIMOE_V_PIPE=3 timeout 900 python -m pytest tests -m gpu -q -x -k "sliced or fullsize_sliced or layer_c5 or whole_batch_routing_layer" > gpurun_out/pytest_pipe.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pipe.log
for v in 0 2 3 4; do OMNIMOE_V_PIPE=$v timeout 600 python bench.py --config C3a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>&1; echo "pipe $v"; python tools/summ.py gpurun_out/b.json; done
for v in 0 3; do OMNIMOE_V_PIPE=$v timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>&1; echo "pipe $v"; python tools/summ.py gpurun_out/b.json; done

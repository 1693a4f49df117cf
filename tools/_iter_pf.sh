cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
python -m paper_2602_05711_b200.build --measure > /dev/null 2>&1
export OMNIMOE_LIB=$PWD/paper_2602_05711_b200/libomnimoe_measure.so
OMNIMOE_V_VARIANT=1 timeout 900 python -m pytest tests -m gpu -q -x -k "sliced or layer_c5" > gpurun_out/pytest_pf.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pf.log
for v in 0 1 2; do for c in C3a C5; do OMNIMOE_V_VARIANT=$v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>&1; echo "variant $v"; python tools/summ.py gpurun_out/b.json; done; done

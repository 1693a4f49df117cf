cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
python -m paper_2602_05711_b200.build --measure > /dev/null 2>&1
export OMNIMOE_LIB=$PWD/paper_2602_05711_b200/libomnimoe_measure.so
for v in 0 1 2 3; do echo "variant $v"; OMNIMOE_ACCUM_VARIANT=$v python tools/bwd_prof.py C3a 2>&1 | grep -v -i warn | grep accum; done
OMNIMOE_ACCUM_VARIANT=1 python -m pytest tests -m gpu -q -x -k "bwd" 2>&1 | tail -1

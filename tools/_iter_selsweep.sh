cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); from paper_2602_05711_b200 import build; build.build(measure=True)" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -k "${TESTS:-route or whole_batch or layer}" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
export OMNIMOE_LIB=$PWD/paper_2602_05711_b200/libomnimoe_measure.so
for cfg in ${CONFIGS:-C3a C4}; do
for v in ${VARIANTS:-"OMNIMOE_SELECT_CLASSES=0" "OMNIMOE_SELECT_CLASSES=1"}; do
  echo "$cfg $v: $(env $v python tools/layer_prof.py $cfg sliced 5 2>&1 | grep select_bucket)"
done; done

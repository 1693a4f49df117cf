cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x -k "${TESTS:-route or logits or layer}" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
M=$PWD/paper_2602_05711_b200/libomnimoe_measure.so
for c in ${CONFIGS:-C3b C5s C2}; do for v in 0 1; do
  OMNIMOE_LIB=$M OMNIMOE_ROUTE_FUSED=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_${c}_$v.json 2>/dev/null
  echo "== $c fused=$v: $(python tools/summ.py gpurun_out/b_${c}_$v.json | cut -c1-120)"
done; done

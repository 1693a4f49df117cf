cd $GRAFT_REPO_ROOT
M=$PWD/paper_2602_05711_b200/libomnimoe_measure.so
H=$PWD/build_ab/libomnimoe_head.so
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest tests -m gpu -q -x -k "$TESTS" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ab.log; fi
for c in ${CONFIGS:-C3a C5 C4 C4pp}; do
for lib in $H $M; do
  OMNIMOE_LIB=$lib timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>/dev/null
  echo "== $c $(basename $lib): $(python tools/summ.py gpurun_out/b.json | cut -c1-70)"
done; done

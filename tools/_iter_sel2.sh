cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -k "route or whole_batch" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
for c in ${CONFIGS:-C3a C4}; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>&1; python tools/summ.py gpurun_out/b.json; done
python tools/layer_prof.py C3a sliced 5 2>&1 | grep -v Warn | grep -v warn | head -8

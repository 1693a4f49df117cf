cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "schedule or sliced or fullsize or layer or bwd or load_stats or ep" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_iter.log
run() { env $1 timeout 600 python bench.py --config ${2:-C3a} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $3 > gpurun_out/b.json 2>&1; echo "$1 ${2:-C3a} $3"; python tools/summ.py gpurun_out/b.json; }
run "X=0"
run "X=0" C5
python tools/layer_prof.py C3a sliced 5 2>&1 | grep -v Warn | tail -22

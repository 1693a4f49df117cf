cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "sliced or fullsize or layer" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_iter.log
run() { env $1 timeout 600 python bench.py --config ${2:-C3a} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $3 > gpurun_out/b.json 2>&1; echo "$1 ${2:-C3a} $3"; python tools/summ.py gpurun_out/b.json; }
run "OMNIMOE_Z256=0"
run "OMNIMOE_ZV=0"
run "OMNIMOE_ZV=1"
run "OMNIMOE_ZV=2"
run "OMNIMOE_ZV=0" C5

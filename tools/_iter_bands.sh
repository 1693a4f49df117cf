cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { env $1 timeout 600 python bench.py --config ${2:-C3a} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>&1; echo "$1 ${2:-C3a}"; python tools/summ.py gpurun_out/b.json; }
for v in "OMNIMOE_Z_MINB=3 OMNIMOE_Z_TIF=2" "OMNIMOE_Z_MINB=2 OMNIMOE_Z_TIF=2" "OMNIMOE_Z_MINB=3 OMNIMOE_Z_TIF=3" "OMNIMOE_Z_MINB=2 OMNIMOE_Z_TIF=3" "OMNIMOE_Z_MINB=3 OMNIMOE_Z_TIF=4" "OMNIMOE_Z_MINB=2 OMNIMOE_Z_TIF=4" "OMNIMOE_Z_MINB=1 OMNIMOE_Z_TIF=4" "OMNIMOE_V_MINB=3" "OMNIMOE_V_MINB=2"; do run "$v"; done
run "OMNIMOE_V_MINB=3" C5
run "OMNIMOE_V_MINB=4" C5

cd $GRAFT_REPO_ROOT
M=$PWD/paper_2602_05711_b200/libomnimoe_measure.so
for c in ${CONFIGS:-C3a C5 C4pp C2}; do for rep in 1 2; do for v in ${VALS:-0 5}; do
  OMNIMOE_LIB=$M OMNIMOE_V_CONFIG=$v timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>/dev/null
  echo "== $c cfg=$v: $(python tools/summ.py gpurun_out/b.json | grep -o "C[0-9a-z]*: [0-9.]* ms\|'a6_pass_v': [0-9.]*" | tr '\n' ' ')"
done; done; done

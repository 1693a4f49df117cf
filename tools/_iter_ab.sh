cd $GRAFT_REPO_ROOT
M=$PWD/paper_2602_05711_b200/libomnimoe_measure.so
H=$PWD/build_ab/libomnimoe_head.so
for c in ${CONFIGS:-C3a C5 C4 C4pp}; do
for v in "$H X=0" $(for x in ${VALS:-0 1}; do echo "$M ${KNOB}=$x"; done | tr ' ' '|'); do
  lib=$(echo $v | tr '|' ' ' | cut -d' ' -f1); kv=$(echo $v | tr '|' ' ' | cut -d' ' -f2)
  OMNIMOE_LIB=$lib env $kv timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>/dev/null
  echo "== $c $(basename $lib) $kv: $(python tools/summ.py gpurun_out/b.json | cut -c1-100)"
done; done

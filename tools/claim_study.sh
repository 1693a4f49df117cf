#!/bin/bash
# pass-V claim pipeline: parity of the executors, then C5/C3a per-kernel times with the
# executor's work counters at the committed offset and shifted by 4 KB / 14 KB
cd "$(dirname "$0")/.."
# OMNIMOE_* knobs are read only by the measurement build (csrc/tuning.cuh)
python -m paper_2602_05711_b200.build --measure > /dev/null
export OMNIMOE_LIB=$(pwd)/paper_2602_05711_b200/libomnimoe_measure.so
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
OUT=gpurun_out/${TAG:-claim}
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "sliced or layer or vslice or group" > $OUT/pytest_sliced.log 2>&1
echo "pytest rc=$? $(tail -1 $OUT/pytest_sliced.log)"
for c in C5 C3a; do
  for pad in none 4096 14336; do
    if [ $pad = none ]; then unset OMNIMOE_WS_PAD_COUNTERS; else export OMNIMOE_WS_PAD_COUNTERS=$pad; fi
    timeout 300 python tools/layer_prof.py $c sliced 5 > $OUT/prof_${c}_pad$pad.log 2>&1
    echo "$c pad=$pad: $(grep -i "vslice\|layer\|total" $OUT/prof_${c}_pad$pad.log | head -4 | tr '\n' ' ')"
  done
done
unset OMNIMOE_WS_PAD_COUNTERS

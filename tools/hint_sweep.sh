#!/bin/bash
# a6 time for L2 hint bitmasks x (group size : token blocks) specs
cd "$(dirname "$0")/.."
# OMNIMOE_* knobs are read only by the measurement build (csrc/tuning.cuh)
python -m paper_2602_05711_b200.build --measure > /dev/null
export OMNIMOE_LIB=$(pwd)/paper_2602_05711_b200/libomnimoe_measure.so
for h in ${HINTS:-0 2 6 7 3}; do
  echo "hints=$h"; OMNIMOE_L2_HINTS=$h python tools/sweep_group.py ${CONFIG:-C3a} ${SPECS:-1024:1,1024:2,8192:1,8192:2} 2>&1 | grep -v "^{"
done

#!/bin/bash
# one `ncu --set full` capture of kernel $KERN during a layer forward of $CONFIG ($LAYOUT)
#   KERN=select_kernel CONFIG=C3a bash tools/ncu_full.sh
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
OUT=gpurun_out/full_${KERN}_${CONFIG:-C3a}${TAG}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KERN}" -s ${SKIP:-0} -c 1 -o $OUT \
  python tools/layer_once.py ${CONFIG:-C3a} ${LAYOUT:-sliced} 1 $EXTRA > ${OUT}.log 2>&1
tail -2 ${OUT}.log

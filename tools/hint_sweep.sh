#!/bin/bash
# a6 time for L2 hint bitmasks x (group size : token blocks) specs
cd "$(dirname "$0")/.."
for h in ${HINTS:-0 2 6 7 3}; do
  echo "hints=$h"; OMNIMOE_L2_HINTS=$h python tools/sweep_group.py ${CONFIG:-C3a} ${SPECS:-1024:1,1024:2,8192:1,8192:2} 2>&1 | grep -v "^{"
done
